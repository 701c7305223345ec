// chain.cu -- persistent decode-chain executor (sm_100a).
//
// A decode token runs the PQ linear layers of a model as a chain of grouped
// GEMVs (q/k/v, o, gate/up, down per block; every layer packed separately,
// P:219).  Launching one kernel per step pays, per step, a launch, the first
// stage's memory latency and a grid-wide completion before the next step may
// read its x.  This executor runs the whole chain in ONE persistent kernel
// (one CTA per SM, cooperative launch):
//
//  * the per-step work (row tile x K-range of groups) is planned once on the
//    host into a [steps][CTAs][items] table;
//  * the producer warp of every CTA streams the codebook/index stages of ALL
//    its steps back to back through the SMEM ring -- weights do not depend on
//    x, so the ring keeps filling while the consumers wait for the previous
//    step (no pipeline drain at step boundaries);
//  * there is NO grid-wide barrier between steps: every output element is a
//    "counted accumulator" (gemv_core.cuh): an int64 red.add target that
//    carries the fixed-point sum (units 2^-32, exact and order-independent
//    -> deterministic) AND the number of contributions; a consumer polls
//    exactly the words it needs until each shows the producer's count.
//
// Besides PQ GEMV steps the kernel runs the non-linear glue of a decoder
// block (whole-model decode, llama.cu): an EMBED step (the embedding row of
// the token the previous run's lm_head chose), RMSNorm and SwiGLU as input
// transforms of a PQ step, the residual connection fused into the PQ epilogue
// (an exact integer add of the residual words), and an ATTN step (RoPE,
// KV-cache append, softmax attention, split over the cache length).
//
// Cross-run / cross-rank protocol (tail words of the arena allocation):
//  * run index r = (CTA entry counter) / nctas; parity r & 1 selects the
//    arena buffer the run accumulates into; the run zeroes the other buffer
//    for run r+1 (no memset node, graph replays need no host bookkeeping);
//  * world > 1: a rank starts zeroing only after EVERY rank finished run r-1
//    (each rank adds 1 to every rank's DONE word when its last CTA exits),
//    so a slow peer's late stores can never hit a zeroed buffer and a fast
//    peer can never write into a buffer before it was zeroed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "chain_kernel.cuh"

namespace fasq {
using namespace chainimpl;

namespace {

// counted accumulator words of the LAST run -> value (units 2^-32) -> fp16 /
// fp32 / FASQ_ACC_I64.  The last run is (entry counter / nctas) - 1 (read on
// the device: graph replays need no host bookkeeping).  Every word is polled
// until it carries its `ks` contributions (peers' red.adds of the last step
// may still be in flight when this rank's kernel ends).  A run that raised
// the out-of-range flag yields NaN (float outputs).
// With a lazy base (off2 >= 0) the value is the sum of both words; with
// RMSNorm slots (sc_off >= 0) it is multiplied by the scale every consumer
// applies (warp_norm_scale's fixed summation order, emulated serially).
__global__ void k_counted_convert(const unsigned long long* __restrict__ arenas, long long arena_words, int nctas,
                                  long long off, int64_t n, int ks, void* out, int dtype, int sys, long long off2,
                                  int ks2, long long sc_off, int sc_n, int sc_F, float sc_eps, int64_t ld) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long* tail = arenas + 2 * arena_words;
    const unsigned long long runs = tail[T_ENTRY] / (unsigned long long)nctas;
    const unsigned last = (unsigned)((runs + 1ull) & 1ull);   // parity of run (runs - 1)
    const unsigned long long* buf = arenas + (long long)last * arena_words;
    long long v = core::poll_value(buf + off + i, ks, sys != 0);
    if (off2 >= 0) v += core::poll_value(buf + off2 + i, ks2, sys != 0);
    double sc = 1.0;
    if (sc_off >= 0) {
        const int b = (int)(i / ld);
        float a[32];
        for (int k = 0; k < 32; ++k) {
            float t = 0.f;
            if (k < sc_n) t += word_f32(buf[sc_off + b * 64 + k]);
            if (k + 32 < sc_n) t += word_f32(buf[sc_off + b * 64 + k + 32]);
            a[k] = t;
        }
        for (int m = 16; m >= 1; m >>= 1) {
            float na[32];
            for (int k = 0; k < 32; ++k) na[k] = a[k] + a[k ^ m];
            for (int k = 0; k < 32; ++k) a[k] = na[k];
        }
        sc = (double)(1.0f / sqrtf(a[0] / (float)sc_F + sc_eps));
    }
    const bool bad = tail[T_OVF] != 0ull;
    const double val = (double)v * core::kAccInv * sc;
    if (dtype == FASQ_ACC_I64) reinterpret_cast<long long*>(out)[i] = sc_off >= 0 ? __double2ll_rn(val * 4294967296.0) : v;
    else if (dtype == FASQ_F32) reinterpret_cast<float*>(out)[i] = bad ? __int_as_float(0x7fc00000) : (float)val;
    else reinterpret_cast<__half*>(out)[i] = bad ? __ushort_as_half((unsigned short)0x7e00) : __double2half(val);
}

// Attention output of the LAST run (ATTN step partials [B][heads][P][hd + 2])
// merged exactly as stage_x_attn merges them, as fp16 / fp32 / FASQ_ACC_I64
// [B][heads * hd].
__global__ void k_attn_convert(const unsigned long long* __restrict__ arenas, long long arena_words, int nctas,
                               long long off, int B, int heads, int hd, int P, void* out, int dtype) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)B * heads * hd;
    if (i >= n) return;
    const unsigned long long* tail = arenas + 2 * arena_words;
    const unsigned long long runs = tail[T_ENTRY] / (unsigned long long)nctas;
    const unsigned last = (unsigned)((runs + 1ull) & 1ull);
    const int b = (int)(i / ((int64_t)heads * hd)), col = (int)(i % ((int64_t)heads * hd));
    const int head = col / hd, e = col - head * hd;
    const unsigned long long* hb = arenas + (long long)last * arena_words + off + ((size_t)b * heads + head) * P * (hd + 2);
    float M = -INFINITY;
    for (int q = 0; q < P; ++q) M = fmaxf(M, word_f32(hb[(size_t)q * (hd + 2) + hd]));
    float den = 0.f, num = 0.f;
    for (int q = 0; q < P; ++q) {
        const unsigned long long* pb = hb + (size_t)q * (hd + 2);
        const float m = word_f32(pb[hd]);
        const float f = m == -INFINITY ? 0.f : expf(m - M);
        den += f * word_f32(pb[hd + 1]);
        num += f * word_f32(pb[e]);
    }
    const float v = num / den;
    if (dtype == FASQ_ACC_I64) reinterpret_cast<long long*>(out)[i] = __float2ll_rn(v * core::kAccScale);
    else if (dtype == FASQ_F32) reinterpret_cast<float*>(out)[i] = v;
    else reinterpret_cast<__half*>(out)[i] = __float2half_rn(v);
}

void destroy_chain(fasq_chain* c) {
    if (!c) return;
    for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
    if (c->arenas) {
        if (c->arena_ipc) cudaFree(c->arenas);
        else dev_free(c->arenas, 0);
    }
    dev_free(c->peers_dev, 0);
    dev_free(c->items, 0);
    dev_free(c->phases, 0);
    delete c;
}

fasq_status upload_peers(fasq_chain* c, const std::vector<unsigned long long*>& bases) {
    FASQ_CUDA_TRY(cudaMemcpy(c->peers_dev, bases.data(), bases.size() * sizeof(void*), cudaMemcpyHostToDevice));
    c->peers_ready = true;
    return FASQ_OK;
}

}  // namespace

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

// ---- planner (host only) ------------------------------------------------------
// K-split count per layer of one step: every layer's work (row tiles x groups)
// gets a share of the `nctas` CTAs proportional to its index bytes; a layer
// with rt row tiles is split into k = share / rt K-ranges (K ranges may differ
// by one group), capped by its group count and by the 6-bit count field of the
// counted words (<= 63).  While the step needs more CTAs than it has, the
// largest split shrinks.
std::vector<int> plan_step_ks(const std::vector<int64_t>& F_out_pad, const std::vector<int>& n_groups, int nctas,
                              int R, bool even) {
    const int nl = (int)F_out_pad.size();
    double W = 0;
    for (int l = 0; l < nl; ++l) W += (double)F_out_pad[l] * n_groups[l];
    std::vector<int> rt(nl), ks(nl);
    int total = 0;
    for (int l = 0; l < nl; ++l) {
        rt[l] = (int)((F_out_pad[l] + R - 1) / R);
        const double share = nctas * ((double)F_out_pad[l] * n_groups[l]) / W;
        int k = std::max(1, (int)(share / rt[l]));
        k = std::min(k, n_groups[l]);
        k = std::min(k, 63);
        if (even) {
            const int gper = (n_groups[l] + k - 1) / k;
            k = (n_groups[l] + gper - 1) / gper;
        }
        ks[l] = k;
        total += rt[l] * k;
    }
    while (total > nctas) {
        int lm = -1;
        for (int l = 0; l < nl; ++l)
            if (ks[l] > 1 && (lm < 0 || ks[l] * rt[l] > ks[lm] * rt[lm])) lm = l;
        if (lm < 0) break;
        total -= rt[lm];
        ks[lm] -= 1;
    }
    return ks;
}

static int chain_rows_per_cta(int d, int B, int nw) {
    const int NB = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : 8;
    const int rw = d <= 2 ? 64 : (NB == 1 ? 64 : NB == 2 ? 32 : NB == 4 ? 16 : 8);
    return rw * nw;
}

fasq_status chain_build(const std::vector<StepDesc>& steps, int B, int world, int rank, int max_ctas, bool det,
                        const ChainModel* model, cudaStream_t st, fasq_chain** out) {
    *out = nullptr;
    const int n_steps = (int)steps.size();
    if (n_steps < 1) return FASQ_E_ARG;
    if (world < 1 || world > 8 || rank < 0 || rank >= world || max_ctas < 0) return FASQ_E_ARG;
    if (B < 1 || B > 8) return FASQ_E_UNSUPPORTED;
    for (const StepDesc& sd : steps)
        for (const fasq_layer* L : sd.layers)
            if (L && (L->bits || L->dim0)) {   // NEXT-2 packed / NEXT-4 dim = 0: per-launch fasq_gemv only
                set_error("chain: packed-index and dim = 0 layers run through fasq_gemv, not the decode chain");
                return FASQ_E_UNSUPPORTED;
            }
    const int NB = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : 8;
    fasq_chain* c = new fasq_chain();
    auto fail = [&](fasq_status s, const std::string& msg) {
        if (!msg.empty()) set_error("chain: " + msg);
        destroy_chain(c);
        return s;
    };
    c->n_steps = n_steps;
    c->B = B;
    c->world = world;
    c->rank = rank;
    const int sms = sm_count();
    c->nctas = sms;
    if (max_ctas > 0) c->nctas = std::min(c->nctas, (int)max_ctas);
    c->nw = 16;
    c->st = 3;
    if (const char* e = getenv("FASQ_CHAIN_CFG")) {   // experiments: "nw,st"
        int a = 0, b = 0;
        if (sscanf(e, "%d,%d", &a, &b) == 2) { c->nw = a; c->st = b; }
    }
    if (model) { c->model = *model; c->has_model = true; }
    // ---- validate + arena layout ----
    int64_t words = 0;
    c->acc_off.resize(n_steps);
    c->acc_ld.resize(n_steps);
    c->acc_ks.resize(n_steps);
    c->kinds.resize(n_steps);
    c->nsq_off.assign(n_steps, -1);
    c->nsq_n.assign(n_steps, 0);
    c->nsq_F.assign(n_steps, 0);
    c->nsq_eps.assign(n_steps, 0.f);
    c->nsq_epi.assign(n_steps, 0);
    c->lazy.assign(n_steps, -1);
    c->attn_hd.assign(n_steps, 0);
    c->attn_heads.assign(n_steps, 0);
    std::vector<int> pq_F_in(n_steps, 0);
    for (int s = 0; s < n_steps; ++s) {
        const StepDesc& S = steps[s];
        c->kinds[s] = S.kind;
        if (S.kind == SK_PQ) {
            if (S.layers.empty() || S.layers.size() > 4) return fail(FASQ_E_ARG, "a PQ step needs 1..4 layers");
            const int64_t F_in = S.layers[0]->F_in;
            for (const fasq_layer* L : S.layers) {
                if (!L) return fail(FASQ_E_ARG, "null layer");
                if (L->F_in != F_in) return fail(FASQ_E_SHAPE, "layers of a step must share F_in");
                if (c->d == 0) c->d = L->d;
                if (L->d != c->d) return fail(FASQ_E_UNSUPPORTED, "all layers of a chain need the same d");
                c->maxC = std::max(c->maxC, L->C);
                const int64_t ld = S.kshard ? L->F_out : (S.out_all ? L->F_out * world : L->F_out);
                c->acc_off[s].push_back(words);
                c->acc_ld[s].push_back(ld);
                words += (int64_t)B * ld;
            }
            pq_F_in[s] = (int)F_in;
            if (S.lazy_step >= 0) {
                if (S.lazy_step >= s || S.layers.size() != 1 || steps[S.lazy_step].kind == SK_ATTN)
                    return fail(FASQ_E_ARG, "lazy residual base must be an earlier PQ/EMBED step (1-layer steps)");
                c->lazy[s] = S.lazy_step;
            }
            if (S.in_mode == IN_RMSNORM) {   // sum-of-squares slots [B][64]
                c->nsq_off[s] = words;
                words += (int64_t)B * 64;
            }
        } else if (S.kind == SK_EMBED) {
            if (!model || !S.embed || S.hidden < 1) return fail(FASQ_E_ARG, "EMBED step needs a model and a table");
            c->acc_off[s].push_back(words);
            c->acc_ld[s].push_back(S.hidden);
            c->acc_ks[s].push_back(1);
            words += (int64_t)B * S.hidden;
        } else if (S.kind == SK_ATTN) {
            if (!model || !S.kc || !S.vc || S.head_dim < 8 || S.head_dim > 128 || S.head_dim % 8 || S.n_kv < 1 ||
                S.n_heads % S.n_kv)
                return fail(FASQ_E_UNSUPPORTED, "ATTN step: head_dim must be a multiple of 8 in 8..128");
            if (S.q_step < 0 || S.q_step >= s || steps[S.q_step].kind != SK_PQ || steps[S.q_step].layers.size() != 3)
                return fail(FASQ_E_ARG, "ATTN step needs an earlier q/k/v step");
            if (model->attn_parts < 1 || model->attn_parts > 4)
                return fail(FASQ_E_UNSUPPORTED, "attention cache parts must be 1..4");
            // partials [B][heads][parts][hd + 2] (logical output width heads * hd)
            c->acc_off[s].push_back(words);
            c->acc_ld[s].push_back((int64_t)S.n_heads * S.head_dim);
            c->acc_ks[s].push_back(1);
            c->attn_hd[s] = S.head_dim;
            c->attn_heads[s] = S.n_heads;
            words += (int64_t)B * S.n_heads * model->attn_parts * (S.head_dim + 2);
        } else {
            return fail(FASQ_E_ARG, "unknown step kind");
        }
    }
    if (c->d == 0) return fail(FASQ_E_ARG, "a chain needs at least one PQ step");
    const bool pair = c->d <= 2;
    if (model && !pair) return fail(FASQ_E_UNSUPPORTED, "whole-model chains need d <= 2");
    c->rw = pair ? 64 : (NB == 1 ? 64 : NB == 2 ? 32 : NB == 4 ? 16 : 8);
    const int E = entry_bytes(c->d);
    const size_t cbb_max = (size_t)c->maxC * 32 * E;
    auto cbring = [&](int stg) { return pair ? (size_t)kChainCS * kPairSlot : (size_t)stg * cbb_max; };
    auto ring = [&](int stg, int nw) { return cbring(stg) + (size_t)stg * c->rw * nw * 32; };
    while (c->st > 1 && ring(c->st, c->nw) > kChainSmem) --c->st;   // 16 consumer warps; shallower ring first
    if (ring(c->st, c->nw) > kChainSmem) return fail(FASQ_E_UNSUPPORTED, "SMEM plan too large");
    c->R = c->rw * c->nw;
    // d = 2, B >= 4: the tensor-core path reads the XOR codebook images (built once per layer)
    const bool mma = c->d == 2 && NB == 8 && !FASQ_CHAIN_NO_MMA;
    if (mma)
        for (const StepDesc& S : steps)
            for (const fasq_layer* L : S.layers) {
                fasq_status e = ensure_cbimg_x(L, st);
                if (e != FASQ_OK) return fail(e, "XOR codebook image");
            }
    words = (words + 1) & ~(int64_t)1;   // 16-B zeroing stores
    c->arena_words = words;
    // ---- work plan: per step a list of items, dealt to the CTAs round-robin ----
    std::vector<std::vector<ChainItem>> per_step(n_steps);
    std::vector<ChainPhase> phases(n_steps);
    for (int s = 0; s < n_steps; ++s) {
        const StepDesc& S = steps[s];
        ChainPhase& P = phases[s];
        std::memset(&P, 0, sizeof(P));
        P.kind = S.kind;
        P.res_off = -1;
        P.res2_off = -1;
        P.x2_off = -1;
        P.sc_off = -1;
        // the RMSNorm scale of a normed source step (applied by this consumer)
        auto set_scale = [&](int src) {
            if (src >= 0 && c->nsq_off[src] >= 0 && !c->nsq_epi[src]) {
                P.sc_off = c->nsq_off[src];
                P.sc_n = c->nsq_n[src];
                P.sc_F = c->nsq_F[src];
                P.sc_eps = c->nsq_eps[src];
            }
        };
        if (S.kind == SK_EMBED) {
            P.embed = S.embed;
            P.e_off = c->acc_off[s][0];
            P.hidden = S.hidden;
            ChainItem w{};
            w.kind = SK_EMBED;
            per_step[s].push_back(w);
            continue;
        }
        if (S.kind == SK_ATTN) {
            const StepDesc& Q = steps[S.q_step];
            const int hd = S.head_dim;
            for (int l = 0; l < 3; ++l) {
                const int64_t want = (int64_t)(l == 0 ? S.n_heads : S.n_kv) * hd;
                if (c->acc_ld[S.q_step][l] != want) return fail(FASQ_E_SHAPE, "q/k/v widths do not match the heads");
            }
            P.q_off = c->acc_off[S.q_step][0];
            P.k_off = c->acc_off[S.q_step][1];
            P.v_off = c->acc_off[S.q_step][2];
            P.q_ks = c->acc_ks[S.q_step][0];
            P.k_ks = c->acc_ks[S.q_step][1];
            P.v_ks = c->acc_ks[S.q_step][2];
            P.q_ld = S.n_heads * hd;
            P.kv_ld = S.n_kv * hd;
            P.o_off = c->acc_off[s][0];
            P.kc = S.kc;
            P.vc = S.vc;
            P.n_heads = S.n_heads;
            P.n_kv = S.n_kv;
            P.hd = hd;
            P.parts = model->attn_parts;
            set_scale(S.q_step);
            (void)Q;
            for (int h = 0; h < S.n_heads; ++h)
                for (int q = 0; q < P.parts; ++q) {
                    ChainItem w{};
                    w.kind = SK_ATTN;
                    w.head = h;
                    w.kidx = q;
                    w.nsq = -1;
                    per_step[s].push_back(w);
                }
            continue;
        }
        // ---- PQ ----
        const int nl = (int)S.layers.size();
        std::vector<int64_t> fop(nl), fop_plan(nl);
        std::vector<int> ngr(nl);
        for (int l = 0; l < nl; ++l) {
            fop[l] = S.layers[l]->F_out_pad;
            ngr[l] = S.layers[l]->n_groups;
            // deterministic TP: K ranges as the unsharded (world 1) plan on a full
            // GPU would cut them -> bit-identical to one GPU
            fop_plan[l] = det && world > 1 && !S.kshard
                              ? (S.layers[l]->F_out * world + kRowBlock - 1) / kRowBlock * kRowBlock
                              : fop[l];
        }
        const bool even = getenv("FASQ_CHAIN_EVEN") != nullptr;
        std::vector<int> ks = plan_step_ks(fop_plan, ngr, det && world > 1 ? sms : c->nctas, c->R, even);
        for (int l = 0; l < nl; ++l) c->acc_ks[s].push_back(S.kshard ? ks[l] * world : ks[l]);
        // input
        P.F_in = pq_F_in[s];
        P.in_mode = S.in_mode;
        if (S.in_mode == IN_EXT) {
            if (c->ext_F_in == 0) c->ext_F_in = P.F_in;
            if (c->ext_F_in != P.F_in) return fail(FASQ_E_SHAPE, "external-input steps need the same F_in");
        } else {
            const int src = S.src_step;
            if (src < 0 || src >= s) return fail(FASQ_E_ARG, "input must come from an earlier step");
            if (S.in_mode == IN_SILU) {
                if (steps[src].kind != SK_PQ || steps[src].layers.size() < 2) return fail(FASQ_E_ARG, "SILU input needs gate/up");
                if (c->acc_ld[src][0] != P.F_in || c->acc_ld[src][1] != P.F_in) return fail(FASQ_E_SHAPE, "gate/up width != F_in");
                P.x_off = c->acc_off[src][0];
                P.x_ks = c->acc_ks[src][0];
                P.x2_off = c->acc_off[src][1];
                P.x2_ks = c->acc_ks[src][1];
                P.x_sys = steps[src].out_all && world > 1;
                set_scale(src);
            } else if (S.in_mode == IN_ATTN) {
                if (steps[src].kind != SK_ATTN) return fail(FASQ_E_ARG, "ATTN input needs an ATTN step");
                if (c->acc_ld[src][0] != P.F_in) return fail(FASQ_E_SHAPE, "attention width != F_in");
                P.x_off = c->acc_off[src][0];
                P.a_heads = c->attn_heads[src];
                P.a_hd = c->attn_hd[src];
                P.a_parts = model->attn_parts;
            } else {
                if (S.src_layer < 0 || S.src_layer >= (int)c->acc_off[src].size())
                    return fail(FASQ_E_ARG, "input layer out of range");
                if (c->acc_ld[src][S.src_layer] != P.F_in) return fail(FASQ_E_SHAPE, "input width != F_in");
                P.x_off = c->acc_off[src][S.src_layer];
                P.x_ks = c->acc_ks[src][S.src_layer];
                P.x_sys = steps[src].kind == SK_PQ && steps[src].out_all && world > 1;
                if (S.in_mode == IN_RMSNORM) {
                    if (!pair || !S.gamma) return fail(FASQ_E_UNSUPPORTED, "RMSNorm input needs d <= 2 and gamma");
                    P.gamma = S.gamma;
                    P.eps = S.eps;
                    P.nsq_off = c->nsq_off[s];
                    P.nsq_n = ks[0];
                    c->nsq_n[s] = ks[0];
                    c->nsq_F[s] = P.F_in;
                    c->nsq_eps[s] = S.eps;
                    c->nsq_epi[s] = S.scale_epilogue ? 1 : 0;
                    P.epi_scale = S.scale_epilogue ? 1 : 0;
                    if (c->lazy[src] >= 0) {   // h = words + lazy base words
                        P.x2_off = c->acc_off[c->lazy[src]][0];
                        P.x2_ks = c->acc_ks[c->lazy[src]][0];
                        if (steps[c->lazy[src]].kind == SK_PQ && steps[c->lazy[src]].out_all && world > 1) P.x_sys = 1;
                    }
                }
            }
            if (S.in_mode != IN_WORDS && !pair) return fail(FASQ_E_UNSUPPORTED, "input transforms need d <= 2");
        }
        if (S.res_step >= 0) {
            if (!pair) return fail(FASQ_E_UNSUPPORTED, "residual epilogue needs d <= 2");
            if (S.res_step >= s || S.res_layer >= (int)c->acc_off[S.res_step].size())
                return fail(FASQ_E_ARG, "residual must come from an earlier step");
            if (c->acc_ld[S.res_step][S.res_layer] != c->acc_ld[s][0] || nl != 1)
                return fail(FASQ_E_SHAPE, "residual width != output width (single-layer steps only)");
            P.res_off = c->acc_off[S.res_step][S.res_layer];
            P.res_ks = c->acc_ks[S.res_step][S.res_layer];
            P.res_here = S.res_here ? 1 : 0;
            P.res_sys = steps[S.res_step].kind == SK_PQ && steps[S.res_step].out_all && world > 1;
            const int lz = c->lazy[S.res_step];
            if (lz >= 0 && S.res_layer == 0) {
                P.res2_off = c->acc_off[lz][0];
                P.res2_ks = c->acc_ks[lz][0];
                if (steps[lz].kind == SK_PQ && steps[lz].out_all && world > 1) P.res_sys = 1;
            }
        }
        P.out_all = S.out_all && world > 1;
        for (int l = 0; l < nl; ++l) {
            const fasq_layer* L = S.layers[l];
            const int rt = (L->F_out_pad + c->R - 1) / c->R;
            for (int r = 0; r < rt; ++r)
                for (int k = 0; k < ks[l]; ++k) {
                    ChainItem w{};
                    w.kind = SK_PQ;
                    w.idx = L->idx;
                    w.cbimg = L->cbimg;
                    w.cbmap = L->cbmap;
                    w.cbmap_x = mma ? L->cbmap_x : nullptr;
                    w.y_off = c->acc_off[s][l];
                    w.F_out = (int)L->F_out;
                    w.ld = (int)c->acc_ld[s][l];
                    w.row0_g = (S.out_all && !S.kshard) ? (int)(L->F_out * rank) : 0;
                    w.F_out_pad = L->F_out_pad;
                    w.N_ss = L->N_ss;
                    w.C = L->C;
                    w.r0 = r * c->R;
                    w.rows_valid = std::min(c->R, L->F_out_pad - w.r0);
                    w.g_begin = (int)((int64_t)k * L->n_groups / ks[l]);
                    w.g_end = (int)((int64_t)(k + 1) * L->n_groups / ks[l]);
                    w.kidx = k;
                    w.kn = ks[l];
                    // (layer 0, row tile 0) K ranges cover F_in once: they contribute the RMSNorm sum of squares
                    w.nsq = (S.in_mode == IN_RMSNORM && l == 0 && r == 0) ? k : -1;
                    c->gmax = std::max(c->gmax, w.g_end - w.g_begin);
                    per_step[s].push_back(w);
                }
        }
    }
    if (c->ext_F_in == 0 && !model) return fail(FASQ_E_ARG, "the chain needs an external input");
    c->mi = 1;
    for (const auto& v : per_step) c->mi = std::max(c->mi, (int)((v.size() + c->nctas - 1) / c->nctas));
    std::vector<ChainItem> items((size_t)n_steps * c->nctas * c->mi);
    for (auto& w : items) { w = ChainItem{}; w.kind = -1; }
    for (int s = 0; s < n_steps; ++s)
        for (size_t q = 0; q < per_step[s].size(); ++q)
            items[((size_t)s * c->nctas + q % c->nctas) * c->mi + q / c->nctas] = per_step[s][q];
    const size_t xg = (pair && NB == 8 && !mma) ? (size_t)32 * NB * c->d * 4 : (size_t)32 * NB * E;   // k_chain XG
    auto smem_of = [&](int stg) {   // k_chain's layout: rings, x staging, mbarriers, s_sq [nw][NB], scratch
        return cbring(stg) + (size_t)stg * c->R * 32 + (size_t)c->gmax * xg + 16 * (stg + kChainCS) +
               (size_t)c->nw * NB * 4 + kChainScratch;
    };
    while (c->st > 1 && smem_of(c->st) > kChainSmem) --c->st;
    c->smem = smem_of(c->st);
    if (c->smem > kChainSmem) return fail(FASQ_E_UNSUPPORTED, "SMEM plan too large");
    if (getenv("FASQ_CHAIN_VERBOSE"))
        fprintf(stderr, "chain plan: %d steps, %d CTAs, nw=%d st=%d R=%d gmax=%d mi=%d smem=%zu arena_words=%lld\n",
                n_steps, c->nctas, c->nw, c->st, c->R, c->gmax, c->mi, c->smem, (long long)words);
    if (model) {   // attention scratch lives in a 64 KiB pair slot
        for (int s = 0; s < n_steps; ++s)
            if (steps[s].kind == SK_ATTN) {
                // attn_item's scratch after the staged cache rows (the rows fall back to
                // global loads when they do not fit; the scratch must)
                const int Tp = (model->max_T + model->attn_parts - 1) / model->attn_parts + 1;
                const size_t need = B == 1 ? kAttnKV + kAttnScratchFixed + (size_t)(Tp + 4) * 4
                                           : (size_t)attn_batched_scratch(B, Tp);
                if (need > kPairSlot) return fail(FASQ_E_UNSUPPORTED, "attention scratch exceeds a pair slot (max_T)");
            }
    }
    const size_t bytes = ((size_t)words * 2 + kTailWords) * 8;
    // the arena of a tensor-parallel chain is exported with CUDA IPC: a whole
    // cudaMalloc allocation; everything else through the library allocator
    c->arena_ipc = world > 1;
    if (c->arena_ipc) {
        if (cudaMalloc(&c->arenas, bytes) != cudaSuccess) { cudaGetLastError(); return fail(FASQ_E_OOM, ""); }
    } else if (dev_alloc_t(&c->arenas, bytes, st) != FASQ_OK) {
        return fail(FASQ_E_OOM, "");
    }
    if (dev_alloc_t(&c->peers_dev, 8 * sizeof(void*), st) != FASQ_OK ||
        dev_alloc(&c->items, items.size() * sizeof(ChainItem), st) != FASQ_OK ||
        dev_alloc(&c->phases, phases.size() * sizeof(ChainPhase), st) != FASQ_OK)
        return fail(FASQ_E_OOM, "");
    cudaError_t e = cudaMemcpyAsync(c->items, items.data(), items.size() * sizeof(ChainItem), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->phases, phases.data(), phases.size() * sizeof(ChainPhase), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->arenas, 0, bytes, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // host vectors go out of scope
    if (e != cudaSuccess) { fasq_status s = cuda_fail(e, "chain upload"); destroy_chain(c); return s; }
    std::vector<unsigned long long*> bases(world, nullptr);
    bases[rank] = c->arenas;
    fasq_status s = upload_peers(c, bases);
    if (s != FASQ_OK) { destroy_chain(c); return s; }
    c->peers_ready = world == 1;
    *out = c;
    return FASQ_OK;
}

fasq_status chain_launch(fasq_chain* c, const void* x_dev, cudaStream_t st) {
    if (!c->peers_ready) { set_error("chain: world > 1 needs fasq_chain_set_peers first"); return FASQ_E_ARG; }
    ChainParams p{};
    p.items = static_cast<const ChainItem*>(c->items);
    p.phases = static_cast<const ChainPhase*>(c->phases);
    p.x_ext = static_cast<const __half*>(x_dev);
    p.trace = c->trace;
    p.peers = c->peers_dev;
    p.arena_words = c->arena_words;
    p.world = c->world;
    p.rank = c->rank;
    p.pf = 0;
    if (const char* e = getenv("FASQ_CHAIN_PF")) p.pf = atoi(e);
    p.attn_pf = 1;
    if (const char* e = getenv("FASQ_ATTN_PF")) p.attn_pf = atoi(e);
    p.dbg = 0;
    if (const char* e = getenv("FASQ_CHAIN_DBG")) p.dbg = atoi(e);
    p.backoff = 0;
    if (const char* e = getenv("FASQ_CHAIN_BACKOFF")) p.backoff = atoi(e);
    p.n_steps = c->n_steps;
    p.nctas = c->nctas;
    p.B = c->B;
    p.gmax = c->gmax;
    p.mi = c->mi;
    p.cbb_max = c->maxC * 32 * entry_bytes(c->d);
    if (c->has_model) {
        p.model = 1;
        p.rope = c->model.rope;
        p.max_T = c->model.max_T;
        p.pos_wrap = c->model.pos_wrap;
        p.tok_hist = c->model.tok_hist;
        p.tok_expect = c->model.tok_expect;
    }
    switch (c->B <= 1 ? 1 : c->B <= 2 ? 2 : c->B <= 4 ? 4 : 8) {
        case 1: return chain_dispatch<1>(c, p, st);
        case 2: return chain_dispatch<2>(c, p, st);
        case 4: return chain_dispatch<4>(c, p, st);
        default: return chain_dispatch<8>(c, p, st);
    }
}

fasq_status chain_output(const fasq_chain* c, int step, int layer, void* y_dev, fasq_dtype dtype, cudaStream_t st) {
    if (step < 0 || step >= c->n_steps) return FASQ_E_ARG;
    if (layer < 0 || layer >= (int)c->acc_off[step].size()) return FASQ_E_ARG;
    if (dtype != FASQ_F16 && dtype != FASQ_F32 && dtype != FASQ_ACC_I64) return FASQ_E_ARG;
    const int64_t n = (int64_t)c->B * c->acc_ld[step][layer];
    if (n <= 0) return FASQ_OK;
    if (c->kinds[step] == SK_ATTN) {
        k_attn_convert<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(c->arenas, c->arena_words, c->nctas,
                                                                     c->acc_off[step][0], c->B, c->attn_heads[step],
                                                                     c->attn_hd[step], c->model.attn_parts, y_dev,
                                                                     (int)dtype);
        FASQ_CUDA_TRY(cudaGetLastError());
        return FASQ_OK;
    }
    const int lz = layer == 0 ? c->lazy[step] : -1;
    const long long off2 = lz >= 0 ? c->acc_off[lz][0] : -1;
    const int ks2 = lz >= 0 ? c->acc_ks[lz][0] : 0;
    const long long sc_off = c->nsq_epi[step] ? -1 : c->nsq_off[step];
    k_counted_convert<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        c->arenas, c->arena_words, c->nctas, c->acc_off[step][layer], n, c->acc_ks[step][layer], y_dev, (int)dtype,
        c->world > 1, off2, ks2, sc_off, c->nsq_n[step], c->nsq_F[step], c->nsq_eps[step], c->acc_ld[step][layer]);
    FASQ_CUDA_TRY(cudaGetLastError());
    return FASQ_OK;
}

void chain_destroy(fasq_chain* c) { destroy_chain(c); }

}  // namespace fasq

using namespace fasq;

extern "C" {

fasq_status fasq_chain_create_tp(const fasq_chain_step* steps, int32_t n_steps, int32_t B, int32_t world,
                                 int32_t rank, int32_t max_ctas, void* stream, fasq_chain** out) {
    if (!out) return FASQ_E_ARG;
    *out = nullptr;
    if (!steps || n_steps < 1) return FASQ_E_ARG;
    std::vector<StepDesc> v(n_steps);
    for (int s = 0; s < n_steps; ++s) {
        const fasq_chain_step& S = steps[s];
        if (!S.layers || S.n_layers < 1 || S.n_layers > 4) return FASQ_E_ARG;
        v[s].kind = SK_PQ;
        v[s].layers.assign(S.layers, S.layers + S.n_layers);
        for (const fasq_layer* L : v[s].layers)
            if (!L) return FASQ_E_ARG;
        if (S.input_step < 0) {
            v[s].in_mode = IN_EXT;
        } else {
            if (S.input_step >= s) return FASQ_E_ARG;
            v[s].in_mode = IN_WORDS;
            v[s].src_step = S.input_step;
            v[s].src_layer = S.input_layer;
        }
        v[s].out_all = world > 1;   // row shards, gathered into every rank's arena
    }
    // deterministic TP (default): K ranges of the unsharded plan -> sharded
    // outputs bit-identical to one GPU; FASQ_CHAIN_FAST=1 plans per rank
    const bool det = getenv("FASQ_CHAIN_FAST") == nullptr;
    return chain_build(v, B, world, rank, max_ctas, det, nullptr, (cudaStream_t)stream, out);
}

fasq_status fasq_chain_create(const fasq_chain_step* steps, int32_t n_steps, int32_t B, void* stream,
                              fasq_chain** out) {
    return fasq_chain_create_tp(steps, n_steps, B, 1, 0, 0, stream, out);
}

fasq_status fasq_chain_ipc_handle(const fasq_chain* c, void* handle_out) {
    if (!c || !handle_out) return FASQ_E_ARG;
    cudaIpcMemHandle_t h;
    FASQ_CUDA_TRY(cudaIpcGetMemHandle(&h, c->arenas));
    std::memcpy(handle_out, &h, sizeof(h));
    return FASQ_OK;
}

fasq_status fasq_chain_set_peers(fasq_chain* c, const void* handles) {
    if (!c || !handles) return FASQ_E_ARG;
    std::vector<unsigned long long*> bases(c->world, nullptr);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) { bases[r] = c->arenas; continue; }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)r * sizeof(h), sizeof(h));
        void* q = nullptr;
        FASQ_CUDA_TRY(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(q);
        bases[r] = static_cast<unsigned long long*>(q);
    }
    return upload_peers(c, bases);
}

fasq_status fasq_chain_set_peer_chains(fasq_chain* c, const fasq_chain* const* chains) {
    if (!c || !chains) return FASQ_E_ARG;
    std::vector<unsigned long long*> bases(c->world, nullptr);
    for (int r = 0; r < c->world; ++r) {
        const fasq_chain* o = chains[r];
        if (!o || o->world != c->world || o->arena_words != c->arena_words || o->n_steps != c->n_steps)
            return FASQ_E_ARG;
        bases[r] = o->arenas;
    }
    if (bases[c->rank] != c->arenas) return FASQ_E_ARG;
    return upload_peers(c, bases);
}

fasq_status fasq_chain_run(fasq_chain* c, const void* x_dev, void* stream) {
    if (!c || !x_dev) return FASQ_E_ARG;
    fasq_status s = chain_launch(c, x_dev, (cudaStream_t)stream);
    if (s == FASQ_OK) set_launch_count(1);
    return s;
}

fasq_status fasq_chain_run_host(fasq_chain* c, const void* x_host, void* y_host, int32_t step, int32_t layer,
                                fasq_dtype dtype, void* stream) {
    if (!c || !x_host || !y_host) return FASQ_E_ARG;
    if (step < 0 || step >= c->n_steps || layer < 0 || layer >= (int)c->acc_off[step].size()) return FASQ_E_ARG;
    if (dtype != FASQ_F16 && dtype != FASQ_F32) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t xb = (size_t)c->B * c->ext_F_in * 2;
    const size_t yb = (size_t)c->B * c->acc_ld[step][layer] * (dtype == FASQ_F32 ? 4 : 2);
    void *xd = nullptr, *yd = nullptr;
    if (dev_alloc(&xd, xb, st) != FASQ_OK || dev_alloc(&yd, yb, st) != FASQ_OK) {
        dev_free(xd, st);
        return FASQ_E_OOM;
    }
    fasq_status s = FASQ_OK;
    cudaError_t e = cudaMemcpyAsync(xd, x_host, xb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) s = cuda_fail(e, "H2D x");
    if (s == FASQ_OK) s = chain_launch(c, xd, st);
    if (s == FASQ_OK) s = chain_output(c, step, layer, yd, dtype, st);
    if (s == FASQ_OK) {
        e = cudaMemcpyAsync(y_host, yd, yb, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = cuda_fail(e, "D2H y");
    }
    dev_free(xd, st);
    dev_free(yd, st);
    e = cudaStreamSynchronize(st);
    if (s == FASQ_OK && e != cudaSuccess) s = cuda_fail(e, "chain_run_host sync");
    if (s == FASQ_OK) set_launch_count(2);
    return s;
}

fasq_status fasq_chain_output(const fasq_chain* c, int32_t step, int32_t layer, void* y_dev, fasq_dtype dtype,
                              void* stream) {
    if (!c || !y_dev) return FASQ_E_ARG;
    fasq_status s = chain_output(c, step, layer, y_dev, dtype, (cudaStream_t)stream);
    if (s == FASQ_OK) set_launch_count(1);
    return s;
}

fasq_status fasq_chain_check(fasq_chain* c, void* stream) {
    if (!c) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long f = 0;
    FASQ_CUDA_TRY(cudaMemcpyAsync(&f, c->tail() + T_OVF, 8, cudaMemcpyDeviceToHost, st));
    FASQ_CUDA_TRY(cudaStreamSynchronize(st));
    if (f) {
        FASQ_CUDA_TRY(cudaMemsetAsync(c->tail() + T_OVF, 0, 8, st));
        FASQ_CUDA_TRY(cudaStreamSynchronize(st));
        set_error("chain: a counted partial exceeded |v| < 2^18 (outputs of that run are NaN)");
        return FASQ_E_RANGE;
    }
    return FASQ_OK;
}

int32_t fasq_chain_plan_ks(const int64_t* F_out, const int64_t* n_groups, int32_t n, int32_t nctas, int32_t d,
                           int32_t B, int32_t* ks_out) {
    if (!F_out || !n_groups || !ks_out || n < 1 || nctas < 1) return FASQ_E_ARG;
    std::vector<int64_t> fop(n);
    std::vector<int> ngr(n);
    for (int i = 0; i < n; ++i) {
        fop[i] = (F_out[i] + kRowBlock - 1) / kRowBlock * kRowBlock;
        ngr[i] = (int)n_groups[i];
    }
    std::vector<int> ks = plan_step_ks(fop, ngr, nctas, chain_rows_per_cta(d, B, 16), false);
    for (int i = 0; i < n; ++i) ks_out[i] = ks[i];
    return FASQ_OK;
}

fasq_status fasq_chain_trace(fasq_chain* c, void* trace_dev) {
    if (!c) return FASQ_E_ARG;
    c->trace = static_cast<unsigned long long*>(trace_dev);
    return FASQ_OK;
}

int32_t fasq_chain_ctas(const fasq_chain* c) { return c ? c->nctas : -1; }

void fasq_chain_free(fasq_chain* c) {
    if (!c) return;
    cudaDeviceSynchronize();
    destroy_chain(c);
}

}  // extern "C"
