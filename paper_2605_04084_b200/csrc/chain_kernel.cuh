// chain_kernel.cuh -- device side of the persistent decode-chain executor
// (sm_100a): work-item / phase descriptors, the step kinds' device code and
// the k_chain kernel template.  Instantiated per batch width in
// chain_k{1,2,4,8}.cu (parallel compilation); the host planner is chain.cu.
// See chain.cu for the design.
#pragma once
#include <cmath>
#include <mutex>
#include <string>

#include "chain_internal.cuh"
#include "gemv_core.cuh"

#ifndef FASQ_CHAIN_NO_MMA
#define FASQ_CHAIN_NO_MMA 0   // 1: batched decode on the FHFMA/FFMA2 row-set path (A/B experiments)
#endif

namespace fasq {
namespace chainimpl {

// Work item of one CTA in one step.  The consumer fields come first (loaded
// by value at the item start, next to the phase); the epilogue fields are
// re-read through the item pointer after the gather loop (same 128-B line,
// an L1 hit) instead of occupying registers across it.
struct alignas(128) ChainItem {
    int kind;                   // SK_* ; -1: no item
    int g_begin, g_end, rows_valid;
    int N_ss, r0, kidx, head;   // kidx: PQ K-range index in its row tile (0 adds the residual); ATTN: cache part
    int nsq;                    // PQ: RMSNorm sum-of-squares slot this item contributes (-1: none)
    int kn;                     // PQ: K ranges of this item's row tile (the residual of warp w's rows
                                //     is added by the range kidx == w % kn)
    int F_out, ld, row0_g;      // local rows, words per batch row of the output, output index of local row 0
    long long y_off;            // word offset of the output [B][ld] in a buffer
    // producer
    const uint8_t* idx;
    const uint8_t* cbimg;
    const void* cbmap;          // d <= 2: 3-D tensor map {32 words, n_groups, C} over cbimg (pair boxes)
    const void* cbmap_x;        // d = 2, B >= 4: the same over the XOR image cbimg_x (tensor-core path)
    int F_out_pad, C;
};

// Per-step description.  The PQ fields fill the first 128-B line.
struct alignas(128) ChainPhase {
    int kind, in_mode, F_in, x_ks;
    long long x_off, x2_off;    // input words (WORDS/NORM/ATTN: x; SILU: gate x, up x2; NORM: x2 = lazy base, < 0: none)
    int x2_ks, x_sys, res_ks, res_here;   // x_sys: input words written by peers (system-scope polls)
    const __half* gamma;        // IN_RMSNORM
    long long res_off;          // residual words (< 0: none), same [B][ld] indexing as the output
    long long nsq_off;          // IN_RMSNORM: sum-of-squares slots [B][64]
    int nsq_n, res_sys, out_all, a_heads;   // out_all: outputs red.add'ed into every rank's arena
    float eps;
    int a_hd, a_parts;          // IN_ATTN: layout of the source attention partials
    long long res2_off;         // lazy base of the residual (< 0: none)
    int res2_ks;
    int sc_n;                   // SILU input / ATTN: RMSNorm scale of the source step, from its
    long long sc_off;           //   sum-of-squares slots (sc_off < 0: none)
    int sc_F;
    float sc_eps;
    int epi_scale;              // IN_RMSNORM: the scale is applied in this step's epilogue
    // ATTN
    long long q_off, k_off, v_off, o_off;
    int q_ks, k_ks, v_ks, q_ld, kv_ld;
    __half* kc;
    __half* vc;
    int n_heads, n_kv, hd, parts;
    // EMBED
    const __half* embed;
    long long e_off;
    int hidden;
};

// Epilogue parameters of the current item, kept in SMEM (one copy per CTA)
// rather than in 512 threads' registers across the gather loop: with 227 KiB
// of SMEM the L1 left for register spills is small, and spills in the loop
// cost more than the loop saves.
struct EpiParams {
    long long y_off, res_off, res2_off, nsq_off;
    int row0_g, ld, F_out, r0;
    int add_res, res_ks, res_sys, out_all;
    int kidx, kn;
    int res2_ks, epi_scale, nsq_n, F_in;
    float eps;
    int pad;
};

struct ChainParams {
    const ChainItem* items;
    const ChainPhase* phases;
    const __half* x_ext;        // [B][F_in of the first step]
    unsigned long long* trace;  // optional [n_steps][nctas][4] globaltimer stamps (fasq_chain_trace)
    unsigned long long* const* peers;   // [world] allocation bases (2 buffers + tail each); peers[rank] = local
    long long arena_words;      // words per buffer
    int world, rank;
    int n_steps, nctas, B, gmax, cbb_max;
    int mi;                     // work items per (step, CTA): [n_steps][nctas][mi]
    int pf;                     // producer: L2-prefetch this many groups of the next step's item
    int attn_pf;                // producer: L2-prefetch the next attention item's cache rows (FASQ_ATTN_PF, default 1)
    int backoff;                // ns slept between input polls (FASQ_CHAIN_BACKOFF, default 0)
    int dbg;                    // experiments only (FASQ_CHAIN_DBG): bit 0 = consumers skip the gather
                                // loop, bit 1 = producer skips the copies (compute on stale SMEM),
                                // bit 2 = producer skips the codebook copies only
    // model (llama.cu)
    int model;
    const float2* rope;
    int max_T, pos_wrap;
    int* tok_hist;
    long long tok_expect;
};

template <int D>
struct ChainPair {
    static constexpr bool value = D <= 2;
};
constexpr int kChainCS = kPairSlots;
// ATTN items: a codebook pair slot (64 KiB) holds the item's K/V cache rows
// (prefetched by the producer warp while earlier steps run) in its first
// kAttnKV bytes and the attention scratch after them.
constexpr uint32_t kAttnKV = 40 * 1024;
constexpr uint32_t kAttnScratchFixed = 5 * 128 * 4 + 4 * 128 * 4 + 64;   // q, k, v, q', k/v new, o row groups, m/l

__device__ __forceinline__ void consumer_bar(int nt) { asm volatile("bar.sync 1, %0;" :: "r"(nt) : "memory"); }

__device__ __forceinline__ unsigned long long cnt_word(long long v) {
    return (1ull << core::kCntShift) + (unsigned long long)(core::kCntBias + v);
}
// A single-contributor counted word carrying fp32 bits (count 1).
__device__ __forceinline__ unsigned long long f32_word(float f) {
    return (1ull << core::kCntShift) | (unsigned long long)__float_as_uint(f);
}
__device__ __forceinline__ float word_f32(unsigned long long v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
__device__ __forceinline__ void st_word(unsigned long long* a, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_word(const unsigned long long* a, bool sys) {
    unsigned long long v;
    if (sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}

// Cache rows [t0, t1) of part `part` of P over Tn = pos + 1 positions, and the
// rows [t0, te) (te = min(t1, pos)) that already sit in the cache; whether they
// are staged in SMEM (same decision on the producer and the consumer side).
struct AttnRows {
    int t0, t1, te;
    bool smem;
};
__device__ __forceinline__ AttnRows attn_rows(int part, int P, int pos, int B, int hd) {
    AttnRows r;
    const int Tn = pos + 1;
    r.t0 = (int)((long long)part * Tn / P);
    r.t1 = (int)((long long)(part + 1) * Tn / P);
    r.te = min(r.t1, pos);
    const long long kv = (long long)B * max(0, r.te - r.t0) * hd * 4;
    r.smem = B == 1 && r.te > r.t0 && kv <= (long long)kAttnKV &&
             kAttnKV + kAttnScratchFixed + (uint32_t)(r.t1 - r.t0 + 4) * 4u <= kPairSlot;
    return r;
}

// ---- EMBED: h0[b] = embed[token_b] as counted words (count 1) ---------------
// token_b = the key the previous run's lm_head red.max'ed into token slot
// (par_prev, b), once all its contributions arrived; the slot is cleared for
// the run after next and the token is appended to the history.
__device__ __forceinline__ void embed_item(const ChainPhase* ph, unsigned long long* cur, unsigned long long* tail,
                                        int B, unsigned run, int pos, int max_T, int* tok_hist,
                                        long long tok_expect, int NT, int* s_tok) {
    const int tid = threadIdx.x;
    const unsigned pp = (run - 1u) & 1u;
    if (tid < B) {
        unsigned long long* slot = tail + T_TOK + (pp * 8 + tid) * 2;
        unsigned long long cnt;
        const unsigned long long t0 = dev::globaltimer();
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(cnt) : "l"(slot + 1) : "memory");
            if (dev::globaltimer() - t0 > 4000000000ull) __trap();
        } while ((long long)cnt != tok_expect);
        unsigned long long key;
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(key) : "l"(slot) : "memory");
        const unsigned tok = tok_of_key(key);
        s_tok[tid] = (int)tok;
        tok_hist[(size_t)tid * max_T + pos] = (int)tok;
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(slot), "l"(0ull) : "memory");
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(slot + 1), "l"(0ull) : "memory");
    }
    consumer_bar(NT);
    // 8 rows' loads in flight per thread (a load -> store chain per element
    // serialised one HBM round trip per iteration: 7 us at B = 1, 38 us at B = 8)
    const int n = ph->hidden;
    constexpr int U = 8;
    for (int i0 = tid; i0 < B * n; i0 += NT * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * NT;
            v[u] = 0.f;
            if (i < B * n) {
                const int b = i / n, c = i - b * n;
                v[u] = __half2float(ph->embed[(size_t)s_tok[b] * n + c]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * NT;
            if (i < B * n) st_word(cur + ph->e_off + i, cnt_word(__float2ll_rn(v[u] * core::kAccScale)));
        }
    }
}

// RMSNorm scale s[b] = 1/sqrt(sum_k slot[b][k] / n + eps) from the n_slots
// sum-of-squares slots of a norm step; every warp computes it the same way
// (lane k and k + 32, xor tree) -> identical in every warp and CTA.
template <int NB>
__device__ __forceinline__ void warp_norm_scale(float (&sc)[NB], const unsigned long long* slots, int n_slots, int n,
                                                float eps, int B, int lane) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        float a = 0.f;
        if (b < B) {
            // both slots of this lane in flight, then the checks
            unsigned long long v0 = 0ull, v1 = 0ull;   // count 0: not yet loaded
            const bool h0 = lane < n_slots, h1 = lane + 32 < n_slots;
            const unsigned long long t0 = dev::globaltimer();
            for (bool done = false; !done;) {
                if (h0 && (v0 >> core::kCntShift) != 1ull) v0 = ld_word(slots + b * 64 + lane, false);
                if (h1 && (v1 >> core::kCntShift) != 1ull) v1 = ld_word(slots + b * 64 + lane + 32, false);
                done = (!h0 || (v0 >> core::kCntShift) == 1ull) && (!h1 || (v1 >> core::kCntShift) == 1ull);
                if (!done && dev::globaltimer() - t0 > 4000000000ull) __trap();
            }
            if (h0) a += word_f32(v0);
            if (h1) a += word_f32(v1);
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
        sc[b] = 1.0f / sqrtf(a / (float)n + eps);
    }
}

// MODEL: the whole-model step kinds and input transforms (EMBED, ATTN,
// RMSNorm / SwiGLU / attention inputs, residual epilogue) are compiled in;
// plain GEMV chains use the MODEL = false instance (fewer live registers in
// the gather loop: the kernel runs at the 96-register cap of 17 warps).
// ---- ATTN: one (local q head, cache part) item ------------------------------
// Llama attention for the token at `pos` (HF LlamaAttention semantics):
// RoPE (rotate-half, cos/sin table) on q and k, the new fp16 k/v appended to
// the KV cache at pos (by the first q head of each KV group, last part),
// scores q.k_t / sqrt(hd) over t <= pos, softmax, o = sum_t p_t v_t.  The
// cache length is split into `parts` ranges over CTAs; each writes its
// unnormalised partial o, max m and sum l (fp32 bits in counted words); the
// consumer (the o projection's x staging, stage_x_attn) merges the parts in
// FIXED order -- no merge round trip here.  slot: a 64 KiB codebook pair slot
// handed over by the producer, holding this item's cache rows [t0, te) for
// every token b (K [B][nk][hd] then V) when r.smem.
__device__ __forceinline__ void attn_item(const ChainPhase* ph, int head, int part, unsigned long long* cur, int B,
                                       int pos, int max_T, const float2* rope, uint8_t* slot, int NT) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int hd = ph->hd, half = hd / 2;
    const int n_heads = ph->n_heads, n_kv = ph->n_kv, P = ph->parts;
    const int grp = n_heads / n_kv, kvh = head / grp;
    const AttnRows r = attn_rows(part, P, pos, B, hd);
    const int nrow = r.t1 - r.t0, nk = max(0, r.te - r.t0);
    const float qk_scale = 1.0f / sqrtf((float)hd);
    // RoPE table row of this position (independent of q/k/v: loaded first)
    const float2 cs = tid < half ? rope[(size_t)pos * half + tid] : make_float2(0.f, 0.f);
    float* s_q = reinterpret_cast<float*>(slot + kAttnKV);   // [128] raw q
    float* s_k = s_q + 128;                                  // [128] raw k
    float* s_v = s_k + 128;                                  // [128] raw v
    float* s_qr = s_v + 128;                                 // [128] rotated q
    __half* s_kn = reinterpret_cast<__half*>(s_qr + 128);    // [128] new k (rotated, fp16)
    __half* s_vn = s_kn + 128;                               // [128] new v (fp16)
    float* s_o = reinterpret_cast<float*>(s_vn + 128);       // [4][128] row-group partials of o
    float* s_ml = s_o + 4 * 128;                             // [2] m, l  (+ pad)
    float* s_sc = s_ml + 16;                                 // [nrow] scores / probabilities
    const __half* kv_k = reinterpret_cast<const __half*>(slot);
    const __half* kv_v = kv_k + (size_t)B * nk * hd;
    unsigned long long* out_base = cur + ph->o_off + (size_t)head * P * (hd + 2) + (size_t)part * (hd + 2);
    const size_t out_bstride = (size_t)n_heads * P * (hd + 2);
    for (int b = 0; b < B; ++b) {
        unsigned long long* ob = out_base + (size_t)b * out_bstride;
        if (nrow <= 0) {   // empty part (Tn < parts): contributes nothing
            if (tid < hd) st_word(ob + tid, f32_word(0.f));
            if (tid == 0) st_word(ob + hd, f32_word(-INFINITY));
            consumer_bar(NT);
            if (tid == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(ob + hd + 1), "l"(f32_word(0.f)) : "memory");
            }
            continue;
        }
        // 1. q (this head), k and v (its KV head) from the counted words
        if (tid < 3 * hd) {
            const int which = tid / hd, e = tid - which * hd;
            const unsigned long long* a =
                which == 0 ? cur + ph->q_off + (size_t)b * ph->q_ld + (size_t)head * hd + e
                           : cur + (which == 1 ? ph->k_off : ph->v_off) + (size_t)b * ph->kv_ld + (size_t)kvh * hd + e;
            const int ks = which == 0 ? ph->q_ks : which == 1 ? ph->k_ks : ph->v_ks;
            const float f = (float)((double)core::poll_value(a, ks, false) * core::kAccInv);
            (which == 0 ? s_q : which == 1 ? s_k : s_v)[e] = f;
        } else if (warp == NT / 32 - 1) {
            // the q/k/v words hold the products of the UNSCALED normed input
            // (chain_internal.cuh): the last warp (idle above, 3 hd <= NT - 32)
            // computes the qkv step's RMSNorm scale of token b meanwhile
            float sc[1] = {1.f};
            if (ph->sc_off >= 0)
                warp_norm_scale<1>(sc, cur + ph->sc_off + (size_t)b * 64, ph->sc_n, ph->sc_F, ph->sc_eps, 1, lane);
            if (lane == 0) s_ml[2] = sc[0];
        }
        consumer_bar(NT);
        const float sb = s_ml[2];
        // 2. RoPE (rotate half): x'[i] = x[i] c - x[i+half] s, x'[i+half] = x[i+half] c + x[i] s
        __half* kc = ph->kc + ((size_t)b * n_kv + kvh) * (size_t)max_T * hd;
        __half* vc = ph->vc + ((size_t)b * n_kv + kvh) * (size_t)max_T * hd;
        const bool writer = head % grp == 0 && r.t1 == pos + 1;   // one cache writer per KV head
        if (tid < half) {
            const float q0 = s_q[tid] * sb, q1 = s_q[tid + half] * sb, k0 = s_k[tid] * sb, k1 = s_k[tid + half] * sb;
            s_qr[tid] = q0 * cs.x - q1 * cs.y;
            s_qr[tid + half] = q1 * cs.x + q0 * cs.y;
            const __half kn0 = __float2half_rn(k0 * cs.x - k1 * cs.y), kn1 = __float2half_rn(k1 * cs.x + k0 * cs.y);
            s_kn[tid] = kn0;
            s_kn[tid + half] = kn1;
            if (writer) { kc[(size_t)pos * hd + tid] = kn0; kc[(size_t)pos * hd + tid + half] = kn1; }
        } else if (tid < half + hd) {
            const int e = tid - half;
            const __half vn = __float2half_rn(s_v[e] * sb);
            s_vn[e] = vn;
            if (writer) vc[(size_t)pos * hd + e] = vn;
        }
        consumer_bar(NT);
        // 3. scores: 16 lanes per row (8 dims each), NT/16 rows per pass
        {
            const int nch = hd / 8;
            const int c = tid & 15, rr = tid >> 4, rpi = NT / 16;
            float qv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) qv[i] = c < nch ? s_qr[c * 8 + i] : 0.f;
            for (int base = 0; base < nrow; base += rpi) {
                const int t = r.t0 + base + rr;
                uint4 kv = make_uint4(0u, 0u, 0u, 0u);
                if (c < nch && t < r.t1) {
                    if (t == pos) kv = *reinterpret_cast<const uint4*>(s_kn + c * 8);
                    else if (r.smem) kv = *reinterpret_cast<const uint4*>(kv_k + ((size_t)b * nk + (t - r.t0)) * hd + c * 8);
                    else kv = __ldcg(reinterpret_cast<const uint4*>(kc + (size_t)t * hd + c * 8));
                }
                const __half* kh = reinterpret_cast<const __half*>(&kv);
                float dsum = 0.f;
#pragma unroll
                for (int i = 0; i < 8; ++i) dsum += qv[i] * __half2float(kh[i]);
#pragma unroll
                for (int m = 8; m >= 1; m >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, m);
                if (c == 0 && t < r.t1) s_sc[t - r.t0] = dsum * qk_scale;
            }
        }
        consumer_bar(NT);
        // 4. softmax statistics (warp 0; fixed order: strided per lane, xor tree)
        if (warp == 0) {
            float mx = -INFINITY;
            for (int i = lane; i < nrow; i += 32) mx = fmaxf(mx, s_sc[i]);
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
            float sm = 0.f;
            for (int i = lane; i < nrow; i += 32) {
                const float pe = expf(s_sc[i] - mx);
                s_sc[i] = pe;
                sm += pe;
            }
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, m);
            if (lane == 0) { s_ml[0] = mx; s_ml[1] = sm; }
        }
        consumer_bar(NT);
        // 5. o partial: thread (dim, row group) sums p_t v_t[dim] over its rows
        {
            const int rgs = min(NT / hd, 4);       // row groups (4 at hd >= 128 with 512 threads)
            const int dim = tid % hd, rg = tid / hd;
            float o = 0.f;
            if (rg < rgs) {
                for (int t = r.t0 + rg; t < r.t1; t += rgs) {
                    __half vh;
                    if (t == pos) vh = s_vn[dim];
                    else if (r.smem) vh = kv_v[((size_t)b * nk + (t - r.t0)) * hd + dim];
                    else vh = __ldcg(vc + (size_t)t * hd + dim);
                    o += s_sc[t - r.t0] * __half2float(vh);
                }
                s_o[rg * 128 + dim] = o;
            }
            consumer_bar(NT);
            if (tid < hd) {
                float od = 0.f;
                for (int g = 0; g < rgs; ++g) od += s_o[g * 128 + tid];
                st_word(ob + tid, f32_word(od));
            }
            if (tid == 0) st_word(ob + hd, f32_word(s_ml[0]));
        }
        consumer_bar(NT);
        if (tid == 0) {   // l last, with release (cumulative over the barrier): a reader that sees l final sees o and m
            asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(ob + hd + 1), "l"(f32_word(s_ml[1])) : "memory");
        }
    }
}

// ---- ATTN, B > 1: all tokens of a (q head, cache part) item at once --------
// Same arithmetic as attn_item, per token b, but every phase covers all B
// tokens (5 CTA barriers per item instead of 5 per token): the loop over b
// cost ~9 us per token at B = 8.  The cache rows of B sequences do not fit
// the SMEM prefetch, so they come from L2 (the producer warms them); the whole
// 64 KiB pair slot is scratch: q, k, v, q' [B][128] fp32, k/v new [B][128]
// fp16, scores [B][rows], o row-group partials [4][B][128], (m, l, s) [B].
constexpr uint32_t attn_batched_scratch(int B, int rows) {
    return (uint32_t)B * (4 * 128 * 4 + 2 * 128 * 2 + 4 * 128 * 4 + 16) + (uint32_t)B * (rows + 4) * 4;
}

__device__ __forceinline__ void attn_item_batched(const ChainPhase* ph, int head, int part, unsigned long long* cur,
                                                  int B, int pos, int max_T, const float2* rope, uint8_t* slot,
                                                  int NT) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int hd = ph->hd, half = hd / 2;
    const int n_heads = ph->n_heads, n_kv = ph->n_kv, P = ph->parts;
    const int grp = n_heads / n_kv, kvh = head / grp;
    const AttnRows r = attn_rows(part, P, pos, B, hd);
    const int nrow = r.t1 - r.t0;
    const float qk_scale = 1.0f / sqrtf((float)hd);
    float* s_q = reinterpret_cast<float*>(slot);             // [B][128]
    float* s_k = s_q + B * 128;
    float* s_v = s_k + B * 128;
    float* s_qr = s_v + B * 128;
    __half* s_kn = reinterpret_cast<__half*>(s_qr + B * 128);   // [B][128]
    __half* s_vn = s_kn + B * 128;
    float* s_o = reinterpret_cast<float*>(s_vn + B * 128);      // [4][B][128]
    float* s_ml = s_o + 4 * B * 128;                            // [B][4]: m, l, scale
    float* s_sc = s_ml + 4 * B;                                 // [B][nrow + 4]
    const int scw = nrow + 4;
    const size_t out_bstride = (size_t)n_heads * P * (hd + 2);
    unsigned long long* out_base = cur + ph->o_off + (size_t)head * P * (hd + 2) + (size_t)part * (hd + 2);
    if (nrow <= 0) {
        for (int i = tid; i < B * hd; i += NT) st_word(out_base + (size_t)(i / hd) * out_bstride + i % hd, f32_word(0.f));
        if (tid < B) st_word(out_base + (size_t)tid * out_bstride + hd, f32_word(-INFINITY));
        consumer_bar(NT);
        if (tid < B)
            asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(out_base + (size_t)tid * out_bstride + hd + 1),
                         "l"(f32_word(0.f)) : "memory");
        return;
    }
    // 0. the qkv step's RMSNorm scale of every token: warp b (idle in phase 1's tail)
    if (warp < B) {
        float sc[1] = {1.f};
        if (ph->sc_off >= 0)
            warp_norm_scale<1>(sc, cur + ph->sc_off + (size_t)warp * 64, ph->sc_n, ph->sc_F, ph->sc_eps, 1, lane);
        if (lane == 0) s_ml[warp * 4 + 2] = sc[0];
    }
    // 1. q (this head), k, v (its KV head) of every token, all in flight
    for (int i = tid; i < B * 3 * hd; i += NT) {
        const int b = i / (3 * hd), rem = i - b * 3 * hd, which = rem / hd, e = rem - which * hd;
        const unsigned long long* a =
            which == 0 ? cur + ph->q_off + (size_t)b * ph->q_ld + (size_t)head * hd + e
                       : cur + (which == 1 ? ph->k_off : ph->v_off) + (size_t)b * ph->kv_ld + (size_t)kvh * hd + e;
        const int ks = which == 0 ? ph->q_ks : which == 1 ? ph->k_ks : ph->v_ks;
        (which == 0 ? s_q : which == 1 ? s_k : s_v)[b * 128 + e] = (float)((double)core::poll_value(a, ks, false) * core::kAccInv);
    }
    consumer_bar(NT);
    // 2. RoPE, new k/v (fp16), cache append (one writer per KV head, last part)
    const bool writer = head % grp == 0 && r.t1 == pos + 1;
    for (int i = tid; i < B * hd; i += NT) {
        const int b = i / hd, e = i - b * hd;
        const float sb = s_ml[b * 4 + 2];
        __half* kc = ph->kc + ((size_t)b * n_kv + kvh) * (size_t)max_T * hd;
        __half* vc = ph->vc + ((size_t)b * n_kv + kvh) * (size_t)max_T * hd;
        if (e < half) {
            const float2 cs = rope[(size_t)pos * half + e];
            const float q0 = s_q[b * 128 + e] * sb, q1 = s_q[b * 128 + e + half] * sb;
            const float k0 = s_k[b * 128 + e] * sb, k1 = s_k[b * 128 + e + half] * sb;
            s_qr[b * 128 + e] = q0 * cs.x - q1 * cs.y;
            s_qr[b * 128 + e + half] = q1 * cs.x + q0 * cs.y;
            const __half kn0 = __float2half_rn(k0 * cs.x - k1 * cs.y), kn1 = __float2half_rn(k1 * cs.x + k0 * cs.y);
            s_kn[b * 128 + e] = kn0;
            s_kn[b * 128 + e + half] = kn1;
            if (writer) { kc[(size_t)pos * hd + e] = kn0; kc[(size_t)pos * hd + e + half] = kn1; }
        }
        const __half vn = __float2half_rn(s_v[b * 128 + e] * sb);
        s_vn[b * 128 + e] = vn;
        if (writer) vc[(size_t)pos * hd + e] = vn;
    }
    consumer_bar(NT);
    // 3. scores of every (token, row): 16 lanes per pair, 4 pairs in flight per lane group
    {
        const int nch = hd / 8;
        const int c = tid & 15, gi = tid >> 4, ngr = NT / 16;
        const int npair = B * nrow;
        for (int base = gi; base < npair; base += 4 * ngr) {
            uint4 kv[4];
            float qv[4][8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int pr = base + u * ngr;
                kv[u] = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (int i2 = 0; i2 < 8; ++i2) qv[u][i2] = 0.f;
                if (pr < npair && c < nch) {
                    const int b = pr / nrow, t = r.t0 + pr - b * nrow;
                    const __half* kc = ph->kc + ((size_t)b * n_kv + kvh) * (size_t)max_T * hd;
                    kv[u] = t == pos ? *reinterpret_cast<const uint4*>(s_kn + b * 128 + c * 8)
                                     : __ldcg(reinterpret_cast<const uint4*>(kc + (size_t)t * hd + c * 8));
#pragma unroll
                    for (int i2 = 0; i2 < 8; ++i2) qv[u][i2] = s_qr[b * 128 + c * 8 + i2];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int pr = base + u * ngr;
                const __half* kh = reinterpret_cast<const __half*>(&kv[u]);
                float dsum = 0.f;
#pragma unroll
                for (int i2 = 0; i2 < 8; ++i2) dsum += qv[u][i2] * __half2float(kh[i2]);
#pragma unroll
                for (int m = 8; m >= 1; m >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, m);
                if (c == 0 && pr < npair) {
                    const int b = pr / nrow;
                    s_sc[b * scw + pr - b * nrow] = dsum * qk_scale;
                }
            }
        }
    }
    consumer_bar(NT);
    // 4. softmax statistics of token b: warp b (fixed order: strided per lane, xor tree)
    if (warp < B) {
        float* sc = s_sc + warp * scw;
        float mx = -INFINITY;
        for (int i = lane; i < nrow; i += 32) mx = fmaxf(mx, sc[i]);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
        float sm = 0.f;
        for (int i = lane; i < nrow; i += 32) {
            const float pe = expf(sc[i] - mx);
            sc[i] = pe;
            sm += pe;
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, m);
        if (lane == 0) { s_ml[warp * 4] = mx; s_ml[warp * 4 + 1] = sm; }
    }
    consumer_bar(NT);
    // 5. o partials: task (row group, token, 8-dim chunk) -- one 16-B load per
    // cache row covers 8 dims, 8 rows in flight (the per-dim version issued one
    // dependent 2-B L2 load per row: ~16 serial L2 round trips per item).  Per
    // dim the rows are still added in ascending t (same sums as before).
    {
        const int nc8 = hd / 8;
        for (int i = tid; i < 4 * B * nc8; i += NT) {
            const int rg = i / (B * nc8), rem = i - rg * B * nc8, b = rem / nc8, c8 = rem - b * nc8;
            const __half* vc = ph->vc + ((size_t)b * n_kv + kvh) * (size_t)max_T * hd + c8 * 8;
            const uint4 vnew = *reinterpret_cast<const uint4*>(s_vn + b * 128 + c8 * 8);
            const float* sc = s_sc + b * scw - r.t0;
            float o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = 0.f;
            int t = r.t0 + rg;
            for (; t + 28 < r.t1; t += 32) {
                uint4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int tt = t + 4 * u;
                    v[u] = tt == pos ? vnew : __ldcg(reinterpret_cast<const uint4*>(vc + (size_t)tt * hd));
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float pu = sc[t + 4 * u];
                    const __half* vh = reinterpret_cast<const __half*>(&v[u]);
#pragma unroll
                    for (int e = 0; e < 8; ++e) o[e] += pu * __half2float(vh[e]);
                }
            }
            for (; t < r.t1; t += 4) {
                const uint4 v = t == pos ? vnew : __ldcg(reinterpret_cast<const uint4*>(vc + (size_t)t * hd));
                const float pu = sc[t];
                const __half* vh = reinterpret_cast<const __half*>(&v);
#pragma unroll
                for (int e = 0; e < 8; ++e) o[e] += pu * __half2float(vh[e]);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) s_o[(rg * B + b) * 128 + c8 * 8 + e] = o[e];
        }
    }
    consumer_bar(NT);
    for (int i = tid; i < B * hd; i += NT) {
        const int b = i / hd, dim = i - b * hd;
        float od = 0.f;
        for (int g2 = 0; g2 < 4; ++g2) od += s_o[(g2 * B + b) * 128 + dim];
        st_word(out_base + (size_t)b * out_bstride + dim, f32_word(od));
    }
    if (tid < B) st_word(out_base + (size_t)tid * out_bstride + hd, f32_word(s_ml[tid * 4]));
    consumer_bar(NT);
    if (tid < B)   // l last, with release (cumulative over the barrier)
        asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(out_base + (size_t)tid * out_bstride + hd + 1),
                     "l"(f32_word(s_ml[tid * 4 + 1])) : "memory");
}

// x staging of the o projection from the attention partials of an ATTN step
// (counted words [B][heads][P][hd + 2], count 1): element col of token b is
// head col / hd, dim col % hd; x = fp16(sum_q e_q o_q / sum_q e_q l_q) with
// e_q = exp(m_q - max_q m_q), parts in fixed order (deterministic).  Layout of
// s_x as core::stage_x.
template <int D, int NB, int NW, bool XF>
__device__ __forceinline__ void stage_x_attn(uint8_t* s_x, const unsigned long long* a, int B, int N_ss, int g_begin,
                                             int ng, int heads, int hd, int P) {
    constexpr int E = core::Entry<D>::value;
    const int n_ent = ng * 32 * NB;
    for (int t = threadIdx.x; t < n_ent; t += NW * 32) {
        const int b = t % NB;
        const int ss = (g_begin + t / (NB * 32)) * 32 + ((t / NB) & 31);
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if (b < B && ss < N_ss) {
            const int col = ss * D, head = col / hd, e0 = col - head * hd;
            const unsigned long long* hb = a + ((size_t)b * heads + head) * P * (hd + 2);
            // poll only the l words (written with release after the part's o and m
            // words, attn_item), all parts in flight; then o and m are final.
            // (Polling all 16 words of an entry in one round trip was measured
            // slower: register pressure, 1.44 -> 1.58 ms per token.)
            unsigned long long lv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) lv[q] = 0ull;
            const unsigned long long t_start = dev::globaltimer();
            for (bool done = false; !done;) {
                done = true;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q < P && (lv[q] >> core::kCntShift) != 1ull)
                        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(lv[q]) : "l"(hb + (size_t)q * (hd + 2) + hd + 1) : "memory");
#pragma unroll
                for (int q = 0; q < 4; ++q)   // checks after all loads were issued
                    if (q < P && (lv[q] >> core::kCntShift) != 1ull) done = false;
                if (!done && dev::globaltimer() - t_start > 4000000000ull) __trap();
            }
            float m[8], l[8], o[8][D];   // P <= 4, fully unrolled (registers, not local memory)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const unsigned long long* pb = hb + (size_t)(q & 3) * (hd + 2);
                m[q] = q < P ? word_f32(ld_word(pb + hd, false)) : -INFINITY;
                l[q] = q < P ? word_f32(lv[q & 3]) : 0.f;
#pragma unroll
                for (int e = 0; e < D; ++e) o[q][e] = q < P ? word_f32(ld_word(pb + e0 + e, false)) : 0.f;
            }
            float M = -INFINITY;
#pragma unroll
            for (int q = 0; q < 8; ++q) M = fmaxf(M, m[q]);
            float den = 0.f, num[D];
#pragma unroll
            for (int e = 0; e < D; ++e) num[e] = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q >= P) continue;
                const float f = m[q] == -INFINITY ? 0.f : expf(m[q] - M);
                den += f * l[q];
#pragma unroll
                for (int e = 0; e < D; ++e) num[e] += f * o[q][e];
            }
#pragma unroll
            for (int e = 0; e < D; ++e)
                w[e >> 1] |= (uint32_t)__half_as_ushort(__float2half_rn(num[e] / den)) << (16 * (e & 1));
        }
        if (XF) {
            core::store_x_f32<D, NB>(s_x, t, w);
        } else {
            uint32_t* dst = reinterpret_cast<uint32_t*>(s_x + (size_t)t * E);
#pragma unroll
            for (int q = 0; q < E / 4; ++q) dst[q] = w[q];
        }
    }
}

template <int D, int NB, int NW, int ST, bool MODEL>
__global__ void __launch_bounds__((NW + 1) * 32, 1) k_chain(ChainParams p) {
    constexpr int E = core::Entry<D>::value;
    constexpr bool PAIR = ChainPair<D>::value;
    // d <= 2: row-set mapping, 64 rows per warp at any B (gemv_core.cuh)
    constexpr int RW = PAIR ? 64 : core::RowsPerWarp<NB>::value;
    constexpr int R = RW * NW;
    constexpr int G = NB <= 2 ? 8 : NB == 4 ? 4 : 2;   // lanes per row set (<= 32 accumulators)
    // d = 2, B >= 4: batched decode on the tensor cores (gemv_core.cuh compute_group_mma)
    // (measured: B = 8 2.95 vs 3.52 ms per 32-block step; B = 4 2.48 vs 1.83 -- the FHFMA path wins there)
    constexpr bool MMA = D == 2 && NB == 8 && !FASQ_CHAIN_NO_MMA;
    constexpr bool XF = PAIR && NB == 8 && !MMA;       // x staged as fp32 (FFMA2 path, compute_group_set)
    constexpr int XG = XF ? 32 * NB * D * 4 : 32 * NB * E;
    constexpr int CS = kChainCS;
    constexpr int NT = NW * 32;                        // consumer threads
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* s_cb = smem;                                       // PAIR: CS * 64 KiB, else ST * cbb_max
    uint8_t* s_idx = s_cb + (PAIR ? CS * kPairSlot : ST * p.cbb_max);   // ST * R * 32
    uint8_t* s_x = s_idx + ST * R * 32;                         // gmax * XG
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_x + p.gmax * XG);
    float* s_sq = reinterpret_cast<float*>(bars + 2 * (ST + CS));   // [NW][NB] RMSNorm sum-of-squares partials
    int* s_tok = reinterpret_cast<int*>(s_sq + NW * NB);             // [8] EMBED tokens
    unsigned& s_run = *reinterpret_cast<unsigned*>(s_tok + 8);       // run index
    int& s_pos = *reinterpret_cast<int*>(s_tok + 9);                 // model position
    unsigned long long*& s_tail = *reinterpret_cast<unsigned long long**>(s_tok + 10);   // this rank's tail words
    EpiParams& s_ep = *reinterpret_cast<EpiParams*>(s_tok + 12);     // the current item's epilogue parameters
    const uint32_t cb_u = dev::smem_u32(s_cb), idx_u = dev::smem_u32(s_idx);
    const uint32_t full0 = dev::smem_u32(&bars[0]), empty0 = dev::smem_u32(&bars[ST]);
    const uint32_t cfull0 = dev::smem_u32(&bars[2 * ST]), cempty0 = dev::smem_u32(&bars[2 * ST + CS]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // (the tail pointer is not kept live across the loop: register pressure)
    auto tail_ptr = [&]() { return p.peers[p.rank] + 2 * p.arena_words; };

    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < ST; ++s) {
            dev::mbar_init(full0 + 8 * s, 1);
            dev::mbar_init(empty0 + 8 * s, NW);
        }
        if (PAIR) {
#pragma unroll
            for (int s = 0; s < CS; ++s) {
                dev::mbar_init(cfull0 + 8 * s, 1);
                dev::mbar_init(cempty0 + 8 * s, NW);
            }
        }
        dev::fence_barrier_init();
    }
    __syncthreads();

    if (warp == NW) {
        // producer: every step's stages, back to back (no dependence on x)
        if (lane == 0) {
            int pos = 0;
            if (p.model) pos = (int)ld_word(tail_ptr() + T_POS, false);
            int it = 0, cit = 0;
            for (int phj = 0; phj < p.n_steps * p.mi; ++phj) {
                const int ph = phj / p.mi;
                const ChainItem& w = p.items[((size_t)ph * p.nctas + blockIdx.x) * p.mi + phj % p.mi];
                if (MODEL && w.kind == SK_ATTN) {
                    if (PAIR) {   // a pair slot for the consumers: cache rows + attention scratch
                        const int cs = cit % CS;
                        if (cit >= CS) dev::mbar_wait(cempty0 + 8 * cs, ((cit / CS) + 1) & 1);
                        const ChainPhase& P = p.phases[ph];
                        const AttnRows r = attn_rows(w.kidx, P.parts, pos, p.B, P.hd);
                        if (r.smem) {
                            const int nk = r.te - r.t0, kvh = w.head / (P.n_heads / P.n_kv);
                            const uint32_t rb = (uint32_t)nk * P.hd * 2u;
                            const uint32_t dst = cb_u + (uint32_t)cs * kPairSlot;
                            dev::mbar_arrive_expect_tx(cfull0 + 8 * cs, 2u * rb * (uint32_t)p.B);
                            for (int b = 0; b < p.B; ++b) {
                                const size_t src = (((size_t)b * P.n_kv + kvh) * p.max_T + r.t0) * P.hd;
                                dev::bulk_g2s(dst + (uint32_t)b * rb, P.kc + src, rb, cfull0 + 8 * cs);
                                dev::bulk_g2s(dst + (uint32_t)(p.B + b) * rb, P.vc + src, rb, cfull0 + 8 * cs);
                            }
                        } else {
                            dev::mbar_arrive(cfull0 + 8 * cs);
                        }
                        ++cit;
                    }
                    continue;
                }
                if (w.kind != SK_PQ || w.rows_valid <= 0) continue;
                if (MODEL && p.attn_pf && ph + 1 < p.n_steps && phj % p.mi == 0) {
                    // the next step is attention: warm L2 with this CTA's cache rows now, so the
                    // pair-slot TMA (issued once a slot frees up) hits L2, not HBM
                    const ChainItem& na = p.items[((size_t)(ph + 1) * p.nctas + blockIdx.x) * p.mi];
                    if (na.kind == SK_ATTN) {
                        const ChainPhase& P = p.phases[ph + 1];
                        const AttnRows r = attn_rows(na.kidx, P.parts, pos, p.B, P.hd);
                        if (r.te > r.t0) {
                            const int kvh = na.head / (P.n_heads / P.n_kv);
                            const uint32_t rb = (uint32_t)(r.te - r.t0) * P.hd * 2u;
                            for (int b = 0; b < p.B; ++b) {
                                const size_t src = (((size_t)b * P.n_kv + kvh) * p.max_T + r.t0) * P.hd;
                                dev::bulk_prefetch_l2(P.kc + src, rb);
                                dev::bulk_prefetch_l2(P.vc + src, rb);
                            }
                        }
                    }
                }
                const uint32_t cbb = (uint32_t)w.C * 32u * E;
                const uint32_t chunk = (uint32_t)w.rows_valid * 32u;
                if (p.pf > 0 && ph + 1 < p.n_steps && phj % p.mi == 0) {
                    // warm L2 with the head of the next step's first item
                    const ChainItem& nw = p.items[((size_t)(ph + 1) * p.nctas + blockIdx.x) * p.mi];
                    if (nw.kind == SK_PQ && nw.rows_valid > 0) {
                        const int ge = min(nw.g_end, nw.g_begin + p.pf);
                        for (int g = nw.g_begin; g < ge; ++g)
                            dev::bulk_prefetch_l2(nw.idx + ((size_t)g * nw.F_out_pad + nw.r0) * 32,
                                                  (uint32_t)nw.rows_valid * 32u);
                    }
                }
                for (int g = w.g_begin; g < w.g_end; ++g, ++it) {
                    if (PAIR && ((g - w.g_begin) & 1) == 0) {
                        // groups g, g+1 -> one pair slot (g+1 past the layer: zero fill)
                        const int cs = cit % CS;
                        if (cit >= CS) dev::mbar_wait(cempty0 + 8 * cs, ((cit / CS) + 1) & 1);
                        if (p.dbg & 6) {   // bit 2: codebook copies only skipped (stale SMEM codebooks)
                            dev::mbar_arrive(cfull0 + 8 * cs);
                        } else {
                            dev::mbar_arrive_expect_tx(cfull0 + 8 * cs, 2u * cbb);
                            dev::tma_load_3d(cb_u + (uint32_t)cs * kPairSlot, MMA ? w.cbmap_x : w.cbmap, 0, g, 0,
                                             cfull0 + 8 * cs);
                        }
                        ++cit;
                    }
                    const int slot = it % ST;
                    if (it >= ST) dev::mbar_wait(empty0 + 8 * slot, ((it / ST) + 1) & 1);
                    const uint32_t full = full0 + 8 * slot;
                    if (p.dbg & 2) { dev::mbar_arrive(full); continue; }
                    dev::mbar_arrive_expect_tx(full, PAIR ? chunk : chunk + cbb);
                    if (!PAIR)
                        dev::bulk_g2s(cb_u + (uint32_t)slot * (uint32_t)p.cbb_max, w.cbimg + (size_t)g * cbb, cbb,
                                      full);
                    dev::bulk_g2s(idx_u + (uint32_t)slot * R * 32u, w.idx + ((size_t)g * w.F_out_pad + w.r0) * 32,
                                  chunk, full);
                }
            }
        }
        __syncwarp();
        return;
    }

    // ---- run prologue ----
    if (threadIdx.x == 0) {
        unsigned long long* const tail = tail_ptr();
        s_tail = tail;
        unsigned long long old;
        asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(tail + T_ENTRY) : "memory");
        const unsigned run = (unsigned)(old / (unsigned long long)p.nctas);
        s_run = run;
        if (p.world > 1) {
            // every rank finished run - 1 (its stores into our buffers landed) before we zero
            const unsigned long long want = (unsigned long long)p.world * run, t0 = dev::globaltimer();
            unsigned long long v;
            for (;;) {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(tail + T_DONE) : "memory");
                if (v >= want) break;
                if (dev::globaltimer() - t0 > 4000000000ull) __trap();
            }
        }
        if (p.model) s_pos = (int)ld_word(tail + T_POS, false);
    }
    consumer_bar(NT);
    const unsigned run = s_run;
    const unsigned par = run & 1u;
    unsigned long long* const cur = p.peers[p.rank] + (long long)par * p.arena_words;   // this run's buffer
    // zero this CTA's share of the other buffer for run + 1 (16-B stores;
    // arena_words is even).  Model chains do it after step 0 (the embedding,
    // one CTA): the embedding CTA starts at once, the others zero while they
    // would wait for it anyway.
    auto zero_next = [&]() {
        ulonglong2* nxt = reinterpret_cast<ulonglong2*>(p.peers[p.rank] + (long long)((s_run & 1u) ^ 1u) * p.arena_words);
        const long long n2 = p.arena_words / 2, per = (n2 + p.nctas - 1) / p.nctas;
        const long long zb = per * blockIdx.x, ze = min(n2, zb + per);
        for (long long i = zb + threadIdx.x; i < ze; i += NT) nxt[i] = make_ulonglong2(0ull, 0ull);
    };
    if (!MODEL) zero_next();
    const bool sys_out = p.world > 1;

    const int wrow0 = warp * RW;
    const auto co = core::chunk_offsets<RW>(wrow0, lane);
    const auto qm = core::set_map<G>(wrow0, lane);
    int slot = 0;            // ring position of the next stage (running across steps)
    uint32_t par_ring = 0;   // its mbarrier phase parity
    int cslot = 0;           // PAIR: codebook pair slot and parity
    uint32_t cpar = 0;
    for (int phj = 0; phj < p.n_steps * p.mi; ++phj) {
        const int ph = phj / p.mi, j = phj % p.mi;
        if (MODEL && phj == p.mi) zero_next();   // start of step 1
        const ChainItem* wp = p.items + ((size_t)ph * p.nctas + blockIdx.x) * p.mi + j;
        const ChainPhase* phs = p.phases + ph;
        // item and phase fields by value: their loads issue here, before the
        // barrier -- not as dependent L2 round trips after it
        const ChainItem w = *wp;
        const ChainPhase pv = *phs;
#define FASQ_TR(k) (p.trace + ((size_t)ph * p.nctas + blockIdx.x) * 4 + (k))
        const bool tr = p.trace != nullptr;   // trace stamps (the pointer is recomputed: register pressure)
        if (tr && threadIdx.x == 0 && j == 0) *FASQ_TR(0) = dev::globaltimer();
        if (w.kind < 0) continue;
        // every consumer warp is done with the previous item's SMEM
        consumer_bar(NT);
        if (MODEL && w.kind == SK_EMBED) {
            embed_item(phs, cur, s_tail, p.B, s_run, s_pos, p.max_T, p.tok_hist, p.tok_expect, NT, s_tok);
            if (tr && lane == 0 && warp == 0) { *FASQ_TR(1) = *FASQ_TR(2) = *FASQ_TR(3) = dev::globaltimer(); }
            continue;
        }
        if (MODEL && w.kind == SK_ATTN) {
            if constexpr (PAIR) {
                dev::mbar_wait(cfull0 + 8 * cslot, cpar);
                if (tr && threadIdx.x == 0 && j == 0) *FASQ_TR(1) = *FASQ_TR(2) = dev::globaltimer();
                if (NB == 1)
                    attn_item(phs, w.head, w.kidx, cur, p.B, s_pos, p.max_T, p.rope, s_cb + (size_t)cslot * kPairSlot,
                              NT);
                else
                    attn_item_batched(phs, w.head, w.kidx, cur, p.B, s_pos, p.max_T, p.rope,
                                      s_cb + (size_t)cslot * kPairSlot, NT);
                __syncwarp();
                if (lane == 0) dev::mbar_arrive(cempty0 + 8 * cslot);
                if (++cslot == CS) { cslot = 0; cpar ^= 1u; }
            }
            if (tr && lane == 0 && warp == 0) *FASQ_TR(3) = dev::globaltimer();
            continue;
        }
        const int ng = w.g_end - w.g_begin;
        const int in_mode = pv.in_mode;
        const bool xsys = pv.x_sys != 0;
        if (in_mode == IN_EXT) {
            core::stage_x<D, NB, NW, XF>(s_x, p.x_ext, 0, pv.F_in, p.B, w.N_ss, w.g_begin, ng);
        } else if (in_mode == IN_WORDS) {
            core::stage_x_counted<D, NB, NW, XF>(s_x, cur + pv.x_off, pv.x_ks, pv.F_in, p.B, w.N_ss, w.g_begin,
                                                 ng, xsys, p.backoff);
        } else if constexpr (PAIR && MODEL) {
            if (in_mode == IN_RMSNORM) {
                if (pv.x2_off >= 0)   // source = a lazily materialised residual sum (x + x2)
                    core::stage_x_counted<D, NB, NW, XF, core::XM_GAMMA2>(s_x, cur + pv.x_off, pv.x_ks, pv.F_in, p.B,
                                                                          w.N_ss, w.g_begin, ng, xsys, 0,
                                                                          cur + pv.x2_off, pv.x2_ks,
                                                                          w.nsq >= 0 ? s_sq : nullptr, pv.gamma);
                else
                    core::stage_x_counted<D, NB, NW, XF, core::XM_GAMMA>(s_x, cur + pv.x_off, pv.x_ks, pv.F_in, p.B,
                                                                         w.N_ss, w.g_begin, ng, xsys, 0, nullptr, 0,
                                                                         w.nsq >= 0 ? s_sq : nullptr, pv.gamma);
            } else if (in_mode == IN_SILU) {
                // gate/up hold the products of the unscaled normed input: the
                // RMSNorm scale of their input (slots, warp_norm_scale) applies here
                float sc[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) sc[b] = 1.f;
                if (pv.sc_off >= 0) warp_norm_scale<NB>(sc, cur + pv.sc_off, pv.sc_n, pv.sc_F, pv.sc_eps, p.B, lane);
                core::stage_x_counted<D, NB, NW, XF, core::XM_SILU>(s_x, cur + pv.x_off, pv.x_ks, pv.F_in, p.B,
                                                                    w.N_ss, w.g_begin, ng, xsys, 0,
                                                                    cur + pv.x2_off, pv.x2_ks, nullptr, nullptr,
                                                                    pv.sc_off >= 0 ? sc : nullptr);
            } else {
                stage_x_attn<D, NB, NW, XF>(s_x, cur + pv.x_off, p.B, w.N_ss, w.g_begin, ng, pv.a_heads, pv.a_hd,
                                            pv.a_parts);
            }
        }
        if (tr && threadIdx.x == 0 && j == 0) *FASQ_TR(1) = dev::globaltimer();
        if (threadIdx.x == 0) {   // epilogue parameters -> SMEM (read after the gather loop)
            EpiParams e;
            e.y_off = wp->y_off;
            e.res_off = phs->res_off;
            e.res2_off = phs->res2_off;
            e.res2_ks = phs->res2_ks;
            e.epi_scale = phs->epi_scale;
            e.nsq_off = phs->nsq_off;
            e.nsq_n = phs->nsq_n;
            e.F_in = phs->F_in;
            e.eps = phs->eps;
            e.row0_g = wp->row0_g;
            e.ld = wp->ld;
            e.F_out = wp->F_out;
            e.r0 = wp->r0;
            // the residual is spread over the row tile's K ranges (warp w's rows: range
            // w % kn) -- a single range polling all 1024 rows' residual words was the
            // slowest CTA of the o / down steps (at B = 8: 1.6x the median item)
            e.add_res = e.res_off >= 0 && phs->res_here;
            e.kidx = w.kidx;
            e.kn = w.kn > 0 ? w.kn : 1;
            e.res_ks = phs->res_ks;
            e.res_sys = phs->res_sys;
            e.out_all = phs->out_all;
            s_ep = e;
        }
        consumer_bar(NT);
        if (tr && threadIdx.x == 0 && j == 0) *FASQ_TR(2) = dev::globaltimer();
        if (PAIR && MODEL && in_mode == IN_RMSNORM && w.nsq >= 0 && threadIdx.x < p.B) {
            // this K range's sum of squares of h (all warps' partials, fixed order)
            float a = 0.f;
            for (int q = 0; q < NW; ++q) a += s_sq[q * NB + threadIdx.x];
            st_word(cur + pv.nsq_off + threadIdx.x * 64 + w.nsq, f32_word(a));
        }
        const bool active = wrow0 < w.rows_valid;
        if constexpr (PAIR) {
            if constexpr (MMA) {
                // tensor-core path: 16 fp32 accumulators per lane (64 rows x 8 tokens per warp)
                float acc[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q] = 0.f;
                const bool run_loop = active && !(p.dbg & 1);
                const uint32_t blk = (uint32_t)(wrow0 >> 6) * 2048u;
                for (int i = 0; i < ng; i += 2) {
                    dev::mbar_wait(cfull0 + 8 * cslot, cpar);
                    const uint32_t lbs = (uint32_t)cslot << 16;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (h == 1 && i + 1 >= ng) break;
                        dev::mbar_wait(full0 + 8 * slot, par_ring);
                        if (run_loop)
                            core::compute_group_mma<NB>(acc, s_idx + slot * R * 32, blk, lane, s_cb,
                                                        lbs + ((uint32_t)h << 7), s_x + (i + h) * XG);
                        __syncwarp();
                        if (lane == 0) dev::mbar_arrive(empty0 + 8 * slot);
                        if (++slot == ST) { slot = 0; par_ring ^= 1u; }
                    }
                    if (lane == 0) dev::mbar_arrive(cempty0 + 8 * cslot);
                    if (++cslot == CS) { cslot = 0; cpar ^= 1u; }
                }
                if (active) {
                    float sc[NB];
                    const bool scl = MODEL && s_ep.epi_scale;
                    if (scl) warp_norm_scale<NB>(sc, cur + s_ep.nsq_off, s_ep.nsq_n, s_ep.F_in, s_ep.eps, p.B, lane);
                    const int row0_g = s_ep.row0_g, ld = s_ep.ld, F_out = s_ep.F_out, r0 = s_ep.r0;
                    long long qv[16];
                    const long long off = (long long)(s_run & 1u) * p.arena_words + s_ep.y_off + row0_g;
                    core::mma_values<NB>(acc, qv, r0 + wrow0, lane, F_out, p.B, scl ? sc : nullptr,
                                         MODEL && s_ep.add_res && warp % s_ep.kn == s_ep.kidx
                                             ? cur + s_ep.res_off + row0_g : nullptr, ld,
                                         s_ep.res_ks, s_ep.res_sys != 0, s_tail + T_OVF,
                                         MODEL && s_ep.res2_off >= 0 ? cur + s_ep.res2_off + row0_g : nullptr,
                                         s_ep.res2_ks);
                    if (s_ep.out_all) {
                        for (int q = 0; q < p.world; ++q)
                            core::counted_store_mma(qv, p.peers[q] + off, r0 + wrow0, lane, F_out, ld, p.B, sys_out);
                    } else {
                        core::counted_store_mma(qv, p.peers[p.rank] + off, r0 + wrow0, lane, F_out, ld, p.B, false);
                    }
                }
            } else {
                // pair stages: row-set mapping (gemv_core.cuh), 2G*NB accumulators
                // per lane, G-lane row reduction
                float acc[2 * G * NB];
#pragma unroll
                for (int q = 0; q < 2 * G * NB; ++q) acc[q] = 0.f;
                const bool run_loop = active && !(p.dbg & 1);
                for (int i = 0; i < ng; i += 2) {
                    dev::mbar_wait(cfull0 + 8 * cslot, cpar);
                    const uint32_t lbs = (uint32_t)cslot << 16;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (h == 1 && i + 1 >= ng) break;
                        dev::mbar_wait(full0 + 8 * slot, par_ring);
                        if (run_loop)
                            core::compute_group_set<D, NB, G>(acc, s_idx + slot * R * 32, qm, s_cb,
                                                              lbs + ((uint32_t)h << 7), s_x + (i + h) * XG);
                        __syncwarp();
                        if (lane == 0) dev::mbar_arrive(empty0 + 8 * slot);
                        if (++slot == ST) { slot = 0; par_ring ^= 1u; }
                    }
                    if (lane == 0) dev::mbar_arrive(cempty0 + 8 * cslot);
                    if (++cslot == CS) { cslot = 0; cpar ^= 1u; }
                }
                core::reduce_set<NB, G>(acc, lane);
                if (active) {
                    if (MODEL && s_ep.epi_scale) {
                        float sc[NB];
                        warp_norm_scale<NB>(sc, cur + s_ep.nsq_off, s_ep.nsq_n, s_ep.F_in, s_ep.eps, p.B, lane);
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int b = 0; b < NB; ++b) acc[h * NB + b] *= sc[b];
                    }
                    const int row0_g = s_ep.row0_g, ld = s_ep.ld, F_out = s_ep.F_out, r0 = s_ep.r0;
                    long long qv[2 * NB];
                    const long long off = (long long)(s_run & 1u) * p.arena_words + s_ep.y_off + row0_g;
                    core::set_values<NB, G>(acc, qv, r0 + wrow0, lane, F_out, p.B,
                                            MODEL && s_ep.add_res && warp % s_ep.kn == s_ep.kidx
                                                ? cur + s_ep.res_off + row0_g : nullptr, ld,
                                            s_ep.res_ks, s_ep.res_sys != 0, s_tail + T_OVF,
                                            MODEL && s_ep.res2_off >= 0 ? cur + s_ep.res2_off + row0_g : nullptr,
                                            s_ep.res2_ks);
                    if (s_ep.out_all) {
                        for (int q = 0; q < p.world; ++q)
                            core::counted_store_q<NB>(qv, p.peers[q] + off, r0 + wrow0, lane, F_out, ld, p.B, sys_out);
                    } else {
                        core::counted_store_q<NB>(qv, p.peers[p.rank] + off, r0 + wrow0, lane, F_out, ld, p.B, false);
                    }
                }
            }
        } else {
            float acc[RW][NB];
#pragma unroll
            for (int q = 0; q < RW; ++q)
#pragma unroll
                for (int b = 0; b < NB; ++b) acc[q][b] = 0.f;
            // d = 4, 8: lane = subspace over 64/B rows per warp
            for (int i = 0; i < ng; ++i) {
                dev::mbar_wait(full0 + 8 * slot, par_ring);
                if (active && !(p.dbg & 1)) {
                    uint32_t xv[NB][E / 4];
                    core::load_x<D, NB>(xv, s_x + i * XG, lane);
                    core::compute_group<D, NB, RW>(acc, s_idx + slot * R * 32, co, s_cb + slot * p.cbb_max, xv, lane);
                }
                __syncwarp();
                if (lane == 0) dev::mbar_arrive(empty0 + 8 * slot);
                if (++slot == ST) { slot = 0; par_ring ^= 1u; }
            }
            core::RowTotals<NB, RW> tot;
            core::reduce_rows<NB, RW>(acc, tot, lane);
            if (active) {
                const long long off = (long long)(s_run & 1u) * p.arena_words + s_ep.y_off + s_ep.row0_g;
                const bool oa = s_ep.out_all != 0;
                const int nq = oa ? p.world : 1;
                for (int q = 0; q < nq; ++q)
                    core::counted_store<NB, RW>(tot, p.peers[oa ? q : p.rank] + off, s_ep.r0 + wrow0, s_ep.F_out,
                                                s_ep.ld, p.B, s_tail + T_OVF);
            }
        }
        if (tr && lane == 0 && warp == 0) *FASQ_TR(3) = dev::globaltimer();
    }
#undef FASQ_TR
    // ---- run epilogue: exit count; the last CTA publishes the run to every rank ----
    consumer_bar(NT);
    if (threadIdx.x == 0) {
        unsigned long long* const tail = s_tail;
        __threadfence_system();
        unsigned long long old;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(tail + T_EXIT) : "memory");
        if (old + 1 == (unsigned long long)(run + 1) * (unsigned long long)p.nctas) {
            if (p.model) {
                const int np = s_pos + 1 < p.max_T ? s_pos + 1 : p.pos_wrap;
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(tail + T_POS), "l"((unsigned long long)np)
                             : "memory");
            }
            __threadfence_system();
            for (int q = 0; q < p.world; ++q) {
                unsigned long long* dn = p.peers[q] + 2 * p.arena_words + T_DONE;
                asm volatile("red.release.sys.global.add.u64 [%0], %1;" :: "l"(dn), "l"(1ull) : "memory");
            }
        }
    }
}

constexpr size_t kChainSmem = kSmemMax;
constexpr size_t kChainScratch = 8 * 4 + 16 + sizeof(EpiParams);   // s_tok, run/pos words, s_ep (after the mbarriers and s_sq)

template <int D, int NB, int NW, int ST, bool MODEL>
fasq_status launch_chain_t(const ChainParams& p, size_t smem, int grid, cudaStream_t st) {
    auto kern = k_chain<D, NB, NW, ST, MODEL>;
    static size_t lim = 0;
    static std::once_flag once;
    std::call_once(once, [&] { lim = set_max_dyn_smem(kern); });
    if (lim < smem) {
        set_error("chain: dynamic SMEM plan (" + std::to_string(smem) + " B) exceeds the device limit (" +
                  std::to_string(lim) + " B)");
        return FASQ_E_UNSUPPORTED;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3((NW + 1) * 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident (consumers spin on producers' words)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FASQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    return FASQ_OK;
}

template <int D, int NB>
fasq_status chain_cfg(const fasq_chain* c, const ChainParams& p, cudaStream_t st) {
    // nw = 16 always fits at C <= 256 (the planner lowers the index-ring depth
    // instead); the whole-model (MODEL) instances exist for the pair path d <= 2
#define FASQ_CHAIN_CASE(NW_, ST_)                                                                      \
    if (c->nw == NW_ && c->st == ST_) {                                                                \
        if constexpr (D <= 2)                                                                          \
            if (c->has_model) return launch_chain_t<D, NB, NW_, ST_, true>(p, c->smem, c->nctas, st); \
        return launch_chain_t<D, NB, NW_, ST_, false>(p, c->smem, c->nctas, st);                       \
    }
    FASQ_CHAIN_CASE(16, 3)
    FASQ_CHAIN_CASE(16, 2)
    FASQ_CHAIN_CASE(16, 1)
#undef FASQ_CHAIN_CASE
    set_error("chain: no kernel instantiated for this tiling (nw=" + std::to_string(c->nw) + ", st=" +
              std::to_string(c->st) + ")");
    return FASQ_E_UNSUPPORTED;
}

// Launch of the chain kernel for batch width NB (defined in chain_k<NB>.cu).
template <int NB>
fasq_status chain_dispatch(const fasq_chain* c, const ChainParams& p, cudaStream_t st);

#define FASQ_CHAIN_DISPATCH_DEF(NB_)                                                          \
    template <>                                                                               \
    fasq_status chain_dispatch<NB_>(const fasq_chain* c, const ChainParams& p, cudaStream_t st) { \
        switch (c->d) {                                                                       \
            case 1: return chain_cfg<1, NB_>(c, p, st);                                       \
            case 2: return chain_cfg<2, NB_>(c, p, st);                                       \
            case 4: return chain_cfg<4, NB_>(c, p, st);                                       \
            case 8: return chain_cfg<8, NB_>(c, p, st);                                       \
        }                                                                                     \
        return FASQ_E_UNSUPPORTED;                                                            \
    }

}  // namespace chainimpl
}  // namespace fasq
