// llama.cu -- whole-model Llama-shaped decode on FASQ layers (sm_100a).
//
// The paper's end-to-end experiment (Table 4) decodes
// Llama-3-8B with every linear layer of the 32 decoder blocks (q, k, v, o,
// gate, up, down) product-quantized, embeddings and lm_head kept fp16
// (SURVEY App. A).  One decode token here is TWO kernel launches:
//
//  1. the persistent decode chain (chain.cu) with the model's step list:
//        EMBED -> per block: {q,k,v} <- RMSNorm(h) ; ATTN ; o (+h) ;
//                            {gate,up} <- RMSNorm(h') ; down <- silu(gate)*up (+h')
//     where "(+h)" is the residual connection fused into the GEMV epilogue;
//  2. k_lm_head: final RMSNorm + the fp16 lm_head GEMV on the tensor cores
//     (mma.sync, the B <= 8 tokens as the M side) + argmax, red.max'ed into a
//     token slot of every rank that the next run's EMBED step reads.
//
// Tensor parallelism (world > 1, Megatron layout): q/k/v and gate/up are row
// shards (this rank's heads / ffn slice, outputs local), o and down are K
// shards (subspaces of the local heads / ffn slice; every rank red.adds its
// partial sums of ALL rows into every rank's arena -- the all-reduce fused
// into the counted stores), the residual is added by rank 0 only, lm_head is
// a vocab shard with the argmax reduced across ranks by red.max.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <initializer_list>
#include <type_traits>
#include <vector>

#include "chain_internal.cuh"
#include "gemv_core.cuh"

namespace fasq {
fasq_status chain_launch(fasq_chain* c, const void* x_dev, cudaStream_t st);
fasq_status chain_output(const fasq_chain* c, int step, int layer, void* y_dev, fasq_dtype dtype, cudaStream_t st);
void chain_destroy(fasq_chain* c);
int sm_count();
}  // namespace fasq

struct fasq_llama {
    fasq_llama_desc desc{};
    fasq_chain* chain = nullptr;
    std::vector<__half*> kc, vc;       // per layer [B][n_kv_local][max_T][hd]
    float2* rope = nullptr;
    int* tok_hist = nullptr;
    float* logits = nullptr;           // optional debug output (fasq_llama_logits)
    int* tok_dev = nullptr;            // staging for fasq_llama_step_host / reset
    int* tok_pin = nullptr;            // pinned host staging [16] (in 0..7, out 8..15) of fasq_llama_step_io
    cudaGraphExec_t io_exec = nullptr; // fasq_llama_step_io at pos < 0: the whole step as one graph launch
    int lm_ctas = 0;
    int n_heads_l = 0, n_kv_l = 0, ffn_l = 0, vocab_l = 0;
    int last_step = 0;                 // chain step of the last down projection
    size_t lm_smem = 0;
    // fasq_llama_prefill: persistent buffers for up to pf_cap tokens, the staged
    // tokens / pos0, a private capture stream and the graph of the last M
    int pf_cap = 0;
    uint8_t* pf_buf = nullptr;
    int* pf_tok = nullptr;             // [pf_cap] prompt tokens, [pf_cap] = pos0
    cudaStream_t pf_stream = nullptr;
    cudaEvent_t pf_ev[2] = {nullptr, nullptr};
    cudaGraphExec_t pf_exec = nullptr;
    int pf_exec_M = 0;
};

namespace fasq {
namespace {

constexpr int kLmNW = 16;

// ---- lm_head: final RMSNorm + fp16 GEMV (mma.sync) + argmax -----------------
// Work unit = a strip of 8 vocab rows x the whole hidden dim, per warp.  The
// contraction is a plain dense product, so it runs on the tensor cores:
// mma.sync.m16n8k16 with A = x (tokens as M, B <= 8 real rows, rows 8..15
// zero) and B = the strip's weights (N = 8 rows).  The k order inside an MMA
// is permuted consistently on both operands (the sum is order-free): lane
// (g, t) loads 32 contiguous bytes of weight row g per 64-column chunk (two
// LDG.128; a warp reads full 128-B lines) and the matching 32 bytes of x[g].
// Ties in the argmax go to the lowest token id (tok_key).
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1)
k_lm_head(const __half* __restrict__ W, int V_local, int v0, int hidden, long long h_off, int h_ks, int h_sys,
          const __half* __restrict__ gamma, float eps, int B, unsigned long long* const* peers, int rank,
          long long arena_words, int world, int nctas_chain, float* logits) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ float s_red[NW * 8];
    __shared__ float s_scale[8];
    __shared__ unsigned long long s_best[NW][8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NT = NW * 32;
    const int pitch = hidden + 8;   // halves; +16 B keeps the x fragment loads conflict-free
    __half* xs = reinterpret_cast<__half*>(smem);
    unsigned long long* const base = peers[rank];
    const unsigned long long runs = base[2 * arena_words + T_ENTRY] / (unsigned long long)nctas_chain;
    const unsigned par = (unsigned)((runs + 1ull) & 1ull);   // parity of the finished run (runs - 1)
    const unsigned long long* h_words = base + (long long)par * arena_words + h_off;
    // 1. final RMSNorm -> x fp16 [B][pitch] in SMEM (every CTA, same fixed order)
    core::norm_scale<8, NW>(h_words, h_ks, hidden, B, eps, h_sys != 0, s_red, s_scale);
    for (int i = tid; i < B * hidden; i += NT) {
        const int b = i / hidden, c = i - b * hidden;
        const long long v = core::poll_value(h_words + i, h_ks, h_sys != 0);
        const float f = (float)((double)v * core::kAccInv) * s_scale[b];
        xs[(size_t)b * pitch + c] = __float2half_rn(f * __half2float(gamma[c]));
    }
    __syncthreads();
    // 2. strips of 8 rows, dealt over all warps of the grid
    const int g = lane >> 2, t = lane & 3;
    const int n_strips = (V_local + 7) / 8;
    const int gw = blockIdx.x * NW + warp, nwarps = gridDim.x * NW;
    unsigned long long best = 0ull;   // key for token g (lanes with g < B)
    const bool tok_lane = g < B;
    const int nchunk = hidden / 64;
    for (int s = gw; s < n_strips; s += nwarps) {
        const int row = s * 8 + g;
        const bool rv = row < V_local;
        const uint4* wr = reinterpret_cast<const uint4*>(W + (size_t)(rv ? row : 0) * hidden) + t * 2;
        const uint4* xr = reinterpret_cast<const uint4*>(xs + (size_t)(tok_lane ? g : 0) * pitch) + t * 2;
        float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
        constexpr int U = 8;
        for (int k0 = 0; k0 < nchunk; k0 += U) {
            uint4 wv[U][2];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (k0 + u < nchunk && rv) {
                    wv[u][0] = __ldcs(wr + (size_t)(k0 + u) * 8);
                    wv[u][1] = __ldcs(wr + (size_t)(k0 + u) * 8 + 1);
                } else {
                    wv[u][0] = wv[u][1] = make_uint4(0u, 0u, 0u, 0u);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (k0 + u >= nchunk) break;
                uint4 xv0 = make_uint4(0u, 0u, 0u, 0u), xv1 = xv0;
                if (tok_lane) {
                    xv0 = xr[(size_t)(k0 + u) * 8];
                    xv1 = xr[(size_t)(k0 + u) * 8 + 1];
                }
                const uint32_t a[4][2] = {{xv0.x, xv0.y}, {xv0.z, xv0.w}, {xv1.x, xv1.y}, {xv1.z, xv1.w}};
                const uint32_t bw[4][2] = {{wv[u][0].x, wv[u][0].y}, {wv[u][0].z, wv[u][0].w},
                                           {wv[u][1].x, wv[u][1].y}, {wv[u][1].z, wv[u][1].w}};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    asm volatile(
                        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                        "{%0,%1,%2,%3};"
                        : "+f"(c0), "+f"(c1), "+f"(c2), "+f"(c3)
                        : "r"(a[j][0]), "r"(0u), "r"(a[j][1]), "r"(0u), "r"(bw[j][0]), "r"(bw[j][1]));
            }
        }
        // c0, c1 = logits of token g for rows s*8 + 2t, 2t + 1
        if (tok_lane) {
            const int r0 = s * 8 + 2 * t;
            if (r0 < V_local) {
                if (logits) logits[(size_t)g * V_local + r0] = c0;
                best = max(best, tok_key(c0, (unsigned)(v0 + r0)));
            }
            if (r0 + 1 < V_local) {
                if (logits) logits[(size_t)g * V_local + r0 + 1] = c1;
                best = max(best, tok_key(c1, (unsigned)(v0 + r0 + 1)));
            }
        }
    }
    // 3. reduce: the 4 lanes of token g, then warps, then one red.max per token and CTA
    best = max(best, __shfl_xor_sync(0xffffffffu, best, 1));
    best = max(best, __shfl_xor_sync(0xffffffffu, best, 2));
    if (t == 0) s_best[warp][g] = best;
    __syncthreads();
    if (tid < B) {
        unsigned long long bb = 0ull;
        for (int w = 0; w < NW; ++w) bb = max(bb, s_best[w][tid]);
        for (int q = 0; q < world; ++q) {
            unsigned long long* slot = peers[q] + 2 * arena_words + T_TOK + (par * 8 + tid) * 2;
            asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" :: "l"(slot), "l"(bb) : "memory");
            asm volatile("red.release.sys.global.add.u64 [%0], %1;" :: "l"(slot + 1), "l"(1ull) : "memory");
        }
    }
}

// (Re)starts decoding: the next run embeds tokens[b] at position pos (pos < 0:
// keep the position).  Writes the token slot the next run reads (parity of
// the previous run, derived on the device) as if an lm_head had chosen it.
__global__ void k_llama_reset(unsigned long long* tail, int nctas, const int* tokens, int B, int pos,
                              long long expect, const int* pos_base = nullptr) {
    const int b = threadIdx.x;
    if (pos_base) pos += *pos_base;   // prefill: pos = pos0 (device-resident) + M
    const unsigned long long runs = tail[T_ENTRY] / (unsigned long long)nctas;
    const unsigned pp = (unsigned)((runs + 1ull) & 1ull);   // (runs - 1) & 1
    if (b < 8) {
        unsigned long long* slot = tail + T_TOK + (pp * 8 + b) * 2;
        slot[0] = b < B ? tok_key(0.f, (unsigned)tokens[b]) : 0ull;
        slot[1] = b < B ? (unsigned long long)expect : 0ull;
        unsigned long long* other = tail + T_TOK + ((pp ^ 1u) * 8 + b) * 2;
        other[0] = 0ull;
        other[1] = 0ull;
    }
    if (b == 0 && pos >= 0) tail[T_POS] = (unsigned long long)pos;
}

// Token chosen by the last step's lm_head (waits for all contributions).
__global__ void k_llama_tokens(const unsigned long long* tail, int nctas, int B, long long expect, int* out) {
    const int b = threadIdx.x;
    if (b >= B) return;
    const unsigned long long runs = tail[T_ENTRY] / (unsigned long long)nctas;
    const unsigned par = (unsigned)((runs + 1ull) & 1ull);
    const unsigned long long* slot = tail + T_TOK + (par * 8 + b) * 2;
    unsigned long long cnt;
    const unsigned long long t0 = dev::globaltimer();
    do {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(cnt) : "l"(slot + 1) : "memory");
        if (dev::globaltimer() - t0 > 4000000000ull) __trap();
    } while ((long long)cnt != expect);
    unsigned long long key;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(key) : "l"(slot) : "memory");
    out[b] = (int)tok_of_key(key);
}

void destroy_model(fasq_llama* m) {
    if (!m) return;
    if (m->chain) chain_destroy(m->chain);
    for (__half* p : m->kc) dev_free(p, 0);
    for (__half* p : m->vc) dev_free(p, 0);
    dev_free(m->rope, 0);
    dev_free(m->tok_hist, 0);
    dev_free(m->logits, 0);
    dev_free(m->tok_dev, 0);
    if (m->tok_pin) cudaFreeHost(m->tok_pin);
    if (m->io_exec) cudaGraphExecDestroy(m->io_exec);
    if (m->pf_stream) cudaStreamSynchronize(m->pf_stream);   // no prefill in flight below
    if (m->pf_exec) cudaGraphExecDestroy(m->pf_exec);
    if (m->pf_buf) dev_free(m->pf_buf, 0);
    for (cudaEvent_t e : m->pf_ev)
        if (e) cudaEventDestroy(e);
    if (m->pf_stream) cudaStreamDestroy(m->pf_stream);
    delete m;
}

fasq_status lm_launch(fasq_llama* m, cudaStream_t st) {
    const fasq_llama_desc& D = m->desc;
    fasq_chain* c = m->chain;
    static bool attr_set = false;
    if (!attr_set) {
        size_t lim = set_max_dyn_smem(k_lm_head<kLmNW>);
        if (lim < m->lm_smem) { set_error("lm_head: SMEM plan exceeds the device limit"); return FASQ_E_UNSUPPORTED; }
        attr_set = true;
    }
    const int ds = m->last_step;
    k_lm_head<kLmNW><<<m->lm_ctas, kLmNW * 32, m->lm_smem, st>>>(
        static_cast<const __half*>(D.lm_head), m->vocab_l, m->vocab_l * D.rank, D.hidden, c->acc_off[ds][0],
        c->acc_ks[ds][0], D.world > 1, static_cast<const __half*>(D.final_norm), D.rms_eps, D.B, c->peers_dev,
        D.rank, c->arena_words, D.world, c->nctas, m->logits);
    FASQ_CUDA_TRY(cudaGetLastError());
    return FASQ_OK;
}

}  // namespace
}  // namespace fasq

using namespace fasq;


// ---- whole-model PREFILL (the paper's E2E protocol: a 128-token prompt) ----
// M prompt tokens of sequence 0 through every block with the prefill products
// (fasq_gemm AUTO: the tcgen05 decode kernel for M <= 128, EXPAND above) and
// plain kernels for the glue; it writes the KV cache of positions [pos0, pos0+M)
// and hands the decode chain the greedy token of the last prompt position at
// position pos0 + M.  Same arithmetic as the decode step (HF Llama, R14): fp32
// residual stream, fp16 PQ inputs and KV cache, RMSNorm as x = fp16(h * r * gamma).
namespace fasq {
namespace {

// one CTA per row m = row0 + blockIdx.x: the residual update, then the RMSNorm
// of the updated row, x[m - row0] = fp16(h[m] / sqrt(mean(h[m]^2) + eps) * gamma);
// the update is h[m] = E[tok[m]] (tok != null: the embedding, block 0's input),
// h[m] += y[m] (y != null: the previous product's residual add) or none.  n % 4
// == 0; each thread keeps up to PF_NV float4 groups of the row in registers (all
// loads issued before the reduction: one row per SM is latency-, not
// bandwidth-bound), the rest of a longer row streams through L1
constexpr int PF_NV = 8;
__global__ void __launch_bounds__(256) k_pf_resid_norm(float* __restrict__ h, const float* __restrict__ y,
                                                       const int* __restrict__ tok, const __half* __restrict__ E,
                                                       const __half* __restrict__ gamma, __half* __restrict__ x,
                                                       int n, float eps, int row0) {
    const int m = row0 + (int)blockIdx.x, n4 = n / 4;
    float4* hr = reinterpret_cast<float4*>(h + (size_t)m * n);
    const float4* yr = y ? reinterpret_cast<const float4*>(y + (size_t)m * n) : nullptr;
    const uint2* er = tok ? reinterpret_cast<const uint2*>(E + (size_t)tok[m] * n) : nullptr;
    auto update = [&](int c4) -> float4 {
        float4 v;
        if (er) {
            const uint2 e = er[c4];
            const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&e.x));
            const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&e.y));
            v = make_float4(a.x, a.y, b.x, b.y);
        } else {
            v = hr[c4];
            if (yr) {
                const float4 d = yr[c4];
                v.x += d.x; v.y += d.y; v.z += d.z; v.w += d.w;
            }
        }
        return v;
    };
    const uint2* gr = reinterpret_cast<const uint2*>(gamma);
    float4 vals[PF_NV];
    uint2 gv[PF_NV];   // gamma with the row (not one more round trip after the reduction)
#pragma unroll
    for (int k = 0; k < PF_NV; ++k) {
        const int c4 = threadIdx.x + k * blockDim.x;
        vals[k] = c4 < n4 ? update(c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        gv[k] = c4 < n4 ? gr[c4] : make_uint2(0u, 0u);
    }
    float a = 0.f;
    const bool write = er || yr;
#pragma unroll
    for (int k = 0; k < PF_NV; ++k) {
        const int c4 = threadIdx.x + k * blockDim.x;
        const float4 v = vals[k];
        a += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        if (write && c4 < n4) hr[c4] = v;
    }
    for (int c4 = threadIdx.x + PF_NV * blockDim.x; c4 < n4; c4 += blockDim.x) {
        const float4 v = update(c4);
        a += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        if (write) hr[c4] = v;
    }
    __shared__ float red[32];
    for (int o = 16; o >= 1; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
        float b = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
        for (int o = 16; o >= 1; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
        if (threadIdx.x == 0) red[0] = b;
    }
    __syncthreads();
    const float r = 1.0f / sqrtf(red[0] / (float)n + eps);
    uint2* xr = reinterpret_cast<uint2*>(x + (size_t)(m - row0) * n);
    auto emit = [&](int c4, float4 v, uint2 gg) {
        const float2 g0 = __half22float2(*reinterpret_cast<const __half2*>(&gg.x));
        const float2 g1 = __half22float2(*reinterpret_cast<const __half2*>(&gg.y));
        __half2 o[2] = {__floats2half2_rn(v.x * r * g0.x, v.y * r * g0.y),
                        __floats2half2_rn(v.z * r * g1.x, v.w * r * g1.y)};
        xr[c4] = *reinterpret_cast<const uint2*>(o);
    };
#pragma unroll
    for (int k = 0; k < PF_NV; ++k) {
        const int c4 = threadIdx.x + k * blockDim.x;
        if (c4 < n4) emit(c4, vals[k], gv[k]);
    }
    for (int c4 = threadIdx.x + PF_NV * blockDim.x; c4 < n4; c4 += blockDim.x) emit(c4, hr[c4], gr[c4]);   // own writes
}

// RoPE on q (in place, fp32) and k; the new k (rotated) / v enter the cache as fp16
__global__ void k_pf_rope_cache(float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
                                __half* __restrict__ kc, __half* __restrict__ vc, const float2* __restrict__ rope,
                                int M, const int* __restrict__ pos0_p, int H, int KV, int hd, int max_T) {
    const int pos0 = *pos0_p;   // device-resident: the cached prefill graph serves any pos0
    const int half = hd / 2;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int per = (H + 2 * KV) * half;   // rotation pairs (q, k) and v pairs per token
    if (i >= (int64_t)M * per) return;
    const int m = (int)(i / per), r = (int)(i - (int64_t)m * per);
    const int pos = pos0 + m;
    if (r < H * half) {
        const int hh = r / half, e = r - hh * half;
        const float2 cs = rope[(size_t)pos * half + e];
        float* qr = q + (size_t)m * H * hd + (size_t)hh * hd;
        const float q0 = qr[e], q1 = qr[e + half];
        qr[e] = q0 * cs.x - q1 * cs.y;
        qr[e + half] = q1 * cs.x + q0 * cs.y;
    } else if (r < (H + KV) * half) {
        const int j = (r - H * half) / half, e = (r - H * half) - j * half;
        const float2 cs = rope[(size_t)pos * half + e];
        const float* kr = k + (size_t)m * KV * hd + (size_t)j * hd;
        const float k0 = kr[e], k1 = kr[e + half];
        __half* dst = kc + ((size_t)j * max_T + pos) * hd;
        dst[e] = __float2half_rn(k0 * cs.x - k1 * cs.y);
        dst[e + half] = __float2half_rn(k1 * cs.x + k0 * cs.y);
    } else {
        const int j = (r - (H + KV) * half) / half, e = (r - (H + KV) * half) - j * half;
        const float* vr = v + (size_t)m * KV * hd + (size_t)j * hd;
        __half* dst = vc + ((size_t)j * max_T + pos) * hd;
        dst[e] = __float2half_rn(vr[e]);
        dst[e + half] = __float2half_rn(vr[e + half]);
    }
}

// causal GQA attention: one warp per (token m, G q heads of one KV head),
// positions t <= pos0 + m in chunks of 32 with an online softmax over chunks.
// Scores: lane L takes position t0 + L (its K row in 16-B loads, converted once
// and dotted with the G queries broadcast from shared memory); P.V: lane L holds
// DPL = hd / 32 consecutive output dims of each head and walks the chunk's V rows
// (loaded once for the G heads).  The chunk's K and V rows are in flight together.
template <int DPL, int G>
__global__ void __launch_bounds__(128, 3) k_pf_attn(const float* __restrict__ q, const __half* __restrict__ kc,
                                                    const __half* __restrict__ vc, __half* __restrict__ out, int M,
                                                    const int* __restrict__ pos0_p, int H, int KV, int max_T) {
    constexpr int hd = 32 * DPL;
    __shared__ __align__(16) float qs[4][G][hd];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int HG = H / G, wg = (int)blockIdx.x * 4 + w;
    if (wg >= M * HG) return;
    // the longest rows (last tokens) first: the tail wave holds the short ones
    const int mi = wg / HG, m = M - 1 - mi, hh0 = (wg - mi * HG) * G, j = hh0 / (H / KV), pos = *pos0_p + m;
    const float sc = 1.0f / sqrtf((float)hd);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float* qr = q + (size_t)m * H * hd + (size_t)(hh0 + g) * hd;
#pragma unroll
        for (int e = 0; e < DPL; ++e) qs[w][g][e * 32 + lane] = qr[e * 32 + lane];
    }
    __syncwarp();
    const __half* K = kc + (size_t)j * max_T * hd;
    const __half* V = vc + (size_t)j * max_T * hd + DPL * lane;
    float mx[G], l[G], o[G][DPL];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        mx[g] = -INFINITY;
        l[g] = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[g][e] = 0.f;
    }
    using VT = typename std::conditional<DPL == 4, uint2, unsigned>::type;
    for (int t0 = 0; t0 <= pos; t0 += 32) {
        const int t = t0 + lane;
        // rows past pos are clamped to pos (finite cache data) and weighted by p = 0
        VT vr[32];
#pragma unroll
        for (int tt = 0; tt < 32; ++tt)
            vr[tt] = *reinterpret_cast<const VT*>(V + (size_t)min(t0 + tt, pos) * hd);
        float s[G];
#pragma unroll
        for (int g = 0; g < G; ++g) s[g] = -INFINITY;
        if (t <= pos) {
            const uint4* kr = reinterpret_cast<const uint4*>(K + (size_t)t * hd);
            uint4 kv[hd / 8];
#pragma unroll
            for (int c = 0; c < hd / 8; ++c) kv[c] = kr[c];
            float acc[G];
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] = 0.f;
#pragma unroll
            for (int c = 0; c < hd / 8; ++c) {
                const __half2* k2 = reinterpret_cast<const __half2*>(&kv[c]);
                const float2 k0 = __half22float2(k2[0]), k1 = __half22float2(k2[1]);
                const float2 k2f = __half22float2(k2[2]), k3 = __half22float2(k2[3]);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float4 qa = *reinterpret_cast<const float4*>(&qs[w][g][8 * c]);
                    const float4 qb = *reinterpret_cast<const float4*>(&qs[w][g][8 * c + 4]);
                    acc[g] += qa.x * k0.x + qa.y * k0.y + qa.z * k1.x + qa.w * k1.y;
                    acc[g] += qb.x * k2f.x + qb.y * k2f.y + qb.z * k3.x + qb.w * k3.y;
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) s[g] = acc[g] * sc;
        }
        float p[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float cm = s[g];
            for (int off = 16; off >= 1; off >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, off));
            const float mn = fmaxf(mx[g], cm), cf = expf(mx[g] - mn);
            p[g] = t <= pos ? expf(s[g] - mn) : 0.f;
            float ps = p[g];
            for (int off = 16; off >= 1; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
            l[g] = l[g] * cf + ps;
#pragma unroll
            for (int e = 0; e < DPL; ++e) o[g][e] *= cf;
            mx[g] = mn;
        }
#pragma unroll
        for (int tt = 0; tt < 32; ++tt) {
            const __half* vh = reinterpret_cast<const __half*>(&vr[tt]);
            float vf[DPL];
#pragma unroll
            for (int e = 0; e < DPL; ++e) vf[e] = __half2float(vh[e]);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float pt = __shfl_sync(0xffffffffu, p[g], tt);
#pragma unroll
                for (int e = 0; e < DPL; ++e) o[g][e] += pt * vf[e];
            }
        }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
        __half* dst = out + (size_t)m * H * hd + (size_t)(hh0 + g) * hd + DPL * lane;
        const float inv = 1.0f / l[g];
#pragma unroll
        for (int e = 0; e < DPL; ++e) dst[e] = __float2half_rn(o[g][e] * inv);
    }
}

// ---- causal GQA attention on the tensor cores (mma.sync.m16n8k16, fp16 in, fp32
// accumulate), FlashAttention-2 style: a warp owns 16 consecutive tokens x one
// q head; S = Q K^T over 32-position chunks of its KV head's cache (staged in
// shared memory by the CTA, shared by its 4 warps = 4 (token block, head) items
// of that KV head), an online softmax over chunks in registers, P (fp16) re-used
// in registers as the A operand of O += P V (V fragments by ldmatrix.trans).
// Scores are scaled by 1/sqrt(hd) in fp32; q, P and the cache are fp16.
__device__ __forceinline__ void pf_mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pf_h2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

template <int HD>
__global__ void __launch_bounds__(128) k_pf_attn_tc(const float* __restrict__ q, const __half* __restrict__ kc,
                                                    const __half* __restrict__ vc, __half* __restrict__ out, int M,
                                                    const int* __restrict__ pos0_p, int H, int KV, int max_T) {
    constexpr int LD = HD + 8;   // halves per staged row (+16 B: conflict-free fragment loads)
    __shared__ __align__(16) __half Kbuf[2][32 * LD];   // double-buffered chunk staging (cp.async)
    __shared__ __align__(16) __half Vbuf[2][32 * LD];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int G = H / KV, NTB = (M + 15) / 16, n_items = NTB * G, ipj = (n_items + 3) / 4;
    const int j = (int)blockIdx.x / ipj, ib = (int)blockIdx.x - j * ipj;
    const int pos0 = *pos0_p;
    const int item = ib * 4 + warp;
    const bool active = item < n_items;
    const int tb = active ? item / G : 0, hh = j * G + (active ? item - (item / G) * G : 0);
    const int last_item = min(ib * 4 + 3, n_items - 1);
    const int pos_hi = pos0 + min(M - 1, (last_item / G) * 16 + 15);   // the CTA's last position
    const int r0 = tb * 16 + g, r1 = r0 + 8;                             // this thread's two rows (tokens)
    const int pr0 = pos0 + min(r0, M - 1), pr1 = pos0 + min(r1, M - 1);  // their last positions
    const float sc = 1.0f / sqrtf((float)HD);
    uint32_t qa[HD / 16][4];
    {
        const float* q0 = q + ((size_t)r0 * H + hh) * HD;
        const float* q1 = q + ((size_t)r1 * H + hh) * HD;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
            const int c = kk * 16 + 2 * t;
            float2 a = make_float2(0.f, 0.f), b = a, cc = a, d = a;
            if (active && r0 < M) {
                a = *reinterpret_cast<const float2*>(q0 + c);
                cc = *reinterpret_cast<const float2*>(q0 + c + 8);
            }
            if (active && r1 < M) {
                b = *reinterpret_cast<const float2*>(q1 + c);
                d = *reinterpret_cast<const float2*>(q1 + c + 8);
            }
            qa[kk][0] = pf_h2(a.x, a.y);
            qa[kk][1] = pf_h2(b.x, b.y);
            qa[kk][2] = pf_h2(cc.x, cc.y);
            qa[kk][3] = pf_h2(d.x, d.y);
        }
    }
    float o[HD / 8][4];
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
    float mx0 = -INFINITY, mx1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    const __half* K = kc + (size_t)j * max_T * HD;
    const __half* V = vc + (size_t)j * max_T * HD;
    // chunk c's rows [32 c, 32 c + 32) -> buffer c & 1 with cp.async (16 B each; rows
    // past the CTA's last position are zero-filled: src-size 0, never NaN garbage)
    auto stage = [&](int c) {
        const int t0s = c * 32;
        __half* ks = Kbuf[c & 1];
        __half* vs = Vbuf[c & 1];
        for (int i = threadIdx.x; i < 32 * HD / 8; i += 128) {
            const int r = i / (HD / 8), cc = i - r * (HD / 8);
            const bool ok = t0s + r <= pos_hi;
            const size_t off = (size_t)(ok ? t0s + r : 0) * HD + cc * 8;
            const uint32_t n = ok ? 16u : 0u;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                         :: "r"(dev::smem_u32(ks + r * LD + cc * 8)), "l"(K + off), "r"(n) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                         :: "r"(dev::smem_u32(vs + r * LD + cc * 8)), "l"(V + off), "r"(n) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int n_chunks = pos_hi / 32 + 1;
    stage(0);
    for (int ch = 0; ch < n_chunks; ++ch) {
        const int t0 = ch * 32;
        if (ch + 1 < n_chunks) {   // the next chunk's copies overlap this chunk's math
            stage(ch + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();   // chunk ch staged by every thread
        const __half* Ks = Kbuf[ch & 1];
        const __half* Vs = Vbuf[ch & 1];
        if (active && t0 <= pos0 + min(tb * 16 + 15, M - 1)) {   // warp-uniform: rows left for this warp
            float sv[4][4];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                sv[nt][0] = sv[nt][1] = sv[nt][2] = sv[nt][3] = 0.f;
                const __half* kr = Ks + (nt * 8 + g) * LD + 2 * t;
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk)
                    pf_mma(sv[nt], qa[kk], *reinterpret_cast<const uint32_t*>(kr + kk * 16),
                           *reinterpret_cast<const uint32_t*>(kr + kk * 16 + 8));
            }
            float m0n = mx0, m1n = mx1;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int p = t0 + nt * 8 + 2 * t + e;
                    sv[nt][e] = p <= pr0 ? sv[nt][e] * sc : -INFINITY;
                    sv[nt][2 + e] = p <= pr1 ? sv[nt][2 + e] * sc : -INFINITY;
                    m0n = fmaxf(m0n, sv[nt][e]);
                    m1n = fmaxf(m1n, sv[nt][2 + e]);
                }
            m0n = fmaxf(m0n, __shfl_xor_sync(0xffffffffu, m0n, 1));
            m0n = fmaxf(m0n, __shfl_xor_sync(0xffffffffu, m0n, 2));
            m1n = fmaxf(m1n, __shfl_xor_sync(0xffffffffu, m1n, 1));
            m1n = fmaxf(m1n, __shfl_xor_sync(0xffffffffu, m1n, 2));
            const float c0 = expf(mx0 - m0n), c1 = expf(mx1 - m1n);   // 0 on the first chunk (mx = -inf)
            float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    sv[nt][e] = expf(sv[nt][e] - m0n);
                    sv[nt][2 + e] = expf(sv[nt][2 + e] - m1n);
                    ls0 += sv[nt][e];
                    ls1 += sv[nt][2 + e];
                }
            ls0 += __shfl_xor_sync(0xffffffffu, ls0, 1);
            ls0 += __shfl_xor_sync(0xffffffffu, ls0, 2);
            ls1 += __shfl_xor_sync(0xffffffffu, ls1, 1);
            ls1 += __shfl_xor_sync(0xffffffffu, ls1, 2);
            l0 = l0 * c0 + ls0;
            l1 = l1 * c1 + ls1;
            mx0 = m0n;
            mx1 = m1n;
#pragma unroll
            for (int nd = 0; nd < HD / 8; ++nd) {
                o[nd][0] *= c0;
                o[nd][1] *= c0;
                o[nd][2] *= c1;
                o[nd][3] *= c1;
            }
#pragma unroll
            for (int k2 = 0; k2 < 2; ++k2) {   // 16 positions per k-step
                const uint32_t pa[4] = {pf_h2(sv[2 * k2][0], sv[2 * k2][1]), pf_h2(sv[2 * k2][2], sv[2 * k2][3]),
                                        pf_h2(sv[2 * k2 + 1][0], sv[2 * k2 + 1][1]),
                                        pf_h2(sv[2 * k2 + 1][2], sv[2 * k2 + 1][3])};
                const int vr = k2 * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
                for (int nd = 0; nd < HD / 8; nd += 2) {
                    const uint32_t va = dev::smem_u32(Vs + vr * LD + 8 * (nd + (lane >> 4)));
                    uint32_t b0, b1, b2, b3;
                    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3) : "r"(va));
                    pf_mma(o[nd], pa, b0, b1);
                    pf_mma(o[nd + 1], pa, b2, b3);
                }
            }
        }
        __syncthreads();   // buffer ch & 1 is re-staged by the next iteration's copy of chunk ch + 2
    }
    if (!active) return;
    const float i0 = 1.0f / l0, i1 = 1.0f / l1;
#pragma unroll
    for (int nd = 0; nd < HD / 8; ++nd) {
        const int c = nd * 8 + 2 * t;
        if (r0 < M)
            *reinterpret_cast<__half2*>(out + ((size_t)r0 * H + hh) * HD + c) =
                __floats2half2_rn(o[nd][0] * i0, o[nd][1] * i0);
        if (r1 < M)
            *reinterpret_cast<__half2*>(out + ((size_t)r1 * H + hh) * HD + c) =
                __floats2half2_rn(o[nd][2] * i1, o[nd][3] * i1);
    }
}

template <int DPL>
void pf_attn_launch(const float* q, const __half* kc, const __half* vc, __half* out, int M, const int* pos0, int H, int KV,
                    int max_T, cudaStream_t st) {
    if (!getenv("FASQ_PF_ATTN_SIMT")) {   // tensor cores (default); the SIMT kernel below is the A/B reference
        const int items = (M + 15) / 16 * (H / KV);
        k_pf_attn_tc<32 * DPL><<<(unsigned)(KV * ((items + 3) / 4)), 128, 0, st>>>(q, kc, vc, out, M, pos0, H, KV,
                                                                                  max_T);
        return;
    }
    const int grp = H / KV;
    const int G = grp % 4 == 0 ? 4 : grp % 2 == 0 ? 2 : 1;
    const unsigned blocks = (unsigned)(((int64_t)M * (H / G) + 3) / 4);
    if (G == 4)
        k_pf_attn<DPL, 4><<<blocks, 128, 0, st>>>(q, kc, vc, out, M, pos0, H, KV, max_T);
    else if (G == 2)
        k_pf_attn<DPL, 2><<<blocks, 128, 0, st>>>(q, kc, vc, out, M, pos0, H, KV, max_T);
    else
        k_pf_attn<DPL, 1><<<blocks, 128, 0, st>>>(q, kc, vc, out, M, pos0, H, KV, max_T);
}

__device__ __forceinline__ float pf_silu_mul(float x, float u) { return x / (1.0f + expf(-x)) * u; }

// a = fp16(silu(g) * u); n4 = n / 4 float4 groups, then the scalar tail
__global__ void k_pf_silu_mul(const float* __restrict__ g, const float* __restrict__ u, __half* __restrict__ a,
                              int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n4 = n / 4;
    if (i < n4) {
        const float4 gv = reinterpret_cast<const float4*>(g)[i], uv = reinterpret_cast<const float4*>(u)[i];
        __half2 r[2] = {__floats2half2_rn(pf_silu_mul(gv.x, uv.x), pf_silu_mul(gv.y, uv.y)),
                        __floats2half2_rn(pf_silu_mul(gv.z, uv.z), pf_silu_mul(gv.w, uv.w))};
        reinterpret_cast<uint2*>(a)[i] = *reinterpret_cast<const uint2*>(r);
    } else if (i < n4 + (n - 4 * n4)) {
        const int64_t k = 4 * n4 + (i - n4);
        a[k] = __float2half_rn(pf_silu_mul(g[k], u[k]));
    }
}

__device__ __forceinline__ unsigned long long pf_key(float f, unsigned tok) {
    const unsigned b = __float_as_uint(f);
    const unsigned ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);   // order-preserving
    return ((unsigned long long)ord << 32) | (unsigned long long)(0xFFFFFFFFu - tok);   // ties -> lowest id
}

// lm_head of ONE token: warps stride over the vocab rows (a lane's first 16
// 16-B loads of a row issued before any use), keep the max of (logit, ~token)
// keys, reduce in the CTA and publish ONE atomicMax per CTA (one per row
// serialises 128 K same-address atomics in L2)
__global__ void __launch_bounds__(256, 1) k_pf_lm_argmax(const __half* __restrict__ W, const __half* __restrict__ x,
                                                         int V, int n, unsigned long long* __restrict__ best) {
    __shared__ unsigned long long s_best[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = (int)blockIdx.x * 8 + warp, nw = (int)gridDim.x * 8;
    const uint4* xr = reinterpret_cast<const uint4*>(x);
    const int n8 = n / 8;
    auto dot8 = [](uint4 wv, uint4 xv) {
        const __half2* w2 = reinterpret_cast<const __half2*>(&wv);
        const __half2* x2 = reinterpret_cast<const __half2*>(&xv);
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 wf = __half22float2(w2[e]), xf = __half22float2(x2[e]);
            a += wf.x * xf.x + wf.y * xf.y;
        }
        return a;
    };
    constexpr int NL = 16;
    unsigned long long kb = 0ull;
    for (int row = gw; row < V; row += nw) {
        const uint4* wr = reinterpret_cast<const uint4*>(W + (size_t)row * n);
        float a = 0.f;
        int c0 = lane;
        if (n8 >= 32 * NL) {
            uint4 wv[NL];
#pragma unroll
            for (int k = 0; k < NL; ++k) wv[k] = __ldcs(wr + lane + 32 * k);
#pragma unroll
            for (int k = 0; k < NL; ++k) a += dot8(wv[k], xr[lane + 32 * k]);
            c0 += 32 * NL;
        }
        for (int c = c0; c < n8; c += 32) a += dot8(__ldcs(wr + c), xr[c]);
        for (int o = 16; o >= 1; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        kb = max(kb, pf_key(a, (unsigned)row));
    }
    if (lane == 0) s_best[warp] = kb;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long b = 0ull;
        for (int w = 0; w < 8; ++w) b = max(b, s_best[w]);
        if (b) atomicMax(best, b);
    }
}

__global__ void k_pf_token(const unsigned long long* __restrict__ best, int* __restrict__ tok) {
    tok[0] = (int)(0xFFFFFFFFu - (unsigned)(*best & 0xFFFFFFFFull));
}

inline unsigned pf_blocks(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

__global__ void k_pf_set(int* __restrict__ dst, int v) { *dst = v; }

}  // namespace
}  // namespace fasq

extern "C" {

fasq_status fasq_llama_create(const fasq_llama_desc* d, void* stream, fasq_llama** out) {
    if (!out) return FASQ_E_ARG;
    *out = nullptr;
    if (!d) return FASQ_E_ARG;
    const fasq_llama_desc& D = *d;
    if (D.n_layers < 1 || D.hidden < 64 || D.hidden % 64 || D.n_heads < 1 || D.n_kv_heads < 1 ||
        D.n_heads % D.n_kv_heads || D.head_dim < 8 || D.head_dim > 128 || D.head_dim % 8 || D.ffn < 1 ||
        D.vocab < 1 || D.max_T < 2 || D.B < 1 || D.B > 8 || D.world < 1 || D.world > 8 || D.rank < 0 ||
        D.rank >= D.world || D.max_ctas < 0)
        return FASQ_E_ARG;
    if (D.n_heads * D.head_dim != D.hidden || D.n_kv_heads % D.world || D.vocab % D.world || D.ffn % D.world)
        return FASQ_E_SHAPE;
    if (!D.q || !D.k || !D.v || !D.o || !D.gate || !D.up || !D.down || !D.attn_norm || !D.mlp_norm ||
        !D.final_norm || !D.embed || !D.lm_head)
        return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    fasq_llama* m = new fasq_llama();
    m->desc = D;
    const int W = D.world, hd = D.head_dim;
    m->n_heads_l = D.n_heads / W;
    m->n_kv_l = D.n_kv_heads / W;
    m->ffn_l = D.ffn / W;
    m->vocab_l = D.vocab / W;
    auto fail = [&](fasq_status s, const std::string& msg) {
        if (!msg.empty()) set_error("llama: " + msg);
        destroy_model(m);
        return s;
    };
    // shapes of this rank's shards
    const int64_t qo = (int64_t)m->n_heads_l * hd, kvo = (int64_t)m->n_kv_l * hd;
    for (int l = 0; l < D.n_layers; ++l) {
        const fasq_layer* Ls[7] = {D.q[l], D.k[l], D.v[l], D.o[l], D.gate[l], D.up[l], D.down[l]};
        const int64_t fo[7] = {qo, kvo, kvo, D.hidden, m->ffn_l, m->ffn_l, D.hidden};
        const int64_t fi[7] = {D.hidden, D.hidden, D.hidden, qo, D.hidden, D.hidden, m->ffn_l};
        for (int i = 0; i < 7; ++i) {
            if (!Ls[i]) return fail(FASQ_E_ARG, "null layer");
            if (Ls[i]->F_out != fo[i] || Ls[i]->F_in != fi[i])
                return fail(FASQ_E_SHAPE, "layer " + std::to_string(l) + "/" + std::to_string(i) +
                                              " is not this rank's shard shape");
            if (Ls[i]->d > 2) return fail(FASQ_E_UNSUPPORTED, "whole-model decode needs d <= 2");
        }
        if (!D.attn_norm[l] || !D.mlp_norm[l]) return fail(FASQ_E_ARG, "null norm weight");
    }
    // device buffers: KV caches, RoPE table, token history, attention partials
    const size_t cache_elems = (size_t)D.B * m->n_kv_l * D.max_T * hd;
    m->kc.assign(D.n_layers, nullptr);
    m->vc.assign(D.n_layers, nullptr);
    for (int l = 0; l < D.n_layers; ++l) {
        if (dev_alloc_t(&m->kc[l], cache_elems * 2, st) != FASQ_OK || dev_alloc_t(&m->vc[l], cache_elems * 2, st) != FASQ_OK)
            return fail(FASQ_E_OOM, "");
        if (cudaMemsetAsync(m->kc[l], 0, cache_elems * 2, st) != cudaSuccess ||
            cudaMemsetAsync(m->vc[l], 0, cache_elems * 2, st) != cudaSuccess)
            return fail(FASQ_E_CUDA, "cache memset");
    }
    {
        // RoPE (HF Llama rotate-half): inv_freq_i = theta^(-2i/hd), angle = pos * inv_freq_i
        std::vector<float2> tab((size_t)D.max_T * (hd / 2));
        for (int p = 0; p < D.max_T; ++p)
            for (int i = 0; i < hd / 2; ++i) {
                const double a = (double)p * std::pow((double)D.rope_theta, -2.0 * i / hd);
                tab[(size_t)p * (hd / 2) + i] = make_float2((float)std::cos(a), (float)std::sin(a));
            }
        if (dev_alloc_t(&m->rope, tab.size() * sizeof(float2), st) != FASQ_OK) return fail(FASQ_E_OOM, "");
        if (cudaMemcpyAsync(m->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(FASQ_E_CUDA, "rope upload");
    }
    const int sms = D.max_ctas > 0 ? std::min(D.max_ctas, sm_count()) : sm_count();
    int parts = 1;   // split the cache length so that heads x parts fill the GPU (<= 4: the o staging polls them at once)
    while (parts < 4 && m->n_heads_l * parts * 2 <= sms) parts *= 2;
    if (const char* e = getenv("FASQ_ATTN_PARTS")) parts = std::max(1, std::min(4, atoi(e)));
    if (dev_alloc_t(&m->tok_hist, (size_t)D.B * D.max_T * 4, st) != FASQ_OK || dev_alloc_t(&m->tok_dev, 64, st) != FASQ_OK)
        return fail(FASQ_E_OOM, "");
    if (cudaHostAlloc(&m->tok_pin, 64, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return fail(FASQ_E_OOM, "pinned token staging");
    }
    cudaMemsetAsync(m->tok_hist, 0, (size_t)D.B * D.max_T * 4, st);
    // step list: 0 = EMBED; block l: 1+5l qkv, 2+5l attn, 3+5l o(+h), 4+5l gate/up, 5+5l down(+h')
    std::vector<StepDesc> steps;
    StepDesc e;
    e.kind = SK_EMBED;
    e.embed = static_cast<const __half*>(D.embed);
    e.hidden = D.hidden;
    steps.push_back(e);
    int h_step = 0;   // step whose layer 0 holds the current residual stream h
    for (int l = 0; l < D.n_layers; ++l) {
        StepDesc qkv;
        qkv.kind = SK_PQ;
        qkv.layers = {D.q[l], D.k[l], D.v[l]};
        qkv.in_mode = IN_RMSNORM;
        qkv.src_step = h_step;
        qkv.gamma = static_cast<const __half*>(D.attn_norm[l]);
        qkv.eps = D.rms_eps;
        const int s_qkv = (int)steps.size();
        steps.push_back(qkv);
        StepDesc at;
        at.kind = SK_ATTN;
        at.q_step = s_qkv;
        at.n_heads = m->n_heads_l;
        at.n_kv = m->n_kv_l;
        at.head_dim = hd;
        at.kc = m->kc[l];
        at.vc = m->vc[l];
        const int s_at = (int)steps.size();
        steps.push_back(at);
        StepDesc o;
        o.kind = SK_PQ;
        o.layers = {D.o[l]};
        o.in_mode = IN_ATTN;
        o.src_step = s_at;
        o.lazy_step = h_step;   // h' = o + h, materialised by its consumers (chain_internal.cuh)
        o.out_all = W > 1;
        o.kshard = W > 1;
        const int s_o = (int)steps.size();
        steps.push_back(o);
        StepDesc gu;
        gu.kind = SK_PQ;
        gu.layers = {D.gate[l], D.up[l]};
        gu.in_mode = IN_RMSNORM;
        gu.src_step = s_o;
        gu.gamma = static_cast<const __half*>(D.mlp_norm[l]);
        // the scale of gate/up is applied by down's SwiGLU staging (measured: 1.440 ms/token vs 1.471
        // with scale_epilogue = true, where the slot round trip sits in the gate/up epilogue)
        gu.scale_epilogue = false;
        gu.eps = D.rms_eps;
        const int s_gu = (int)steps.size();
        steps.push_back(gu);
        StepDesc dn;
        dn.kind = SK_PQ;
        dn.layers = {D.down[l]};
        dn.in_mode = IN_SILU;
        dn.src_step = s_gu;
        dn.res_step = s_o;
        dn.res_here = D.rank == 0;
        dn.out_all = W > 1;
        dn.kshard = W > 1;
        h_step = (int)steps.size();
        steps.push_back(dn);
    }
    m->last_step = h_step;
    m->lm_ctas = sms;
    ChainModel cm;
    cm.rope = m->rope;
    cm.max_T = D.max_T;
    cm.pos_wrap = std::max(0, std::min(D.pos_wrap, D.max_T - 1));
    cm.tok_hist = m->tok_hist;
    cm.tok_expect = (long long)W * m->lm_ctas;
    cm.attn_parts = parts;
    fasq_status s = chain_build(steps, D.B, W, D.rank, D.max_ctas, false, &cm, st, &m->chain);
    if (s != FASQ_OK) return fail(s, "");
    m->lm_smem = (size_t)D.B * (D.hidden + 8) * 2;
    if (m->lm_smem > 200 * 1024) return fail(FASQ_E_UNSUPPORTED, "lm_head x staging exceeds SMEM");
    *out = m;
    return FASQ_OK;
}

fasq_status fasq_llama_ipc_handle(const fasq_llama* m, void* handle_out) {
    if (!m) return FASQ_E_ARG;
    return fasq_chain_ipc_handle(m->chain, handle_out);
}

fasq_status fasq_llama_set_peers(fasq_llama* m, const void* handles) {
    if (!m) return FASQ_E_ARG;
    return fasq_chain_set_peers(m->chain, handles);
}

fasq_status fasq_llama_set_peer_models(fasq_llama* m, const fasq_llama* const* models) {
    if (!m || !models) return FASQ_E_ARG;
    std::vector<const fasq_chain*> cs(m->desc.world);
    for (int r = 0; r < m->desc.world; ++r) {
        if (!models[r]) return FASQ_E_ARG;
        cs[r] = models[r]->chain;
    }
    return fasq_chain_set_peer_chains(m->chain, cs.data());
}

const fasq_chain* fasq_llama_chain(const fasq_llama* m) { return m ? m->chain : nullptr; }

fasq_status fasq_llama_kv_cache(const fasq_llama* m, int32_t layer, void** k_dev, void** v_dev) {
    if (!m || layer < 0 || layer >= m->desc.n_layers || !k_dev || !v_dev) return FASQ_E_ARG;
    *k_dev = m->kc[layer];
    *v_dev = m->vc[layer];
    return FASQ_OK;
}

fasq_status fasq_llama_reset(fasq_llama* m, const int32_t* tokens_host, int32_t pos, void* stream) {
    if (!m || !tokens_host) return FASQ_E_ARG;
    if (pos >= m->desc.max_T) return FASQ_E_ARG;
    for (int b = 0; b < m->desc.B; ++b)
        if (tokens_host[b] < 0 || tokens_host[b] >= m->desc.vocab) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    FASQ_CUDA_TRY(cudaMemcpyAsync(m->tok_dev, tokens_host, (size_t)m->desc.B * 4, cudaMemcpyHostToDevice, st));
    k_llama_reset<<<1, 32, 0, st>>>(m->chain->tail(), m->chain->nctas, m->tok_dev, m->desc.B, pos,
                                    (long long)m->desc.world * m->lm_ctas);
    FASQ_CUDA_TRY(cudaGetLastError());
    FASQ_CUDA_TRY(cudaStreamSynchronize(st));   // tokens_host may go away
    set_launch_count(1);
    return FASQ_OK;
}

fasq_status fasq_llama_step(fasq_llama* m, void* stream) {
    if (!m) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    fasq_status s = chain_launch(m->chain, m->rope /* unused external input */, st);
    if (s == FASQ_OK) s = lm_launch(m, st);
    if (s == FASQ_OK) set_launch_count(2);
    return s;
}

fasq_status fasq_llama_step_ex(fasq_llama* m, void* stream, int32_t part) {
    if (!m || part < 0 || part > 2) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    fasq_status s = FASQ_OK;
    if (part != 2) s = chain_launch(m->chain, m->rope /* unused external input */, st);
    if (s == FASQ_OK && part != 1) s = lm_launch(m, st);
    if (s == FASQ_OK) set_launch_count(part == 0 ? 2 : 1);
    return s;
}

fasq_status fasq_llama_tokens(const fasq_llama* m, int32_t* tokens_dev, void* stream) {
    if (!m || !tokens_dev) return FASQ_E_ARG;
    k_llama_tokens<<<1, 32, 0, (cudaStream_t)stream>>>(m->chain->tail(), m->chain->nctas, m->desc.B,
                                                       (long long)m->desc.world * m->lm_ctas, tokens_dev);
    FASQ_CUDA_TRY(cudaGetLastError());
    set_launch_count(1);
    return FASQ_OK;
}

fasq_status fasq_llama_step_host(fasq_llama* m, int32_t* tokens_out_host, void* stream) {
    if (!m || !tokens_out_host) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    fasq_status s = chain_launch(m->chain, m->rope, st);
    if (s == FASQ_OK) s = lm_launch(m, st);
    if (s == FASQ_OK) {
        k_llama_tokens<<<1, 32, 0, st>>>(m->chain->tail(), m->chain->nctas, m->desc.B,
                                         (long long)m->desc.world * m->lm_ctas, m->tok_dev);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpyAsync(tokens_out_host, m->tok_dev, (size_t)m->desc.B * 4,
                                                  cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) s = cuda_fail(e, "llama step_host");
    }
    if (s == FASQ_OK) set_launch_count(3);
    return s;
}

fasq_status fasq_llama_step_io(fasq_llama* m, const int32_t* tokens_in_host, int32_t pos, int32_t* tokens_out_host,
                               void* stream) {
    if (!m || !tokens_in_host || !tokens_out_host) return FASQ_E_ARG;
    if (pos >= m->desc.max_T) return FASQ_E_ARG;
    const int B = m->desc.B;
    for (int b = 0; b < B; ++b)
        if (tokens_in_host[b] < 0 || tokens_in_host[b] >= m->desc.vocab) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    // the input tokens go through the model's pinned staging (the copy is truly
    // asynchronous and the caller's buffer is free on return); ONE synchronisation
    // at the end instead of fasq_llama_reset's + fasq_llama_step_host's two
    auto enqueue = [&](cudaStream_t q, int p) -> fasq_status {
        cudaError_t e = cudaMemcpyAsync(m->tok_dev, m->tok_pin, (size_t)B * 4, cudaMemcpyHostToDevice, q);
        if (e != cudaSuccess) return cuda_fail(e, "llama step_io H2D");
        k_llama_reset<<<1, 32, 0, q>>>(m->chain->tail(), m->chain->nctas, m->tok_dev, B, p,
                                       (long long)m->desc.world * m->lm_ctas);
        FASQ_CUDA_TRY(cudaGetLastError());
        fasq_status s = chain_launch(m->chain, m->rope, q);
        if (s == FASQ_OK) s = lm_launch(m, q);
        if (s != FASQ_OK) return s;
        k_llama_tokens<<<1, 32, 0, q>>>(m->chain->tail(), m->chain->nctas, B, (long long)m->desc.world * m->lm_ctas,
                                        m->tok_dev + 8);
        FASQ_CUDA_TRY(cudaGetLastError());
        FASQ_CUDA_TRY(cudaMemcpyAsync(m->tok_pin + 8, m->tok_dev + 8, (size_t)B * 4, cudaMemcpyDeviceToHost, q));
        return FASQ_OK;
    };
    for (int b = 0; b < B; ++b) m->tok_pin[b] = tokens_in_host[b];
    fasq_status s = FASQ_OK;
    if (pos < 0 && getenv("FASQ_LLAMA_IO_GRAPH") == nullptr) {
        // continue at the current position: the six operations as ONE graph launch
        // (captured once on a private stream; the graph's addresses are the model's)
        if (!m->io_exec) {
            cudaStream_t cs;
            FASQ_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            cudaGraph_t g = nullptr;
            cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
            if (e == cudaSuccess) {
                s = enqueue(cs, -1);
                e = cudaStreamEndCapture(cs, &g);
            }
            if (e == cudaSuccess && s == FASQ_OK) e = cudaGraphInstantiate(&m->io_exec, g, 0);
            if (g) cudaGraphDestroy(g);
            cudaStreamDestroy(cs);
            if (s != FASQ_OK) return s;
            if (e != cudaSuccess) { m->io_exec = nullptr; return cuda_fail(e, "llama step_io graph"); }
        }
        FASQ_CUDA_TRY(cudaGraphLaunch(m->io_exec, st));
    } else {
        s = enqueue(st, pos);
    }
    if (s == FASQ_OK) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) s = cuda_fail(e, "llama step_io");
    }
    if (s == FASQ_OK) {
        for (int b = 0; b < B; ++b) tokens_out_host[b] = m->tok_pin[8 + b];
        set_launch_count(4);
    }
    return s;
}

}  // extern "C"

namespace fasq {
namespace {

// prefill working set for M tokens (fp32 residual / products, fp16 inputs)
struct PfBufs {
    float *h, *q, *k, *v, *y, *g, *u;
    __half *x, *a;
    unsigned long long* best;
};

size_t pf_layout(const fasq_llama_desc& D, int M, PfBufs* b, uint8_t* base) {
    const int n = D.hidden, H = D.n_heads, KV = D.n_kv_heads, hd = D.head_dim, ffn = D.ffn;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* p = base ? base + off : nullptr;
        off += (bytes + 255) / 256 * 256;
        return p;
    };
    const size_t Mn = (size_t)M * n;
    PfBufs t;
    t.h = reinterpret_cast<float*>(take(Mn * 4));
    t.q = reinterpret_cast<float*>(take((size_t)M * H * hd * 4));
    t.k = reinterpret_cast<float*>(take((size_t)M * KV * hd * 4));
    t.v = reinterpret_cast<float*>(take((size_t)M * KV * hd * 4));
    t.y = reinterpret_cast<float*>(take(Mn * 4));
    t.g = reinterpret_cast<float*>(take((size_t)M * ffn * 4));
    t.u = reinterpret_cast<float*>(take((size_t)M * ffn * 4));
    t.x = reinterpret_cast<__half*>(take((size_t)M * std::max(n, std::max(ffn, H * hd)) * 2));
    t.a = reinterpret_cast<__half*>(take((size_t)M * std::max(ffn, H * hd) * 2));
    t.best = reinterpret_cast<unsigned long long*>(take(8));
    if (b) *b = t;
    return off;
}

// The whole prefill as stream work on st: tokens / pos0 read from device memory
// (so the captured graph serves any prompt and position of M tokens).
fasq_status pf_enqueue(fasq_llama* m, const int* tok, const int* pos0_p, int M, const PfBufs& B, cudaStream_t st) {
    const fasq_llama_desc& D = m->desc;
    const int n = D.hidden, H = D.n_heads, KV = D.n_kv_heads, hd = D.head_dim, ffn = D.ffn;
    float *h = B.h, *q = B.q, *k = B.k, *v = B.v, *y = B.y, *g = B.g, *u = B.u;
    __half *x = B.x, *a = B.a;
    fasq_status s = FASQ_OK;
    auto check = [&](cudaError_t e, const char* w) { if (s == FASQ_OK && e != cudaSuccess) s = cuda_fail(e, w); };
    auto gemm = [&](const fasq_layer* L, const __half* X, float* Y) {
        if (s == FASQ_OK) s = fasq_gemm(L, X, M, Y, FASQ_F32, FASQ_GEMM_AUTO, st);
    };
    // products sharing their input (q / k / v, gate / up): one EXPAND launch above the short-L crossover
    auto gemm_group = [&](std::initializer_list<const fasq_layer*> Ls, const __half* X,
                          std::initializer_list<float*> Ys) {
        const fasq_layer* lv[4];
        void* yv[4];
        int c = 0;
        for (const fasq_layer* L : Ls) lv[c++] = L;
        c = 0;
        for (float* Y : Ys) yv[c++] = Y;
        if (s == FASQ_OK) s = fasq_gemm_grouped(lv, c, X, M, yv, FASQ_F32, FASQ_GEMM_AUTO, st);
    };
    for (int l = 0; l < D.n_layers && s == FASQ_OK; ++l) {
        // block 0: h = embedding; block l > 0: h += the previous block's down product
        k_pf_resid_norm<<<M, 256, 0, st>>>(h, l ? y : nullptr, l ? nullptr : tok, static_cast<const __half*>(D.embed),
                                           static_cast<const __half*>(D.attn_norm[l]), x, n, D.rms_eps, 0);
        check(cudaGetLastError(), "prefill rmsnorm");
        gemm_group({D.q[l], D.k[l], D.v[l]}, x, {q, k, v});
        if (s != FASQ_OK) break;
        k_pf_rope_cache<<<pf_blocks((int64_t)M * (H + 2 * KV) * (hd / 2), 256), 256, 0, st>>>(
            q, k, v, m->kc[l], m->vc[l], m->rope, M, pos0_p, H, KV, hd, D.max_T);
        check(cudaGetLastError(), "prefill rope");
        if (hd == 128)
            pf_attn_launch<4>(q, m->kc[l], m->vc[l], a, M, pos0_p, H, KV, D.max_T, st);
        else
            pf_attn_launch<2>(q, m->kc[l], m->vc[l], a, M, pos0_p, H, KV, D.max_T, st);
        check(cudaGetLastError(), "prefill attention");
        gemm(D.o[l], a, y);
        if (s != FASQ_OK) break;
        k_pf_resid_norm<<<M, 256, 0, st>>>(h, y, nullptr, nullptr, static_cast<const __half*>(D.mlp_norm[l]), x, n,
                                           D.rms_eps, 0);
        check(cudaGetLastError(), "prefill mlp norm");
        gemm_group({D.gate[l], D.up[l]}, x, {g, u});
        if (s != FASQ_OK) break;
        k_pf_silu_mul<<<pf_blocks((int64_t)M * ffn / 4 + 3, 256), 256, 0, st>>>(g, u, a, (int64_t)M * ffn);
        check(cudaGetLastError(), "prefill swiglu");
        gemm(D.down[l], a, y);
    }
    if (s == FASQ_OK) {
        // the last prompt position's greedy token -> the decode chain's token slot;
        // only the last position's residual is still needed: its final add + norm
        k_pf_resid_norm<<<1, 256, 0, st>>>(h, y, nullptr, nullptr, static_cast<const __half*>(D.final_norm), x, n,
                                           D.rms_eps, M - 1);
        check(cudaMemsetAsync(B.best, 0, 8, st), "prefill argmax");
        k_pf_lm_argmax<<<std::min<int64_t>(pf_blocks(D.vocab, 8), (int64_t)sm_count() * 2), 256, 0, st>>>(
            static_cast<const __half*>(D.lm_head), x, D.vocab, n, B.best);
        k_pf_token<<<1, 1, 0, st>>>(B.best, m->tok_dev);
        k_llama_reset<<<1, 32, 0, st>>>(m->chain->tail(), m->chain->nctas, m->tok_dev, 1, M,
                                        (long long)D.world * m->lm_ctas, pos0_p);
        check(cudaGetLastError(), "prefill token");
    }
    return s;
}

}  // namespace
}  // namespace fasq

extern "C" {

fasq_status fasq_llama_prefill(fasq_llama* m, const int32_t* tokens_dev, int32_t M, int32_t pos0, void* stream) {
    if (!m || !tokens_dev || M < 1 || pos0 < 0) return FASQ_E_ARG;
    const fasq_llama_desc& D = m->desc;
    if (pos0 + M > D.max_T) return FASQ_E_ARG;
    if (D.B != 1 || D.world != 1 || (D.head_dim != 128 && D.head_dim != 64) || D.hidden % 8) {
        set_error("llama prefill: one sequence (B = 1), one GPU, head_dim 64 or 128");
        return FASQ_E_UNSUPPORTED;
    }
    cudaStream_t st = (cudaStream_t)stream;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    FASQ_CUDA_TRY(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone || getenv("FASQ_PREFILL_EAGER")) {
        // the caller is capturing (or asked for eager launches): per-call working
        // set and staging (stream-ordered allocations become graph memory nodes)
        PfBufs B;
        const size_t bytes = pf_layout(D, M, nullptr, nullptr);
        uint8_t* base = nullptr;
        int* pos_d = nullptr;
        fasq_status s = dev_alloc_t(&base, bytes, st);
        if (s == FASQ_OK) s = dev_alloc_t(&pos_d, sizeof(int), st);
        if (s == FASQ_OK) {
            pf_layout(D, M, &B, base);
            k_pf_set<<<1, 1, 0, st>>>(pos_d, pos0);
            s = pf_enqueue(m, tokens_dev, pos_d, M, B, st);
        }
        dev_free(pos_d, st);
        dev_free(base, st);
        if (s == FASQ_OK) set_launch_count(1 + 8 * D.n_layers + 5);
        return s;
    }
    // Not capturing: the prefill of M tokens runs as ONE cached CUDA graph on a
    // private stream joined to `stream` (the ~230 launches of a Llama-3-8B
    // prefill cost ~0.5 ms of host launch time eagerly).  The first call for a
    // given M runs eagerly on that stream -- which also sizes its split-K
    // workspaces -- and captures the graph for the next calls; tokens and pos0
    // are staged into device memory the graph reads.
    if (!m->pf_stream) {
        FASQ_CUDA_TRY(cudaStreamCreateWithFlags(&m->pf_stream, cudaStreamNonBlocking));
        FASQ_CUDA_TRY(cudaEventCreateWithFlags(&m->pf_ev[0], cudaEventDisableTiming));
        FASQ_CUDA_TRY(cudaEventCreateWithFlags(&m->pf_ev[1], cudaEventDisableTiming));
    }
    cudaStream_t ps = m->pf_stream;
    FASQ_CUDA_TRY(cudaEventRecord(m->pf_ev[0], st));
    FASQ_CUDA_TRY(cudaStreamWaitEvent(ps, m->pf_ev[0], 0));
    fasq_status s = FASQ_OK;
    if (M > m->pf_cap) {   // grow the persistent working set; the old graph referenced the old one
        if (m->pf_exec) {
            cudaStreamSynchronize(ps);   // rare path: no launch of the old graph in flight
            cudaGraphExecDestroy(m->pf_exec);
            m->pf_exec = nullptr;
            m->pf_exec_M = 0;
        }
        dev_free(m->pf_buf, ps);
        m->pf_buf = nullptr;
        m->pf_cap = 0;
        const size_t bytes = pf_layout(D, M, nullptr, nullptr) + (size_t)(M + 1) * sizeof(int) + 256;
        s = dev_alloc_t(&m->pf_buf, bytes, ps);
        if (s == FASQ_OK) {
            m->pf_cap = M;
            m->pf_tok = reinterpret_cast<int*>(m->pf_buf + pf_layout(D, M, nullptr, nullptr));
        }
    }
    if (s == FASQ_OK) {
        PfBufs B;
        pf_layout(D, m->pf_cap, &B, m->pf_buf);
        int* pos_d = m->pf_tok + m->pf_cap;
        cudaError_t e = cudaMemcpyAsync(m->pf_tok, tokens_dev, (size_t)M * sizeof(int), cudaMemcpyDeviceToDevice, ps);
        if (e != cudaSuccess) s = cuda_fail(e, "prefill tokens");
        if (s == FASQ_OK) {
            k_pf_set<<<1, 1, 0, ps>>>(pos_d, pos0);
            if (m->pf_exec && m->pf_exec_M == M) {
                e = cudaGraphLaunch(m->pf_exec, ps);
                if (e != cudaSuccess) s = cuda_fail(e, "prefill graph launch");
                if (s == FASQ_OK) set_launch_count(2);
            } else {
                s = pf_enqueue(m, m->pf_tok, pos_d, M, B, ps);   // this call's prefill, eagerly
                if (s == FASQ_OK) {
                    // capture the same sequence for the next calls with this M
                    if (m->pf_exec) cudaGraphExecDestroy(m->pf_exec);
                    m->pf_exec = nullptr;
                    m->pf_exec_M = 0;
                    cudaGraph_t gr = nullptr;
                    e = cudaStreamBeginCapture(ps, cudaStreamCaptureModeThreadLocal);
                    if (e == cudaSuccess) {
                        const fasq_status sc = pf_enqueue(m, m->pf_tok, pos_d, M, B, ps);
                        e = cudaStreamEndCapture(ps, &gr);
                        if (sc == FASQ_OK && e == cudaSuccess &&
                            cudaGraphInstantiate(&m->pf_exec, gr, 0) == cudaSuccess)
                            m->pf_exec_M = M;
                        if (gr) cudaGraphDestroy(gr);
                    }
                    cudaGetLastError();   // a failed capture only leaves the next call eager
                    set_launch_count(1 + 8 * D.n_layers + 5);
                }
            }
        }
    }
    FASQ_CUDA_TRY(cudaEventRecord(m->pf_ev[1], ps));
    FASQ_CUDA_TRY(cudaStreamWaitEvent(st, m->pf_ev[1], 0));
    return s;
}

fasq_status fasq_llama_logits(fasq_llama* m, int32_t enable, void** logits_dev) {
    if (!m) return FASQ_E_ARG;
    if (enable && !m->logits) {
        if (dev_alloc_t(&m->logits, (size_t)m->desc.B * m->vocab_l * 4, 0) != FASQ_OK) return FASQ_E_OOM;
        FASQ_CUDA_TRY(cudaStreamSynchronize(0));
    }
    if (!enable && m->logits) {
        cudaDeviceSynchronize();
        dev_free(m->logits, 0);
        m->logits = nullptr;
    }
    if (logits_dev) *logits_dev = m->logits;
    return FASQ_OK;
}

fasq_status fasq_llama_token_history(const fasq_llama* m, int32_t* hist_dev, void* stream) {
    if (!m || !hist_dev) return FASQ_E_ARG;
    FASQ_CUDA_TRY(cudaMemcpyAsync(hist_dev, m->tok_hist, (size_t)m->desc.B * m->desc.max_T * 4,
                                  cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return FASQ_OK;
}

void fasq_llama_free(fasq_llama* m) {
    if (!m) return;
    cudaDeviceSynchronize();
    destroy_model(m);
}

}  // extern "C"
