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
                              long long expect) {
    const int b = threadIdx.x;
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

__global__ void k_pf_embed(const int* __restrict__ tok, const __half* __restrict__ E, float* __restrict__ h, int M,
                           int n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)M * n) return;
    const int m = (int)(i / n), c = (int)(i - (int64_t)m * n);
    h[i] = __half2float(E[(size_t)tok[m] * n + c]);
}

// one CTA per row: x[m] = fp16(h[m] / sqrt(mean(h[m]^2) + eps) * gamma)
__global__ void k_pf_rmsnorm(const float* __restrict__ h, const __half* __restrict__ gamma, __half* __restrict__ x,
                             int n, float eps, int row0) {
    const int m = row0 + (int)blockIdx.x;
    const float* hr = h + (size_t)m * n;
    float a = 0.f;
    for (int c = threadIdx.x; c < n; c += blockDim.x) a += hr[c] * hr[c];
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
    for (int c = threadIdx.x; c < n; c += blockDim.x)
        x[(size_t)(m - row0) * n + c] = __float2half_rn(hr[c] * r * __half2float(gamma[c]));
}

// RoPE on q (in place, fp32) and k; the new k (rotated) / v enter the cache as fp16
__global__ void k_pf_rope_cache(float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
                                __half* __restrict__ kc, __half* __restrict__ vc, const float2* __restrict__ rope,
                                int M, int pos0, int H, int KV, int hd, int max_T) {
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

// causal GQA attention: one warp per (token m, q head); lane holds DPL = hd / 32
// consecutive dims (hd = 64 or 128); one pass over the positions t <= pos0 + m
// with an online softmax
template <int DPL>
__global__ void k_pf_attn(const float* __restrict__ q, const __half* __restrict__ kc, const __half* __restrict__ vc,
                          __half* __restrict__ out, int M, int pos0, int H, int KV, int max_T) {
    constexpr int hd = 32 * DPL;
    const int wg = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (wg >= M * H) return;
    const int m = wg / H, hh = wg - m * H, j = hh / (H / KV), pos = pos0 + m;
    const float sc = 1.0f / sqrtf((float)hd);
    const float* qr = q + (size_t)m * H * hd + (size_t)hh * hd + DPL * lane;
    float qv[DPL], o[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) { qv[e] = qr[e]; o[e] = 0.f; }
    const __half* K = kc + (size_t)j * max_T * hd + DPL * lane;
    const __half* V = vc + (size_t)j * max_T * hd + DPL * lane;
    float mx = -INFINITY, l = 0.f;
    for (int t = 0; t <= pos; ++t) {
        __half kh[DPL], vh[DPL];
#pragma unroll
        for (int e = 0; e < DPL; e += 2) {
            *reinterpret_cast<__half2*>(kh + e) = *reinterpret_cast<const __half2*>(K + (size_t)t * hd + e);
            *reinterpret_cast<__half2*>(vh + e) = *reinterpret_cast<const __half2*>(V + (size_t)t * hd + e);
        }
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) s += qv[e] * __half2float(kh[e]);
        for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        s *= sc;
        const float mn = fmaxf(mx, s), cf = expf(mx - mn), p = expf(s - mn);
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[e] = o[e] * cf + p * __half2float(vh[e]);
        l = l * cf + p;
        mx = mn;
    }
    __half* dst = out + (size_t)m * H * hd + (size_t)hh * hd + DPL * lane;
    const float inv = 1.0f / l;
#pragma unroll
    for (int e = 0; e < DPL; ++e) dst[e] = __float2half_rn(o[e] * inv);
}

__global__ void k_pf_silu_mul(const float* __restrict__ g, const float* __restrict__ u, __half* __restrict__ a,
                              int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float x = g[i];
    a[i] = __float2half_rn(x / (1.0f + expf(-x)) * u[i]);
}

__global__ void k_pf_add(float* __restrict__ h, const float* __restrict__ y, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) h[i] += y[i];
}

__device__ __forceinline__ unsigned long long pf_key(float f, unsigned tok) {
    const unsigned b = __float_as_uint(f);
    const unsigned ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);   // order-preserving
    return ((unsigned long long)ord << 32) | (unsigned long long)(0xFFFFFFFFu - tok);   // ties -> lowest id
}

// lm_head of ONE token: a warp per vocab row (16-B loads), max of (logit, ~token) keys
__global__ void k_pf_lm_argmax(const __half* __restrict__ W, const __half* __restrict__ x, int V, int n,
                               unsigned long long* __restrict__ best) {
    const int row = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (row >= V) return;
    const uint4* wr = reinterpret_cast<const uint4*>(W + (size_t)row * n);
    const uint4* xr = reinterpret_cast<const uint4*>(x);
    float a = 0.f;
    for (int c = lane; c < n / 8; c += 32) {
        const uint4 wv = __ldg(wr + c), xv = xr[c];
        const __half2* w2 = reinterpret_cast<const __half2*>(&wv);
        const __half2* x2 = reinterpret_cast<const __half2*>(&xv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 wf = __half22float2(w2[e]), xf = __half22float2(x2[e]);
            a += wf.x * xf.x + wf.y * xf.y;
        }
    }
    for (int o = 16; o >= 1; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) atomicMax(best, pf_key(a, (unsigned)row));
}

__global__ void k_pf_token(const unsigned long long* __restrict__ best, int* __restrict__ tok) {
    tok[0] = (int)(0xFFFFFFFFu - (unsigned)(*best & 0xFFFFFFFFull));
}

inline unsigned pf_blocks(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

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

fasq_status fasq_llama_prefill(fasq_llama* m, const int32_t* tokens_dev, int32_t M, int32_t pos0, void* stream) {
    if (!m || !tokens_dev || M < 1 || pos0 < 0) return FASQ_E_ARG;
    const fasq_llama_desc& D = m->desc;
    if (pos0 + M > D.max_T) return FASQ_E_ARG;
    if (D.B != 1 || D.world != 1 || (D.head_dim != 128 && D.head_dim != 64) || D.hidden % 8) {
        set_error("llama prefill: one sequence (B = 1), one GPU, head_dim 64 or 128");
        return FASQ_E_UNSUPPORTED;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int n = D.hidden, H = D.n_heads, KV = D.n_kv_heads, hd = D.head_dim, ffn = D.ffn;
    const int64_t Mn = (int64_t)M * n;
    float *h = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *y = nullptr, *g = nullptr, *u = nullptr;
    __half *x = nullptr, *a = nullptr;
    unsigned long long* best = nullptr;
    fasq_status s = dev_alloc_t(&h, (size_t)Mn * 4, st);
    if (s == FASQ_OK) s = dev_alloc_t(&q, (size_t)M * H * hd * 4, st);
    if (s == FASQ_OK) s = dev_alloc_t(&k, (size_t)M * KV * hd * 4, st);
    if (s == FASQ_OK) s = dev_alloc_t(&v, (size_t)M * KV * hd * 4, st);
    if (s == FASQ_OK) s = dev_alloc_t(&y, (size_t)Mn * 4, st);
    if (s == FASQ_OK) s = dev_alloc_t(&g, (size_t)M * ffn * 4, st);
    if (s == FASQ_OK) s = dev_alloc_t(&u, (size_t)M * ffn * 4, st);
    if (s == FASQ_OK) s = dev_alloc_t(&x, (size_t)M * std::max(n, std::max(ffn, H * hd)) * 2, st);
    if (s == FASQ_OK) s = dev_alloc_t(&a, (size_t)M * std::max(ffn, H * hd) * 2, st);
    if (s == FASQ_OK) s = dev_alloc_t(&best, 8, st);
    auto check = [&](cudaError_t e, const char* w) { if (s == FASQ_OK && e != cudaSuccess) s = cuda_fail(e, w); };
    auto gemm = [&](const fasq_layer* L, const __half* X, float* Y) {
        if (s == FASQ_OK) s = fasq_gemm(L, X, M, Y, FASQ_F32, FASQ_GEMM_AUTO, st);
    };
    if (s == FASQ_OK) {
        k_pf_embed<<<pf_blocks(Mn, 256), 256, 0, st>>>(tokens_dev, static_cast<const __half*>(D.embed), h, M, n);
        check(cudaGetLastError(), "prefill embed");
    }
    for (int l = 0; l < D.n_layers && s == FASQ_OK; ++l) {
        k_pf_rmsnorm<<<M, 256, 0, st>>>(h, static_cast<const __half*>(D.attn_norm[l]), x, n, D.rms_eps, 0);
        check(cudaGetLastError(), "prefill rmsnorm");
        gemm(D.q[l], x, q);
        gemm(D.k[l], x, k);
        gemm(D.v[l], x, v);
        if (s != FASQ_OK) break;
        k_pf_rope_cache<<<pf_blocks((int64_t)M * (H + 2 * KV) * (hd / 2), 256), 256, 0, st>>>(
            q, k, v, m->kc[l], m->vc[l], m->rope, M, pos0, H, KV, hd, D.max_T);
        check(cudaGetLastError(), "prefill rope");
        if (hd == 128)
            k_pf_attn<4><<<pf_blocks((int64_t)M * H * 32, 256), 256, 0, st>>>(q, m->kc[l], m->vc[l], a, M, pos0, H, KV,
                                                                               D.max_T);
        else
            k_pf_attn<2><<<pf_blocks((int64_t)M * H * 32, 256), 256, 0, st>>>(q, m->kc[l], m->vc[l], a, M, pos0, H, KV,
                                                                               D.max_T);
        check(cudaGetLastError(), "prefill attention");
        gemm(D.o[l], a, y);
        if (s != FASQ_OK) break;
        k_pf_add<<<pf_blocks(Mn, 256), 256, 0, st>>>(h, y, Mn);
        k_pf_rmsnorm<<<M, 256, 0, st>>>(h, static_cast<const __half*>(D.mlp_norm[l]), x, n, D.rms_eps, 0);
        check(cudaGetLastError(), "prefill mlp norm");
        gemm(D.gate[l], x, g);
        gemm(D.up[l], x, u);
        if (s != FASQ_OK) break;
        k_pf_silu_mul<<<pf_blocks((int64_t)M * ffn, 256), 256, 0, st>>>(g, u, a, (int64_t)M * ffn);
        check(cudaGetLastError(), "prefill swiglu");
        gemm(D.down[l], a, y);
        if (s != FASQ_OK) break;
        k_pf_add<<<pf_blocks(Mn, 256), 256, 0, st>>>(h, y, Mn);
        check(cudaGetLastError(), "prefill residual");
    }
    if (s == FASQ_OK) {
        // the last prompt position's greedy token -> the decode chain's token slot
        k_pf_rmsnorm<<<1, 256, 0, st>>>(h, static_cast<const __half*>(D.final_norm), x, n, D.rms_eps, M - 1);
        check(cudaMemsetAsync(best, 0, 8, st), "prefill argmax");
        k_pf_lm_argmax<<<pf_blocks((int64_t)D.vocab * 32, 256), 256, 0, st>>>(
            static_cast<const __half*>(D.lm_head), x, D.vocab, n, best);
        k_pf_token<<<1, 1, 0, st>>>(best, m->tok_dev);
        k_llama_reset<<<1, 32, 0, st>>>(m->chain->tail(), m->chain->nctas, m->tok_dev, 1, pos0 + M,
                                        (long long)D.world * m->lm_ctas);
        check(cudaGetLastError(), "prefill token");
    }
    for (void* p : {(void*)h, (void*)q, (void*)k, (void*)v, (void*)y, (void*)g, (void*)u, (void*)x, (void*)a,
                    (void*)best})
        dev_free(p, st);
    if (s == FASQ_OK) set_launch_count(0);
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
