// chain_internal.cuh -- host-side description of a decode chain, shared by the
// generic chain API (chain.cu) and the whole-model Llama executor (llama.cu).
#pragma once
#include <cstring>
#include <vector>

#include "fasq_internal.cuh"

namespace fasq {

// Step kinds of the persistent decode-chain kernel.
enum ChainStepKind : int {
    SK_PQ = 0,      // grouped PQ GEMV (Eq. 3): 1..4 layers sharing one input
    SK_EMBED = 1,   // h0 = embedding row of the token the previous run's lm_head chose
    SK_ATTN = 2     // RoPE + KV-cache append + softmax attention over the cache (one token)
};
// Input transforms of a PQ step (how its fp16 x is formed from counted words).
enum ChainInMode : int {
    IN_EXT = 0,     // the chain's external fp16 input x
    IN_WORDS = 1,   // output words of (src_step, src_layer), rounded to fp16
    IN_RMSNORM = 2, // RMSNorm(words of src) * gamma, the scale folded into the epilogue (below)
    IN_SILU = 3,    // silu(layer 0 of src_step) * (layer 1 of src_step) (gate/up)
    IN_ATTN = 4     // the merged attention partials of an ATTN step (src_step)
};
// RMSNorm folding (IN_RMSNORM): RMSNorm(h) = s * (h (.) gamma) with the scalar
// s = 1/sqrt(mean(h^2) + eps) per token, and the PQ product is linear in x
// (Eq. 3), so a step stages x = fp16(h (.) gamma) over its own K range only and
// multiplies its fp32 partials by s in the epilogue.  The sum of squares is
// contributed by the K ranges of (layer 0, row tile 0) -- they cover F_in
// exactly once -- into per-range slots (fp32 bits in counted words, count 1);
// every warp sums the slots in a fixed order, so every CTA applies the same s.
// The scale is applied by the CONSUMERS of the normed step's outputs (the
// attention step for q/k/v, the SwiGLU staging for gate/up, chain outputs):
// their slot loads overlap their own input waits, while in the producing
// epilogue they were one more L2 round trip on the critical path.
// Attention output (SK_ATTN): per (token, head, cache part) the unnormalised
// o [hd], the running max m and the sum l, fp32 bits in counted words
// [B][heads][parts][hd + 2]; the consumer merges the parts in fixed order.

struct StepDesc {
    int kind = SK_PQ;
    std::vector<const fasq_layer*> layers;   // SK_PQ
    int in_mode = IN_EXT;
    int src_step = -1, src_layer = 0;
    const __half* gamma = nullptr;           // IN_RMSNORM weight [F_in]
    float eps = 1e-5f;
    bool scale_epilogue = false;             // IN_RMSNORM: apply the scale in this step's epilogue (its
                                             // consumers cannot hide the slot loads) instead of in the consumers
    int res_step = -1, res_layer = 0;        // SK_PQ: residual added to layer 0's output
    int lazy_step = -1;                      // SK_PQ, 1 layer: the VALUE of this output is its words + the
                                             // layer-0 words of lazy_step (a residual sum materialised by
                                             // its consumers: norm staging, residual epilogue, outputs)
    bool res_here = true;                    // this rank adds the residual (K-sharded steps: one rank)
    // outputs: local (false) or written into every rank's arena (true).  With
    // kshard, every rank holds a K slice (subspaces) of the layer and writes
    // partial sums for ALL rows (all-reduce fused into the counted stores);
    // without it, a rank holds a row shard (rows gathered).
    bool out_all = false;
    bool kshard = false;
    // SK_ATTN: q/k/v are layers 0/1/2 of q_step (this rank's heads)
    int q_step = -1;
    int n_heads = 0, n_kv = 0, head_dim = 0;
    __half* kc = nullptr;                    // [B][n_kv][max_T][head_dim] fp16 (this layer)
    __half* vc = nullptr;
    // SK_EMBED
    const __half* embed = nullptr;           // fp16 [vocab][hidden]
    int hidden = 0;
};

// Model-level extras of a chain (llama.cu); zero for plain GEMV chains.
struct ChainModel {
    const float2* rope = nullptr;            // [max_T][head_dim/2] (cos, sin)
    int max_T = 0, pos_wrap = 0;
    int* tok_hist = nullptr;                 // [B][max_T] tokens chosen by the runs (int32)
    long long tok_expect = 0;                // contributions per token slot (all ranks' lm_head CTAs)
    int attn_parts = 1;                      // cache parts per head (items per head of an ATTN step)
};

fasq_status chain_build(const std::vector<StepDesc>& steps, int B, int world, int rank, int max_ctas, bool det,
                        const ChainModel* model, cudaStream_t st, fasq_chain** out);

// Arena tail words (after the two double-buffered arenas; IPC-shared):
constexpr int kTailWords = 64;
constexpr int T_ENTRY = 0;     // CTA entry counter (monotonic, u64): run index = entry / nctas
constexpr int T_EXIT = 1;      // CTA exit counter
constexpr int T_DONE = 2;      // finished runs x ranks (every rank adds 1 to every rank's word per run)
constexpr int T_OVF = 3;       // sticky: a counted partial was out of range (values poisoned)
constexpr int T_POS = 4;       // model: position of the token this run decodes
constexpr int T_TOK = 16;      // model: token slots [2 parities][8 sequences][key, count]

// Token slot key: orderable logit in the high 32 bits, ~token in the low 32
// (red.max picks the largest logit, ties -> the lowest token id).
__host__ __device__ inline unsigned long long tok_key(float logit, unsigned token) {
    unsigned u;
#ifdef __CUDA_ARCH__
    u = __float_as_uint(logit);
#else
    std::memcpy(&u, &logit, 4);
#endif
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - token);
}
__host__ __device__ inline unsigned tok_of_key(unsigned long long k) {
    return 0xFFFFFFFFu - (unsigned)(k & 0xFFFFFFFFull);
}

}  // namespace fasq

// The chain object (opaque behind the ABI).
struct fasq_chain {
    int n_steps = 0, B = 0, d = 0, nctas = 0;
    int world = 1, rank = 0;
    int rw = 0, nw = 0, st = 0, R = 0, gmax = 1, maxC = 1, mi = 1;
    size_t smem = 0;
    std::vector<std::vector<int64_t>> acc_off;   // per step, per output: word offset in one arena buffer
    std::vector<std::vector<int64_t>> acc_ld;    // per step, per output: words per batch row
    std::vector<std::vector<int>> acc_ks;        // per step, per output: contributions per word
    std::vector<long long> nsq_off;              // per step: RMSNorm sum-of-squares slots [B][64] (-1: none)
    std::vector<int> nsq_n;                      // per step: slots per token (K ranges of layer 0)
    std::vector<int> nsq_F;                      // per step: F_in (the normed width)
    std::vector<float> nsq_eps;
    std::vector<char> nsq_epi;                   // per step: the scale is applied in the epilogue (outputs are final)
    std::vector<int> lazy;                       // per step: lazy base step (-1: none)
    std::vector<int> attn_hd, attn_heads;        // per ATTN step: head dim, local heads (output layout)
    int ext_F_in = 0;
    unsigned long long* arenas = nullptr;        // [2][arena_words] + tail (ONE allocation, IPC-exportable)
    bool arena_ipc = false;                      // cudaMalloc'ed (world > 1) rather than from the library allocator
    int64_t arena_words = 0;
    unsigned long long** peers_dev = nullptr;    // device [world]: every rank's `arenas`
    std::vector<void*> ipc_opened;
    bool peers_ready = true;
    void* items = nullptr;
    void* phases = nullptr;
    unsigned long long* trace = nullptr;
    fasq::ChainModel model{};
    bool has_model = false;
    std::vector<int> kinds;
    unsigned long long* tail() const { return arenas + 2 * arena_words; }
};
