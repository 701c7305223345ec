/*
 * include/fasq.h -- C ABI of the B200-native FASQ library (libfasq.so).
 *
 * FASQ (arXiv 2605.04084, /root/reference/PAPER.md cited as P:<line>) stores
 * each FP16 linear-layer weight W [F_out][F_in] (y = W.x, the nn.Linear
 * convention) as product-quantized codebooks + uint8 index tables and computes
 * products directly on them (Eq. 3):
 *
 *     y[b][j] = sum_{ss=0}^{N_ss-1} dot( x[b][ss*d : ss*d+d],
 *                                        T_cluster[ss/group][T_index[ss][j]] )
 *
 * Symbols: d = SZ_ss (sub-vector size), C = K_s (codebook cardinality),
 * N_ss = F_in/d subspaces over the INPUT axis (Eq. 3 / Alg. 2, P:267-268;
 * DESIGN.md reading R1), and `group` consecutive subspaces share one codebook
 * (N_cb = N_ss/group; group = 1 is the paper's Alg. 1).
 *
 * Logical arrays (the only layouts that cross this ABI):
 *   W         fp16 [F_out][F_in]            row major
 *   codebooks fp16 [N_cb][C][d]             T_cluster
 *   indices   uint8 [N_ss][F_out]           T_index  ("1 B index" P:274);
 *             uint16 when C > 256 (C <= 1024: Eq. 4's ceil(log2 K_s)-bit indices,
 *             P:224-231, Table 2's 2-512 / 2-1024 points P:479-488)
 *   x / X     fp16 [B or M][F_in]           row major
 *   y / Y     fp16 or fp32 [B or M][F_out]  row major
 * A layer stores these in a private physical layout tuned for the kernels
 * (DESIGN.md "Data layout in HBM"); fasq_export returns the logical form.
 *
 * Conventions for every call:
 *   - Pointers named *_dev are CUDA device pointers; *_host are host pointers.
 *     The caller owns all buffers it passes; the library owns each layer's
 *     storage (allocated on the current device at creation, released by
 *     fasq_free).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls that
 *     take a stream are stream-ordered and asynchronous unless documented.
 *   - Layers are immutable after creation and may be shared across streams
 *     and host threads: split-K workspaces are per call (allocated in stream
 *     order from the library allocator, fasq_set_allocator), never per layer.
 *   - No exception crosses the ABI.  Argument errors are returned
 *     synchronously before anything is enqueued.  CUDA launch/allocation
 *     failures return FASQ_E_CUDA / FASQ_E_OOM; asynchronous device faults
 *     surface as FASQ_E_CUDA on a later call.  fasq_last_error_message()
 *     describes the last failure on the calling thread.
 *   - There is no CPU fallback: every compute step runs in this library's
 *     sm_100a kernels; without a usable CUDA device every compute call fails
 *     with FASQ_E_CUDA.
 */
#ifndef FASQ_H_
#define FASQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FASQ_ABI_VERSION 4

typedef enum {
    FASQ_OK = 0,
    FASQ_E_ARG = -1,              /* null pointer / non-positive size / bad enum        */
    FASQ_E_NONDIVISIBLE = -2,     /* F_in % d != 0 or N_ss % group != 0 (Eq. 2) */
    FASQ_E_CLUSTER_OVERFLOW = -3, /* C > group*F_out points per codebook    */
    FASQ_E_NONFINITE = -4,        /* W holds inf/NaN (SPEC S:73 DegenerateInput)         */
    FASQ_E_SHAPE = -5,            /* operand shape mismatch          */
    FASQ_E_UNSUPPORTED = -6,      /* d not in {1,2,4,8}, C > 1024 (or > 256 unpacked), B > 8, n_pts > 2^23 */
    FASQ_E_CUDA = -7,             /* CUDA runtime / launch error, or no device           */
    FASQ_E_OOM = -8,              /* device allocation failed                            */
    FASQ_E_RANGE = -9             /* a counted partial left its |v| < 2^18 range (fasq_chain_check) */
} fasq_status;

typedef enum {
    FASQ_F16 = 0,
    FASQ_F32 = 1,
    FASQ_ACC_I64 = 2   /* int64 fixed point in units of 2^-32.  As an OUTPUT of the GEMVs the
                          result is ADDED into the caller-zeroed buffer with integer atomics
                          (associative -> deterministic, no split-K merge phase); as an INPUT
                          (FASQ_FLAG_X_ACC) it is rounded to fp16 once per element. */
} fasq_dtype;

typedef enum {
    FASQ_GEMM_AUTO = 0,      /* library picks (EXPAND_TC when shapes allow) */
    FASQ_GEMM_LUT = 1,       /* Alg. 3-style LUT build + gather               */
    FASQ_GEMM_EXPAND_TC = 2  /* centroid expansion into SMEM tiles + tcgen05 MMA  */
} fasq_gemm_algo;

/* Flags for the *_ex calls. */
#define FASQ_FLAG_PDL 1u     /* launch with programmatic dependent launch: the kernel's
                                 codebook/index prefetch may start before the previous
                                 kernel on the stream finishes (x is read only after
                                 griddepcontrol.wait).  Only valid when the layer was
                                 NOT written by the immediately preceding kernel. */

#define FASQ_FLAG_X_ACC 2u   /* x_dev holds FASQ_ACC_I64 values [B][F_in] (a previous GEMV's
                                 accumulator output) instead of fp16 */

/* Pack parameters (Alg. 1). */
typedef struct {
    int32_t d;        /* SZ_ss: 1, 2, 4 or 8                                     */
    int32_t C;        /* K_s: 1..256 (uint8 indices); 257..1024 packed (d = 2)    */
    int32_t group;    /* consecutive subspaces per codebook (1 = paper)           */
    int32_t iters;    /* T >= 0: maximum assign+update rounds (25 = default)      */
    uint64_t seed;    /* seeded init (splitmix64)                                 */
    int32_t init;     /* 0: seeded distinct sample (reading R3); 1: exact-integer
                         k-means++ (reading R17)                      */
    int32_t empty;    /* 0: an empty cluster keeps its centroid (R5); 1: reseed it
                         from the farthest point (reading R18)        */
    uint32_t layout;  /* FASQ_LAYOUT_* bits (0 = Eq. 3's input-axis subspaces,
                         uint8 indices).  FASQ_LAYOUT_PACKED is forced for
                         C > 256.                                                 */
} fasq_pack_params;

/* Layout flags (fasq_pack_params.layout, fasq_import_ex).  Layers with either
 * flag run fasq_gemv / fasq_gemv_ex / fasq_gemv_host (B <= 8), a one-layer
 * fasq_gemv_grouped, and fasq_gemm (FASQ_GEMM_AUTO, as 8-token GEMV slices);
 * the decode chain, fasq_llama_* and (FASQ_LAYOUT_DIM0) fasq_shard_rows
 * return FASQ_E_UNSUPPORTED for them. */
#define FASQ_LAYOUT_PACKED 1u   /* NEXT-2 (Eq. 4): ceil(log2 C)-bit packed
                                   indices, d = 2, C = 2..1024 (Table 2's 2-128 ...
                                   2-1024)                                  */
#define FASQ_LAYOUT_DIM0 2u     /* NEXT-4: the paper's dim = 0 partition (Eq. 2 first
                                   case P:174-186; its experiments): subspace
                                   ss = OUTPUT rows [ss*d, ss*d+d), N_ss = F_out/d,
                                   indices [N_ss][F_in] (the datapoints are W's
                                   columns), y[ss*d+e] = sum_j x[j] *
                                   T_cluster[ss/group][T_index[ss][j]][e].  uint8
                                   indices (C <= 256); not combinable with PACKED.     */

typedef struct fasq_layer fasq_layer; /* opaque */

typedef struct {
    int64_t F_out, F_in;
    int32_t d, C, group, N_ss, N_cb;
    int32_t row_offset;          /* first output row held (fasq_shard_rows), else 0 */
    int64_t index_bytes;         /* Eq. 4 index table: ceil(N_ss*F_out*index_bits/8) */
    int64_t codebook_bytes;      /* logical: N_cb * C * d * 2                     */
    int64_t device_bytes;        /* physical HBM bytes this layer owns            */
    double bits_per_weight;      /* 8*(index+codebook bytes)/(F_out*F_in)         */
    double eff_bits_W;           /* paper #W = ceil(log2 C)/d             */
    int32_t index_bits;          /* stored bits per index: 8 (uint8 layout) or
                                    ceil(log2 C) (packed, NEXT-2)                 */
    uint32_t layout;             /* FASQ_LAYOUT_* bits of the layer               */
} fasq_layer_info;

/* ---- creation --------------------------------------------------------- */

/* Packs W (fp16 [F_out][F_in], device) into a new layer with the GPU k-means
 * packer.  Output is bit-identical to the CPU oracle's fasq_ref_pack for the
 * same params.  W is read during the call's stream work only; it may be freed
 * after the stream reaches this point.  Synchronises `stream` once (to size
 * the unique-key sets).  *out is NULL on failure. */
fasq_status fasq_pack(const void* W_dev, int64_t F_out, int64_t F_in,
                      const fasq_pack_params* params, void* stream, fasq_layer** out);

/* Creates a layer from logical codebooks (fp16 [N_cb][C][d]) and indices
 * (uint8 [N_ss][F_out]; uint16 when C > 256), both device pointers, e.g. an
 * oracle-packed layer.  C > 256 makes a packed layer (as fasq_import_packed
 * with packed = 1).  Indices >= C are a caller error (undefined results for
 * uint8 layers).  Asynchronous. */
fasq_status fasq_import(const void* codebooks_dev, const void* indices_dev,
                        int64_t F_out, int64_t F_in, int32_t d, int32_t C, int32_t group,
                        void* stream, fasq_layer** out);

/* The same with a chosen layout (FASQ_LAYOUT_* bits): FASQ_LAYOUT_PACKED stores
 * ceil(log2 C) bits per index (NEXT-2, e.g. 7 bits for Table 2's 2-128,
 * P:496); FASQ_LAYOUT_DIM0 reads indices_dev as [F_out/d][F_in] (the dim = 0
 * partition, NEXT-4).  For a packed layer indices >= C return FASQ_E_ARG
 * (checked on the device; the call then synchronises `stream`). */
fasq_status fasq_import_ex(const void* codebooks_dev, const void* indices_dev,
                           int64_t F_out, int64_t F_in, int32_t d, int32_t C, int32_t group,
                           uint32_t layout, void* stream, fasq_layer** out);

/* Writes the layer's logical codebooks / indices to device buffers of
 * N_cb*C*d fp16 and N_ss*F_out uint8 (uint16 when C > 256) elements (either
 * pointer may be NULL). */
fasq_status fasq_export(const fasq_layer* layer, void* codebooks_dev, void* indices_dev,
                        void* stream);

/* Row shard for multi-GPU: a new layer holding output rows
 * [rank*F_out/world, (rank+1)*F_out/world) and ALL codebooks, created on the
 * current device.  Requires F_out % world == 0. */
fasq_status fasq_shard_rows(const fasq_layer* layer, int32_t rank, int32_t world,
                            void* stream, fasq_layer** out);

fasq_status fasq_layer_info_get(const fasq_layer* layer, fasq_layer_info* info);
void fasq_free(fasq_layer* layer);       /* synchronises the device; NULL is a no-op */

/* Deduplication ("removing repeated centroids within each subspace"):
 * *distinct = the number of distinct fp16 centroids summed over the layer's
 * codebooks (at most N_cb * C); the deduplicated codebook size is
 * distinct * d * 2 bytes.  Indices already reference only the first copy of a
 * repeated centroid (nearest-centroid ties go to the lowest k, reading R5), so
 * removing the later copies needs no index rewrite.  Synchronous. */
fasq_status fasq_layer_distinct_centroids(const fasq_layer* layer, int64_t* distinct, void* stream);

/* ---- products ------------------------------------------------------------ */

/* Decode GEMV (Alg. 2's math): y[b] = W_hat . x[b].
 * x_dev fp16 [B][F_in], y_dev [B][F_out] of y_dtype.  fp32 accumulation of
 * exact fp16 products; the split-K merge is deterministic (fixed order).
 * B in 1..8 runs the decode GEMV kernels; B > 8 (the paper's future work:
 * adaptive GEMV <-> tensor-core dispatch for B = 16..64) is the same
 * product through fasq_gemm (AUTO), with flags == 0 only (else
 * FASQ_E_UNSUPPORTED). */
fasq_status fasq_gemv(const fasq_layer* layer, const void* x_dev, int32_t B, void* y_dev,
                      fasq_dtype y_dtype, void* stream);
fasq_status fasq_gemv_ex(const fasq_layer* layer, const void* x_dev, int32_t B, void* y_dev,
                         fasq_dtype y_dtype, uint32_t flags, void* stream);

/* Options of fasq_gemv_grouped (all fields may be zero / NULL). */
typedef struct {
    uint32_t flags;                          /* FASQ_FLAG_PDL | FASQ_FLAG_X_ACC                     */
    const fasq_layer* const* next_layers;    /* layers of the NEXT launch of a decode chain: the
                                                kernel warms L2 with their first stages while it
                                                finishes (performance hint; results unchanged)   */
    int32_t n_next;                          /* 0..4                                               */
    void* zero_dev;                          /* side job: zero this device range during the launch
                                                (e.g. the FASQ_ACC_I64 outputs of the launch two
                                                steps back in a chain); must not alias this
                                                launch's inputs or outputs                          */
    int64_t zero_bytes;                      /* multiple of 8                                      */
} fasq_gemv_opts;

/* Grouped decode GEMV: n (1..4) layers that share the input x (q/k/v or
 * gate/up of a transformer block -- each packed separately) in ONE
 * launch: ys[l] = W_hat_l . x.  All layers must have the same F_in and d
 * (FASQ_E_SHAPE otherwise).  y_dtype FASQ_F16/F32: same numerics as n
 * separate fasq_gemv calls.  y_dtype FASQ_ACC_I64: ys[l] are int64 [B][F_out]
 * buffers the result is added to.  opts may be NULL. */
fasq_status fasq_gemv_grouped(const fasq_layer* const* layers, int32_t n, const void* x_dev, int32_t B,
                              void* const* ys_dev, fasq_dtype y_dtype, const fasq_gemv_opts* opts,
                              void* stream);

/* Converts n FASQ_ACC_I64 values to fp16 / fp32 (out_dtype). */
fasq_status fasq_acc_convert(const void* acc_dev, int64_t n, void* out_dev, fasq_dtype out_dtype, void* stream);

/* ---- decode chain (persistent executor) --------------------------------- */

/* One step of a decode chain: 1..4 layers sharing one input (q/k/v, o,
 * gate/up, down ...).  input_step = -1: the chain's external fp16 input x;
 * otherwise the output of layer `input_layer` of the earlier step
 * `input_step` (its F_out must equal this step's F_in). */
typedef struct {
    const fasq_layer* const* layers;
    int32_t n_layers;
    int32_t input_step;
    int32_t input_layer;
} fasq_chain_step;

typedef struct fasq_chain fasq_chain; /* opaque */

/* Plans a chain of grouped decode GEMVs (all layers: same d, B in 1..8) for
 * ONE persistent kernel (one CTA per SM, cooperative launch): every CTA
 * streams the codebook/index stages of all its steps through its SMEM ring
 * without draining at step boundaries.  There is no grid-wide barrier:
 * every output element is a counted accumulator (int64 fixed-point sum in
 * FASQ_ACC_I64 units plus the number of K-split contributions), and a step
 * polls only the words of its own K range until they are final.  Each K
 * range's fp32 partial is rounded once to FASQ_ACC_I64 units, so results
 * depend on the K-range plan (SM count; see fasq_chain_plan_ks) but not on
 * arrival order: repeated runs are bit-identical.
 * The layers must outlive the chain.  Synchronises `stream`.
 * A step with more row tiles than SMs gives several work items per CTA.
 * FASQ_E_UNSUPPORTED: the SMEM plan does not fit. */
fasq_status fasq_chain_create(const fasq_chain_step* steps, int32_t n_steps, int32_t B, void* stream,
                              fasq_chain** out);

/* Tensor-parallel chain (north_star "splitting output rows across GPUs with
 * an all-gather"), one process (or chain) per GPU: every layer of
 * `steps` is THIS rank's row shard (rows [rank*F_out, (rank+1)*F_out) of a
 * layer with world*F_out rows, rank-major, all codebooks replicated -- as
 * fasq_shard_rows produces), and every step's input is the full
 * world*F_out-wide output of its producer.  The all-gather is fused into the
 * GEMV: each rank red.adds its rows' counted accumulators into EVERY rank's
 * arena (NVLink peer memory), so a step's consumers on every GPU wait only for
 * their own K range -- no NCCL call and no host round trip between steps.
 * Deterministic by default: the K ranges are those the unsharded (world = 1)
 * chain would use on this GPU, so when every shard's F_out is a multiple of 64
 * the gathered outputs are bit-identical to the single-GPU chain's
 * (environment FASQ_CHAIN_FAST=1: plan each rank on its own shard instead).
 * world in 1..8; max_ctas > 0 caps the CTAs (e.g. several ranks sharing one
 * GPU in tests), 0 = one per SM.  Before the first run every rank must call
 * fasq_chain_set_peers (handles from every rank's fasq_chain_ipc_handle,
 * exchanged by the caller) or, for chains of one process,
 * fasq_chain_set_peer_chains.  All ranks must run their chains the same
 * number of times; run n on a rank starts writing only after every rank
 * finished run n-1 (a per-run DONE word every rank increments in every rank's
 * arena tail), and a rank that never delivers turns into a kernel error
 * (trap) after ~4 s instead of a hang. */
fasq_status fasq_chain_create_tp(const fasq_chain_step* steps, int32_t n_steps, int32_t B, int32_t world,
                                 int32_t rank, int32_t max_ctas, void* stream, fasq_chain** out);
/* Writes this chain's arena IPC handle (cudaIpcMemHandle_t, 64 bytes). */
fasq_status fasq_chain_ipc_handle(const fasq_chain* chain, void* handle_out);
/* handles: world x 64 bytes, rank-major (this rank's entry is ignored). */
fasq_status fasq_chain_set_peers(fasq_chain* chain, const void* handles);
/* In-process peers: chains[r] is rank r's chain (chains[rank] == chain). */
fasq_status fasq_chain_set_peer_chains(fasq_chain* chain, const fasq_chain* const* chains);

/* Runs the whole chain on x_dev (fp16 [B][F_in of the external-input steps]):
 * ONE kernel launch (the accumulators are double-buffered; each run zeroes the
 * buffer of the next run in-kernel, the run index lives on the device, so
 * graph replays work).  A chain instance must not run concurrently with itself. */
fasq_status fasq_chain_run(fasq_chain* chain, const void* x_dev, void* stream);

/* End-to-end run with HOST buffers: copies x_host (fp16 [B][F_in], ideally
 * pinned) to the device, runs the chain, converts the output of (step, layer)
 * to fp16/fp32 and copies it to y_host.  Synchronous. */
fasq_status fasq_chain_run_host(fasq_chain* chain, const void* x_host, void* y_host, int32_t step, int32_t layer,
                                fasq_dtype dtype, void* stream);

/* Output of layer `layer` of step `step` after the last run, as fp16 / fp32 /
 * FASQ_ACC_I64 [B][width] (width = world*F_out for gathered row shards;
 * valid until the next run).  Waits on the device until every word carries
 * all its contributions (peers' stores of the last step may still be in
 * flight).  fp16/fp32 outputs of a run that raised the range flag are NaN. */
fasq_status fasq_chain_output(const fasq_chain* chain, int32_t step, int32_t layer, void* y_dev,
                              fasq_dtype dtype, void* stream);
/* Synchronises `stream`; FASQ_E_RANGE if any run since the last check had a
 * K-split partial outside |v| < 2^18 (its values were clamped and its float
 * outputs poisoned with NaN); clears the flag. */
fasq_status fasq_chain_check(fasq_chain* chain, void* stream);
/* Host-only planner query: K-split count per layer of one grouped step of
 * n layers (F_out, n_groups = ceil(F_in/d/32)) on nctas CTAs at batch B
 * (what fasq_chain_create uses; <= 63 per layer, the counted-word field). */
int32_t fasq_chain_plan_ks(const int64_t* F_out, const int64_t* n_groups, int32_t n, int32_t nctas, int32_t d,
                           int32_t B, int32_t* ks_out);
/* Diagnostics: when trace_dev is not NULL, every later fasq_chain_run writes
 * per (step, CTA) four %globaltimer stamps (ns) into it, uint64
 * [n_steps][fasq_chain_ctas(chain)][4]: step entry, inputs final and staged
 * (dataflow wait done), CTA synchronised, outputs stored (CTAs without work
 * in a step write only the first).  The buffer is the caller's
 * and must stay allocated while tracing is on; NULL turns tracing off. */
fasq_status fasq_chain_trace(fasq_chain* chain, void* trace_dev);
int32_t fasq_chain_ctas(const fasq_chain* chain);   /* CTAs (= SMs) the chain runs on; -1 for NULL */
void fasq_chain_free(fasq_chain* chain);   /* synchronises the device; NULL is a no-op */

/* ---- whole-model decode (Llama-shaped; the paper's E2E setting) ---- */

/* A decoder-only model whose every linear layer is a FASQ layer (the
 * embedding, norms and lm_head stay fp16).  HF Llama semantics: pre-norm
 * blocks h' = h + o(Attn(RMSNorm(h))), h'' = h' + down(silu(gate(x)) * up(x))
 * with x = RMSNorm(h'); RoPE rotate-half with theta; GQA (n_heads / n_kv_heads
 * query heads per KV head); greedy argmax over the lm_head logits.
 * Tensor parallelism (world > 1, Megatron): q/k/v are row shards holding
 * this rank's n_heads/world heads (n_kv_heads/world KV heads), o is a K shard
 * (its F_in = this rank's heads x head_dim), gate/up row shards of ffn/world,
 * down a K shard (F_in = ffn/world); embed is the full table, lm_head this
 * rank's vocab/world rows.  Pointer arrays have n_layers entries; every
 * pointer is a device pointer owned by the caller and must outlive the model. */
typedef struct {
    int32_t n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab;
    float rms_eps, rope_theta;
    int32_t max_T;       /* KV-cache positions per sequence                                   */
    int32_t pos_wrap;    /* a step at position max_T-1 is followed by pos_wrap (benchmarks)   */
    int32_t B;           /* sequences decoded together, 1..8                                  */
    int32_t world, rank;
    const fasq_layer* const* q;
    const fasq_layer* const* k;
    const fasq_layer* const* v;
    const fasq_layer* const* o;
    const fasq_layer* const* gate;
    const fasq_layer* const* up;
    const fasq_layer* const* down;
    const void* const* attn_norm;   /* fp16 [hidden] per layer */
    const void* const* mlp_norm;    /* fp16 [hidden] per layer */
    const void* final_norm;         /* fp16 [hidden]           */
    const void* embed;              /* fp16 [vocab][hidden]    */
    const void* lm_head;            /* fp16 [vocab/world][hidden] */
    int32_t max_ctas;               /* 0 = one CTA per SM; > 0 caps the CTAs (ranks sharing a GPU in tests) */
} fasq_llama_desc;

typedef struct fasq_llama fasq_llama; /* opaque */

/* Builds the decode executor: one persistent chain (EMBED, then per block
 * qkv <- RMSNorm, ATTN, o + residual, gate/up <- RMSNorm, down <- SwiGLU +
 * residual) and the lm_head kernel; allocates the fp16 KV caches
 * ([B][n_kv_heads/world][max_T][head_dim] per layer, zeroed).  Chain step
 * numbering (fasq_llama_chain + fasq_chain_output): 0 = embedding h0; block l:
 * 1+5l = q/k/v (layers 0/1/2), 2+5l = attention output, 3+5l = h after the
 * attention residual, 4+5l = gate/up, 5+5l = h after the MLP residual.
 * Synchronises `stream`. */
fasq_status fasq_llama_create(const fasq_llama_desc* desc, void* stream, fasq_llama** out);
fasq_status fasq_llama_ipc_handle(const fasq_llama* model, void* handle_out);   /* world > 1: as fasq_chain_* */
fasq_status fasq_llama_set_peers(fasq_llama* model, const void* handles);
/* In-process peers: models[r] is rank r's model (models[rank] == model). */
fasq_status fasq_llama_set_peer_models(fasq_llama* model, const fasq_llama* const* models);
const fasq_chain* fasq_llama_chain(const fasq_llama* model);
/* This rank's KV cache of a layer: fp16 [B][n_kv_heads/world][max_T][head_dim]. */
fasq_status fasq_llama_kv_cache(const fasq_llama* model, int32_t layer, void** k_dev, void** v_dev);
/* The next step decodes tokens_host[b] (B entries) at position pos (pos < 0:
 * keep the current position); positions < pos must be in the KV cache.
 * Synchronous. */
fasq_status fasq_llama_reset(fasq_llama* model, const int32_t* tokens_host, int32_t pos, void* stream);
/* One greedy decode step of every sequence: TWO launches (chain, lm_head);
 * the chosen tokens feed the next step on the device (graph-replayable). */
fasq_status fasq_llama_step(fasq_llama* model, void* stream);
/* Whole-model PREFILL of a prompt (the paper's E2E protocol: prompt 128)
 * for a one-sequence, one-GPU model (B = 1, world = 1, head_dim 64 or 128): the M
 * tokens tokens_dev (int32, device) at positions [pos0, pos0 + M) go through
 * every block -- RMSNorm, PQ q/k/v (fasq_gemm_grouped AUTO), RoPE, the KV
 * cache write, causal GQA attention over positions <= each token's, PQ o +
 * residual, RMSNorm, PQ gate/up, SwiGLU, PQ down + residual -- and the greedy
 * token of the last prompt position becomes the next fasq_llama_step's input
 * at position pos0 + M.  Cache positions < pos0 must already hold the earlier
 * context.  Stream-ordered with respect to `stream`.  Outside stream capture
 * the work runs on a model-private stream joined to `stream` by events: the
 * first call for a given M launches eagerly and captures a CUDA graph that the
 * next calls with that M replay (tokens and pos0 are staged into device memory
 * it reads; the model keeps a working set for the largest M seen).  Inside a
 * caller's capture (or with FASQ_PREFILL_EAGER set) every call launches its
 * kernels on `stream` with a per-call working set from the library allocator.
 * tokens_dev may be overwritten by work ordered after the call on `stream`.
 * Not thread-safe per model. */
fasq_status fasq_llama_prefill(fasq_llama* model, const int32_t* tokens_dev, int32_t M, int32_t pos0, void* stream);
/* One step in parts, for per-kernel timing: part 0 = both launches
 * (fasq_llama_step), 1 = the chain kernel only, 2 = the lm_head kernel only.
 * A part-1 call must be followed by a part-2 call on the same stream before
 * the next step (the next chain run waits for the lm_head's token).
 * FASQ_E_ARG for another part. */
fasq_status fasq_llama_step_ex(fasq_llama* model, void* stream, int32_t part);
/* The tokens the last step chose (int32 [B], device). */
fasq_status fasq_llama_tokens(const fasq_llama* model, int32_t* tokens_dev, void* stream);
/* End to end with a HOST buffer: one step, then the chosen tokens are copied
 * to tokens_out_host (int32 [B]).  Synchronous. */
fasq_status fasq_llama_step_host(fasq_llama* model, int32_t* tokens_out_host, void* stream);
/* End to end in one call: the B tokens tokens_in_host (int32, host) are decoded
 * at position pos (< 0: the current position) -- fasq_llama_reset + one step +
 * the chosen tokens to tokens_out_host -- with a single synchronisation (the
 * inputs go through the model's pinned staging).  Synchronous. */
fasq_status fasq_llama_step_io(fasq_llama* model, const int32_t* tokens_in_host, int32_t pos,
                               int32_t* tokens_out_host, void* stream);
/* Diagnostics: enable (1) / disable (0) writing the lm_head logits (fp32
 * [B][vocab/world]) of every later step; *logits_dev receives the buffer. */
fasq_status fasq_llama_logits(fasq_llama* model, int32_t enable, void** logits_dev);
/* Copies the token history (int32 [B][max_T]: the token each step embedded,
 * at its position) to hist_dev. */
fasq_status fasq_llama_token_history(const fasq_llama* model, int32_t* hist_dev, void* stream);
void fasq_llama_free(fasq_llama* model);   /* synchronises the device; NULL is a no-op */

/* Same product with HOST buffers (end-to-end path): copies x_host (fp16
 * [B][F_in], ideally pinned) to the device, runs fasq_gemv and copies y back
 * to y_host.  Synchronous: returns after y_host is written. */
fasq_status fasq_gemv_host(const fasq_layer* layer, const void* x_host, int32_t B,
                           void* y_host, fasq_dtype y_dtype, void* stream);

/* Prefill GEMM (Alg. 3's math): Y = X . W_hat^T for M >= 1 rows.
 * X_dev fp16 [M][F_in], Y_dev [M][F_out] of y_dtype.  On a packed-index layer
 * (NEXT-2) only FASQ_GEMM_AUTO is accepted and the product runs as packed
 * GEMVs over 8-token slices (no tensor-core kernel reads the packed layout). */
fasq_status fasq_gemm(const fasq_layer* layer, const void* X_dev, int64_t M, void* Y_dev,
                      fasq_dtype y_dtype, fasq_gemm_algo algo, void* stream);

/* Prefill GEMMs of n layers reading the same X (a block's q / k / v, or gate /
 * up): Y_dev[l] = X . W_hat_l^T, each as fasq_gemm(layers[l], ...) computes
 * it, except that a grouped launch may split K differently (its tile count
 * differs), so the fp32 sums can differ in the last bits; the result is still
 * deterministic for a given (layers, M).  layers[]
 * and Y_dev[] are host arrays of n pointers (n >= 1); every layer has the same
 * F_in (FASQ_E_SHAPE otherwise); Y_dev[l] is [M][F_out_l] of y_dtype.  When
 * every layer would run EXPAND on its own (AUTO above the short-L crossover,
 * or FASQ_GEMM_EXPAND_TC) and n <= 4 layers share K groups, C and d, ONE
 * launch covers all their row tiles; otherwise the layers run one fasq_gemm
 * each, in order.  Errors as fasq_gemm. */
fasq_status fasq_gemm_grouped(const fasq_layer* const* layers, int32_t n, const void* X_dev, int64_t M,
                              void* const* Y_dev, fasq_dtype y_dtype, fasq_gemm_algo algo, void* stream);

/* ---- diagnostics ---------------------------------------------------------- */

/* Number of kernel launches the last successful compute call on this host
 * thread enqueued (bench.py's gpu_launches accounting). */
int32_t fasq_last_launch_count(void);
const char* fasq_status_string(fasq_status status);
const char* fasq_last_error_message(void);
int32_t fasq_abi_version(void);

/* ---- device memory (north_star: "PyTorch is used only for device memory") ---- */

/* Caller allocator: alloc(ctx, bytes, stream) returns a device pointer on the
 * current device, 256-B aligned, usable in stream order on `stream` (a
 * cudaStream_t; NULL = legacy default stream), or NULL on failure;
 * free(ctx, ptr, stream) releases it in stream order.  Both are called from
 * the calling host thread of the library call that needs the memory. */
typedef void* (*fasq_alloc_fn)(void* ctx, size_t bytes, void* stream);
typedef void (*fasq_free_fn)(void* ctx, void* ptr, void* stream);
/* Routes every device buffer the library owns -- layer storage, chain arenas
 * and plans, KV caches, per-call split-K workspaces, pack scratch -- through
 * alloc/free from now on (a pointer is always released by the allocator that
 * produced it).  alloc = free = NULL restores the default (CUDA's
 * stream-ordered allocator, cudaMallocAsync / cudaFreeAsync).  Exception: the
 * arena of a tensor-parallel chain (world > 1) is always a cudaMalloc
 * allocation (CUDA IPC exports whole allocations).
 * FASQ_E_ARG if exactly one of alloc / free is NULL. */
fasq_status fasq_set_allocator(fasq_alloc_fn alloc, fasq_free_fn free, void* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FASQ_H_ */
