// fasq_internal.cuh -- shared definitions of the product library (CUDA, sm_100a).
// Nothing here is shared with oracle/ (which is independent test infrastructure).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/fasq.h"

namespace fasq {

constexpr int kGroupSubs = 32;   // subspaces per "group" = one per lane of a warp
constexpr int kRowBlock = 64;    // rows per index block (F_out_pad is a multiple)

// ---------------------------------------------------------------------------
// The layer object (opaque behind the ABI).  Physical layout (DESIGN.md
// "Data layout in HBM"):
//
//  idx    [n_groups][F_out_pad/64][32 subspaces][64 rows] uint8: per group g
//         and 64-row block, subspace-major, so that lane s of a warp (= the
//         group's subspace s) loads the indices of 16 rows with one LDS.128.
//         The four 16-row chunks of a (block, subspace) segment are rotated
//         by s/2: chunk c (rows 16c..16c+15) sits at 16-B position
//         (c + (s >> 1)) & 3, which makes the LDS.128 of a quarter-warp hit 8
//         distinct 16-B bank groups (conflict-free).  Rows [r0, r0 + n) of a
//         group with r0, n multiples of 64 are ONE contiguous range of n*32
//         bytes at (g*F_out_pad + r0)*32.  Padded subspaces (>= N_ss) and rows
//         (>= F_out) hold 0.  idx_offset() below is the definition.
//  cbimg  [n_groups][C][32][E] bytes, E = entry bytes (4 for d<=2 -- d=1 is
//         padded to (c,0) --, 8 for d=4, 16 for d=8): the codebook of each
//         lane's subspace, k-major so that one k-row is 32*E contiguous bytes
//         and lane s reads bank(s) whatever k is.  Padded subspaces hold 0.
//  cb     [N_cb][C][d] fp16, the logical codebooks (export / GEMM staging).
// ---------------------------------------------------------------------------
__host__ __device__ inline int64_t idx_offset(int64_t g, int64_t r, int s, int64_t F_out_pad) {
    return (g * F_out_pad + (r & ~(int64_t)63)) * 32 + s * 64 + 16 * ((((r >> 4) & 3) + (s >> 1)) & 3) + (r & 15);
}
}  // namespace fasq

struct fasq_layer {
    int64_t F_out = 0, F_in = 0;
    int32_t d = 0, C = 0, group = 0, N_ss = 0, N_cb = 0;
    int32_t row_offset = 0;
    int32_t F_out_pad = 0;     // multiple of kRowBlock (64)
    int32_t n_groups = 0;      // ceil(N_ss / 32)
    int32_t E = 0;             // cbimg entry bytes
    int device = 0;
    uint8_t* idx = nullptr;    // physical indices
    uint8_t* cbimg = nullptr;  // GEMV codebook image
    void* cbmap = nullptr;     // d <= 2: device CUtensorMap {32 words, n_groups, C} over cbimg, strides
                               // {C*128, 128} B: a box {32, 2, C} at group g lands in SMEM as the
                               // codebook PAIR [C][g, g+1][32 words] (256-B k-rows, gemv_core.cuh)
    __half* cb = nullptr;      // logical codebooks
    int64_t idx_bytes = 0, cbimg_bytes = 0, cb_bytes = 0;
    // d = 2, batched decode on the tensor cores (gemv_core.cuh compute_group_mma):
    // the codebook image with word s of k-row k at position s ^ ((k & 7) << 2)
    // (8 lanes that gather one subspace's codebook spread over 8 banks), and its
    // pair tensor map.  Derived from cbimg on first use (ensure_cbimg_x).
    uint8_t* cbimg_x = nullptr;
    void* cbmap_x = nullptr;
    // NEXT-2 packed indices (Eq. 4: ceil(log2 K_s) bits per index).
    // bits = 0: the uint8 layout above (C <= 256).  bits > 0: `idx` holds
    // [n_groups][F_out_pad/64][32 subspaces][seg bytes], one segment per (group,
    // 64-row block, subspace) = the LSB-first bitstream of its 64 rows' codes
    // (row r at bits [r*bits, r*bits + bits)), seg = 8*bits bytes; rows
    // [r0, r0 + n) of a group (multiples of 64) are ONE contiguous range.  The
    // logical table that crosses the ABI is uint8 for C <= 256, uint16 above.
    int32_t bits = 0;
    int32_t seg = 0;
    int32_t idx_w = 1;         // logical index element bytes (1: C <= 256, 2: C <= 1024)
    // NEXT-4 dim = 0 (FASQ_LAYOUT_DIM0): subspace ss = output rows [ss*d, ss*d+d),
    // N_ss = F_out/d, datapoints = the F_in columns.  `idx` holds
    // [n_groups][K_pad/16][32 subspaces][16 columns] uint8 (lane s = subspace s
    // loads 16 columns' indices with one LDS.128; a (group, column range) chunk
    // is ONE contiguous range); cbimg/cbmap/cb as above (per subspace).
    int32_t dim0 = 0;
    int32_t K_pad = 0;         // dim0: F_in rounded up to 64
};

namespace fasq {

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string& msg);
fasq_status cuda_fail(cudaError_t e, const char* what);
void set_launch_count(int n);
void add_launch_count(int n);

#define FASQ_CUDA_TRY(expr)                                       \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return ::fasq::cuda_fail(_e, #expr); \
    } while (0)

inline int entry_bytes(int d) { return d <= 2 ? 4 : d * 2; }

// Opt a kernel into the largest dynamic SMEM the device allows next to its
// static SMEM; returns that byte count (0 on failure).
template <class K>
inline size_t set_max_dyn_smem(K kern) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) { cudaGetLastError(); return 0; }
    const size_t lim = (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return lim;
}
constexpr size_t kSmemBudget = 227 * 1024 - 2048;   // dynamic-SMEM planning budget (static SMEM headroom)
constexpr size_t kSmemMax = 226 * 1024 - 64;        // opt-in maximum (227 KiB) minus the 1 KiB the kernels report as static SMEM
// codebook PAIR ring (d <= 2): slots of [<= 256][2][32] words, 64 KiB stride so
// that the slot is byte 2 of the gather's PRMT constant
constexpr int kPairSlots = 2;
constexpr uint32_t kPairSlot = 65536;

// ---- layout kernels (layout.cu) ---------------------------------------------
fasq_status alloc_layer_storage(fasq_layer* L, cudaStream_t st);
fasq_status ensure_cbimg_x(const fasq_layer* L, cudaStream_t st);   // d = 2 only; synchronises st
fasq_status count_distinct_centroids(const fasq_layer* L, int64_t* distinct, cudaStream_t st);   // layout.cu   // idx, cbimg, cb and (d <= 2) cbmap
// idx_logical: uint8 or (L->idx_w == 2) uint16 [N_ss][F_out]
fasq_status build_physical_from_logical(fasq_layer* L, const __half* cb_logical,
                                        const void* idx_logical, cudaStream_t st);
fasq_status build_cbimg(fasq_layer* L, cudaStream_t st);
fasq_status idx16_to_8(const uint16_t* a, uint8_t* b, int64_t n, cudaStream_t st);
fasq_status export_logical(const fasq_layer* L, __half* cb_out, void* idx_out, cudaStream_t st);
// layout: FASQ_LAYOUT_* bits (PACKED: ceil(log2 C)-bit indices, C <= 1024; DIM0: output-axis subspaces)
fasq_status init_layer_shape(fasq_layer* L, int64_t F_out, int64_t F_in, int32_t d, int32_t C, int32_t group,
                             uint32_t layout);
uint32_t layer_layout(const fasq_layer* L);
// NEXT-4: decode GEMV on a dim = 0 layer (gemv_dim0.cu), B = 1..8
fasq_status gemv_dim0_launch(const fasq_layer* L, const __half* x, int B, void* y, fasq_dtype yt, uint32_t flags,
                             cudaStream_t st);
// out[j][i] = in[i][j] for fp16 [rows][cols] (dim = 0 pack)
fasq_status transpose_f16(const __half* in, __half* out, int64_t rows, int64_t cols, cudaStream_t st);
// G5 / NEXT-3: batched decode (B <= 64) on tcgen05, weights as the UMMA A operand (gemv_tc.cu)
bool gemv_tc_supported(const fasq_layer* L, int B);
constexpr int kGemvTcMinBatch = 5;   // measured crossover (profiles/r02/gemv_tc_sweep.jsonl)
int gemv_tc_min_batch();
fasq_status gemv_tc_launch(const fasq_layer* L, const __half* X, int B, void* y, fasq_dtype yt, uint32_t flags,
                           cudaStream_t st);
// NEXT-2: decode GEMV on a packed layer (gemv_packed.cu), B = 1..8
fasq_status gemv_packed_launch(const fasq_layer* L, const __half* x, int B, void* y, fasq_dtype yt, uint32_t flags,
                               cudaStream_t st);
fasq_status copy_rows(const fasq_layer* src, fasq_layer* dst, int32_t row0, cudaStream_t st);
// Device memory through the library allocator (alloc.cu, fasq_set_allocator).
fasq_status dev_alloc(void** p, size_t bytes, cudaStream_t st);
void dev_free(void* p, cudaStream_t st);
enum { WS_GEMV = 0, WS_GEMM_TC = 1, WS_GEMM_LUT = 2, WS_GEMV_TC = 3, WS_KINDS = 4 };
fasq_status stream_workspace(cudaStream_t st, int purpose, size_t bytes, void** out);   // alloc.cu
template <class T>
inline fasq_status dev_alloc_t(T** p, size_t bytes, cudaStream_t st) {
    void* q = nullptr;
    fasq_status s = dev_alloc(&q, bytes, st);
    *p = static_cast<T*>(q);
    return s;
}

// ---- compute entry points ---------------------------------------------------
fasq_status gemv_launch(const fasq_layer* L, const __half* x, int B, void* y, fasq_dtype yt,
                        uint32_t flags, cudaStream_t st);
struct GemvOpts {
    uint32_t flags = 0;
    int x_acc = 0, y_acc = 0;
    void* zero_ptr = nullptr;
    int64_t zero_bytes = 0;
    const fasq_layer* const* next = nullptr;
    int n_next = 0;
};
fasq_status gemv_grouped_launch2(const fasq_layer* const* Ls, int nl, const void* x, int B, void* const* ys,
                                 fasq_dtype yt, const GemvOpts& o, cudaStream_t st);
fasq_status acc_convert_launch(const void* acc, int64_t n, void* out, fasq_dtype yt, cudaStream_t st);
fasq_status gemv_grouped_launch(const fasq_layer* const* Ls, int nl, const __half* x, int B, void* const* ys,
                                fasq_dtype yt, uint32_t flags, cudaStream_t st,
                                const fasq_layer* const* next = nullptr, int n_next = 0);
fasq_status gemm_lut_launch(const fasq_layer* L, const __half* X, int64_t M, void* Y,
                            fasq_dtype yt, cudaStream_t st);
fasq_status gemm_tc_launch(const fasq_layer* L, const __half* X, int64_t M, void* Y,
                           fasq_dtype yt, cudaStream_t st);
bool gemm_tc_supported(const fasq_layer* L, int64_t M);
bool gemm_tc_groupable(const fasq_layer* const* Ls, int n, int64_t M);
fasq_status gemm_tc_launch_grouped(const fasq_layer* const* Ls, int n, const __half* X, int64_t M, void* const* Ys,
                                   fasq_dtype yt, cudaStream_t st);
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda);
// nullptr if unavailable (gemm_tc.cu).
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode();
fasq_status pack_run(const __half* W, fasq_layer* L, const fasq_pack_params* p, cudaStream_t st,
                     __half* cb_logical_out, uint16_t* idx_logical_out);   // uint16 indices for every C

// ---- device helpers -----------------------------------------------------------
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
// acc += c.lo*x.lo + c.hi*x.hi with exact fp16 products, fp32 accumulation
// (fma.rn.f32.f16 -> SASS FHFMA).
__device__ __forceinline__ float fhfma2(uint32_t c, uint32_t x, float acc) {
    asm("{.reg .f16 a, b, e, f;\n\t"
        "mov.b32 {a, b}, %1;\n\t"
        "mov.b32 {e, f}, %2;\n\t"
        "fma.rn.f32.f16 %0, a, e, %0;\n\t"
        "fma.rn.f32.f16 %0, b, f, %0;}"
        : "+f"(acc) : "r"(c), "r"(x));
    return acc;
}
// (a0, a1) += c * (x0, x1): fma.rn.f32x2 with a scalar broadcast (SASS FFMA2).
__device__ __forceinline__ void ffma2(float& a0, float& a1, float c, float x0, float x1) {
    asm("{.reg .b64 a, b, d;\n\t"
        "mov.b64 a, {%2, %2};\n\t"
        "mov.b64 b, {%3, %4};\n\t"
        "mov.b64 d, {%0, %1};\n\t"
        "fma.rn.f32x2 d, a, b, d;\n\t"
        "mov.b64 {%0, %1}, d;}"
        : "+f"(a0), "+f"(a1) : "f"(c), "f"(x0), "f"(x1));
}
__device__ __forceinline__ float fhfma1(uint32_t c, uint32_t x, float acc) {
    asm("{.reg .f16 a, b, e, f;\n\t"
        "mov.b32 {a, b}, %1;\n\t"
        "mov.b32 {e, f}, %2;\n\t"
        "fma.rn.f32.f16 %0, a, e, %0;}"
        : "+f"(acc) : "r"(c), "r"(x));
    return acc;
}

// ---- mbarrier / bulk copy (TMA engine) -------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
// try_wait with a suspend-time hint: the waiting warp sleeps in hardware
// until the phase completes (or the hint expires) instead of re-issuing the
// probe -- spinning consumers would steal issue slots from the warps that
// are still computing on the previous stage.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;}"
        : "=r"(ok) : "r"(bar), "r"(parity), "r"(1000000u) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait_sleep(bar, parity)) {
    }
}
// acquire at CLUSTER scope: the phase was completed by a remote arrive from the
// other CTA of a cluster (release.cluster), whose prior writes must be visible
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;}"
            : "=r"(ok) : "r"(bar), "r"(parity), "r"(1000000u) : "memory");
    }
}
// 1-D bulk async copy global -> shared (this CTA), completion on mbarrier.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        :: "r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(policy) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// 3-D tiled TMA load (tensor map in global memory, 64-B aligned), completion
// on mbarrier.  Out-of-range box elements are zero-filled and still counted.
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        :: "r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
// L2 prefetch through the TMA engine (no SMEM destination).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"(bytes) : "memory");
}
// Programmatic dependent launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

}  // namespace dev
}  // namespace fasq
