// gemv_tc.cu -- batched decode (B = 2..64 tokens) on tcgen05: the weights as the
// UMMA A operand, the tokens as N (sm_100a).
//
// SURVEY 8(d.1) G5 and NEXT-3 ("adaptive GEMV <-> tensor-core dispatch for
// B = 16-64").  The per-launch GEMVs do B FMAs per gathered centroid on
// the CUDA cores (B = 8: 16 FHFMA per index) and the prefill EXPAND kernel is
// shaped for thousands of tokens (2 x 128-token accumulators: at M = 16 it
// runs 94 % empty MMAs and moves 512 KiB of split-K partials per CTA).  Here a
// CTA owns 384 weight rows (three 128-row UMMA M tiles) x a K range:
//
//   L producer   : per 64-wide K chunk (one group of 32 subspaces at d = 2) the
//                  codebook image and the 384 rows' index chunk (two bulk copies);
//   X producer   : the chunk's X tile [NT tokens][64] (TMA, 128B swizzle; rows
//                  past B are zero-filled) -- the UMMA B operand;
//   12 expansion : lane = subspace (the GEMV mapping: one LDS.128 = 16 rows'
//     warps        indices, lane s gathers from bank s), centroids stored into
//                  the K-major SWIZZLE_128B A tile (conflict-free STS rows);
//   MMA thread   : 4 K-steps x 3 tiles of tcgen05.mma.cta_group::1.kind::f16
//                  (M = 128 rows, N = NT tokens, K = 16) into 3 TMEM accumulators;
//   epilogue     : tcgen05.ld (32x32b: lane = row, registers = tokens) -> y[tok][row];
//                  split-K over K ranges: fp32 partial tiles in a per-stream
//                  workspace; the co-resident CTAs of a row tile meet on a
//                  counter and each sums a 1/ks slice in fixed order
//                  (deterministic).
// The MMA work is negligible (a 128x16x64 MMA is ~32 tensor cycles); the kernel
// is an expansion engine: per index 4 B gather + 4 B STS + 4 B UMMA A read,
// independent of B -- the CUDA-core GEMV's B-fold FMA work is gone.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "fasq_internal.cuh"

namespace fasq {
namespace {

constexpr int TT_K = 64;             // K per chunk (one 128-B swizzle row of fp16)
constexpr int TT_MS = 3;             // 128-row UMMA M tiles per CTA
constexpr int TT_R = 128 * TT_MS;    // weight rows per CTA
constexpr int TT_EXP = 12;           // expansion / epilogue warps (32 rows each; 3 per TMEM lane quarter)
constexpr int TT_THREADS = (3 + TT_EXP) * 32;
constexpr int TT_S = 2;              // stages of both rings

struct TtParams {
    const uint8_t* idx;     // [n_groups][F_out_pad/64][32][64]
    const uint8_t* cbimg;   // [n_groups][C][32][4]
    void* y;                // [B][F_out] f16 / f32
    float* ws;              // ks > 1: partial tiles [ks][row_tiles][NT][TT_R]
    unsigned* tickets;      // ks > 1: [row_tiles][arrive, depart] (zero between launches)
    int B, F_out, F_out_pad, n_groups, C, y_f32, row_tiles;
};

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    // K-major SWIZZLE_128B: start >> 4, LBO 0, SBO = 1024 >> 4, version 1, layout 2
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)(1024u >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
constexpr uint32_t idesc_f16(int M, int N) {   // D f32, A = B = f16, K-major, N >> 3, M >> 4
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr int tmem_cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }

template <int NT>
__global__ void __launch_bounds__(TT_THREADS, 1) k_gemv_tc(const __grid_constant__ CUtensorMap xmap, TtParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_SUB = 128 * TT_K * 2;                // 16 KiB per 128-row tile
    constexpr int A_BYTES = TT_MS * A_SUB;               // 48 KiB
    constexpr int X_BYTES = NT * TT_K * 2;               // 2..8 KiB (multiple of 1 KiB)
    constexpr int I_BYTES = TT_R * 32;                   // 12 KiB
    constexpr int TCOLS = tmem_cols(TT_MS * NT);
    const int CB_BYTES = p.C * 128;
    uint8_t* sA = smem;                                  // TT_S x A
    uint8_t* sX = sA + TT_S * A_BYTES;                   // TT_S x X
    uint8_t* sI = sX + TT_S * X_BYTES;                   // TT_S x idx
    uint8_t* sC = sI + TT_S * I_BYTES;                   // TT_S x codebook image
    uint64_t* bars = reinterpret_cast<uint64_t*>(sC + TT_S * CB_BYTES);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5 * TT_S + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = (int)blockIdx.x, n0 = tile * TT_R;
    const int ksplit = (int)gridDim.y, kz = (int)blockIdx.y;
    const int kb = (int)((int64_t)kz * p.n_groups / ksplit);
    const int nk = (int)((int64_t)(kz + 1) * p.n_groups / ksplit) - kb;
    const int rows_valid = min(TT_R, p.F_out_pad - n0);   // multiple of 64
    const uint32_t bar0 = dev::smem_u32(bars);
    auto xfull = [&](int s) { return bar0 + 8u * s; };                 // X tile landed (tx)
    auto afull = [&](int s) { return bar0 + 8u * (TT_S + s); };        // A tile expanded (8 warps)
    auto empty = [&](int s) { return bar0 + 8u * (2 * TT_S + s); };    // MMA done with X and A slot
    auto lfull = [&](int s) { return bar0 + 8u * (3 * TT_S + s); };    // codebook + indices landed (tx)
    auto lempty = [&](int s) { return bar0 + 8u * (4 * TT_S + s); };   // expansion done with them
    const uint32_t accum = bar0 + 8u * (5 * TT_S);

    if (threadIdx.x == 0) {
        for (int s = 0; s < TT_S; ++s) {
            dev::mbar_init(xfull(s), 1);
            dev::mbar_init(afull(s), TT_EXP);
            dev::mbar_init(empty(s), 1);
            dev::mbar_init(lfull(s), 1);
            dev::mbar_init(lempty(s), TT_EXP);
        }
        dev::mbar_init(accum, 1);
        dev::fence_barrier_init();
        dev::pdl_launch_dependents();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(dev::smem_u32(tmem_slot)), "n"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------ X producer -----------------------------
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
            dev::pdl_wait();   // x is the previous kernel's output
            for (int i = 0; i < nk; ++i) {
                const int s = i % TT_S;
                if (i >= TT_S) dev::mbar_wait(empty(s), ((i / TT_S) + 1) & 1);
                dev::mbar_arrive_expect_tx(xfull(s), (uint32_t)X_BYTES);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                    :: "r"(dev::smem_u32(sX + s * X_BYTES)), "l"(reinterpret_cast<uint64_t>(&xmap)),
                       "r"((kb + i) * TT_K), "r"(0), "r"(xfull(s)) : "memory");
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ---------------------- codebook + index producer ----------------------
        if (lane == 0) {
            const uint32_t ib = (uint32_t)rows_valid * 32u;
            for (int i = 0; i < nk; ++i) {
                const int s = i % TT_S;
                if (i >= TT_S) dev::mbar_wait(lempty(s), ((i / TT_S) + 1) & 1);
                dev::mbar_arrive_expect_tx(lfull(s), ib + (uint32_t)CB_BYTES);
                dev::bulk_g2s(dev::smem_u32(sI + s * I_BYTES), p.idx + ((size_t)(kb + i) * p.F_out_pad + n0) * 32, ib,
                              lfull(s));
                dev::bulk_g2s(dev::smem_u32(sC + (size_t)s * CB_BYTES), p.cbimg + (size_t)(kb + i) * CB_BYTES,
                              (uint32_t)CB_BYTES, lfull(s));
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------ MMA issuer -----------------------------
        constexpr uint32_t idesc = idesc_f16(128, NT);
        for (int i = 0; i < nk; ++i) {
            const int s = i % TT_S;
            const uint32_t ph = (i / TT_S) & 1;
            dev::mbar_wait(xfull(s), ph);
            dev::mbar_wait(afull(s), ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                const uint32_t a_base = dev::smem_u32(sA + s * A_BYTES), x_base = dev::smem_u32(sX + s * X_BYTES);
#pragma unroll
                for (int kk = 0; kk < TT_K / 16; ++kk) {
                    const uint64_t bd = desc_sw128(x_base + kk * 32);
#pragma unroll
                    for (int m = 0; m < TT_MS; ++m) {
                        const uint64_t ad = desc_sw128(a_base + m * A_SUB + kk * 32);
                        const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{.reg .pred p;\n\t"
                            "setp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                            :: "r"(tmem + (uint32_t)(m * NT)), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             :: "r"(empty(s)) : "memory");
                if (i == nk - 1)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 :: "r"(accum) : "memory");
            }
            __syncwarp();
        }
    } else {
        // ------------------------------ expansion ------------------------------
        // warp ew: rows [32 ew, 32 ew + 32) = two 16-row chunks; lane = subspace s
        // writes K columns (2s, 2s+1) of each row: 16-B chunk s/4 of the 128-B row at
        // chunk ((s/4) ^ (row & 7)) (K-major SWIZZLE_128B), word s & 3
        const int ew = warp - 3;
        uint32_t xo[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) xo[q] = ((uint32_t)(((lane >> 2) ^ q) << 4)) | ((uint32_t)(lane & 3) << 2);
        const uint32_t rot = (uint32_t)(lane >> 1);
        for (int i = 0; i < nk; ++i) {
            const int s = i % TT_S;
            const uint32_t ph = (i / TT_S) & 1;
            dev::mbar_wait(lfull(s), ph);
            if (i >= TT_S) dev::mbar_wait(empty(s), ((i / TT_S) + 1) & 1);   // A slot free
            const uint32_t ibase = dev::smem_u32(sI + s * I_BYTES) + (uint32_t)lane * 64u;
            const uint32_t cbl = dev::smem_u32(sC + (size_t)s * CB_BYTES) + (uint32_t)lane * 4u;
            const uint32_t abase = dev::smem_u32(sA + s * A_BYTES);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r0 = 32 * ew + 16 * h;                 // first row of the 16-row chunk
                const uint32_t c = (uint32_t)((r0 & 63) >> 4);
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (r0 < rows_valid) v = dev::lds128(ibase + (uint32_t)(r0 >> 6) * 2048u + 16u * ((c + rot) & 3u));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                const uint32_t arow = abase + (uint32_t)(r0 >> 7) * A_SUB + (uint32_t)(r0 & 127) * 128u;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t k = dev::prmt(w[j >> 2], 0u, 0x4440u | (uint32_t)(j & 3));
                    const uint32_t cv = dev::lds32(cbl + (k << 7));
                    asm volatile("st.shared.u32 [%0], %1;" :: "r"(arow + (uint32_t)j * 128u + xo[j & 7]), "r"(cv) : "memory");
                }
            }
            dev::fence_proxy_async();   // generic-proxy STS -> visible to the tensor core (async proxy)
            __syncwarp();
            if (lane == 0) {
                dev::mbar_arrive(afull(s));
                dev::mbar_arrive(lempty(s));
            }
        }
        // ------------------------------ epilogue -------------------------------
        dev::mbar_wait(accum, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int q = warp & 3;                                // TMEM lane quarter of this warp
        const int grp = ew >> 2;                               // 3 warps per quarter: tile grp
        for (int m = grp; m < TT_MS; m += TT_EXP / 4) {
            const int rl = m * 128 + q * 32 + lane;            // row within the CTA tile
            const int row = n0 + rl;
            // 16 token columns at a time: TMEM -> registers -> y (or the split-K
            // partial tile); bounded registers for NT up to 128
#pragma unroll 1
            for (int c0 = 0; c0 < NT; c0 += 16) {
                if (c0 >= p.B) break;
                uint32_t r[16];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(m * NT + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                    "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                      "=r"(r[14]), "=r"(r[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (ksplit == 1) {
                    if (row < p.F_out) {
#pragma unroll
                        for (int v = 0; v < 16; ++v) {
                            const int t = c0 + v;
                            if (t >= p.B) break;
                            const float fv = __uint_as_float(r[v]);
                            if (p.y_f32) reinterpret_cast<float*>(p.y)[(size_t)t * p.F_out + row] = fv;
                            else reinterpret_cast<__half*>(p.y)[(size_t)t * p.F_out + row] = __float2half_rn(fv);
                        }
                    }
                } else {
                    float* wr = p.ws + ((size_t)kz * p.row_tiles + tile) * NT * TT_R;
#pragma unroll
                    for (int v = 0; v < 16; ++v)
                        if (c0 + v < p.B) __stcg(wr + (size_t)(c0 + v) * TT_R + rl, __uint_as_float(r[v]));
                }
            }
        }
        if (ksplit > 1) {
            // all ks CTAs of a row tile are co-resident (grid <= #SMs): arrive, wait for
            // the others, then each sums a 1/ks slice of the tile's rows over z = 0..ks-1
            // in fixed order (deterministic).  The last CTA to leave resets both
            // counters for the next launch on this stream.
            __threadfence();
            asm volatile("bar.sync 1, %0;" :: "n"(TT_EXP * 32) : "memory");
            unsigned* arrive = p.tickets + 2 * tile;
            unsigned* depart = arrive + 1;
            if (ew == 0 && lane == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(arrive) : "memory");
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(arrive) : "memory");
                } while (v < (unsigned)ksplit);
                unsigned old;
                asm volatile("atom.add.relaxed.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(depart) : "memory");
                if (old == (unsigned)ksplit - 1u) {   // every CTA has seen arrive == ks
                    *arrive = 0u;
                    *depart = 0u;
                }
            }
            asm volatile("bar.sync 1, %0;" :: "n"(TT_EXP * 32) : "memory");
            const int r_lo = (int)((int64_t)kz * TT_R / ksplit), r_hi = (int)((int64_t)(kz + 1) * TT_R / ksplit);
            const int nr = r_hi - r_lo;
            for (int e = (ew * 32 + lane); e < p.B * nr; e += TT_EXP * 32) {
                const int t = e / nr, rl = r_lo + (e - t * nr), row = n0 + rl;
                if (row >= p.F_out) continue;
                float sum = 0.f;
                for (int z = 0; z < ksplit; ++z)
                    sum += __ldcg(p.ws + (((size_t)z * p.row_tiles + tile) * NT + t) * TT_R + rl);
                if (p.y_f32) reinterpret_cast<float*>(p.y)[(size_t)t * p.F_out + row] = sum;
                else reinterpret_cast<__half*>(p.y)[(size_t)t * p.F_out + row] = __float2half_rn(sum);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(TCOLS));
    }
}

size_t tt_smem(int NT, int C) {
    return 1024 + (size_t)TT_S * (TT_MS * 128 * TT_K * 2 + (size_t)NT * TT_K * 2 + TT_R * 32 + (size_t)C * 128) +
           8 * (5 * TT_S + 1) + 16;
}

int num_sms_tt() {
    static int n = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    });
    return n;
}

template <int NT>
fasq_status launch_tt(const CUtensorMap& map, const TtParams& p, dim3 grid, size_t smem, uint32_t flags,
                      cudaStream_t st) {
    auto kern = k_gemv_tc<NT>;
    static size_t lim = 0;
    static std::once_flag once;
    std::call_once(once, [&] { lim = set_max_dyn_smem(kern); });
    if (lim < smem) { set_error("gemv (tcgen05): SMEM"); return FASQ_E_UNSUPPORTED; }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(TT_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (flags & FASQ_FLAG_PDL) ? 1 : 0;
    FASQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, map, p));
    return FASQ_OK;
}

}  // namespace

bool gemv_tc_supported(const fasq_layer* L, int B) {
    return L->d == 2 && L->C <= 256 && !L->bits && !L->dim0 && (L->F_in % 64) == 0 && B >= 1 && B <= 128 &&
           tt_smem(B <= 16 ? 16 : B <= 32 ? 32 : B <= 64 ? 64 : 128, L->C) <= kSmemMax && get_encode() != nullptr;
}

fasq_status gemv_tc_launch(const fasq_layer* L, const __half* X, int B, void* y, fasq_dtype yt, uint32_t flags,
                           cudaStream_t st) {
    if (!gemv_tc_supported(L, B)) return FASQ_E_UNSUPPORTED;
    if ((reinterpret_cast<uintptr_t>(X) & 15) != 0) return FASQ_E_ARG;
    const int NT = B <= 16 ? 16 : B <= 32 ? 32 : B <= 64 ? 64 : 128;
    PFN_encodeTiled enc = get_encode();
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)L->F_in, (cuuint64_t)B};
    cuuint64_t gstride[1] = {(cuuint64_t)L->F_in * 2};
    cuuint32_t box[2] = {TT_K, (cuuint32_t)NT};   // rows B..NT-1 of the box are zero-filled
    cuuint32_t estr[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(X), gdim, gstride, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        set_error("gemv (tcgen05): tensor map encode failed");
        return FASQ_E_CUDA;
    }
    TtParams p{};
    p.idx = L->idx;
    p.cbimg = L->cbimg;
    p.y = y;
    p.B = B;
    p.F_out = (int)L->F_out;
    p.F_out_pad = L->F_out_pad;
    p.n_groups = L->n_groups;
    p.C = L->C;
    p.y_f32 = yt == FASQ_F32;
    p.row_tiles = (L->F_out_pad + TT_R - 1) / TT_R;
    // K split: about one CTA per SM, equal groups per range (FASQ_GEMV_TC_KS forces it)
    if (p.row_tiles > num_sms_tt()) return FASQ_E_UNSUPPORTED;   // the split-K merge needs co-residency
    int ks = std::max(1, std::min(num_sms_tt() / p.row_tiles, L->n_groups));
    if (const char* e = getenv("FASQ_GEMV_TC_KS"))
        ks = std::max(1, std::min({atoi(e), L->n_groups, num_sms_tt() / p.row_tiles}));
    const int gper = (L->n_groups + ks - 1) / ks;
    ks = (L->n_groups + gper - 1) / gper;
    uint8_t* ws_call = nullptr;
    if (ks > 1) {
        // a FIXED ticket header (row_tiles <= #SMs): a header sized by this call's
        // row tiles would move and could overlap an earlier call's partials on
        // the shared stream workspace (garbage counters)
        const size_t tkb = 4096;
        if ((size_t)p.row_tiles * 8 > tkb) return FASQ_E_UNSUPPORTED;
        const size_t need = tkb + (size_t)ks * p.row_tiles * NT * TT_R * sizeof(float);
        uint8_t* ws = nullptr;
        fasq_status s = stream_workspace(st, WS_GEMV_TC, need, reinterpret_cast<void**>(&ws));
        if (s != FASQ_OK) return s;
        if (!ws) {   // first use inside stream capture: per-call workspace with zeroed tickets
            s = dev_alloc_t(&ws_call, need, st);
            if (s != FASQ_OK) return s;
            cudaError_t e = cudaMemsetAsync(ws_call, 0, tkb, st);
            if (e != cudaSuccess) { dev_free(ws_call, st); return cuda_fail(e, "gemv (tcgen05) workspace"); }
            ws = ws_call;
        }
        p.tickets = reinterpret_cast<unsigned*>(ws);
        p.ws = reinterpret_cast<float*>(ws + tkb);
    }
    const dim3 grid((unsigned)p.row_tiles, (unsigned)ks, 1);
    const size_t smem = tt_smem(NT, L->C);
    fasq_status s;
    switch (NT) {
        case 16: s = launch_tt<16>(map, p, grid, smem, flags, st); break;
        case 32: s = launch_tt<32>(map, p, grid, smem, flags, st); break;
        case 64: s = launch_tt<64>(map, p, grid, smem, flags, st); break;
        default: s = launch_tt<128>(map, p, grid, smem, flags, st); break;
    }
    dev_free(ws_call, st);
    if (s == FASQ_OK) set_launch_count(1);
    return s;
}

}  // namespace fasq
