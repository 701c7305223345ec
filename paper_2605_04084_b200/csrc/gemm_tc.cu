// gemm_tc.cu -- FASQ prefill GEMM, centroid-EXPAND variant on tcgen05 (sm_100a).
//
// Y[M][F_out] = X[M][F_in] . W_hat^T computed as a dense fp16 contraction on
// the 5th-gen tensor cores WITHOUT materialising W_hat in HBM: the paper's
// future-work direction (1), "a pipelined reconstruction kernel that rebuilds
// FP16 weight tiles in parallel with tensor-core GEMM, avoiding full
// materialization".  Per CTA tile (2 x 128 tokens x 256 weight rows)
// and per K-chunk of 64 input features (= one group of 32 subspaces at d=2):
//
//   X producer    : TMA 2-D loads of the two X tiles (128B swizzle); its ring
//                   slot is released by the MMA commit;
//   cb/idx producer: bulk copies of the group's codebook image and the tile's
//                   index chunk into a ring released by the EXPANSION warps (not
//                   the MMA), so the next chunks' loads start one MMA period
//                   earlier -- the coupled single ring left the tensor pipe idle
//                   on load latency (ncu: 47 % tensor-active, expansion warps
//                   waiting on the full barrier); decoupled: +15-32 % TFLOP/s;
//   8 expand warps: lane = subspace (as in the GEMV); gather the centroids of
//                   32 rows from the SMEM codebook image (lane s -> bank s,
//                   conflict-free) and store them into the B tile
//                   in the UMMA K-major SWIZZLE_128B layout (never to HBM);
//   MMA thread    : 2 token tiles x 4 x tcgen05.mma.cta_group::1.kind::f16
//                   (M=128, N=256, K=16) into two TMEM fp32 accumulators (all
//                   512 columns) -- each expanded B tile feeds 256 tokens, which
//                   halves the expansion + codebook SMEM traffic per FLOP;
//                   tcgen05.commit frees the stage;
//   epilogue      : tcgen05.ld (32x32b) -> fp32/fp16 -> Y (8 warps).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "fasq_internal.cuh"

namespace fasq {

namespace {

constexpr int TC_M = 128;          // tokens per accumulator (UMMA M)
constexpr int TC_MT = 2;           // token tiles per CTA sharing each expanded B tile (2 TMEM accumulators)
constexpr int TC_N = 256;          // weight rows per CTA tile (UMMA N)
constexpr int TC_K = 64;           // K elements per chunk (one 128B swizzle atom row)
constexpr int TC_STAGES = 2;
constexpr int TC_EXP_WARPS = 8;    // expansion warps (lane = weight row)
constexpr int TC_THREADS = (3 + TC_EXP_WARPS) * 32;   // + X producer, MMA, codebook/index producer

// One layer of a (grouped) launch: its row tiles are [rt0, next layer's rt0).
constexpr int kTcGroup = 4;
struct TcLayer {
    const uint8_t* idx;      // [n_groups][F_out_pad/64][32][64] (fasq_internal.cuh)
    const uint8_t* cbimg;    // [n_groups][C][32][4]
    void* Y;                 // [M][F_out]
    int F_out, F_out_pad, rt0;
};

struct TcParams {
    TcLayer lay[kTcGroup];   // layers sharing X, F_in, n_groups and C (q/k/v, gate/up): one launch
    int n_lay;
    float* ws;               // split-K (gridDim.z > 1): fp32 partial tiles [ks][tiles][256 tokens][256 rows]
    unsigned* tickets;       // [tiles][2] arrive / depart counters (zero between launches)
    int M, n_groups, C, y_f32;
    int tile0, ntx;          // this launch covers tiles tile0 + blockIdx.x (row tile = tile % ntx)
    int pair_order;          // 1: tiles in pair order (even token-tile count); 0: row-major (tile % ntx, tile / ntx)
};

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    // K-major, SWIZZLE_128B: start>>4 [0,14), LBO=0, SBO=1024>>4 [32,46),
    // version=1 [46,48), layout_type=2 (128B) [61,64)
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)(1024u >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// kind::f16 instruction descriptor: D=f32, A=B=f16, both K-major, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar) : "memory");
}

// PAIR: a 2-CTA cluster shares each 256-row B tile (cta_group::2, M = 256 per
// MMA): CTA r expands weight rows [n0 + 128 r, n0 + 128 r + 128) only, keeps its
// own 2 x 128 tokens (its 1-CTA tile), and the leader (r = 0) issues the pair
// MMAs reading both CTAs' A and B halves -- half the expansion work, B-tile
// SMEM and UMMA B-operand reads per SM (the 1-CTA kernel is SMEM-bandwidth
// bound: TC + LSU + TMA wavefronts ~ 80 % of the SMEM data path, ncu).
template <bool PAIR>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap xmap, TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the swizzled tiles
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int C = p.C;
    constexpr int A_TILE = TC_M * TC_K * 2;       // 16 KiB per token tile
    constexpr int A_BYTES = TC_MT * A_TILE;       // per stage
    constexpr int NR = PAIR ? TC_N / 2 : TC_N;    // weight rows expanded by this CTA
    constexpr int B_BYTES = NR * TC_K * 2;        // 32 KiB (16 KiB per CTA of a pair)
    constexpr int IDX_BYTES = NR * 32;            // 8 KiB (4 KiB)
    const int CB_BYTES = C * 128;                 // per stage: [C][32][4]
    uint8_t* sA = smem;                                   // STAGES * A
    // SX stages of the X/B ring (PAIR: 3 -- the halved B tile frees the SMEM, and the
    // cross-CTA hand-off per chunk needs the slack), SL of the codebook/index ring
    constexpr int SX = PAIR ? 3 : TC_STAGES, SL = TC_STAGES;
    uint8_t* sB = sA + SX * A_BYTES;                      // SX * B
    uint8_t* sI = sB + SX * B_BYTES;                      // SL * IDX
    uint8_t* sC = sI + SL * IDX_BYTES;                    // SL * [C][32][4] (one bulk copy each)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sC + SL * CB_BYTES);
    // bars: full[S] (X tiles), bfull[S] (B tile expanded), empty[S] (MMA done:
    // X and B slot free), lfull[S] / lempty[S] (codebook + index chunk ring,
    // released by the expansion warps -- not by the MMA -- so the next chunks'
    // loads start one MMA period earlier), accum
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * SX + 2 * SL + 1);   // + pair[SX]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // tiles in PAIR order: tile 2i + r = (row tile (i % ntx), token tile 2 (i / ntx) + r),
    // so the two CTAs of a cluster share the row tile (both kernels use it)
    const int tile_g = p.tile0 + (int)blockIdx.x;            // tile of the whole problem
    const int rank = tile_g & 1;                             // = %cluster_ctarank for PAIR
    // an odd token-tile count without pairs runs row-major: no phantom token tile
    const bool po = PAIR || p.pair_order;
    const int nrt = po ? (tile_g >> 1) % p.ntx : tile_g % p.ntx;
    const int ntt = po ? 2 * ((tile_g >> 1) / p.ntx) + rank : tile_g / p.ntx;
    // the layer owning row tile nrt (static indices: the params stay in the constant bank)
    const uint8_t* g_idx = p.lay[0].idx;
    const uint8_t* g_cb = p.lay[0].cbimg;
    void* g_Y = p.lay[0].Y;
    int F_out = p.lay[0].F_out, F_out_pad = p.lay[0].F_out_pad, rt0 = 0;
#pragma unroll
    for (int l = 1; l < kTcGroup; ++l)
        if (l < p.n_lay && nrt >= p.lay[l].rt0) {
            g_idx = p.lay[l].idx;
            g_cb = p.lay[l].cbimg;
            g_Y = p.lay[l].Y;
            F_out = p.lay[l].F_out;
            F_out_pad = p.lay[l].F_out_pad;
            rt0 = p.lay[l].rt0;
        }
    const int n0t = (nrt - rt0) * TC_N;                      // weight-row tile of its layer (epilogue rows)
    const int n0 = n0t + (PAIR ? rank * NR : 0);             // rows this CTA expands
    const int m0 = ntt * TC_M * TC_MT;                       // first token of this CTA's token tiles
    // token tiles with real tokens: a tile with <= 128 left loads one X tile and
    // issues one accumulator's MMAs (the second would multiply zero-filled rows;
    // at M <= 128 that was half the tensor time of every chunk).  PAIR MMAs span
    // both CTAs' tiles: always both.
    const int nmt = (!PAIR && m0 + TC_M >= p.M) ? 1 : TC_MT;
    // split-K (small M: too few tiles for the SMs): this CTA's K chunks [kb, kb + nk)
    const int ksplit = (int)gridDim.z, kz = (int)blockIdx.z;
    const int kb = (int)((int64_t)kz * p.n_groups / ksplit);
    const int nk = (int)((int64_t)(kz + 1) * p.n_groups / ksplit) - kb;
    const uint32_t bar0 = dev::smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto bfull_bar = [&](int s) { return bar0 + 8u * (SX + s); };
    auto empty_bar = [&](int s) { return bar0 + 8u * (2 * SX + s); };
    auto lfull_bar = [&](int s) { return bar0 + 8u * (3 * SX + s); };
    auto lempty_bar = [&](int s) { return bar0 + 8u * (3 * SX + SL + s); };
    const uint32_t accum_bar = bar0 + 8u * (3 * SX + 2 * SL);
    auto pair_bar = [&](int s) { return bar0 + 8u * (3 * SX + 2 * SL + 1 + s); };   // PAIR leader: peer stage ready

    if (threadIdx.x == 0) {
        for (int s = 0; s < SX; ++s) {
            dev::mbar_init(full_bar(s), 1);
            dev::mbar_init(bfull_bar(s), TC_EXP_WARPS);
            dev::mbar_init(empty_bar(s), 1);
            dev::mbar_init(pair_bar(s), 1);
        }
        for (int s = 0; s < SL; ++s) {
            dev::mbar_init(lfull_bar(s), 1);
            dev::mbar_init(lempty_bar(s), TC_EXP_WARPS);
        }
        dev::mbar_init(accum_bar, 1);
        dev::fence_barrier_init();
    }
    if (warp == 1) {   // TMEM allocation (2 x 256 fp32 columns: the two 128x256 accumulators)
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                         :: "r"(dev::smem_u32(tmem_slot)), "n"(256 * TC_MT));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                         :: "r"(dev::smem_u32(tmem_slot)), "n"(256 * TC_MT));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if constexpr (PAIR) {   // barriers initialised in both CTAs before any remote arrive
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------------------- X producer -----------------------------
        if (lane == 0) asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
        for (int i = 0; i < nk; ++i) {
            const int s = i % SX;
            if (i >= SX) dev::mbar_wait(empty_bar(s), ((i / SX) + 1) & 1);
            if (lane == 0) {
                dev::mbar_arrive_expect_tx(full_bar(s), (uint32_t)(nmt * A_TILE));
#pragma unroll
                for (int t = 0; t < TC_MT; ++t)
                    if (t < nmt)
                        tma_load_2d(dev::smem_u32(sA + s * A_BYTES + t * A_TILE), &xmap, (kb + i) * TC_K,
                                    m0 + t * TC_M, full_bar(s));
            }
            __syncwarp();
        }
    } else if (warp == 2 + TC_EXP_WARPS) {
        // ---------------------- codebook + index producer ----------------------
        const int rows = max(0, min(NR, F_out_pad - n0));      // idx rows present (multiple of 64)
        const uint32_t idx_bytes = (uint32_t)rows * 32u;
        const uint32_t cb_u = dev::smem_u32(sC);
        for (int i = 0; i < nk; ++i) {
            const int s = i % SL;
            if (i >= SL) dev::mbar_wait(lempty_bar(s), ((i / SL) + 1) & 1);
            if (lane == 0) {
                dev::mbar_arrive_expect_tx(lfull_bar(s), idx_bytes + (uint32_t)CB_BYTES);
                if (idx_bytes)
                    dev::bulk_g2s(dev::smem_u32(sI + s * IDX_BYTES),
                                  g_idx + ((size_t)(kb + i) * F_out_pad + n0) * 32, idx_bytes, lfull_bar(s));
                // (a PAIR variant fetching one codebook half per CTA with
                // .multicast::cluster was measured 25 % slower: the shared slot
                // couples the two CTAs' rings; profiles/r02/gemm_pair_ab.txt)
                dev::bulk_g2s(cb_u + (uint32_t)s * (uint32_t)CB_BYTES, g_cb + (size_t)(kb + i) * CB_BYTES,
                              (uint32_t)CB_BYTES, lfull_bar(s));
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer -----------------------------
        if (PAIR && rank == 1) {
            // the peer's relay: once this CTA's X tiles and B half of stage s are
            // in SMEM, arrive (release, cluster scope) on the leader's pair_bar(s)
            for (int i = 0; i < nk; ++i) {
                const int s = i % SX;
                const uint32_t ph = (i / SX) & 1;
                dev::mbar_wait(full_bar(s), ph);
                dev::mbar_wait(bfull_bar(s), ph);
                if (lane == 0) {
                    uint32_t rb;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rb) : "r"(pair_bar(s)));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(rb) : "memory");
                }
                __syncwarp();
            }
        } else {
        constexpr uint32_t idesc = idesc_f16(PAIR ? 2 * TC_M : TC_M, TC_N);
        for (int i = 0; i < nk; ++i) {
            const int s = i % SX;
            const uint32_t ph = (i / SX) & 1;
            dev::mbar_wait(full_bar(s), ph);
            dev::mbar_wait(bfull_bar(s), ph);
            if (PAIR) dev::mbar_wait_cluster(pair_bar(s), ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                const uint32_t b_base = dev::smem_u32(sB + s * B_BYTES);
#pragma unroll
                for (int t = 0; t < TC_MT; ++t) {
                    if (t >= nmt) break;
                    const uint32_t a_base = dev::smem_u32(sA + s * A_BYTES + t * A_TILE);
#pragma unroll
                    for (int kk = 0; kk < TC_K / 16; ++kk) {
                        const uint64_t ad = umma_desc_sw128(a_base + kk * 32);
                        const uint64_t bd = umma_desc_sw128(b_base + kk * 32);
                        const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                        if constexpr (PAIR)
                            asm volatile(
                                "{.reg .pred p;\n\t"
                                "setp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;}"
                                :: "r"(tmem + (uint32_t)(t * TC_N)), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                        else
                            asm volatile(
                                "{.reg .pred p;\n\t"
                                "setp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                                :: "r"(tmem + (uint32_t)(t * TC_N)), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    }
                }
                if constexpr (PAIR) {
                    // frees stage s in BOTH CTAs (X producers and expansion warps)
                    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                                 :: "r"(empty_bar(s)), "h"((unsigned short)3) : "memory");
                    if (i == nk - 1)
                        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                                     :: "r"(accum_bar), "h"((unsigned short)3) : "memory");
                } else {
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 :: "r"(empty_bar(s)) : "memory");
                    if (i == nk - 1)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                     :: "r"(accum_bar) : "memory");
                }
            }
            __syncwarp();
        }
        }
    } else {
        // ------------------------------ expansion ------------------------------
        // warp ew expands weight rows [32*ew, 32*ew + 32) of the tile; lane =
        // subspace s (the GEMV's mapping, gemv_core.cuh): one LDS.128 gives the
        // indices of 16 rows, lane s gathers c_s[k] from bank s (conflict-free
        // whatever k is) and writes K columns (2s, 2s+1) of the row; the 32
        // lanes of one STS fill one 128-B B-tile row (K-major SWIZZLE_128B:
        // 16-B chunk c of row r at c ^ (r & 7)) -> conflict-free.
        const int ew = warp - 2;                 // 0..7
        constexpr int RPW = NR / TC_EXP_WARPS;   // rows per expansion warp (32, PAIR: 16)
        uint32_t xo[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) xo[q] = ((uint32_t)(((lane >> 2) ^ q) << 4)) | ((uint32_t)(lane & 3) << 2);
        const uint32_t cb_u = dev::smem_u32(sC);
        const uint32_t ib0 = (uint32_t)((ew * RPW) >> 6) * 2048u + (uint32_t)lane * 64u;   // 64-row block
        const uint32_t cw0 = (uint32_t)(((ew * RPW) & 63) >> 4);                          // first 16-row chunk
        const uint32_t rot = (uint32_t)(lane >> 1);
        const bool have = n0 + ew * RPW < F_out_pad;     // this warp's rows were loaded (64-row blocks)
        for (int i = 0; i < nk; ++i) {
            const int s = i % SL, sx = i % SX;
            const uint32_t ph = (i / SL) & 1;
            dev::mbar_wait(lfull_bar(s), ph);                                       // codebook + indices
            if (i >= SX) dev::mbar_wait(empty_bar(sx), ((i / SX) + 1) & 1);          // B slot free
            const uint32_t ia = dev::smem_u32(sI + s * IDX_BYTES) + ib0;
            const uint32_t cbl = cb_u + (uint32_t)s * (uint32_t)CB_BYTES + (uint32_t)lane * 4u;
            const uint32_t bst = dev::smem_u32(sB + sx * B_BYTES) + (uint32_t)(ew * RPW) * 128u;
#pragma unroll
            for (int h = 0; h < RPW / 16; ++h) {
                const uint32_t c = cw0 + (uint32_t)h;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (have) v = dev::lds128(ia + 16u * ((c + rot) & 3u));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t k = dev::prmt(w[j >> 2], 0u, 0x4440u | (uint32_t)(j & 3));
                    const uint32_t cv = dev::lds32(cbl + (k << 7));
                    asm volatile("st.shared.u32 [%0], %1;" :: "r"(bst + (uint32_t)(h * 16 + j) * 128u + xo[j & 7]),
                                 "r"(cv) : "memory");
                }
            }
            dev::fence_proxy_async();      // generic-proxy STS -> visible to tcgen05 (async proxy)
            __syncwarp();
            if (lane == 0) {
                dev::mbar_arrive(bfull_bar(sx));
                dev::mbar_arrive(lempty_bar(s));
            }
        }
        // ------------------------------ epilogue -------------------------------
        {
            dev::mbar_wait(accum_bar, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int q = warp & 3;                    // TMEM lane quarter this warp may access
            const int t = ew >> 2;
            // <= 128 real tokens left in this tile (short prefill): the second
            // accumulator is all phantom -> both warp halves drain accumulator 0,
            // each half of its columns; else warp half t drains accumulator t
            const bool one_acc = m0 + TC_M >= p.M;
            const int ta = one_acc ? 0 : t;            // accumulator (token tile) this warp drains
            const int cbeg = one_acc ? t * (TC_N / 2) : 0, cend = one_acc ? cbeg + TC_N / 2 : TC_N;
            const int ml = ta * TC_M + q * 32 + lane;  // token within the CTA tile
            const int m = m0 + ml;                     // token
            constexpr int TT = TC_M * TC_MT;           // tokens per CTA tile (workspace column pitch)
            const int tile = (int)blockIdx.x;         // tile within this launch (workspace / tickets)
            // 32 consecutive outputs (rows n .. n+31) of token m -> Y (fp32 / fp16)
            auto store32 = [&](int n, const float* r) {
                if (m >= p.M || n >= F_out) return;
                const bool full = n + 32 <= F_out;
                if (p.y_f32) {
                    float* yr = reinterpret_cast<float*>(g_Y) + (size_t)m * F_out + n;
                    if (full && (F_out % 4 == 0)) {
#pragma unroll
                        for (int v = 0; v < 8; ++v)
                            reinterpret_cast<float4*>(yr)[v] = make_float4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
                    } else {
                        for (int v = 0; v < 32; ++v)
                            if (n + v < F_out) yr[v] = r[v];
                    }
                } else {
                    __half* yr = reinterpret_cast<__half*>(g_Y) + (size_t)m * F_out + n;
                    if (full && (F_out % 8 == 0)) {
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            __half2 h[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) h[u] = __floats2half2_rn(r[8 * v + 2 * u], r[8 * v + 2 * u + 1]);
                            uint4 o;
                            o.x = *reinterpret_cast<uint32_t*>(&h[0]);
                            o.y = *reinterpret_cast<uint32_t*>(&h[1]);
                            o.z = *reinterpret_cast<uint32_t*>(&h[2]);
                            o.w = *reinterpret_cast<uint32_t*>(&h[3]);
                            reinterpret_cast<uint4*>(yr)[v] = o;
                        }
                    } else {
                        for (int v = 0; v < 32; ++v)
                            if (n + v < F_out) yr[v] = __float2half_rn(r[v]);
                    }
                }
            };
#pragma unroll 1
            for (int c0 = cbeg; c0 < cend; c0 += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ta * TC_N + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                    "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                      "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                      "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float f[32];
#pragma unroll
                for (int v = 0; v < 32; ++v) f[v] = __uint_as_float(r[v]);
                if (ksplit > 1) {
                    // partial tile -> workspace, merged below in fixed ks order
                    // (deterministic).  Column-major [kz][tile][col][token]: one
                    // column of a warp's 32 tokens is one 128-B line (a token-major
                    // row per lane scattered 16-B pieces over 32 lines per store).
                    // Warps holding only phantom tokens skip it (never read).
                    if (m0 + ta * TC_M + q * 32 < p.M) {
                        float* wc = p.ws + ((size_t)kz * gridDim.x + tile) * (size_t)(TT * TC_N) + (size_t)c0 * TT + ml;
#pragma unroll
                        for (int v = 0; v < 32; ++v) __stcg(wc + (size_t)v * TT, f[v]);
                    }
                } else {
                    store32(n0t + c0, f);
                }
            }
            if (ksplit > 1) {
                // all ks CTAs of the tile are co-resident (grid <= #SMs): arrive,
                // wait for the others, then each sums a 1/ks slice of the tile's
                // columns over z = 0..ks-1 in fixed order (deterministic).  The
                // last CTA to leave resets both counters for the next launch.
                __threadfence();
                asm volatile("bar.sync 1, %0;" :: "n"(TC_EXP_WARPS * 32) : "memory");
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
                    if (old == (unsigned)ksplit - 1u) {   // everyone has seen arrive == ks
                        *arrive = 0u;
                        *depart = 0u;
                    }
                }
                asm volatile("bar.sync 1, %0;" :: "n"(TC_EXP_WARPS * 32) : "memory");
                // this CTA's column slice: 32-column chunks [kz * 8 / ks, (kz + 1) * 8 / ks)
                // (ks = 2..8); with one real accumulator the two warp halves (same
                // tokens) split it when it holds >= 2 chunks
                int mb = (kz * (TC_N / 32)) / ksplit * 32, me = ((kz + 1) * (TC_N / 32)) / ksplit * 32;
                if (one_acc) {
                    const int nc = (me - mb) / 32;
                    if (nc >= 2) {
                        const int hc = nc / 2 * 32;
                        if (t) mb += hc;
                        else me = mb + hc;
                    } else if (t) {
                        me = mb;
                    }
                }
                if (m < p.M) {
#pragma unroll 1
                    for (int c0 = mb; c0 < me; c0 += 32) {
                        float f[32];
#pragma unroll
                        for (int v = 0; v < 32; ++v) f[v] = 0.f;
                        for (int z = 0; z < ksplit; ++z) {   // fixed order
                            const float* rd = p.ws + ((size_t)z * gridDim.x + tile) * (size_t)(TT * TC_N) +
                                              (size_t)c0 * TT + ml;
#pragma unroll
                            for (int v = 0; v < 32; ++v) f[v] += __ldcg(rd + (size_t)v * TT);
                        }
                        store32(n0t + c0, f);
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if constexpr (PAIR) {   // both CTAs done with the pair's TMEM before it is released
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(256 * TC_MT));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(256 * TC_MT));
    }
}

size_t tc_smem_bytes(int C, bool pair = false) {
    const size_t nr = pair ? TC_N / 2 : TC_N;
    const size_t sx = pair ? 3 : TC_STAGES, sl = TC_STAGES;
    return 1024 + sx * (TC_MT * TC_M * TC_K * 2 + nr * TC_K * 2) + sl * (nr * 32 + (size_t)C * 128) +
           8 * (4 * sx + 2 * sl + 1) + 16;
}

}  // namespace

PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
        cudaGetLastError();
    });
    return fn;
}

bool gemm_tc_supported(const fasq_layer* L, int64_t M) {
    return L->d == 2 && L->C <= 256 && (L->F_in % 64) == 0 && M >= 1 && M < (1ll << 31) &&
           tc_smem_bytes(L->C) <= kSmemBudget && get_encode() != nullptr;
}

// Layers one grouped launch can take: the same input X (F_in), K groups, C and d.
bool gemm_tc_groupable(const fasq_layer* const* Ls, int n, int64_t M) {
    if (n < 1 || n > kTcGroup) return false;
    for (int l = 0; l < n; ++l) {
        if (!Ls[l] || Ls[l]->bits || Ls[l]->dim0 || !gemm_tc_supported(Ls[l], M)) return false;
        if (Ls[l]->F_in != Ls[0]->F_in || Ls[l]->n_groups != Ls[0]->n_groups || Ls[l]->C != Ls[0]->C ||
            Ls[l]->d != Ls[0]->d)
            return false;
    }
    return true;
}

fasq_status gemm_tc_launch(const fasq_layer* L, const __half* X, int64_t M, void* Y, fasq_dtype yt, cudaStream_t st) {
    return gemm_tc_launch_grouped(&L, 1, X, M, &Y, yt, st);
}

// One EXPAND launch over n layers sharing X: the row tiles of all layers form
// one tile grid (layer l owns [rt0_l, rt0_l + ntx_l)), so the small layers of a
// step (k / v: 4 row tiles) share the SMs with the large ones instead of each
// paying a launch, a pipeline fill and a split-K merge on a mostly idle GPU.
fasq_status gemm_tc_launch_grouped(const fasq_layer* const* Ls, int n, const __half* X, int64_t M, void* const* Ys,
                                   fasq_dtype yt, cudaStream_t st) {
    if (!gemm_tc_groupable(Ls, n, M)) return FASQ_E_UNSUPPORTED;
    const fasq_layer* L = Ls[0];
    PFN_encodeTiled enc = get_encode();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return FASQ_E_CUDA; }
    if ((reinterpret_cast<uintptr_t>(X) & 15) != 0) return FASQ_E_ARG;
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)L->F_in, (cuuint64_t)M};
    cuuint64_t gstride[1] = {(cuuint64_t)L->F_in * 2};
    cuuint32_t box[2] = {TC_K, TC_M};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(X), gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed"); return FASQ_E_CUDA; }
    TcParams p{};
    int ntx = 0;
    for (int l = 0; l < n; ++l) {
        p.lay[l].idx = Ls[l]->idx;
        p.lay[l].cbimg = Ls[l]->cbimg;
        p.lay[l].Y = Ys[l];
        p.lay[l].F_out = (int)Ls[l]->F_out;
        p.lay[l].F_out_pad = Ls[l]->F_out_pad;
        p.lay[l].rt0 = ntx;
        // F_out_pad rows of each idx table exist; a tile past F_out_pad loads none
        ntx += (Ls[l]->F_out_pad + TC_N - 1) / TC_N;
    }
    p.n_lay = n;
    p.M = (int)M;
    p.n_groups = L->n_groups;
    p.C = L->C;
    p.y_f32 = yt == FASQ_F32;
    const size_t smem = tc_smem_bytes(L->C), smem2 = tc_smem_bytes(L->C, true);
    static std::once_flag once;
    static size_t lim = 0, lim2 = 0;
    std::call_once(once, [] {
        lim = set_max_dyn_smem(k_gemm_tc<false>);
        lim2 = set_max_dyn_smem(k_gemm_tc<true>);
    });
    if (lim < smem) { set_error("gemm_tc: SMEM"); return FASQ_E_UNSUPPORTED; }
    // 2-CTA pairs (cta_group::2) for the launches without split-K: opt-in
    // (FASQ_GEMM_PAIR=1) -- measured equal at 4096^2 and 3-5 % slower on the
    // 14336-row / 14336-column shapes (profiles/r02/gemm_pair_ab.txt)
    const char* pe = getenv("FASQ_GEMM_PAIR");
    const bool pair_env = pe && atoi(pe) == 1;
    const bool pair_ok = pair_env && lim2 >= smem2;
    // token tiles: an even count is numbered in pair order (kernel); an odd count
    // runs row-major with the exact count (a phantom tile would expand its weight
    // slab for nothing: half the CTAs at M <= 256), unless 2-CTA pairs are on, which
    // round it up to even (the phantom tile reads zero-filled X and stores nothing)
    const int nty_exact = (int)((M + TC_M * TC_MT - 1) / (TC_M * TC_MT));
    p.pair_order = (nty_exact % 2 == 0 || pair_env) ? 1 : 0;
    const int nty = p.pair_order ? (nty_exact + 1) / 2 * 2 : nty_exact;
    const int tiles_all = ntx * nty;
    p.ntx = ntx;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // Tile scheduling (one CTA per SM; 1-D grids over tile ranges):
    //  * fewer tiles than SMs (small M): split K over gridDim.z for all tiles;
    //  * several waves with a small last wave (e.g. 14336 rows x M = 2048: 448
    //    tiles = 3 x 148 + 4): the full waves in one launch, the tail tiles in
    //    a second launch split over K so the tail takes ~1/ks of a tile.
    // Split-K: fp32 partial tiles through a per-layer workspace, merged in
    // fixed ks order (deterministic), see the kernel epilogue.
    auto pick_ks = [&](int tiles) {
        int ks = 1;
        if (const char* e = getenv("FASQ_GEMM_KSPLIT")) ks = atoi(e);
        else if (tiles < sms) ks = std::min(sms / tiles, L->n_groups / 8);
        ks = std::max(1, std::min(ks, 8));   // the merge deals 8 chunks of 32 columns over the ks CTAs
        while (ks > 1 && (tiles * ks > sms || ks > L->n_groups)) --ks;   // co-resident, >= 1 chunk each
        return ks;
    };
    int launches[2][3];   // {tile0, tiles, ks}
    int nl = 0;
    int tail = tiles_all > sms ? tiles_all % sms : 0;
    if (tail & 1) ++tail;   // the full-wave launch keeps whole pairs
    if (tail > 0 && tail <= sms / 4 && getenv("FASQ_GEMM_KSPLIT") == nullptr) {
        launches[nl][0] = 0; launches[nl][1] = tiles_all - tail; launches[nl][2] = 1; ++nl;
        launches[nl][0] = tiles_all - tail; launches[nl][1] = tail; launches[nl][2] = pick_ks(tail); ++nl;
    } else {
        launches[nl][0] = 0; launches[nl][1] = tiles_all; launches[nl][2] = pick_ks(tiles_all); ++nl;
    }
    // Split-K workspace: a FIXED ticket header (kTicketHdr bytes; launch li's
    // [tiles][arrive, depart] at li * kTicketHdr / 2 -- tiles <= #SMs when ks > 1)
    // followed by the launches' fp32 partial tiles.  The header never moves: a
    // ticket region placed after the partials moved with the call's size and
    // could land on an earlier call's partials (garbage counters on a shared
    // stream workspace); each launch's last CTAs leave its tickets at zero.
    constexpr size_t kTicketHdr = 4096;
    size_t part_off[2] = {0, 0}, total = kTicketHdr;
    for (int li = 0; li < nl; ++li) {
        part_off[li] = total;
        if (launches[li][2] > 1) {
            if ((size_t)2 * launches[li][1] * sizeof(unsigned) > kTicketHdr / 2) return FASQ_E_UNSUPPORTED;
            total += (size_t)launches[li][2] * launches[li][1] * (TC_M * TC_MT) * TC_N * sizeof(float);
        }
    }
    uint8_t* ws = nullptr;
    uint8_t* ws_call = nullptr;
    if (total > kTicketHdr) {
        // the stream's workspace (zero at allocation), else a per-call one (capture)
        fasq_status s = stream_workspace(st, WS_GEMM_TC, total, reinterpret_cast<void**>(&ws));
        if (s != FASQ_OK) return s;
        if (!ws) {
            s = dev_alloc_t(&ws_call, total, st);
            if (s != FASQ_OK) return s;
            cudaError_t e = cudaMemsetAsync(ws_call, 0, kTicketHdr, st);
            if (e != cudaSuccess) { dev_free(ws_call, st); return cuda_fail(e, "gemm workspace tickets"); }
            ws = ws_call;
        }
    }
    for (int li = 0; li < nl; ++li) {
        const int tiles = launches[li][1], ks = launches[li][2];
        dim3 grid((unsigned)tiles, 1, 1);
        p.tile0 = launches[li][0];
        if (ks > 1) {
            p.ws = reinterpret_cast<float*>(ws + part_off[li]);
            p.tickets = reinterpret_cast<unsigned*>(ws + (size_t)li * (kTicketHdr / 2));
            grid.z = (unsigned)ks;
        }
        cudaError_t e;
        if (ks == 1 && pair_ok && p.pair_order && (tiles & 1) == 0 && (p.tile0 & 1) == 0) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = grid;
            cfg.blockDim = dim3(TC_THREADS, 1, 1);
            cfg.dynamicSmemBytes = smem2;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            e = cudaLaunchKernelEx(&cfg, k_gemm_tc<true>, map, p);
        } else {
            k_gemm_tc<false><<<grid, TC_THREADS, smem, st>>>(map, p);
            e = cudaGetLastError();
        }
        if (e != cudaSuccess) {
            dev_free(ws_call, st);
            return cuda_fail(e, "k_gemm_tc launch");
        }
    }
    dev_free(ws_call, st);   // stream-ordered
    set_launch_count(nl);
    return FASQ_OK;
}

}  // namespace fasq
