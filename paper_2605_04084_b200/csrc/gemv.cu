// gemv.cu -- FASQ decode GEMV for sm_100a (batch 1..8).
//
// Computes Eq. 3, y[b][j] = sum_ss dot(x[b]_ss, T_cluster[ss][T_index[ss][j]]),
// directly on the codebooks + indices, never materialising W.  The
// paper's RTX 3090 design (Alg. 2: one thread per output row, the
// subspace codebook through L1, atomicAdd split-K) is prior art only; on
// B200 its 32 lanes all gather from ONE 1 KiB codebook at random rows, i.e.
// ~3 SMEM/L1 wavefronts per warp-gather.  This kernel instead:
//
//  * lane s of a warp owns subspace s of the current 32-subspace group and
//    keeps x_s in registers; the warp owns RW output rows (64 at B = 1).  The
//    group's codebook image sits in SMEM k-major, [C][32 lanes][E bytes], so
//    lane s gathers from bank s whatever the indices are: one wavefront per
//    warp-gather.  The index table is stored subspace-major per 64-row block
//    (layout.cu), so ONE LDS.128 gives a lane the indices of 16 rows; per
//    index the lane issues PRMT (extract k), LEA (address), LDS and two FHFMA
//    (fma.rn.f32.f16: exact fp16 product, fp32 accumulation) at d = 2.  The
//    32 lanes' per-row partials are summed once per K range by a transposed
//    butterfly (gemv_core.cuh);
//  * a producer warp streams each (row tile, group) index chunk and the
//    group's codebook image into a 3-stage SMEM ring with the TMA bulk-copy
//    engine (cp.async.bulk + mbarrier complete_tx); consumers never issue
//    global loads in the hot loop;
//  * split-K over subspace groups (grid.y) is merged deterministically in
//    the same kernel: every CTA publishes its partial sums, the last CTA of
//    a row tile to arrive (atomic ticket) adds them in fixed ks order (the
//    paper's atomicAdd merge, is order-nondeterministic).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "fasq_internal.cuh"
#include "gemv_core.cuh"

namespace fasq {

constexpr int kMaxGroup = 4;   // layers per grouped launch (q/k/v, gate/up)

struct GemvLayerArgs {
    const uint8_t* idx;     // [n_groups][F_out_pad][32]
    const uint8_t* cbimg;   // [n_groups][C][32][E]
    const void* cbmap;      // d <= 2: codebook PAIR tensor map (fasq_layer::cbmap)
    void* y;                // [B][F_out]
    long long* acc;         // ksplit > 1: int64 fixed-point sums [B][F_out_pad] (per-call workspace, zeroed)
    unsigned* cnt;          // ksplit > 1: contributions per output [B][F_out_pad] (zeroed)
    int F_out, F_out_pad, N_ss, n_groups, C, ksplit, cta_begin;
};

// Fixed-point accumulation mode (FASQ_ACC_I64): partial sums are converted
// to int64 in units of 2^-32 (exact scaling, one RN rounding each) and
// red.add'ed -- integer addition is associative, so the result is
// deterministic whatever the arrival order, with no split-K merge phase.
using core::kAccScale;
using core::kAccInv;

struct GemvParams {
    GemvLayerArgs L[kMaxGroup];   // layers sharing x (grouped launch); CTAs are laid out layer-major
    int nl;
    int x_acc;                    // 1: x is int64 [B][F_in] in units of 2^-32 (FASQ_ACC_I64)
    int y_acc;                    // 1: ys are int64 [B][F_out] accumulators (red.add, caller-zeroed)
    unsigned long long* zero_ptr; // side job: zero these words (not used by this launch)
    long long zero_words;
    GemvLayerArgs N[kMaxGroup];   // the NEXT launch of a decode chain (L2 prefetch hints), nn = 0: none
    int nn;
    const __half* x;        // [B][F_in]
    int F_in, B, y_f32;
    int gmax;               // max groups per CTA (x staging capacity)
};

// SMEM layout: cb ring [ST][C][32][E] (one contiguous TMA bulk copy per
// stage -- the microbenchmark in tools/mb_bulk.cu shows 128-B bulk copies
// cap at ~0.6 TB/s while >=16 KiB copies reach ~7 TB/s), index ring
// [ST][R/64][32][64], x [gmax][32][NB][E], mbarriers full[ST], empty[ST].
// Under programmatic dependent launch the NEXT layer's CTAs may become
// resident as soon as SMEM allows and prefetch their codebook/index stages
// (weights do not depend on x); they only wait (griddepcontrol.wait) before
// touching x.
template <int D, int NB, int NW, int ST>
__global__ void __launch_bounds__((NW + 1) * 32, 1) k_gemv(GemvParams p) {
    constexpr int E = core::Entry<D>::value;
    // d <= 2, B = 1: row-set mapping (gemv_core.cuh, G = 8 lanes per row set).
    // B > 1 keeps lane = subspace with 64/B rows per warp here: a per-launch
    // GEMV is dominated by per-CTA fixed costs and wants the finer row tiles
    // (measured: the row-set mapping's 1024-row tiles were 15-30 % slower at
    // B = 2..8 per launch; the decode chain uses row sets at every B).
    constexpr bool PAIR_ = D <= 2 && NB == 1;
    constexpr int RW = core::RowsPerWarp<NB>::value;   // rows per consumer warp
    constexpr int G = 8;
    constexpr int R = RW * NW;                         // rows per CTA tile
    constexpr int XG = 32 * NB * E;                    // x bytes per staged group
    constexpr bool PAIR = D <= 2;                      // codebook PAIR ring (gemv_core.cuh)
    constexpr int CS = kPairSlots;
    extern __shared__ __align__(1024) uint8_t smem[];

    int li = 0;
#pragma unroll
    for (int l = 1; l < kMaxGroup; ++l)
        if (l < p.nl && (int)blockIdx.x >= p.L[l].cta_begin) li = l;
    const GemvLayerArgs& la = p.L[li];
    const int C = la.C;
    const int ksplit = la.ksplit, n_groups = la.n_groups, F_out = la.F_out, F_out_pad = la.F_out_pad;
    const uint32_t CBB = (uint32_t)C * 32u * E;   // codebook image bytes per group
    const int local = (int)blockIdx.x - la.cta_begin;
    const int rt = local / ksplit, ks = local % ksplit;
    const int g_begin = (int)((int64_t)ks * n_groups / ksplit);
    const int g_end = (int)((int64_t)(ks + 1) * n_groups / ksplit);
    const int ng = g_end - g_begin;
    const int r0 = rt * R;
    const int rows_valid = min(R, F_out_pad - r0);   // multiple of 64

    uint8_t* s_cb = smem;                                     // PAIR: CS*64 KiB, else ST*CBB
    uint8_t* s_idx = s_cb + (PAIR ? CS * kPairSlot : ST * CBB);   // ST*R*32
    uint8_t* s_x = s_idx + ST * R * 32;                       // gmax*XG
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_x + p.gmax * XG);   // full[ST], empty[ST], cfull[CS], cempty[CS]
    const uint32_t cb_u = dev::smem_u32(s_cb);
    const uint32_t x_u = dev::smem_u32(s_x);
    const uint32_t idx_u = dev::smem_u32(s_idx);
    const uint32_t full0 = dev::smem_u32(&bars[0]);
    const uint32_t empty0 = dev::smem_u32(&bars[ST]);
    const uint32_t cfull0 = dev::smem_u32(&bars[2 * ST]), cempty0 = dev::smem_u32(&bars[2 * ST + CS]);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

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
        dev::pdl_launch_dependents();   // let the next layer's CTAs start prefetching now
    }
    __syncthreads();

    if (warp == NW) {
        // ------------------------- producer warp -------------------------
        if (lane == 0) {
            const uint32_t idx_chunk = (uint32_t)rows_valid * 32u;
            for (int i = 0; i < ng; ++i) {
                const int g = g_begin + i;
                if (PAIR && (i & 1) == 0) {   // groups g, g+1 -> one pair slot (one 3-D TMA box)
                    const int cs = (i >> 1) % CS;
                    if ((i >> 1) >= CS) dev::mbar_wait(cempty0 + 8 * cs, (((i >> 1) / CS) + 1) & 1);
                    dev::mbar_arrive_expect_tx(cfull0 + 8 * cs, 2u * CBB);
                    dev::tma_load_3d(cb_u + (uint32_t)cs * kPairSlot, la.cbmap, 0, g, 0, cfull0 + 8 * cs);
                }
                const int slot = i % ST;
                if (i >= ST) dev::mbar_wait(empty0 + 8 * slot, ((i / ST) + 1) & 1);
                const uint32_t full = full0 + 8 * slot;
                dev::mbar_arrive_expect_tx(full, PAIR ? idx_chunk : idx_chunk + CBB);
                if (!PAIR) dev::bulk_g2s(cb_u + (uint32_t)slot * CBB, la.cbimg + (size_t)g * CBB, CBB, full);
                dev::bulk_g2s(idx_u + (uint32_t)slot * R * 32u, la.idx + ((size_t)g * F_out_pad + r0) * 32,
                              idx_chunk, full);
                if (i == ng - 1 && p.nn > 0) {
                    // this CTA's counterpart in the next launch of the chain: warm L2 with
                    // its first ST stages while this layer finishes (HBM is otherwise idle
                    // during the split-K merge and the kernel boundary)
                    int nli = 0;
                    for (int l = 1; l < p.nn; ++l)
                        if ((int)blockIdx.x >= p.N[l].cta_begin) nli = l;
                    const GemvLayerArgs& na = p.N[nli];
                    const int nlocal = (int)blockIdx.x - na.cta_begin;
                    const int nrt = nlocal / na.ksplit, nks = nlocal % na.ksplit;
                    const int nr0 = nrt * R;
                    if (nlocal >= 0 && nr0 < na.F_out_pad) {
                        const int nrows = min(R, na.F_out_pad - nr0);
                        const int ng0 = (int)((int64_t)nks * na.n_groups / na.ksplit);
                        const int ng1 = (int)((int64_t)(nks + 1) * na.n_groups / na.ksplit);
                        const uint32_t ncbb = (uint32_t)na.C * 32u * E;
                        for (int gg = ng0; gg < min(ng1, ng0 + ST); ++gg) {
                            dev::bulk_prefetch_l2(na.cbimg + (size_t)gg * ncbb, ncbb);
                            dev::bulk_prefetch_l2(na.idx + ((size_t)gg * na.F_out_pad + nr0) * 32, (uint32_t)nrows * 32u);
                        }
                    }
                }
            }
        }
        __syncwarp();
        return;
    }

    // --------------------------- consumer warps ----------------------------
    // x staging (after the previous kernel's writes are visible).
    dev::pdl_wait();
    {
        core::stage_x<D, NB, NW>(s_x, p.x, p.x_acc, p.F_in, p.B, la.N_ss, g_begin, ng);
        asm volatile("bar.sync 1, %0;" :: "n"(NW * 32) : "memory");
    }

    float acc[PAIR_ ? 1 : RW][NB];        // lane = subspace mapping (d = 4, 8)
    float accs[PAIR_ ? 2 * G * NB : 1];   // row-set mapping (d <= 2)
#pragma unroll
    for (int q = 0; q < (PAIR_ ? 1 : RW); ++q)
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[q][b] = 0.f;
#pragma unroll
    for (int q = 0; q < (PAIR_ ? 2 * G * NB : 1); ++q) accs[q] = 0.f;

    const int wrow0 = warp * RW;
    const bool active = wrow0 < rows_valid;          // rows_valid is a multiple of 64 >= RW
    const auto co = core::chunk_offsets<RW>(wrow0, lane);
    const auto sm = core::set_map<G>(wrow0, lane);
    int slot = 0;
    uint32_t par = 0;
    if constexpr (PAIR) {
        int cslot = 0;
        uint32_t cpar = 0;
        for (int i = 0; i < ng; i += 2) {
            dev::mbar_wait(cfull0 + 8 * cslot, cpar);
            const uint32_t lbs = (uint32_t)cslot << 16;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h == 1 && i + 1 >= ng) break;
                dev::mbar_wait(full0 + 8 * slot, par);
                if (active) {
                    if constexpr (PAIR_) {
                        core::compute_group_set<D, NB, G>(accs, s_idx + slot * R * 32, sm, s_cb,
                                                          lbs + ((uint32_t)h << 7), s_x + (i + h) * XG);
                    } else {
                        uint32_t xv[NB][E / 4];
                        core::load_x<D, NB>(xv, s_x + (i + h) * XG, lane);
                        core::compute_group_pair<D, NB, RW>(acc, s_idx + slot * R * 32, co, s_cb,
                                                            (uint32_t)lane * 4u + lbs + ((uint32_t)h << 7), xv);
                    }
                }
                __syncwarp();
                if (lane == 0) dev::mbar_arrive(empty0 + 8 * slot);
                if (++slot == ST) { slot = 0; par ^= 1u; }
            }
            if (lane == 0) dev::mbar_arrive(cempty0 + 8 * cslot);
            if (++cslot == CS) { cslot = 0; cpar ^= 1u; }
        }
    } else {
        for (int i = 0; i < ng; ++i) {
            dev::mbar_wait(full0 + 8 * slot, par);
            if (active) {
                uint32_t xv[NB][E / 4];
                core::load_x<D, NB>(xv, s_x + i * XG, lane);
                core::compute_group<D, NB, RW>(acc, s_idx + slot * R * 32, co, s_cb + slot * CBB, xv, lane);
            }
            __syncwarp();
            if (lane == 0) dev::mbar_arrive(empty0 + 8 * slot);
            if (++slot == ST) { slot = 0; par ^= 1u; }
        }
    }

    // ------------------------------ epilogue --------------------------------
    if (p.zero_words > 0) {       // side job (e.g. the accumulators of the launch two steps back)
        const long long per = (p.zero_words + gridDim.x - 1) / gridDim.x;
        const long long zb = per * blockIdx.x, ze = min(p.zero_words, zb + per);
        for (long long i = zb + threadIdx.x; i < ze; i += NW * 32) p.zero_ptr[i] = 0ull;
    }
    core::RowTotals<NB, RW> tot;
    if constexpr (PAIR_) {
        // row sets: lane holds rows lane and 32 + lane of the warp (RowTotals of RW = 64)
        core::reduce_set<NB, G>(accs, lane);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int b = 0; b < NB; ++b) tot.v[h][b] = accs[h * NB + b];
        tot.rsel = lane;
        tot.own = true;
    } else {
        core::reduce_rows<NB, RW>(acc, tot, lane);
    }
    constexpr int H = core::RowTotals<NB, RW>::H;
    if (p.y_acc) {
        if (active)
            core::acc_store<NB, RW>(tot, reinterpret_cast<unsigned long long*>(la.y), r0 + wrow0, F_out, p.B);
        return;
    }
    if (ksplit == 1) {
        if (active && tot.own) {
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int row = r0 + wrow0 + h * 32 + tot.rsel;
                if (row >= F_out) continue;
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    if (b >= p.B) continue;
                    if (p.y_f32) reinterpret_cast<float*>(la.y)[(size_t)b * F_out + row] = tot.v[h][b];
                    else reinterpret_cast<__half*>(la.y)[(size_t)b * F_out + row] = __float2half_rn(tot.v[h][b]);
                }
            }
        }
        return;
    }
    // split-K, no merge phase: every K-split CTA adds its partial, rounded once
    // to int64 units of 2^-32 (exact scaling; integer addition is associative
    // -> deterministic), into acc[b][row] and then counts itself in cnt[b][row]
    // with acq_rel; the CTA that brings the count to ksplit is the last
    // contributor of that output: its acquire sees every add, so it converts
    // the sum and stores y.  No barrier, no second pass over partials (the
    // dense-output merge of round 1 cost three L2 round trips per launch).
    if (active && tot.own) {
        // 1. every add, relaxed; 2. ONE fence (orders this thread's adds before
        // its counts); 3. relaxed counts; 4. the last contributor fences
        // (acquire side) and converts.  Per-output acq_rel atomics serialised a
        // full L2 round trip per output.
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const int row = r0 + wrow0 + h * 32 + tot.rsel;
            if (row >= F_out) continue;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                if (b >= p.B) continue;
                const long long v = __float2ll_rn(tot.v[h][b] * kAccScale);
                asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(la.acc + (size_t)b * F_out_pad + row), "l"(v) : "memory");
            }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        unsigned last = 0u;   // bit (h * NB + b): this thread completed that output
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const int row = r0 + wrow0 + h * 32 + tot.rsel;
            if (row >= F_out) continue;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                if (b >= p.B) continue;
                unsigned old;
                asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(la.cnt + (size_t)b * F_out_pad + row) : "memory");
                if (old == (unsigned)ksplit - 1u) last |= 1u << (h * NB + b);
            }
        }
        if (last) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int row = r0 + wrow0 + h * 32 + tot.rsel;
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    if (!(last >> (h * NB + b) & 1u)) continue;
                    const size_t w = (size_t)b * F_out_pad + row;
                    long long sum;
                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(sum) : "l"(la.acc + w) : "memory");
                    la.acc[w] = 0ll;   // self-cleaning for the next launch on this stream
                    la.cnt[w] = 0u;
                    const double val = (double)sum * kAccInv;
                    if (p.y_f32) reinterpret_cast<float*>(la.y)[(size_t)b * F_out + row] = (float)val;
                    else reinterpret_cast<__half*>(la.y)[(size_t)b * F_out + row] = __double2half(val);
                }
            }
        }
    }
}

// ------------------------------- host side ----------------------------------
static int g_num_sms = 0;
static std::mutex g_mu;

static int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        g_num_sms = n > 0 ? n : 148;
    }
    return g_num_sms;
}

struct GemvPlan {
    int rw, nw, st, R;
    int nl;
    int row_tiles[kMaxGroup], ksplit[kMaxGroup];
    int gmax, grid;
    size_t smem;
};

template <int D, int NB, int NW, int ST>
static fasq_status launch_gemv_t(const GemvParams& p, const GemvPlan& pl, uint32_t flags, cudaStream_t st) {
    auto kern = k_gemv<D, NB, NW, ST>;
    static size_t lim = 0;
    static std::once_flag once;
    std::call_once(once, [&] { lim = set_max_dyn_smem(kern); });
    if (lim < pl.smem) { set_error("gemv: dynamic SMEM plan exceeds the device limit"); return FASQ_E_UNSUPPORTED; }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.grid, 1, 1);
    cfg.blockDim = dim3((NW + 1) * 32, 1, 1);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (flags & FASQ_FLAG_PDL) ? 1 : 0;
    FASQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    return FASQ_OK;
}

template <int D, int NB>
static fasq_status dispatch_cfg(const GemvParams& p, const GemvPlan& pl, uint32_t flags, cudaStream_t st) {
#define FASQ_GEMV_CFG_CASE(NW_, ST_) \
    if (pl.nw == NW_ && pl.st == ST_) return launch_gemv_t<D, NB, NW_, ST_>(p, pl, flags, st);
    FASQ_GEMV_CFG_CASE(16, 3)
    FASQ_GEMV_CFG_CASE(16, 2)
    FASQ_GEMV_CFG_CASE(16, 1)
    FASQ_GEMV_CFG_CASE(16, 4)
    FASQ_GEMV_CFG_CASE(8, 3)
    FASQ_GEMV_CFG_CASE(8, 2)
    FASQ_GEMV_CFG_CASE(8, 1)
#undef FASQ_GEMV_CFG_CASE
    set_error("gemv: no kernel instantiated for this tiling");
    return FASQ_E_UNSUPPORTED;
}

template <int D>
static fasq_status dispatch_nb(int NB, const GemvParams& p, const GemvPlan& pl, uint32_t flags, cudaStream_t st) {
    switch (NB) {
        case 1: return dispatch_cfg<D, 1>(p, pl, flags, st);
        case 2: return dispatch_cfg<D, 2>(p, pl, flags, st);
        case 4: return dispatch_cfg<D, 4>(p, pl, flags, st);
        case 8: return dispatch_cfg<D, 8>(p, pl, flags, st);
    }
    return FASQ_E_UNSUPPORTED;
}

// Tiling plan: each layer's work is split into R-row tiles
// x K-ranges of 32-subspace groups; the CTAs of all layers of a (grouped)
// launch add up to about #SMs, one CTA per SM -- the second SM slot is left
// for the NEXT launch's prefetch under PDL (no CTA waits on another: split-K
// outputs are converted by their last contributor, see the epilogue).  CTAs are shared between the
// layers in proportion to their index bytes.  Env FASQ_GEMV_CFG="nw,stages"
// overrides the default tiling (tuning only).
static int gemv_rows_per_warp(int NB) { return NB == 1 ? 64 : NB == 2 ? 32 : NB == 4 ? 16 : 8; }

static GemvPlan plan_gemv(const fasq_layer* const* Ls, int nl, int NB, bool spin_merge = true) {
    GemvPlan pl{};
    pl.nw = 16;
    pl.st = 3;
    pl.rw = gemv_rows_per_warp(NB);
    if (const char* e = getenv("FASQ_GEMV_CFG")) {
        int a = 0, b = 0;
        if (sscanf(e, "%d,%d", &a, &b) == 2) { pl.nw = a; pl.st = b; }
    }
    pl.nl = nl;
    const int E = Ls[0]->E;
    int maxC = 0;
    for (int l = 0; l < nl; ++l) maxC = std::max(maxC, Ls[l]->C);
    // large codebook images (d = 4/8 with C = 256: 64/128 KiB per group): fewer
    // stages, then fewer rows per CTA
    const bool pair = E == 4;   // codebook PAIR ring (d <= 2)
    auto cbring = [&](int st) { return pair ? (size_t)kPairSlots * kPairSlot : (size_t)st * maxC * 32 * E; };
    auto ring = [&](int st, int nw) { return cbring(st) + (size_t)st * pl.rw * nw * 32 + 2 * 1024; };
    while (pl.st > 2 && ring(pl.st, pl.nw) > kSmemMax) --pl.st;
    if (ring(pl.st, pl.nw) > kSmemMax && pl.nw > 8) pl.nw = 8;
    while (pl.st > 1 && ring(pl.st, pl.nw) > kSmemMax) --pl.st;
    pl.R = pl.rw * pl.nw;
    int sms = num_sms();
    if (!spin_merge) {   // ACC outputs: no co-residency requirement; FASQ_GEMV_OCC = CTAs per SM to plan for
        if (const char* e = getenv("FASQ_GEMV_OCC")) sms *= std::max(1, atoi(e));
    }
    double W = 0;
    for (int l = 0; l < nl; ++l) W += (double)Ls[l]->F_out_pad * Ls[l]->n_groups;
    int total = 0;
    for (int l = 0; l < nl; ++l) {
        const fasq_layer* L = Ls[l];
        pl.row_tiles[l] = (L->F_out_pad + pl.R - 1) / pl.R;
        const double share = sms * ((double)L->F_out_pad * L->n_groups) / W;
        int ks = std::max(1, (int)(share / pl.row_tiles[l]));
        ks = std::min(ks, L->n_groups);
        if (getenv("FASQ_GEMV_UNEVEN") == nullptr) {     // balance: equal groups per CTA
            const int gper = (L->n_groups + ks - 1) / ks;
            ks = (L->n_groups + gper - 1) / gper;
        }
        pl.ksplit[l] = ks;
        total += pl.row_tiles[l] * ks;
    }
    // co-residency (the dense-output merge spins on its peers): shrink the
    // largest K-split until all CTAs fit on the SMs
    while (spin_merge && total > sms) {
        int lm = -1;
        for (int l = 0; l < nl; ++l)
            if (pl.ksplit[l] > 1 && (lm < 0 || pl.ksplit[l] * pl.row_tiles[l] > pl.ksplit[lm] * pl.row_tiles[lm])) lm = l;
        if (lm < 0) break;                               // ksplit == 1 everywhere: no spin, waves are fine
        total -= pl.row_tiles[lm];
        pl.ksplit[lm] -= 1;
    }
    pl.grid = total;
    pl.gmax = 1;
    for (int l = 0; l < nl; ++l) pl.gmax = std::max(pl.gmax, (Ls[l]->n_groups + pl.ksplit[l] - 1) / pl.ksplit[l]);
    const size_t xg = (size_t)32 * NB * E;
    auto smem_of = [&](int st) {
        return cbring(st) + (size_t)st * pl.R * 32 + (size_t)pl.gmax * xg + 16 * (st + kPairSlots);
    };
    while (pl.st > 1 && smem_of(pl.st) > kSmemMax) --pl.st;
    pl.smem = smem_of(pl.st);
    return pl;
}

static void fill_layer_args(GemvLayerArgs* a, const fasq_layer* L, const GemvPlan& pl, int l, int cta, void* y,
                            long long* acc = nullptr, unsigned* cnt = nullptr) {
    a->idx = L->idx;
    a->cbimg = L->cbimg;
    a->cbmap = L->cbmap;
    a->y = y;
    a->acc = acc;
    a->cnt = cnt;
    a->F_out = (int)L->F_out;
    a->F_out_pad = L->F_out_pad;
    a->N_ss = L->N_ss;
    a->n_groups = L->n_groups;
    a->C = L->C;
    a->ksplit = pl.ksplit[l];
    a->cta_begin = cta;
}

fasq_status gemv_grouped_launch(const fasq_layer* const* Ls_, int nl, const __half* x, int B, void* const* ys,
                                fasq_dtype yt, uint32_t flags, cudaStream_t st, const fasq_layer* const* next,
                                int n_next) {
    GemvOpts o{};
    o.flags = flags;
    o.next = next;
    o.n_next = n_next;
    return gemv_grouped_launch2(Ls_, nl, x, B, ys, yt, o, st);
}

fasq_status gemv_grouped_launch2(const fasq_layer* const* Ls_, int nl, const void* x_, int B, void* const* ys,
                                 fasq_dtype yt, const GemvOpts& o, cudaStream_t st) {
    const __half* x = static_cast<const __half*>(x_);
    const uint32_t flags = o.flags;
    const fasq_layer* const* next = o.next;
    const int n_next = o.n_next;
    if (nl < 1 || nl > kMaxGroup) return FASQ_E_UNSUPPORTED;
    for (int l = 1; l < nl; ++l)
        if (Ls_[l]->F_in != Ls_[0]->F_in || Ls_[l]->d != Ls_[0]->d) return FASQ_E_SHAPE;
    const int NB = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : 8;
    GemvPlan pl = plan_gemv(Ls_, nl, NB, false);   // no output mode spins on peers any more
    GemvParams p{};
    p.x_acc = o.x_acc;
    p.y_acc = o.y_acc;
    p.zero_ptr = static_cast<unsigned long long*>(o.zero_ptr);
    p.zero_words = o.zero_ptr ? o.zero_bytes / 8 : 0;
    p.nl = nl;
    p.x = x;
    p.F_in = (int)Ls_[0]->F_in;
    p.B = B;
    p.y_f32 = yt == FASQ_F32;
    p.gmax = pl.gmax;
    // split-K with dense outputs: int64 sums + contribution counts per output.
    // Workspace: the calling STREAM's (layers stay immutable; launches on one
    // stream are ordered, and the last contributor of every output zeroes its
    // words again -- no memset per launch); grown outside stream capture.  A
    // first launch inside capture with too small a stream workspace gets a
    // per-call workspace (allocation + memset nodes) instead.
    size_t acc_bytes = 0, cnt_bytes = 0;
    size_t acc_off[kMaxGroup] = {}, cnt_off[kMaxGroup] = {};
    if (!o.y_acc)
        for (int l = 0; l < nl; ++l)
            if (pl.ksplit[l] > 1) {
                acc_off[l] = acc_bytes;
                acc_bytes += (size_t)B * Ls_[l]->F_out_pad * sizeof(long long);
                cnt_off[l] = cnt_bytes;
                cnt_bytes += (size_t)B * Ls_[l]->F_out_pad * sizeof(unsigned);
            }
    uint8_t* ws = nullptr;
    uint8_t* ws_call = nullptr;   // per-call workspace (capture fallback), released after the launch
    if (acc_bytes) {
        fasq_status s = stream_workspace(st, WS_GEMV, acc_bytes + cnt_bytes, reinterpret_cast<void**>(&ws));
        if (s != FASQ_OK) return s;
        if (!ws) {
            s = dev_alloc_t(&ws_call, acc_bytes + cnt_bytes, st);
            if (s != FASQ_OK) return s;
            cudaError_t e = cudaMemsetAsync(ws_call, 0, acc_bytes + cnt_bytes, st);
            if (e != cudaSuccess) { dev_free(ws_call, st); return cuda_fail(e, "gemv workspace"); }
            ws = ws_call;
        }
    }
    int cta = 0;
    for (int l = 0; l < nl; ++l) {
        const bool sk = ws && pl.ksplit[l] > 1;
        fill_layer_args(&p.L[l], Ls_[l], pl, l, cta, ys[l], sk ? reinterpret_cast<long long*>(ws + acc_off[l]) : nullptr,
                        sk ? reinterpret_cast<unsigned*>(ws + acc_bytes + cnt_off[l]) : nullptr);
        cta += pl.row_tiles[l] * pl.ksplit[l];
    }
    // L2-prefetch hints for the next launch of a decode chain (same tiling family)
    if (next && n_next > 0 && n_next <= kMaxGroup) {
        bool ok = true;
        for (int l = 0; l < n_next; ++l) ok = ok && next[l] && next[l]->d == Ls_[0]->d;
        if (ok) {
            GemvPlan pn = plan_gemv(next, n_next, NB, false);
            if (pn.R == pl.R && pn.st == pl.st) {
                int c2 = 0;
                for (int l = 0; l < n_next; ++l) {
                    fill_layer_args(&p.N[l], next[l], pn, l, c2, nullptr);
                    c2 += pn.row_tiles[l] * pn.ksplit[l];
                }
                p.nn = n_next;
            }
        }
    }
    fasq_status s;
    switch (Ls_[0]->d) {
        case 1: s = dispatch_nb<1>(NB, p, pl, flags, st); break;
        case 2: s = dispatch_nb<2>(NB, p, pl, flags, st); break;
        case 4: s = dispatch_nb<4>(NB, p, pl, flags, st); break;
        case 8: s = dispatch_nb<8>(NB, p, pl, flags, st); break;
        default: s = FASQ_E_UNSUPPORTED;
    }
    dev_free(ws_call, st);   // stream-ordered: released after the launch completes
    if (s == FASQ_OK) set_launch_count(1);
    return s;
}

__global__ void k_acc_convert(const long long* __restrict__ acc, int64_t n, void* out, int f32) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = (double)acc[i] * kAccInv;
    if (f32) reinterpret_cast<float*>(out)[i] = (float)v;
    else reinterpret_cast<__half*>(out)[i] = __double2half(v);
}

fasq_status acc_convert_launch(const void* acc, int64_t n, void* out, fasq_dtype yt, cudaStream_t st) {
    if (n <= 0) return FASQ_OK;
    k_acc_convert<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(static_cast<const long long*>(acc), n, out,
                                                                 yt == FASQ_F32);
    FASQ_CUDA_TRY(cudaGetLastError());
    set_launch_count(1);
    return FASQ_OK;
}

int gemv_tc_min_batch() {
    // the smallest decode batch routed to the tcgen05 kernel (FASQ_GEMV_TC_MIN_B overrides;
    // 0 or > 64 disables it); default from profiles/r02/gemv_tc_sweep.jsonl
    const char* e = getenv("FASQ_GEMV_TC_MIN_B");
    const int v = e ? atoi(e) : kGemvTcMinBatch;
    return v <= 0 ? 1 << 30 : v;
}

fasq_status gemv_launch(const fasq_layer* L, const __half* x, int B, void* y, fasq_dtype yt, uint32_t flags,
                        cudaStream_t st) {
    if (L->bits) return gemv_packed_launch(L, x, B, y, yt, flags, st);   // NEXT-2 packed indices
    if (L->dim0) return gemv_dim0_launch(L, x, B, y, yt, flags, st);     // NEXT-4 output-axis subspaces
    // batched decode on tcgen05 (gemv_tc.cu) from B >= FASQ_GEMV_TC_MIN_B (measured default below)
    if (B >= gemv_tc_min_batch() && gemv_tc_supported(L, B)) return gemv_tc_launch(L, x, B, y, yt, flags, st);
    void* ys[1] = {y};
    return gemv_grouped_launch(&L, 1, x, B, ys, yt, flags, st);
}

}  // namespace fasq
