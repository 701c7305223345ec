// gemv_packed.cu -- NEXT-2: decode GEMV on ceil(log2 C)-bit packed indices (sm_100a).
//
// Eq. 4 charges ceil(log2 K_s) bits per index; Table 2
// uses d = 2 with K_s = 128 / 256 / 512 / 1024 (#W 3.5 / 4 / 4.5 / 5).  The
// byte-index kernels (gemv.cu, chain.cu) store 8 bits whatever C is; this
// kernel reads the packed layout of fasq_internal.cuh (per (group, 64-row
// block, subspace) one LSB-first bitstream of 64 codes) and computes the same
// product, Eq. 3: y[b][j] = sum_ss dot(x[b]_ss, T_cluster[ss][k]).
//
// Mapping (the lane = subspace G2 loop of gemv_core.cuh): lane s owns the
// group's subspace s and keeps x_s in registers; a warp owns RW = 64/NB rows.
// Per group the lane loads its codes' bitstream words from SMEM and, per row,
// places the code at bit 7 with one shift/funnel-shift (compile-time bit
// positions: BITS is a template parameter), ORs in its lane offset (LOP3: the
// image is [C][32 lanes][4 B], so lane s reads bank s for any code -- one
// wavefront per warp-gather), gathers the centroid and adds dot(x_s, c) with
// two FHFMA (exact fp16 products, fp32 accumulation).  Per index: SHF, LOP3,
// LDS, 2 x FHFMA at B = 1.
//
// A producer warp streams each group's index chunk (rows [r0, r0 + R), ONE
// bulk copy) into an ST-deep ring and its codebook image (C x 128 B, one bulk
// copy) into a CS-deep ring (CS = 1 for C = 1024: a 128-KiB image).  Split-K
// over groups is merged like gemv.cu (int64 fixed-point red.add, the last
// contributor converts; deterministic).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "fasq_internal.cuh"
#include "gemv_core.cuh"

namespace fasq {
namespace {

constexpr int kPW = 16;   // consumer warps

struct PackedParams {
    const uint8_t* idx;     // packed [n_groups][F_out_pad/64][32][seg]
    const uint8_t* cbimg;   // [n_groups][C][32][4]
    const __half* x;        // [B][F_in]
    void* y;                // [B][F_out] (f16 / f32) or int64 accumulators (y_mode 2)
    long long* acc;         // split-K workspace [B][F_out_pad] (zeroed, self-cleaning)
    unsigned* cnt;          // [B][F_out_pad]
    int F_out, F_out_pad, F_in, N_ss, n_groups, C, ksplit, B, y_mode, cs, st;
    int gmax;               // max groups per CTA (x staging capacity)
};

template <int BITS, int NB>
__global__ void __launch_bounds__((kPW + 1) * 32, 1) k_gemv_packed(PackedParams p) {
    constexpr int RW = core::RowsPerWarp<NB>::value;   // 64 / NB rows per warp
    constexpr int R = RW * kPW;                        // rows per CTA tile (>= 128)
    constexpr int SEG = 8 * BITS;                      // bytes per (block, subspace) segment
    constexpr uint32_t MASK = ((1u << BITS) - 1u) << 7;   // code at bit 7: k-row stride 128 B
    extern __shared__ __align__(1024) uint8_t smem[];

    const int CS = p.cs, ST = p.st;
    const uint32_t CBB = (uint32_t)p.C * 128u;         // codebook image bytes per group
    const int rt = (int)blockIdx.x / p.ksplit, ks = (int)blockIdx.x % p.ksplit;
    const int g_begin = (int)((int64_t)ks * p.n_groups / p.ksplit);
    const int g_end = (int)((int64_t)(ks + 1) * p.n_groups / p.ksplit);
    const int ng = g_end - g_begin;
    const int r0 = rt * R;
    const int rows_valid = min(R, p.F_out_pad - r0);   // multiple of 64
    const uint32_t chunk = (uint32_t)(rows_valid / 64) * 32u * SEG;

    uint8_t* s_cb = smem;                              // CS x CBB
    uint8_t* s_idx = s_cb + (size_t)CS * CBB;          // ST x (R/64 * 32 * SEG)
    constexpr uint32_t IDXB = (uint32_t)(R / 64) * 32u * SEG;
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_idx + (size_t)ST * IDXB);   // full[ST] empty[ST] cfull[CS] cempty[CS]
    const uint32_t cb_u = dev::smem_u32(s_cb), idx_u = dev::smem_u32(s_idx);
    const uint32_t full0 = dev::smem_u32(&bars[0]), empty0 = dev::smem_u32(&bars[ST]);
    const uint32_t cfull0 = dev::smem_u32(&bars[2 * ST]), cempty0 = dev::smem_u32(&bars[2 * ST + CS]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            dev::mbar_init(full0 + 8 * s, 1);
            dev::mbar_init(empty0 + 8 * s, kPW);
        }
        for (int s = 0; s < CS; ++s) {
            dev::mbar_init(cfull0 + 8 * s, 1);
            dev::mbar_init(cempty0 + 8 * s, kPW);
        }
        dev::fence_barrier_init();
        dev::pdl_launch_dependents();
    }
    __syncthreads();

    if (warp == kPW) {
        // ---- producer: weights never depend on x -> stream from kernel entry ----
        if (lane == 0) {
            int slot = 0, cslot = 0;
            uint32_t par = 0, cpar = 0;
            for (int i = 0; i < ng; ++i) {
                const int g = g_begin + i;
                if (i >= ST) dev::mbar_wait(empty0 + 8 * slot, par ^ 1u);
                dev::mbar_arrive_expect_tx(full0 + 8 * slot, chunk);
                dev::bulk_g2s(idx_u + (uint32_t)slot * IDXB,
                              p.idx + ((size_t)g * (p.F_out_pad / 64) + r0 / 64) * 32 * SEG, chunk, full0 + 8 * slot);
                if (i >= CS) dev::mbar_wait(cempty0 + 8 * cslot, cpar ^ 1u);
                dev::mbar_arrive_expect_tx(cfull0 + 8 * cslot, CBB);
                dev::bulk_g2s(cb_u + (uint32_t)cslot * CBB, p.cbimg + (size_t)g * CBB, CBB, cfull0 + 8 * cslot);
                if (++slot == ST) { slot = 0; par ^= 1u; }
                if (++cslot == CS) { cslot = 0; cpar ^= 1u; }
            }
        }
        __syncwarp();
        return;
    }

    // ---- consumers -----------------------------------------------------------
    const int wrow0 = warp * RW;
    const bool active = wrow0 < rows_valid;
    // this warp's code bits inside its 64-row block's segment: byte offset bo
    // (RW >= 8 rows -> RW*BITS bits is a whole number of bytes)
    const int bo = ((wrow0 & 63) * BITS) >> 3;
    const uint32_t fsh = (uint32_t)(bo & 3) * 8u;     // bit shift inside the first word
    const uint32_t seg_off = (uint32_t)((wrow0 >> 6) * 32 + lane) * SEG + (uint32_t)(bo & ~3);
    const uint32_t lane_off = (uint32_t)lane * 4u;

    float acc[RW][NB];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[r][b] = 0.f;

    dev::pdl_wait();   // x (and the outputs we add into) are the previous kernel's
    // x of the whole K range -> SMEM [group][32 lanes][NB] words once (one global
    // load per word, all in flight) instead of per-group loads on the critical
    // path (ncu: long-scoreboard stalls 5 per issue)
    uint32_t* s_x = reinterpret_cast<uint32_t*>(bars + 2 * ST + 2 * CS);
    for (int e = threadIdx.x; e < ng * 32 * NB; e += kPW * 32) {
        const int gl = e / (32 * NB), rem = e - gl * 32 * NB, sl = rem / NB, b = rem - sl * NB;
        const int ss = (g_begin + gl) * 32 + sl;
        s_x[e] = (b < p.B && ss < p.N_ss) ? __ldg(reinterpret_cast<const unsigned int*>(p.x + (size_t)b * p.F_in) + ss)
                                          : 0u;
    }
    asm volatile("bar.sync 1, %0;" :: "n"(kPW * 32) : "memory");

    int slot = 0, cslot = 0;
    uint32_t par = 0, cpar = 0;
    for (int i = 0; i < ng; ++i) {
        uint32_t xv[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) xv[b] = s_x[(i * 32 + lane) * NB + b];
        dev::mbar_wait(full0 + 8 * slot, par);
        dev::mbar_wait(cfull0 + 8 * cslot, cpar);
        if (active) {
            const uint8_t* sp = s_idx + (size_t)slot * IDXB + seg_off;
            const uint8_t* cbs = s_cb + (size_t)cslot * CBB;
            // rows in chunks of CH: only the bitstream words of one chunk are live
            // (loading all 2*BITS words of a 64-row segment up front spilled)
            constexpr int CH = RW < 16 ? RW : 16;
            constexpr int MW = (CH * BITS + 31) / 32 + 1;   // words a chunk can touch
#pragma unroll
            for (int c0 = 0; c0 < RW; c0 += CH) {
                const int a0 = (c0 * BITS) >> 5;                 // first word of the chunk
                const int a1 = ((c0 + CH) * BITS - 1) >> 5;      // last word
                uint32_t w[MW + 1];
#pragma unroll
                for (int q = 0; q <= MW; ++q) w[q] = 0u;
                if constexpr (RW == 64) {   // warp rows start the segment: word aligned
#pragma unroll
                    for (int q = 0; q < MW; ++q)
                        if (a0 + q <= a1) w[q] = core::lds<uint32_t>(sp + 4 * (a0 + q));
                } else {                    // realign by fsh bits (runtime, < 32)
                    uint32_t raw[MW + 1];
#pragma unroll
                    for (int q = 0; q <= MW; ++q)
                        raw[q] = (a0 + q <= a1 + 1) ? core::lds<uint32_t>(sp + 4 * (a0 + q)) : 0u;
#pragma unroll
                    for (int q = 0; q < MW; ++q)
                        if (a0 + q <= a1) w[q] = __funnelshift_r(raw[q], raw[q + 1], fsh);
                }
                constexpr int JB = CH < 8 ? CH : 8;   // gathers in flight before their FMAs
#pragma unroll
                for (int j0 = 0; j0 < CH; j0 += JB) {
                    uint32_t c[JB];
#pragma unroll
                    for (int j = 0; j < JB; ++j) {
                        const int pbit = (c0 + j0 + j) * BITS - 32 * a0, lo = pbit >> 5, sh = pbit & 31;
                        uint32_t v;
                        if (sh + BITS <= 32) v = sh >= 7 ? (w[lo] >> (sh - 7)) : (w[lo] << (7 - sh));
                        else v = __funnelshift_r(w[lo], w[lo + 1], sh - 7);
                        c[j] = core::lds<uint32_t>(cbs + ((v & MASK) | lane_off));
                    }
#pragma unroll
                    for (int j = 0; j < JB; ++j)
#pragma unroll
                        for (int b = 0; b < NB; ++b)
                            acc[c0 + j0 + j][b] = dev::fhfma2(c[j], xv[b], acc[c0 + j0 + j][b]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            dev::mbar_arrive(empty0 + 8 * slot);
            dev::mbar_arrive(cempty0 + 8 * cslot);
        }
        if (++slot == ST) { slot = 0; par ^= 1u; }
        if (++cslot == CS) { cslot = 0; cpar ^= 1u; }
    }

    // ---- epilogue (as gemv.cu) ---------------------------------------------------
    core::RowTotals<NB, RW> tot;
    core::reduce_rows<NB, RW>(acc, tot, lane);
    constexpr int H = core::RowTotals<NB, RW>::H;
    if (!active) return;
    if (p.y_mode == 2) {
        core::acc_store<NB, RW>(tot, reinterpret_cast<unsigned long long*>(p.y), r0 + wrow0, p.F_out, p.B);
        return;
    }
    if (!tot.own) return;
    if (p.ksplit == 1) {
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const int row = r0 + wrow0 + h * 32 + tot.rsel;
            if (row >= p.F_out) continue;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                if (b >= p.B) continue;
                if (p.y_mode == 1) reinterpret_cast<float*>(p.y)[(size_t)b * p.F_out + row] = tot.v[h][b];
                else reinterpret_cast<__half*>(p.y)[(size_t)b * p.F_out + row] = __float2half_rn(tot.v[h][b]);
            }
        }
        return;
    }
    // split-K without a merge phase: int64 fixed-point adds (units 2^-32), one
    // fence, relaxed counts; the last contributor of an output converts it and
    // re-zeroes its words (deterministic: integer addition is associative)
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const int row = r0 + wrow0 + h * 32 + tot.rsel;
        if (row >= p.F_out) continue;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (b >= p.B) continue;
            const long long v = __float2ll_rn(tot.v[h][b] * core::kAccScale);
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(p.acc + (size_t)b * p.F_out_pad + row), "l"(v)
                         : "memory");
        }
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    unsigned last = 0u;
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const int row = r0 + wrow0 + h * 32 + tot.rsel;
        if (row >= p.F_out) continue;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (b >= p.B) continue;
            unsigned old;
            asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old)
                         : "l"(p.cnt + (size_t)b * p.F_out_pad + row) : "memory");
            if (old == (unsigned)p.ksplit - 1u) last |= 1u << (h * NB + b);
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
                const size_t wd = (size_t)b * p.F_out_pad + row;
                long long sum;
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(sum) : "l"(p.acc + wd) : "memory");
                p.acc[wd] = 0ll;
                p.cnt[wd] = 0u;
                const double val = (double)sum * core::kAccInv;
                if (p.y_mode == 1) reinterpret_cast<float*>(p.y)[(size_t)b * p.F_out + row] = (float)val;
                else reinterpret_cast<__half*>(p.y)[(size_t)b * p.F_out + row] = __double2half(val);
            }
        }
    }
}

int num_sms_packed() {
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

template <int BITS, int NB>
fasq_status launch_t(const PackedParams& p, int grid, size_t smem, uint32_t flags, cudaStream_t st) {
    auto kern = k_gemv_packed<BITS, NB>;
    static size_t lim = 0;
    static std::once_flag once;
    std::call_once(once, [&] { lim = set_max_dyn_smem(kern); });
    if (lim < smem) { set_error("gemv (packed): SMEM plan exceeds the device limit"); return FASQ_E_UNSUPPORTED; }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3((kPW + 1) * 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (flags & FASQ_FLAG_PDL) ? 1 : 0;
    FASQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    return FASQ_OK;
}

template <int NB>
fasq_status dispatch_bits(int bits, const PackedParams& p, int grid, size_t smem, uint32_t flags, cudaStream_t st) {
    switch (bits) {
        case 1: return launch_t<1, NB>(p, grid, smem, flags, st);
        case 2: return launch_t<2, NB>(p, grid, smem, flags, st);
        case 3: return launch_t<3, NB>(p, grid, smem, flags, st);
        case 4: return launch_t<4, NB>(p, grid, smem, flags, st);
        case 5: return launch_t<5, NB>(p, grid, smem, flags, st);
        case 6: return launch_t<6, NB>(p, grid, smem, flags, st);
        case 7: return launch_t<7, NB>(p, grid, smem, flags, st);
        case 8: return launch_t<8, NB>(p, grid, smem, flags, st);
        case 9: return launch_t<9, NB>(p, grid, smem, flags, st);
        case 10: return launch_t<10, NB>(p, grid, smem, flags, st);
    }
    return FASQ_E_UNSUPPORTED;
}

}  // namespace

fasq_status gemv_packed_launch(const fasq_layer* L, const __half* x, int B, void* y, fasq_dtype yt, uint32_t flags,
                               cudaStream_t st) {
    if (!L->bits || L->d != 2) return FASQ_E_UNSUPPORTED;
    if (B < 1 || B > 8) return FASQ_E_UNSUPPORTED;
    if (flags & ~FASQ_FLAG_PDL) return FASQ_E_UNSUPPORTED;   // x is fp16 here (no FASQ_FLAG_X_ACC)
    const int NB = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : 8;
    const int RW = 64 / NB, R = RW * kPW;
    const size_t CBB = (size_t)L->C * 128;
    const size_t IDXB = (size_t)(R / 64) * 32 * L->seg;
    // grid: row tiles x K-splits over groups, ~ one CTA per SM, equal groups per CTA
    const int row_tiles = (L->F_out_pad + R - 1) / R;
    int ks = std::max(1, num_sms_packed() / row_tiles);
    ks = std::min(ks, L->n_groups);
    const int gper = (L->n_groups + ks - 1) / ks;
    ks = (L->n_groups + gper - 1) / gper;
    // rings: two codebook slots when they fit next to two index stages, else one;
    // plus the K range's x ([gper][32][NB] words)
    const size_t xbytes = (size_t)gper * 32 * NB * 4;
    int cs = 2, stg = 3;
    auto smem_of = [&](int c, int s) { return (size_t)c * CBB + (size_t)s * IDXB + 16 * (size_t)(c + s) + xbytes; };
    while (stg > 2 && smem_of(cs, stg) > kSmemMax) --stg;
    if (smem_of(cs, stg) > kSmemMax) cs = 1;
    while (stg > 1 && smem_of(cs, stg) > kSmemMax) --stg;
    const size_t smem = smem_of(cs, stg);
    if (smem > kSmemMax) { set_error("gemv (packed): codebook image too large"); return FASQ_E_UNSUPPORTED; }

    PackedParams p{};
    p.idx = L->idx;
    p.cbimg = L->cbimg;
    p.x = x;
    p.y = y;
    p.F_out = (int)L->F_out;
    p.F_out_pad = L->F_out_pad;
    p.F_in = (int)L->F_in;
    p.N_ss = L->N_ss;
    p.n_groups = L->n_groups;
    p.C = L->C;
    p.ksplit = ks;
    p.B = B;
    p.y_mode = yt == FASQ_ACC_I64 ? 2 : yt == FASQ_F32 ? 1 : 0;
    p.cs = cs;
    p.st = stg;
    p.gmax = gper;
    uint8_t* ws_call = nullptr;
    if (ks > 1 && p.y_mode != 2) {
        // per-(stream, purpose) workspace shared with gemv.cu (stream-ordered, self-cleaning)
        const size_t accb = (size_t)B * L->F_out_pad * 8, cntb = (size_t)B * L->F_out_pad * 4;
        uint8_t* ws = nullptr;
        fasq_status s = stream_workspace(st, WS_GEMV, accb + cntb, reinterpret_cast<void**>(&ws));
        if (s != FASQ_OK) return s;
        if (!ws) {   // first use inside stream capture: a per-call zeroed workspace
            s = dev_alloc_t(&ws_call, accb + cntb, st);
            if (s != FASQ_OK) return s;
            cudaError_t e = cudaMemsetAsync(ws_call, 0, accb + cntb, st);
            if (e != cudaSuccess) { dev_free(ws_call, st); return cuda_fail(e, "gemv (packed) workspace"); }
            ws = ws_call;
        }
        p.acc = reinterpret_cast<long long*>(ws);
        p.cnt = reinterpret_cast<unsigned*>(ws + accb);
    }
    const int grid = row_tiles * ks;
    fasq_status s;
    switch (NB) {
        case 1: s = dispatch_bits<1>(L->bits, p, grid, smem, flags, st); break;
        case 2: s = dispatch_bits<2>(L->bits, p, grid, smem, flags, st); break;
        case 4: s = dispatch_bits<4>(L->bits, p, grid, smem, flags, st); break;
        default: s = dispatch_bits<8>(L->bits, p, grid, smem, flags, st); break;
    }
    dev_free(ws_call, st);
    if (s == FASQ_OK) set_launch_count(1);
    return s;
}

}  // namespace fasq
