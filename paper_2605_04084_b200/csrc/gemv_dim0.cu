// gemv_dim0.cu -- NEXT-4: decode GEMV on the paper's dim = 0 partition (sm_100a).
//
// Eq. 2's first case -- the layout of the paper's experiments,
// "dim=0 (quantization along the output dimension)" -- splits W's
// OUTPUT rows into N_ss = F_out/d subspaces; the datapoints are W's columns,
// so T_index is [N_ss][F_in] and
//
//     y[b][ss*d + e] = sum_j x[b][j] * T_cluster[ss/group][T_index[ss][j]][e].
//
// Mapping: a CTA owns one group of 32 subspaces (32*d output rows) and a
// range of columns; lane s of every warp is subspace s.  The group's 32
// codebooks are staged ONCE per CTA ([C][32 lanes][E] image: lane s reads bank
// s for any index -- one wavefront per warp-gather); the index table streams
// through an SMEM ring in 512-column chunks ([16-column block][32][16]: one
// LDS.128 gives a lane its 16 indices) and the warps take the chunk's 16-column
// blocks round-robin.  x[b][j] is the same for every lane (a broadcast load);
// every index costs extract, address, LDS and d*B FHFMA (c_e * x_j: exact fp16
// products, fp32 accumulation), and a lane accumulates only its OWN d outputs
// per token -- no cross-lane reduction at all (the input-axis kernels end every
// K range with a 32-lane butterfly).  The warps' partials are summed through
// SMEM in fixed warp order, then split-K over column ranges is merged like
// gemv.cu (int64 fixed-point red.add, the last contributor converts).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "fasq_internal.cuh"
#include "gemv_core.cuh"

namespace fasq {
namespace {

constexpr int kDW = 16;     // consumer warps
constexpr int kCH = 512;    // columns per index stage (32 blocks of 16)

struct Dim0Params {
    const uint8_t* idx;     // [n_groups][K_pad/16][32][16]
    const uint8_t* cbimg;   // [n_groups][C][32][E]
    const __half* x;        // [B][F_in]
    void* y;
    long long* acc;
    unsigned* cnt;
    int F_out, F_in, K_pad, N_ss, C, ksplit, B, y_mode, st;
    int x_staged;           // 1: the producer stages x[b][stage columns] next to the indices
};

// acc += c_half[CS] * x_half[XS]  (fma.rn.f32.f16: exact product, one fp32 rounding)
template <int CS, int XS>
__device__ __forceinline__ float fma_hh(uint32_t c, uint32_t x, float acc) {
    if constexpr (CS == 0 && XS == 0)
        asm("{.reg .f16 c0, c1, x0, x1;\n\tmov.b32 {c0, c1}, %1;\n\tmov.b32 {x0, x1}, %2;\n\t"
            "fma.rn.f32.f16 %0, c0, x0, %0;}" : "+f"(acc) : "r"(c), "r"(x));
    else if constexpr (CS == 0 && XS == 1)
        asm("{.reg .f16 c0, c1, x0, x1;\n\tmov.b32 {c0, c1}, %1;\n\tmov.b32 {x0, x1}, %2;\n\t"
            "fma.rn.f32.f16 %0, c0, x1, %0;}" : "+f"(acc) : "r"(c), "r"(x));
    else if constexpr (CS == 1 && XS == 0)
        asm("{.reg .f16 c0, c1, x0, x1;\n\tmov.b32 {c0, c1}, %1;\n\tmov.b32 {x0, x1}, %2;\n\t"
            "fma.rn.f32.f16 %0, c1, x0, %0;}" : "+f"(acc) : "r"(c), "r"(x));
    else
        asm("{.reg .f16 c0, c1, x0, x1;\n\tmov.b32 {c0, c1}, %1;\n\tmov.b32 {x0, x1}, %2;\n\t"
            "fma.rn.f32.f16 %0, c1, x1, %0;}" : "+f"(acc) : "r"(c), "r"(x));
    return acc;
}

// (a 2-CTA/SM variant -- launch bounds capping the registers at 56 -- was
// measured slower: the cap serialised the gathers; profiles/r02/dim0_gemv_ab.txt)
template <int D, int NB>
__global__ void __launch_bounds__((kDW + 1) * 32, 1) k_gemv_dim0(Dim0Params p) {
    constexpr int E = core::Entry<D>::value;     // 4 (d <= 2, d = 1 padded), 8, 16 bytes
    constexpr int EW = E / 4;                    // centroid words
    constexpr uint32_t KROW = 32u * E;           // bytes per k-row of the image
    constexpr uint32_t IXB = kCH * 32u;          // index bytes per stage
    constexpr uint32_t XSB = kCH * 2u;           // x bytes per token per stage
    constexpr uint32_t STB = IXB + NB * XSB;     // stage: indices, then x [NB][kCH] fp16
    extern __shared__ __align__(1024) uint8_t smem[];

    const int ST = p.st;
    const uint32_t CBB = (uint32_t)p.C * KROW;
    const int g = (int)blockIdx.x / p.ksplit, ks = (int)blockIdx.x % p.ksplit;
    const int units = p.K_pad / 64;                                   // 64-column units
    const int u0 = (int)((int64_t)ks * units / p.ksplit), u1 = (int)((int64_t)(ks + 1) * units / p.ksplit);
    const int j0 = u0 * 64, j1 = u1 * 64;                             // this CTA's columns
    const int nst = (j1 - j0 + kCH - 1) / kCH;                        // index stages

    uint8_t* s_cb = smem;
    uint8_t* s_idx = smem + CBB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_idx + (size_t)ST * STB);   // cfull, full[ST], empty[ST]
    const uint32_t cfull = dev::smem_u32(&bars[0]);
    const uint32_t full0 = dev::smem_u32(&bars[1]), empty0 = dev::smem_u32(&bars[1 + ST]);
    const uint32_t cb_u = dev::smem_u32(s_cb), idx_u = dev::smem_u32(s_idx);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        dev::mbar_init(cfull, 1);
        for (int s = 0; s < ST; ++s) {
            dev::mbar_init(full0 + 8 * s, 1);
            dev::mbar_init(empty0 + 8 * s, kDW);
        }
        dev::fence_barrier_init();
        dev::pdl_launch_dependents();
    }
    __syncthreads();

    if (warp == kDW) {
        // ---- producer: the group's codebooks once, then per stage the index chunk
        // and (x_staged) the stage's x columns of every token.  Weights do not
        // depend on x: the first ST stages' indices go out before
        // griddepcontrol.wait, their x right after it.
        if (lane == 0) {
            dev::mbar_arrive_expect_tx(cfull, CBB);
            dev::bulk_g2s(cb_u, p.cbimg + (size_t)g * CBB, CBB, cfull);
            auto xbytes = [&](int c0, int cols) {   // valid x bytes of a stage (F_in % 8 == 0 when staged)
                return (uint32_t)max(0, min(cols, p.F_in - c0)) * 2u;
            };
            auto issue_x = [&](int i, int slot) {
                const int c0 = j0 + i * kCH, cols = min(kCH, j1 - c0);
                const uint32_t xb = xbytes(c0, cols);
                if (!xb) return;
                for (int b = 0; b < p.B; ++b)
                    dev::bulk_g2s(idx_u + (uint32_t)slot * STB + IXB + (uint32_t)b * XSB,
                                  p.x + (size_t)b * p.F_in + c0, xb, full0 + 8 * slot);
            };
            const int pre = min(ST, nst);
            for (int i = 0; i < pre; ++i) {
                const int c0 = j0 + i * kCH, cols = min(kCH, j1 - c0);
                const uint32_t xb = p.x_staged ? xbytes(c0, cols) * (uint32_t)p.B : 0u;
                dev::mbar_arrive_expect_tx(full0 + 8 * i, (uint32_t)cols * 32u + xb);
                dev::bulk_g2s(idx_u + (uint32_t)i * STB, p.idx + ((size_t)g * (p.K_pad / 16) + c0 / 16) * 512,
                              (uint32_t)cols * 32u, full0 + 8 * i);
            }
            if (p.x_staged) {
                dev::pdl_wait();
                for (int i = 0; i < pre; ++i) issue_x(i, i);
            }
            int slot = pre % ST;
            uint32_t par = pre == ST ? 1u : 0u;
            for (int i = pre; i < nst; ++i) {
                const int c0 = j0 + i * kCH, cols = min(kCH, j1 - c0);
                const uint32_t xb = p.x_staged ? xbytes(c0, cols) * (uint32_t)p.B : 0u;
                dev::mbar_wait(empty0 + 8 * slot, par ^ 1u);
                dev::mbar_arrive_expect_tx(full0 + 8 * slot, (uint32_t)cols * 32u + xb);
                dev::bulk_g2s(idx_u + (uint32_t)slot * STB, p.idx + ((size_t)g * (p.K_pad / 16) + c0 / 16) * 512,
                              (uint32_t)cols * 32u, full0 + 8 * slot);
                if (p.x_staged) issue_x(i, slot);
                if (++slot == ST) { slot = 0; par ^= 1u; }
            }
        }
        __syncwarp();
        return;
    }

    // ---- consumers -------------------------------------------------------------
    // AS independent accumulator sets (column q -> set q % AS): with only d*B
    // accumulators per lane every FMA would wait on the previous one (4-cycle
    // dependent chains, ~4 indices/clk/SM measured); the sets are added in
    // fixed order at the end
    constexpr int AS = D * NB >= 8 ? 1 : 8 / (D * NB);
    float acc[AS][D][NB];
#pragma unroll
    for (int a = 0; a < AS; ++a)
#pragma unroll
        for (int e = 0; e < D; ++e)
#pragma unroll
            for (int b = 0; b < NB; ++b) acc[a][e][b] = 0.f;
    dev::pdl_wait();
    const uint32_t lane_off = (uint32_t)lane * E;
    // x[b][j .. j+8) for every token: 4 words each, the same for all lanes
    auto load_x = [&](int j, uint32_t (&xv)[NB][4]) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (b < p.B && j < p.F_in) {
                // F_in is a multiple of d; columns past F_in read 0 (their indices are 0 too)
                if (j + 8 <= p.F_in && ((p.F_in & 7) == 0)) {
                    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p.x + (size_t)b * p.F_in + j));
                    xv[b][0] = a.x; xv[b][1] = a.y; xv[b][2] = a.z; xv[b][3] = a.w;
                } else {
                    const unsigned short* h = reinterpret_cast<const unsigned short*>(p.x + (size_t)b * p.F_in);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t lo = j + 2 * q < p.F_in ? (uint32_t)__ldg(h + j + 2 * q) : 0u;
                        const uint32_t hi = j + 2 * q + 1 < p.F_in ? (uint32_t)__ldg(h + j + 2 * q + 1) : 0u;
                        xv[b][q] = lo | (hi << 16);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) xv[b][q] = 0u;
            }
        }
    };
    dev::mbar_wait(cfull, 0);
    int slot = 0;
    uint32_t par = 0;
    for (int i = 0; i < nst; ++i) {
        const int c0 = j0 + i * kCH, nblk = min(kCH, j1 - c0) / 16;
        dev::mbar_wait(full0 + 8 * slot, par);
        const uint8_t* stg = s_idx + (size_t)slot * STB;
        uint4 iv_next = make_uint4(0u, 0u, 0u, 0u);
        if (warp < nblk) iv_next = core::lds<uint4>(stg + (warp * 32 + lane) * 16);
        for (int blk = warp; blk < nblk; blk += kDW) {
            // this block's 16 indices were loaded one block ahead (the next block's
            // LDS overlaps this block's gathers)
            const uint4 iv = iv_next;
            if (blk + kDW < nblk) iv_next = core::lds<uint4>(stg + ((blk + kDW) * 32 + lane) * 16);
            const uint32_t iw[4] = {iv.x, iv.y, iv.z, iv.w};
            // columns per x load: the whole block when d*B is small (16 gathers in flight)
            constexpr int JB = D * NB <= 4 ? 16 : 8;
#pragma unroll
            for (int q0 = 0; q0 < 16; q0 += JB) {
                uint32_t xv[NB][JB / 2];
                const int jc = c0 + blk * 16 + q0;
#pragma unroll
                for (int h = 0; h < JB / 8; ++h) {
                    uint32_t xh[NB][4];
                    if (p.x_staged) {   // broadcast LDS.128 per token (columns >= F_in read as 0)
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            uint4 a = make_uint4(0u, 0u, 0u, 0u);
                            if (b < p.B && jc + 8 * h < p.F_in)
                                a = core::lds<uint4>(stg + IXB + b * XSB + (jc + 8 * h - c0) * 2);
                            xh[b][0] = a.x; xh[b][1] = a.y; xh[b][2] = a.z; xh[b][3] = a.w;
                        }
                    } else {
                        load_x(jc + 8 * h, xh);
                    }
#pragma unroll
                    for (int b = 0; b < NB; ++b)
#pragma unroll
                        for (int w = 0; w < 4; ++w) xv[b][4 * h + w] = xh[b][w];
                }
                // gathers in flight before their FMAs: 8, or 2 when d*B accumulators are many
                constexpr int JG = D * NB >= 32 ? 2 : JB;
#pragma unroll
                for (int q1 = 0; q1 < JB; q1 += JG) {
                    uint32_t c[JG][EW];
#pragma unroll
                    for (int q = 0; q < JG; ++q) {
                        const int qq = q0 + q1 + q;
                        const uint32_t k = (iw[qq >> 2] >> (8 * (qq & 3))) & 0xffu;
                        const uint8_t* a = s_cb + k * KROW + lane_off;
                        if constexpr (EW == 1) {
                            c[q][0] = core::lds<uint32_t>(a);
                        } else if constexpr (EW == 2) {
                            const uint2 v = core::lds<uint2>(a);
                            c[q][0] = v.x;
                            c[q][EW > 1 ? 1 : 0] = v.y;
                        } else {
                            const uint4 v = core::lds<uint4>(a);
                            c[q][0] = v.x;
                            c[q][1 % EW] = v.y;
                            c[q][2 % EW] = v.z;
                            c[q][3 % EW] = v.w;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < JG; ++q) {
                        const int jq = q1 + q;   // column within the 8-column half: x word jq/2, half jq&1
                        float (&A)[D][NB] = acc[jq % AS];
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            const uint32_t xw = xv[b][jq >> 1];
#pragma unroll
                            for (int e = 0; e < D; ++e) {
                                if ((jq & 1) == 0) {
                                    if ((e & 1) == 0) A[e][b] = fma_hh<0, 0>(c[q][e >> 1], xw, A[e][b]);
                                    else A[e][b] = fma_hh<1, 0>(c[q][e >> 1], xw, A[e][b]);
                                } else {
                                    if ((e & 1) == 0) A[e][b] = fma_hh<0, 1>(c[q][e >> 1], xw, A[e][b]);
                                    else A[e][b] = fma_hh<1, 1>(c[q][e >> 1], xw, A[e][b]);
                                }
                            }
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(empty0 + 8 * slot);
        if (++slot == ST) { slot = 0; par ^= 1u; }
    }

#pragma unroll
    for (int a = 1; a < AS; ++a)
#pragma unroll
        for (int e = 0; e < D; ++e)
#pragma unroll
            for (int b = 0; b < NB; ++b) acc[0][e][b] += acc[a][e][b];

    // ---- cross-warp sum in fixed warp order (through the drained index ring) ----
    // scratch [kDW warps][32 lanes][16 values]; D*NB values per lane in rounds of 16
    asm volatile("bar.sync 1, %0;" :: "n"(kDW * 32) : "memory");   // every warp is past the ring
    float* scr = reinterpret_cast<float*>(s_idx);
    constexpr int V = D * NB;
    const int tid = threadIdx.x;                       // 0 .. kDW*32-1
    const int o_lane = tid >> 4, o_v = tid & 15;       // output (lane, value) summed by this thread
#pragma unroll
    for (int v0 = 0; v0 < V; v0 += 16) {
#pragma unroll
        for (int v = 0; v < 16; ++v)
            if (v0 + v < V) scr[(warp * 32 + lane) * 16 + v] = acc[0][(v0 + v) / NB][(v0 + v) % NB];
        asm volatile("bar.sync 1, %0;" :: "n"(kDW * 32) : "memory");
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < kDW; ++w) sum += scr[(w * 32 + o_lane) * 16 + o_v];
        asm volatile("bar.sync 1, %0;" :: "n"(kDW * 32) : "memory");
        const int v = v0 + o_v;
        if (v >= V) continue;
        const int e = v / NB, b = v % NB;
        const int ss = g * 32 + o_lane;
        if (ss >= p.N_ss || b >= p.B) continue;
        const int row = ss * D + e;
        if (p.y_mode == 2) {
            const long long q = __float2ll_rn(sum * core::kAccScale);
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(reinterpret_cast<unsigned long long*>(p.y) +
                                                                           (size_t)b * p.F_out + row), "l"(q) : "memory");
        } else if (p.ksplit == 1) {
            if (p.y_mode == 1) reinterpret_cast<float*>(p.y)[(size_t)b * p.F_out + row] = sum;
            else reinterpret_cast<__half*>(p.y)[(size_t)b * p.F_out + row] = __float2half_rn(sum);
        } else {
            // split-K without a merge phase (as gemv.cu): add, fence, count; the last
            // contributor converts and re-zeroes the words
            const size_t wd = (size_t)b * p.F_out + row;
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(p.acc + wd),
                         "l"(__float2ll_rn(sum * core::kAccScale)) : "memory");
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            unsigned old;
            asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.cnt + wd) : "memory");
            if (old == (unsigned)p.ksplit - 1u) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                long long tot;
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(tot) : "l"(p.acc + wd) : "memory");
                p.acc[wd] = 0ll;
                p.cnt[wd] = 0u;
                const double val = (double)tot * core::kAccInv;
                if (p.y_mode == 1) reinterpret_cast<float*>(p.y)[wd] = (float)val;
                else reinterpret_cast<__half*>(p.y)[wd] = __double2half(val);
            }
        }
    }
}

int num_sms_dim0() {
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

template <int D, int NB>
fasq_status launch_t(const Dim0Params& p, int grid, size_t smem, uint32_t flags, cudaStream_t st) {
    auto kern = k_gemv_dim0<D, NB>;
    static size_t lim = 0;
    static std::once_flag once;
    std::call_once(once, [&] { lim = set_max_dyn_smem(kern); });
    if (lim < smem) { set_error("gemv (dim 0): SMEM plan exceeds the device limit"); return FASQ_E_UNSUPPORTED; }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3((kDW + 1) * 32, 1, 1);
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

template <int D>
fasq_status dispatch_nb(int NB, const Dim0Params& p, int grid, size_t smem, uint32_t flags, cudaStream_t st) {
    switch (NB) {
        case 1: return launch_t<D, 1>(p, grid, smem, flags, st);
        case 2: return launch_t<D, 2>(p, grid, smem, flags, st);
        case 4: return launch_t<D, 4>(p, grid, smem, flags, st);
        default: return launch_t<D, 8>(p, grid, smem, flags, st);
    }
}

}  // namespace

fasq_status gemv_dim0_launch(const fasq_layer* L, const __half* x, int B, void* y, fasq_dtype yt, uint32_t flags,
                             cudaStream_t st) {
    if (!L->dim0) return FASQ_E_UNSUPPORTED;
    if (B < 1 || B > 8) return FASQ_E_UNSUPPORTED;
    if (flags & ~FASQ_FLAG_PDL) return FASQ_E_UNSUPPORTED;
    const int NB = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : 8;
    const size_t CBB = (size_t)L->C * 32 * L->E;
    const size_t stb = (size_t)kCH * 32 + (size_t)NB * kCH * 2;
    int stg = 4;
    auto smem_of = [&](int s) { return CBB + (size_t)s * stb + 8 * (size_t)(1 + 2 * s); };
    while (stg > 2 && smem_of(stg) > kSmemMax) --stg;
    // the cross-warp scratch (kDW x 32 x 16 floats = 32 KiB) reuses the ring
    if (smem_of(stg) > kSmemMax || (size_t)stg * stb < (size_t)kDW * 32 * 16 * 4) {
        set_error("gemv (dim 0): codebook image too large");
        return FASQ_E_UNSUPPORTED;
    }
    // grid: subspace groups x column splits.  Makespan model: the busiest SM runs
    // ceil(n*ks/SMs) CTAs of (fixed cost ~ 512 columns + K/ks columns) each --
    // every split re-stages the group's codebooks and adds a split-K merge
    const int n = L->n_groups, units = L->K_pad / 64, sms = num_sms_dim0();
    int ks = 1;
    double best = 1e30;
    for (int k = 1; k <= std::min(16, units); ++k) {
        const double t = (double)((n * k + sms - 1) / sms) * (512.0 + (double)L->K_pad / k);
        if (t < best * 0.97) { best = t; ks = k; }
    }
    Dim0Params p{};
    p.idx = L->idx;
    p.cbimg = L->cbimg;
    p.x = x;
    p.y = y;
    p.F_out = (int)L->F_out;
    p.F_in = (int)L->F_in;
    p.K_pad = L->K_pad;
    p.N_ss = L->N_ss;
    p.C = L->C;
    p.ksplit = ks;
    p.B = B;
    p.y_mode = yt == FASQ_ACC_I64 ? 2 : yt == FASQ_F32 ? 1 : 0;
    p.st = stg;
    // x rows through the TMA engine (16-B aligned chunks) when F_in % 8 == 0
    p.x_staged = (L->F_in % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) ? 1 : 0;
    uint8_t* ws_call = nullptr;
    if (ks > 1 && p.y_mode != 2) {
        const size_t accb = (size_t)B * L->F_out * 8, cntb = (size_t)B * L->F_out * 4;
        uint8_t* ws = nullptr;
        fasq_status s = stream_workspace(st, WS_GEMV, accb + cntb, reinterpret_cast<void**>(&ws));
        if (s != FASQ_OK) return s;
        if (!ws) {
            s = dev_alloc_t(&ws_call, accb + cntb, st);
            if (s != FASQ_OK) return s;
            cudaError_t e = cudaMemsetAsync(ws_call, 0, accb + cntb, st);
            if (e != cudaSuccess) { dev_free(ws_call, st); return cuda_fail(e, "gemv (dim 0) workspace"); }
            ws = ws_call;
        }
        p.acc = reinterpret_cast<long long*>(ws);
        p.cnt = reinterpret_cast<unsigned*>(ws + accb);
    }
    const int grid = n * ks;
    const size_t smem = smem_of(stg);
    fasq_status s;
    switch (L->d) {
        case 1: s = dispatch_nb<1>(NB, p, grid, smem, flags, st); break;
        case 2: s = dispatch_nb<2>(NB, p, grid, smem, flags, st); break;
        case 4: s = dispatch_nb<4>(NB, p, grid, smem, flags, st); break;
        default: s = dispatch_nb<8>(NB, p, grid, smem, flags, st); break;
    }
    dev_free(ws_call, st);
    if (s == FASQ_OK) set_launch_count(1);
    return s;
}

}  // namespace fasq
