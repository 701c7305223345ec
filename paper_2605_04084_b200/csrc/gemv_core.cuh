// gemv_core.cuh -- device building blocks of the FASQ decode GEMV, shared by
// the per-launch kernel (gemv.cu) and the persistent decode-chain kernel
// (chain.cu).  See gemv.cu for the design; everything here is the hot loop
// of Eq. 3 on the rotated lane = row layout.
#pragma once
#include "fasq_internal.cuh"

namespace fasq {
namespace core {

constexpr float kAccScale = 4294967296.0f;      // FASQ_ACC_I64 units: 2^-32
constexpr double kAccInv = 1.0 / 4294967296.0;

// x staging for a K-range of ng groups: [gl][64 entries][NB][E] -- the 32
// subspaces of each group twice so the rotated index (s + rot) needs no wrap.
// x is fp16 [B][F_in] or (x_acc) FASQ_ACC_I64 [B][F_in] rounded to fp16 here.
template <int D, int NB, int NW>
__device__ __forceinline__ void stage_x(uint8_t* s_x, const __half* x, int x_acc, int F_in, int B, int N_ss,
                                        int g_begin, int ng) {
    constexpr int E = D <= 2 ? 4 : 2 * D;
    const int tid = threadIdx.x;
    const int n_ent = ng * 64 * NB;   // entries of E bytes
    // all global loads first (one round trip), then the SMEM stores
    constexpr int XPT = 4;            // entries per thread per pass
    for (int t0 = tid; t0 < n_ent; t0 += NW * 32 * XPT) {
        uint32_t w[XPT][4];
#pragma unroll
        for (int u = 0; u < XPT; ++u) {
            const int t = t0 + u * NW * 32;
            w[u][0] = w[u][1] = w[u][2] = w[u][3] = 0u;
            if (t >= n_ent) continue;
            const int b = t % NB;
            const int e64 = (t / NB) % 64;
            const int gl = t / (NB * 64);
            const int ss = (g_begin + gl) * 32 + (e64 & 31);
            if (b < B && ss < N_ss && x_acc) {
                const long long* src = reinterpret_cast<const long long*>(x) + (size_t)b * F_in + (size_t)ss * D;
#pragma unroll
                for (int e = 0; e < D; ++e) {
                    const long long v = __ldcg(src + e);
                    const uint32_t h = __half_as_ushort(__double2half((double)v * kAccInv));
                    w[u][e >> 1] |= h << (16 * (e & 1));
                }
            } else if (b < B && ss < N_ss) {
                const __half* src = x + (size_t)b * F_in + (size_t)ss * D;
                if (D == 1) {
                    w[u][0] = (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(src));
                } else if (D == 2) {
                    w[u][0] = __ldg(reinterpret_cast<const unsigned int*>(src));
                } else if (D == 4) {
                    const uint2 v = __ldg(reinterpret_cast<const uint2*>(src));
                    w[u][0] = v.x; w[u][1] = v.y;
                } else {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(src));
                    w[u][0] = v.x; w[u][1] = v.y; w[u][2] = v.z; w[u][3] = v.w;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < XPT; ++u) {
            const int t = t0 + u * NW * 32;
            if (t >= n_ent) continue;
            uint32_t* dst = reinterpret_cast<uint32_t*>(s_x + (size_t)t * E);
#pragma unroll
            for (int q = 0; q < E / 4; ++q) dst[q] = w[u][q];
        }
    }
}

struct LaneConsts {
    int hA, rot;
    uint32_t Lr[16];
};

// Lane constants: the conflict-free LDS.128 half order (hA), the lane's
// subspace rotation, and the prmt lowbytes L[w] = [8*sub(2w), 8*sub(2w+1), 0, 0]
// so that prmt(idx word, L, sel) = k*256 + 8*sub (E=4: >>1 -> k*128 + 4*sub;
// E=8: as is; E=16: <<1 -> k*512 + 16*sub).
__device__ __forceinline__ void lane_consts(int lane, LaneConsts& lc) {
    lc.hA = (lane >> 2) & 1;
    lc.rot = (lane + 16 * lc.hA) & 31;
#pragma unroll
    for (int w = 0; w < 16; ++w)
        lc.Lr[w] = (uint32_t)(((2 * w + lc.rot) & 31) * 8) | ((uint32_t)(((2 * w + 1 + lc.rot) & 31) * 8) << 8);
}

// One 32-subspace group for this lane's RPL rows: acc[q][b] += sum over the
// group's subspaces of dot(x_ss, c[k]) (PRMT, LEA, LDS, FHFMA per index).
template <int D, int NB, int RPL>
__device__ __forceinline__ void compute_group(float (&acc)[RPL][NB], uint32_t idx_slot, uint32_t cbs, uint32_t x_grp,
                                              int warp_row0, int rows_valid, int lane, const LaneConsts& lc) {
    constexpr int E = D <= 2 ? 4 : 2 * D;
    uint32_t iw[RPL][8];
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int rl = warp_row0 + q * 32 + lane;
        const uint32_t a = idx_slot + (uint32_t)rl * 32u;
        if (warp_row0 + q * 32 < rows_valid) {
            uint4 v0 = dev::lds128(a + 16u * lc.hA);
            uint4 v1 = dev::lds128(a + 16u * (1 - lc.hA));
            iw[q][0] = v0.x; iw[q][1] = v0.y; iw[q][2] = v0.z; iw[q][3] = v0.w;
            iw[q][4] = v1.x; iw[q][5] = v1.y; iw[q][6] = v1.z; iw[q][7] = v1.w;
        } else {
#pragma unroll
            for (int w = 0; w < 8; ++w) iw[q][w] = 0u;
        }
    }
    const uint32_t xb = x_grp + (uint32_t)lc.rot * (NB * E);
#pragma unroll
    for (int s = 0; s < 32; ++s) {
        uint32_t xv[NB][E / 4];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const uint32_t xa = xb + (uint32_t)(s * NB * E + b * E);
            if (E == 4) {
                xv[b][0] = dev::lds32(xa);
            } else if (E == 8) {
                uint2 t2 = dev::lds64(xa);
                xv[b][0] = t2.x; xv[b][1 % (E / 4)] = t2.y;
            } else {
                uint4 t4 = dev::lds128(xa);
                xv[b][0] = t4.x; xv[b][1 % (E / 4)] = t4.y;
                xv[b][2 % (E / 4)] = t4.z; xv[b][3 % (E / 4)] = t4.w;
            }
        }
        const int wi = s >> 2, j = s & 3, lw = s >> 1, lj = s & 1;
        // byte0 = L byte lj (8*sub), byte1 = idx byte j (k), bytes 2,3 = L byte 2 (0)
        const uint32_t sel = (uint32_t)(4 + lj) | ((uint32_t)j << 4) | (6u << 8) | (6u << 12);
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            if (warp_row0 + q * 32 >= rows_valid) continue;
            uint32_t addr = dev::prmt(iw[q][wi], lc.Lr[lw], sel);
            if (E == 4) addr >>= 1;
            if (E == 16) addr <<= 1;
            if (E == 4) {
                const uint32_t c = dev::lds32(cbs + addr);
#pragma unroll
                for (int b = 0; b < NB; ++b)
                    acc[q][b] = (D == 1) ? dev::fhfma1(c, xv[b][0], acc[q][b]) : dev::fhfma2(c, xv[b][0], acc[q][b]);
            } else if (E == 8) {
                const uint2 c = dev::lds64(cbs + addr);
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    acc[q][b] = dev::fhfma2(c.x, xv[b][0], acc[q][b]);
                    acc[q][b] = dev::fhfma2(c.y, xv[b][1 % (E / 4)], acc[q][b]);
                }
            } else {
                const uint4 c = dev::lds128(cbs + addr);
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    acc[q][b] = dev::fhfma2(c.x, xv[b][0], acc[q][b]);
                    acc[q][b] = dev::fhfma2(c.y, xv[b][1 % (E / 4)], acc[q][b]);
                    acc[q][b] = dev::fhfma2(c.z, xv[b][2 % (E / 4)], acc[q][b]);
                    acc[q][b] = dev::fhfma2(c.w, xv[b][3 % (E / 4)], acc[q][b]);
                }
            }
        }
    }
}

// FASQ_ACC_I64 output: round each fp32 partial to int64 units of 2^-32 and
// red.add it (integer addition is associative -> deterministic).
template <int RPL, int NB>
__device__ __forceinline__ void acc_store(const float (&acc)[RPL][NB], unsigned long long* y, int r0, int warp_row0,
                                          int rows_valid, int F_out, int B, int lane) {
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int row = r0 + warp_row0 + q * 32 + lane;
        if (warp_row0 + q * 32 >= rows_valid || row >= F_out) continue;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (b >= B) continue;
            const long long v = __float2ll_rn(acc[q][b] * kAccScale);
            unsigned long long* dst = y + (size_t)b * F_out + row;
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(dst), "l"(v) : "memory");
        }
    }
}

}  // namespace core
}  // namespace fasq
