// gemv_core.cuh -- device building blocks of the FASQ decode GEMV, shared by
// the per-launch kernel (gemv.cu) and the persistent decode-chain kernel
// (chain.cu): the hot loop of Eq. 3 on the lane = SUBSPACE
// mapping.
//
// A warp owns RW output rows and, per 32-subspace group, lane s owns the
// group's subspace s: it keeps x_s in registers, loads the indices of 16 rows
// with one LDS.128 (sub-major index layout, fasq_internal.cuh), and for each
// row gathers centroid T_cluster[s][k] from the SMEM codebook image
// [C][32][E] -- lane s always hits bank s, so every warp-gather is one
// wavefront whatever the indices are -- and accumulates dot(x_s, c) into the
// row's register.  After the K range, the 32 lanes' per-row partial sums are
// added by a transposed butterfly (fixed order -> deterministic).
#pragma once
#include "fasq_internal.cuh"

namespace fasq {
namespace core {

constexpr float kAccScale = 4294967296.0f;      // FASQ_ACC_I64 units: 2^-32

// Plain C++ shared-memory loads (pointers derived from the kernel's
// __shared__ buffer -> LDS): unlike asm volatile they can be scheduled freely
// between the mbarrier waits/arrivals, which are asm volatile with a memory
// clobber and therefore order them.
template <class T>
__device__ __forceinline__ T lds(const uint8_t* p) { return *reinterpret_cast<const T*>(p); }
constexpr double kAccInv = 1.0 / 4294967296.0;

// Rows per consumer warp for an NB-wide batch (acc registers RW*NB = 64).
template <int NB>
struct RowsPerWarp {
    static constexpr int value = NB == 1 ? 64 : NB == 2 ? 32 : NB == 4 ? 16 : 8;
};

template <int D>
struct Entry {
    static constexpr int value = D <= 2 ? 4 : 2 * D;
};

// x staging for a K-range of ng groups: [gl][32 subspaces][NB][E] bytes.
// x is fp16 [B][F_in] or (x_acc) FASQ_ACC_I64 [B][F_in] rounded to fp16 here.
// XF (row-set FFMA2 path, B = 8): instead store x as fp32
// [gl][e < D][NB/4][32 subspaces][4 tokens] (the fp16 values converted
// exactly): one LDS.128 per (e, 4 tokens) and the 32 lanes' subspaces are
// consecutive 16-B blocks -> conflict-free.  See compute_group_set.
template <int D, int NB>
__device__ __forceinline__ void store_x_f32(uint8_t* s_x, int t, const uint32_t (&w)[4]) {
    const int b = t % NB, e32 = (t / NB) & 31, gl = t / (NB * 32);
    float* g = reinterpret_cast<float*>(s_x) + (size_t)gl * 32 * D * NB;
#pragma unroll
    for (int e = 0; e < D; ++e)
        g[((e * (NB / 4) + b / 4) * 32 + e32) * 4 + (b & 3)] =
            __half2float(__ushort_as_half((unsigned short)(w[e >> 1] >> (16 * (e & 1)))));
}

template <int D, int NB, int NW, bool XF = false>
__device__ __forceinline__ void stage_x(uint8_t* s_x, const __half* x, int x_acc, int F_in, int B, int N_ss,
                                        int g_begin, int ng) {
    constexpr int E = Entry<D>::value;
    const int tid = threadIdx.x;
    const int n_ent = ng * 32 * NB;   // entries of E bytes
    // all global loads of a pass first (one round trip), then the SMEM stores
    constexpr int XPT = 4;            // entries per thread per pass
    for (int t0 = tid; t0 < n_ent; t0 += NW * 32 * XPT) {
        uint32_t w[XPT][4];
#pragma unroll
        for (int u = 0; u < XPT; ++u) {
            const int t = t0 + u * NW * 32;
            w[u][0] = w[u][1] = w[u][2] = w[u][3] = 0u;
            if (t >= n_ent) continue;
            const int b = t % NB;
            const int e32 = (t / NB) & 31;
            const int gl = t / (NB * 32);
            const int ss = (g_begin + gl) * 32 + e32;
            if (b < B && ss < N_ss && x_acc) {
                const long long* src = reinterpret_cast<const long long*>(x) + (size_t)b * F_in + (size_t)ss * D;
                long long v[D];
                if (D == 1) {
                    v[0] = __ldcg(src);
                } else {
#pragma unroll
                    for (int e = 0; e < D; e += 2) {
                        const longlong2 t2 = __ldcg(reinterpret_cast<const longlong2*>(src + e));
                        v[e] = t2.x;
                        v[(e + 1) % D] = t2.y;
                    }
                }
#pragma unroll
                for (int e = 0; e < D; ++e) {
                    const uint32_t h = __half_as_ushort(__double2half((double)v[e] * kAccInv));
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
            if (XF) {
                store_x_f32<D, NB>(s_x, t, w[u]);
                continue;
            }
            uint32_t* dst = reinterpret_cast<uint32_t*>(s_x + (size_t)t * E);
#pragma unroll
            for (int q = 0; q < E / 4; ++q) dst[q] = w[u][q];
        }
    }
}

// This lane's x_s for every batch row of staged group gl.
template <int D, int NB>
__device__ __forceinline__ void load_x(uint32_t (&xv)[NB][Entry<D>::value / 4], const uint8_t* x_grp, int lane) {
    constexpr int E = Entry<D>::value;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const uint8_t* a = x_grp + (lane * NB + b) * E;
        if (E == 4) {
            xv[b][0] = lds<uint32_t>(a);
        } else if (E == 8) {
            const uint2 t = lds<uint2>(a);
            xv[b][0] = t.x;
            xv[b][1 % (E / 4)] = t.y;
        } else {
            const uint4 t = lds<uint4>(a);
            xv[b][0] = t.x;
            xv[b][1 % (E / 4)] = t.y;
            xv[b][2 % (E / 4)] = t.z;
            xv[b][3 % (E / 4)] = t.w;
        }
    }
}

// SMEM byte offset of this warp's first index chunk inside an index stage
// (rows [wrow0, wrow0 + RW) of the stage's row tile, lane = subspace).
__device__ __forceinline__ uint32_t idx_lane_off(int wrow0, int lane) {
    return (uint32_t)(wrow0 >> 6) * 2048u + (uint32_t)lane * 64u;
}

// Per-lane byte offsets of the warp's 16-row index chunks inside an index
// stage (chunk c of the warp's 64-row block at 16 * ((c + s/2) & 3); RW = 8:
// + 8 for the odd half).  Loop-invariant: computed once per kernel.
template <int RW>
struct ChunkOffs {
    static constexpr int N = RW >= 16 ? RW / 16 : 1;
    uint32_t o[N];
};
template <int RW>
__device__ __forceinline__ ChunkOffs<RW> chunk_offsets(int wrow0, int lane) {
    ChunkOffs<RW> c;
    const int c0 = (wrow0 >> 4) & 3;
#pragma unroll
    for (int ci = 0; ci < ChunkOffs<RW>::N; ++ci)
        c.o[ci] = idx_lane_off(wrow0, lane) + 16u * (((uint32_t)(c0 + ci) + (uint32_t)(lane >> 1)) & 3u) +
                  (RW == 8 ? (uint32_t)(wrow0 & 8) : 0u);
    return c;
}

// One 32-subspace group: acc[j][b] += dot(x[b]_s, c_s[k_s(row j)]) for the
// warp's RW rows (lane s = subspace s).  idx_stage = index stage base, co =
// chunk_offsets(); cbs = codebook image stage base.
template <int D, int NB, int RW>
__device__ __forceinline__ void compute_group(float (&acc)[RW][NB], const uint8_t* idx_stage, const ChunkOffs<RW>& co,
                                              const uint8_t* cbs, const uint32_t (&xv)[NB][Entry<D>::value / 4],
                                              int lane) {
    constexpr int E = Entry<D>::value;
    constexpr int NCH = ChunkOffs<RW>::N;              // 16-row chunks per warp
    // E = 4: address = cbs + 4*s + (k << 7)        (PRMT extracts k, LEA scales)
    // E = 8: address = cbs + (k << 8 | 8*s)        (one PRMT)
    // E = 16: address = cbs + (k << 8 | 8*s) << 1  (PRMT + shift)
    const uint8_t* cbl = cbs + lane * 4;
    const uint32_t L8 = (uint32_t)lane * 8u;
#pragma unroll
    for (int ci = 0; ci < NCH; ++ci) {
        const uint8_t* ca = idx_stage + co.o[ci];
        uint32_t w[4];
        if (RW >= 16) {
            const uint4 v = lds<uint4>(ca);
            w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
        } else {   // RW = 8: half a chunk
            const uint2 v = lds<uint2>(ca);
            w[0] = v.x; w[1] = v.y; w[2] = 0u; w[3] = 0u;
        }
        // all gathers of a batch first, then the FMAs: keeps LDS_BATCH loads in
        // flight per warp (ptxas otherwise serialises gather -> use)
        constexpr int NJ = RW >= 16 ? 16 : RW;
        constexpr int JB = E == 4 ? NJ : 8;                // rows per gather batch
#pragma unroll
        for (int j0 = 0; j0 < NJ; j0 += JB) {
            if (E == 4) {
                uint32_t c[JB];
#pragma unroll
                for (int j = 0; j < JB; ++j) {
                    const uint32_t k = dev::prmt(w[(j0 + j) >> 2], 0u, 0x4440u | (uint32_t)((j0 + j) & 3));
                    c[j] = lds<uint32_t>(cbl + (k << 7));
                }
#pragma unroll
                for (int j = 0; j < JB; ++j)
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        float& a = acc[ci * 16 + j0 + j][b];
                        a = (D == 1) ? dev::fhfma1(c[j], xv[b][0], a) : dev::fhfma2(c[j], xv[b][0], a);
                    }
            } else if (E == 8) {
                uint2 c[JB];
#pragma unroll
                for (int j = 0; j < JB; ++j) {
                    const uint32_t ad = dev::prmt(w[(j0 + j) >> 2], L8, 0x7704u | ((uint32_t)((j0 + j) & 3) << 4));
                    c[j] = lds<uint2>(cbs + ad);
                }
#pragma unroll
                for (int j = 0; j < JB; ++j)
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        float& a = acc[ci * 16 + j0 + j][b];
                        a = dev::fhfma2(c[j].x, xv[b][0], a);
                        a = dev::fhfma2(c[j].y, xv[b][1 % (E / 4)], a);
                    }
            } else {
                uint4 c[JB];
#pragma unroll
                for (int j = 0; j < JB; ++j) {
                    const uint32_t ad = dev::prmt(w[(j0 + j) >> 2], L8, 0x7704u | ((uint32_t)((j0 + j) & 3) << 4)) << 1;
                    c[j] = lds<uint4>(cbs + ad);
                }
#pragma unroll
                for (int j = 0; j < JB; ++j)
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        float& a = acc[ci * 16 + j0 + j][b];
                        a = dev::fhfma2(c[j].x, xv[b][0], a);
                        a = dev::fhfma2(c[j].y, xv[b][1 % (E / 4)], a);
                        a = dev::fhfma2(c[j].z, xv[b][2 % (E / 4)], a);
                        a = dev::fhfma2(c[j].w, xv[b][3 % (E / 4)], a);
                    }
            }
        }
    }
}

// E = 4 (d <= 2) over a codebook PAIR stage: two consecutive groups staged
// as [C][2][32] words (one 3-D TMA box, chain.cu), i.e. 256-B k-rows.  The
// gather address (k << 8) | (h*128 + 4*s) is then ONE PRMT of the index word
// with the lane constant lb = h*128 + 4*s (byte 0) -- no IMAD/LEA -- and the
// LDS adds the uniform ring base cbs; lbv's byte 2 may carry the slot (64 KiB
// units): PRMT, LDS, FHFMA x d per index.  Lane s still reads bank s for any
// k (one wavefront per warp-gather).
template <int D, int NB, int RW>
__device__ __forceinline__ void compute_group_pair(float (&acc)[RW][NB], const uint8_t* idx_stage,
                                                   const ChunkOffs<RW>& co, const uint8_t* cbs, uint32_t lbv,
                                                   const uint32_t (&xv)[NB][1]) {
    constexpr int NCH = ChunkOffs<RW>::N;
#pragma unroll
    for (int ci = 0; ci < NCH; ++ci) {
        const uint8_t* ca = idx_stage + co.o[ci];
        uint32_t w[4];
        if (RW >= 16) {
            const uint4 v = lds<uint4>(ca);
            w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
        } else {
            const uint2 v = lds<uint2>(ca);
            w[0] = v.x; w[1] = v.y; w[2] = 0u; w[3] = 0u;
        }
        constexpr int NJ = RW >= 16 ? 16 : RW;
        uint32_t c[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            c[j] = lds<uint32_t>(cbs + dev::prmt(w[j >> 2], lbv, 0x7604u | ((uint32_t)(j & 3) << 4)));
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                float& a = acc[ci * 16 + j][b];
                a = (D == 1) ? dev::fhfma1(c[j], xv[b][0], a) : dev::fhfma2(c[j], xv[b][0], a);
            }
    }
}

// ---- row-set mapping (decode chain, pair stages, any B) ---------------------
// The 32-lane reduction of the lane = subspace mapping moves 31 values per row
// through SHFL (SHFL-bound, ~0.5 us per work item on a full CTA), and at B > 1
// the 64-accumulator budget shrank the rows per warp (RW = 64/B) and with them
// the rows per codebook stage.  Here a warp always owns 64 rows, split into
// K = 32/G row sets: lane l = G*a + u owns the 2G rows {G*a + t, 32 + G*a + t :
// t < G} and, in phase p = 0..K-1 of every group, subspace
// sigma_p = G*((a + p) % K) + u.  Every phase is a permutation of the 32
// subspaces over the 32 lanes -> 32 distinct banks per warp-gather; a lane
// keeps 2G x B accumulators (G = 8 for B <= 2, 4 for B = 4, 2 for B = 8: <= 32); a row
// total is a reduction over the G lanes of its set (log2 G butterfly rounds),
// after which lane l holds rows l and 32 + l for every token (contiguous
// counted stores).  The index bytes of (sigma_p, G rows) are G bytes of the
// existing layout (two LDS per phase; G = 8 conflict-free per half-warp, G = 4
// and 2 at most 2-way -- checked exhaustively for the s/2 chunk rotation).
template <int G>
struct SetMap {
    static constexpr int K = 32 / G;
    uint32_t blk;   // byte offset of the warp's 64-row block inside an index stage
    uint32_t a, u;  // row set, lane within the set
    // phase ph: subspace, and the index-byte offsets of the set's two row runs
    __device__ __forceinline__ uint32_t sg(int ph) const { return G * ((a + (uint32_t)ph) % K) + u; }
    __device__ __forceinline__ uint32_t ia(uint32_t s) const {
        const uint32_t r0 = G * a;
        return blk + s * 64u + 16u * (((r0 >> 4) + (s >> 1)) & 3u) + (r0 & 15u);
    }
    __device__ __forceinline__ uint32_t ib(uint32_t s) const {
        const uint32_t r1 = 32u + G * a;
        return blk + s * 64u + 16u * (((r1 >> 4) + (s >> 1)) & 3u) + (r1 & 15u);
    }
};
template <int G>
__device__ __forceinline__ SetMap<G> set_map(int wrow0, int lane) {
    SetMap<G> m;
    m.blk = (uint32_t)(wrow0 >> 6) * 2048u;
    m.a = (uint32_t)lane / G;
    m.u = (uint32_t)lane % G;
    return m;
}

// One group on a codebook pair stage (half h and slot bits in lbs).  Value
// (row t of the set, token b) accumulates in register (2*(t % G) + t / G)*NB + b
// (t < G: row G*a + t, else 32 + G*a + t - G).  x_grp: the group's staged x
// [32 subspaces][NB][4 B].
template <int D, int NB, int G>
__device__ __forceinline__ void compute_group_set(float (&acc)[2 * G * NB], const uint8_t* idx_stage,
                                                  const SetMap<G>& m, const uint8_t* cbs, uint32_t lbs,
                                                  const uint8_t* x_grp) {
    constexpr int K = 32 / G;
    if constexpr (NB == 8) {
        // B = 8: x staged as fp32 (store_x_f32 layout); each centroid half is converted
        // once (HADD2.F32) and FFMA2 (fma.rn.f32x2, scalar broadcast) updates
        // two tokens per instruction -- the same exact products and fp32 sums
        // in the same order as the FHFMA path, half the FMA instructions
        // (measured: 3.49 -> 3.39 ms per B = 8 step; at B = 4 the FHFMA path
        // is faster, 1.85 vs 2.09 ms).
#pragma unroll
        for (int ph = 0; ph < K; ++ph) {
            const uint32_t sg = m.sg(ph);
            float xf[D][NB];
            const float4* xa = reinterpret_cast<const float4*>(x_grp) + sg;
#pragma unroll
            for (int e = 0; e < D; ++e)
#pragma unroll
                for (int b = 0; b < NB; b += 4) {
                    const float4 t = *(xa + (e * (NB / 4) + b / 4) * 32);
                    xf[e][b] = t.x; xf[e][b + 1] = t.y; xf[e][b + 2] = t.z; xf[e][b + 3] = t.w;
                }
            constexpr int NWD = G >= 4 ? G / 2 : 1;
            uint32_t w[NWD];
            if (G == 8) {
                const uint2 va = lds<uint2>(idx_stage + m.ia(sg));
                const uint2 vb = lds<uint2>(idx_stage + m.ib(sg));
                w[0] = va.x; w[1 % NWD] = va.y; w[2 % NWD] = vb.x; w[3 % NWD] = vb.y;
            } else if (G == 4) {
                w[0] = lds<uint32_t>(idx_stage + m.ia(sg));
                w[1 % NWD] = lds<uint32_t>(idx_stage + m.ib(sg));
            } else {
                w[0] = (uint32_t)lds<uint16_t>(idx_stage + m.ia(sg)) |
                       ((uint32_t)lds<uint16_t>(idx_stage + m.ib(sg)) << 16);
            }
            const uint32_t lbv = lbs + sg * 4u;
            uint32_t c[2 * G];
#pragma unroll
            for (int t = 0; t < 2 * G; ++t)
                c[t] = lds<uint32_t>(cbs + dev::prmt(w[t >> 2], lbv, 0x7604u | ((uint32_t)(t & 3) << 4)));
#pragma unroll
            for (int t = 0; t < 2 * G; ++t) {
                const int base = (2 * (t % G) + t / G) * NB;
#pragma unroll
                for (int e = 0; e < D; ++e) {
                    const float ce = __half2float(__ushort_as_half((unsigned short)(c[t] >> (16 * e))));
#pragma unroll
                    for (int b = 0; b < NB; b += 2) dev::ffma2(acc[base + b], acc[base + b + 1], ce, xf[e][b], xf[e][b + 1]);
                }
            }
        }
        return;
    }
#pragma unroll
    for (int ph = 0; ph < K; ++ph) {
        const uint32_t sg = m.sg(ph);
        uint32_t xv[NB];
        const uint8_t* xa = x_grp + sg * 4u * NB;
        if (NB == 1) {
            xv[0] = lds<uint32_t>(xa);
        } else if (NB == 2) {
            const uint2 t = lds<uint2>(xa);
            xv[0] = t.x; xv[1 % NB] = t.y;
        } else {
#pragma unroll
            for (int b = 0; b < NB; b += 4) {
                const uint4 t = lds<uint4>(xa + 4 * b);
                xv[b] = t.x; xv[(b + 1) % NB] = t.y; xv[(b + 2) % NB] = t.z; xv[(b + 3) % NB] = t.w;
            }
        }
        constexpr int NWD = G >= 4 ? G / 2 : 1;   // index words: rows t < G in the first G/4 (or half) words
        uint32_t w[NWD];
        if (G == 8) {
            const uint2 va = lds<uint2>(idx_stage + m.ia(sg));
            const uint2 vb = lds<uint2>(idx_stage + m.ib(sg));
            w[0] = va.x; w[1 % NWD] = va.y; w[2 % NWD] = vb.x; w[3 % NWD] = vb.y;
        } else if (G == 4) {
            w[0] = lds<uint32_t>(idx_stage + m.ia(sg));
            w[1 % NWD] = lds<uint32_t>(idx_stage + m.ib(sg));
        } else {   // G = 2: two 16-bit halves in one word
            w[0] = (uint32_t)lds<uint16_t>(idx_stage + m.ia(sg)) | ((uint32_t)lds<uint16_t>(idx_stage + m.ib(sg)) << 16);
        }
        const uint32_t lbv = lbs + sg * 4u;
        uint32_t c[2 * G];
#pragma unroll
        for (int t = 0; t < 2 * G; ++t)
            c[t] = lds<uint32_t>(cbs + dev::prmt(w[t >> 2], lbv, 0x7604u | ((uint32_t)(t & 3) << 4)));
#pragma unroll
        for (int t = 0; t < 2 * G; ++t)
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                float& r = acc[(2 * (t % G) + t / G) * NB + b];
                r = (D == 1) ? dev::fhfma1(c[t], xv[b], r) : dev::fhfma2(c[t], xv[b], r);
            }
    }
}

// Row totals of a set: transposed butterfly over its G lanes (xor G/2 .. 1,
// fixed order).  Afterwards v[h*NB + b] = row (lane + 32h) of the warp, token b.
template <int NB, int G>
__device__ __forceinline__ void reduce_set(float (&v)[2 * G * NB], int lane) {
#pragma unroll
    for (int msk = G / 2, half = G * NB; msk >= 1; msk >>= 1, half >>= 1) {
        const bool up = (lane & msk) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = up ? v[i] : v[i + half];
            const float keep = up ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, msk);
        }
    }
}

// Transposed butterfly over the 32 lanes: v[i] (i < N, N = 32/16/8) holds
// this lane's partial of row i; afterwards v[0] holds the total of row
// (lane >> (5 - log2 N)) (each row on 32/N lanes).  Fixed order.
template <int N>
__device__ __forceinline__ void transpose_reduce(float (&v)[N], int lane) {
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const int m = 16 >> r;
        const int n = N >> r;          // live values before this round (compile-time after unrolling)
        if (n > 1) {
            const int half = n >> 1;
            const bool up = (lane & m) != 0;
#pragma unroll
            for (int i = 0; i < half; ++i) {
                const float send = up ? v[i] : v[i + half];
                const float keep = up ? v[i + half] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
            }
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
        }
    }
}

// Row totals of the warp: out[h][b] = total of row h*32 + rsel (RW = 64: two
// halves) where rsel = lane >> shift; `own` = this lane writes those rows.
template <int NB, int RW>
struct RowTotals {
    static constexpr int H = RW > 32 ? RW / 32 : 1;
    static constexpr int N = RW > 32 ? 32 : RW;
    float v[H][NB];
    int rsel;
    bool own;
};

template <int NB, int RW>
__device__ __forceinline__ void reduce_rows(const float (&acc)[RW][NB], RowTotals<NB, RW>& t, int lane) {
    constexpr int H = RowTotals<NB, RW>::H, N = RowTotals<NB, RW>::N;
    constexpr int shift = N == 32 ? 0 : N == 16 ? 1 : 2;
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            float v[N];
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = acc[h * 32 + i][b];
            transpose_reduce<N>(v, lane);
            t.v[h][b] = v[0];
        }
    t.rsel = lane >> shift;
    t.own = (lane & ((1 << shift) - 1)) == 0;
}

// FASQ_ACC_I64 output: round each fp32 row total to int64 units of 2^-32 and
// red.add it (integer addition is associative -> deterministic).
template <int NB, int RW>
__device__ __forceinline__ void acc_store(const RowTotals<NB, RW>& t, unsigned long long* y, int row0, int F_out,
                                          int B) {
    if (!t.own) return;
#pragma unroll
    for (int h = 0; h < RowTotals<NB, RW>::H; ++h) {
        const int row = row0 + h * 32 + t.rsel;
        if (row >= F_out) continue;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (b >= B) continue;
            const long long v = __float2ll_rn(t.v[h][b] * kAccScale);
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(y + (size_t)b * F_out + row), "l"(v) : "memory");
        }
    }
}

// ---- counted accumulators (decode-chain dataflow, chain.cu) -----------------
// A chain output word is an int64 red.add target holding BOTH the value and
// the number of contributions: every K-split CTA adds
//     (1 << kCntShift) + kCntBias + v,   v = rn(partial * 2^32), |v| < kCntBias,
// so the low kCntShift bits stay positive and never carry into the count
// (<= 63 contributions x 2^51 < 2^57), and a consumer that reads
// count == ks knows the value is final: sum v = low bits - ks * kCntBias.
// The word is self-validating -> no grid barrier between chain steps.
constexpr int kCntShift = 58;
constexpr long long kCntBias = 1ll << 50;
constexpr unsigned long long kCntMask = (1ull << kCntShift) - 1;

// Out-of-range partials: the value field holds |v| < kCntBias (2^18 in value
// units).  A partial outside it is clamped AND raises the sticky flag *ovf,
// which poisons the run's converted outputs (NaN) and makes fasq_chain_check
// return FASQ_E_RANGE -- never a silently wrong finite number.
__device__ __forceinline__ long long cnt_clamp(long long v, unsigned long long* ovf) {
    if (v >= kCntBias || v <= -kCntBias) {
        if (ovf) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(ovf), "l"(1ull) : "memory");
        v = max(-(kCntBias - 1), min(kCntBias - 1, v));
    }
    return v;
}

// Polls one counted word until it carries `ks` contributions; returns its
// value (units 2^-32).  The watchdog turns a lost producer into a kernel
// error (trap) after 4 s instead of a hang.
__device__ __forceinline__ long long poll_value(const unsigned long long* a, int ks, bool sys) {
    unsigned long long v;
    const unsigned long long t0 = dev::globaltimer();
    for (;;) {
        if (sys)
            asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
        else
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
        if ((v >> kCntShift) == (unsigned long long)ks) break;
        if (dev::globaltimer() - t0 > 4000000000ull) __trap();
    }
    return (long long)(v & kCntMask) - (long long)ks * kCntBias;
}

// y points at this shard's row 0 inside a [B][ld] word array; rows >= F_out
// (the shard's local rows) are padding and skipped.  System-scope reduction:
// y may be a peer GPU's buffer (NVLink, fasq_chain_create_tp).
template <int NB, int RW>
__device__ __forceinline__ void counted_store(const RowTotals<NB, RW>& t, unsigned long long* y, int row0, int F_out,
                                              int ld, int B, unsigned long long* ovf) {
    if (!t.own) return;
#pragma unroll
    for (int h = 0; h < RowTotals<NB, RW>::H; ++h) {
        const int row = row0 + h * 32 + t.rsel;
        if (row >= F_out) continue;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (b >= B) continue;
            const long long v = cnt_clamp(__float2ll_rn(t.v[h][b] * kAccScale), ovf);
            const unsigned long long add = (1ull << kCntShift) + (unsigned long long)(kCntBias + v);
            asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" :: "l"(y + (size_t)b * ld + row), "l"(add) : "memory");
        }
    }
}

// Row totals of the row-set mapping -> fixed-point values: v[h*NB + b] is
// row row0w + 32h + lane, token b.  With `res` (residual words of the same
// [B][ld] indexing, `res_ks` contributions each), the residual value is added
// exactly (integer) to the partial -- the transformer's residual connection
// fused into the GEMV epilogue of ONE K-split CTA per row.
template <int NB, int G>
__device__ __forceinline__ void set_values(const float (&v)[2 * G * NB], long long (&q)[2 * NB], int row0w, int lane,
                                           int F_out, int B, const unsigned long long* res, int res_ld, int res_ks,
                                           bool res_sys, unsigned long long* ovf,
                                           const unsigned long long* res2 = nullptr, int res2_ks = 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int b = 0; b < NB; ++b) q[h * NB + b] = __float2ll_rn(v[h * NB + b] * kAccScale);
    if (res) {
        // residual words (and the lazy base res2, chain_internal.cuh): every
        // word of this lane in flight at once, reloaded until all are final
        constexpr int NR = 4 * NB;
        unsigned long long w[NR];
        bool need[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const int src = i / (2 * NB), h = (i / NB) & 1, b = i % NB;
            const int row = row0w + 32 * h + lane;
            need[i] = row < F_out && b < B && (src == 0 || res2 != nullptr);
            w[i] = 0ull;
        }
        const unsigned long long t0 = dev::globaltimer();
        for (bool done = false; !done;) {
            done = true;
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                const int src = i / (2 * NB), h = (i / NB) & 1, b = i % NB;
                const int ks = src == 0 ? res_ks : res2_ks;
                if (!need[i] || (w[i] >> kCntShift) == (unsigned long long)ks) continue;
                const unsigned long long* a = (src == 0 ? res : res2) + (size_t)b * res_ld + row0w + 32 * h + lane;
                if (res_sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w[i]) : "l"(a) : "memory");
                else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w[i]) : "l"(a) : "memory");
            }
            // check after ALL loads were issued (a check right after each load
            // serialised one L2 round trip per word: +2 us on the residual CTAs)
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                const int ks = i / (2 * NB) == 0 ? res_ks : res2_ks;
                if (need[i] && (w[i] >> kCntShift) != (unsigned long long)ks) done = false;
            }
            if (!done && dev::globaltimer() - t0 > 4000000000ull) __trap();
        }
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const int src = i / (2 * NB);
            const int ks = src == 0 ? res_ks : res2_ks;
            if (need[i]) q[i % (2 * NB)] += (long long)(w[i] & kCntMask) - (long long)ks * kCntBias;
        }
    }
#pragma unroll
    for (int i = 0; i < 2 * NB; ++i) q[i] = cnt_clamp(q[i], ovf);
}

// Counted stores of set_values' results: rows row0w + lane and row0w + 32 +
// lane of every token b < B (word b*ld + row).
template <int NB>
__device__ __forceinline__ void counted_store_q(const long long (&q)[2 * NB], unsigned long long* y, int row0w,
                                                int lane, int F_out, int ld, int B, bool sys) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int row = row0w + 32 * h + lane;
        if (row >= F_out) continue;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            if (b >= B) continue;
            const unsigned long long add = (1ull << kCntShift) + (unsigned long long)(kCntBias + q[h * NB + b]);
            if (sys)   // peer GPU arenas (tensor parallel): system scope
                asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" :: "l"(y + (size_t)b * ld + row), "l"(add) : "memory");
            else
                asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(y + (size_t)b * ld + row), "l"(add) : "memory");
        }
    }
}

// ---- batched decode on the tensor cores (d = 2, B = 4..8) --
// mma.sync.m16n8k16 (fp16 x fp16 -> fp32) with the WEIGHTS as A and the NB <= 8
// tokens as B (N = 8; tokens >= B are zero): a k16 slice is 8 subspaces, and
// A's register a_i of lane (g, t) is exactly one centroid (d = 2 halves):
// rows {g, g+8} x k-slots {t, t+4}.  Lane (g, t) owns the 8 consecutive rows
// 8g..8g+7 of the warp's 64 (MMA tile j: row g -> 8g+2j, row g+8 -> 8g+2j+1),
// so its indices of one subspace are ONE LDS.64 of the physical layout (2
// wavefronts per warp, the minimum for 256 B).  The 8 lanes of a k-slot share
// one subspace's codebook; on the XOR image (word s of k-row k at s ^ ((k&7)<<2),
// fasq_layer::cbimg_x) they spread over 8 banks and the 4 k-slots never
// collide, so a warp-gather costs ~2.6 wavefronts for random indices.  Per
// index: PRMT + SHF + LOP3 + LDS + 1/4 HMMA-equivalent (the FHFMA/FFMA2 path
// needs 4 + B instructions) -- B-independent.  x is staged [group][32
// subspaces][NB] fp16x2 words: B's registers are x_s[token g] (conflict-free).
// The fp16 products are exact and accumulate in fp32 inside the MMA.
__device__ __forceinline__ uint32_t gather_x(const uint8_t* cbs, uint32_t w, uint32_t lc, int byte) {
    uint32_t ad = dev::prmt(w, lc, 0x7604u | ((uint32_t)byte << 4));   // (k << 8) | lane constant (slot, h, 4s)
    ad ^= (ad >> 4) & 0x70u;                                             // XOR image: s ^ ((k & 7) << 2)
    return lds<uint32_t>(cbs + ad);
}

__device__ __forceinline__ void mma_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One group (32 subspaces = 4 k-steps) of the warp's 64 rows on a codebook
// pair slot (XOR image): acc[4j + c] = C[tile j] (c: rows 8g+2j / 8g+2j+1 x
// tokens 2t / 2t+1, see mma_values).  blk = the warp's 64-row block offset in
// the index stage; lbs = slot and half bits of the pair address.
template <int NB>
__device__ __forceinline__ void compute_group_mma(float (&acc)[16], const uint8_t* idx_stage, uint32_t blk, int lane,
                                                  const uint8_t* cbs, uint32_t lbs, const uint8_t* x_grp) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int kst = 0; kst < 4; ++kst) {
        const uint32_t s0 = (uint32_t)(kst * 8 + t), s1 = s0 + 4u;
        const uint2 i0 = lds<uint2>(idx_stage + blk + s0 * 64u + 16u * ((((uint32_t)g >> 1) + (s0 >> 1)) & 3u) +
                                    8u * ((uint32_t)g & 1u));
        const uint2 i1 = lds<uint2>(idx_stage + blk + s1 * 64u + 16u * ((((uint32_t)g >> 1) + (s1 >> 1)) & 3u) +
                                    8u * ((uint32_t)g & 1u));
        uint32_t b0 = 0u, b1 = 0u;
        if (g < NB) {
            b0 = lds<uint32_t>(x_grp + (s0 * NB + (uint32_t)g) * 4u);
            b1 = lds<uint32_t>(x_grp + (s1 * NB + (uint32_t)g) * 4u);
        }
        const uint32_t c0 = lbs + s0 * 4u, c1 = lbs + s1 * 4u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t w0 = j < 2 ? i0.x : i0.y, w1 = j < 2 ? i1.x : i1.y;
            const int r = (2 * j) & 3;
            uint32_t a[4];
            a[0] = gather_x(cbs, w0, c0, r);       // row 8g+2j,   subspace s0
            a[1] = gather_x(cbs, w0, c0, r + 1);   // row 8g+2j+1, subspace s0
            a[2] = gather_x(cbs, w1, c1, r);       // row 8g+2j,   subspace s1
            a[3] = gather_x(cbs, w1, c1, r + 1);   // row 8g+2j+1, subspace s1
            float* cj = acc + 4 * j;
            mma_16816(*reinterpret_cast<float(*)[4]>(cj), a, b0, b1);
        }
    }
}

// The MMA accumulators -> fixed-point values (units 2^-32) with the optional
// RMSNorm scale per token (sc, NB entries) and residual words (res [+ res2],
// [B][res_ld] indexing, polled in parallel); q[4j + c] belongs to row
// row0w + 8g + 2j + (c >> 1), token 2t + (c & 1).
template <int NB>
__device__ __forceinline__ void mma_values(const float (&acc)[16], long long (&q)[16], int row0w, int lane, int F_out,
                                           int B, const float* sc, const unsigned long long* res, int res_ld,
                                           int res_ks, bool res_sys, unsigned long long* ovf,
                                           const unsigned long long* res2 = nullptr, int res2_ks = 0) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int tok = 2 * t + (i & 1);
        float v = acc[i];
        if (sc) {
            float sb = sc[0];
#pragma unroll
            for (int b = 1; b < NB; ++b)
                if (b == tok) sb = sc[b];
            v *= sb;
        }
        q[i] = __float2ll_rn(v * kAccScale);
    }
    if (res) {
        // 4 batches of 4 outputs (8 words in flight): bounded registers at the
        // 96-register cap of the chain kernel
#pragma unroll
        for (int bt = 0; bt < 4; ++bt) {
            unsigned long long w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = 0ull;
            const unsigned long long t0 = dev::globaltimer();
            for (bool done = false; !done;) {
                done = true;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int k = 4 * bt + (i & 3), src = i >> 2;
                    const int row = row0w + 8 * g + 2 * (k >> 2) + ((k >> 1) & 1), tok = 2 * t + (k & 1);
                    const int ks = src == 0 ? res_ks : res2_ks;
                    if (row >= F_out || tok >= B || (src == 1 && !res2)) continue;
                    if ((w[i] >> kCntShift) == (unsigned long long)ks) continue;
                    const unsigned long long* a = (src == 0 ? res : res2) + (size_t)tok * res_ld + row;
                    if (res_sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w[i]) : "l"(a) : "memory");
                    else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w[i]) : "l"(a) : "memory");
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {   // checks after all loads were issued
                    const int k = 4 * bt + (i & 3), src = i >> 2;
                    const int row = row0w + 8 * g + 2 * (k >> 2) + ((k >> 1) & 1), tok = 2 * t + (k & 1);
                    const int ks = src == 0 ? res_ks : res2_ks;
                    if (row >= F_out || tok >= B || (src == 1 && !res2)) continue;
                    if ((w[i] >> kCntShift) != (unsigned long long)ks) done = false;
                }
                if (!done && dev::globaltimer() - t0 > 4000000000ull) __trap();
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int k = 4 * bt + (i & 3), src = i >> 2;
                const int row = row0w + 8 * g + 2 * (k >> 2) + ((k >> 1) & 1), tok = 2 * t + (k & 1);
                const int ks = src == 0 ? res_ks : res2_ks;
                if (row >= F_out || tok >= B || (src == 1 && !res2)) continue;
                q[k] += (long long)(w[i] & kCntMask) - (long long)ks * kCntBias;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) q[i] = cnt_clamp(q[i], ovf);
}

// Counted stores of mma_values' results (word tok * ld + row).
__device__ __forceinline__ void counted_store_mma(const long long (&q)[16], unsigned long long* y, int row0w, int lane,
                                                  int F_out, int ld, int B, bool sys) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int row = row0w + 8 * g + 2 * (i >> 2) + ((i >> 1) & 1), tok = 2 * t + (i & 1);
        if (row >= F_out || tok >= B) continue;
        const unsigned long long add = (1ull << kCntShift) + (unsigned long long)(kCntBias + q[i]);
        if (sys) asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" :: "l"(y + (size_t)tok * ld + row), "l"(add) : "memory");
        else asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(y + (size_t)tok * ld + row), "l"(add) : "memory");
    }
}

// x staging from counted accumulator words [B][F_in] produced by ks K-split
// CTAs of the previous step: every thread polls its words until all carry
// count == ks (one L2 round trip once they are final), then forms fp16 x.
// Layout of s_x as stage_x.  MODE:
//   XM_WORDS  x = fp16(value)                                  (one RN rounding)
//   XM_GAMMA  x = fp16(fp32(value) * gamma[col])               (RMSNorm with the scale folded into
//             the epilogue, chain_internal.cuh); with sq != NULL also the sum of fp32(value)^2 per
//             token over this K range: sq[warp * NB + b] = the warp's partial (fixed order)
//   XM_GAMMA2 as XM_GAMMA of the value (x word + x2 word) (a lazily materialised residual sum)
//   XM_SILU   x = fp16(silu(g) * u), g/u = values of x / x2    (SwiGLU gate * up, fp32), with
//             xs != NULL: g and u scaled by xs[b] first (the RMSNorm scale of the gate/up input)
constexpr int XM_WORDS = 0, XM_GAMMA = 1, XM_SILU = 2, XM_GAMMA2 = 3;

template <int D, int NB, int NW, bool XF = false, int MODE = XM_WORDS>
__device__ __forceinline__ void stage_x_counted(uint8_t* s_x, const unsigned long long* x, int ks, int F_in, int B,
                                                int N_ss, int g_begin, int ng, bool sys = true, int backoff = 0,
                                                const unsigned long long* x2 = nullptr, int ks2 = 0,
                                                float* sq = nullptr, const __half* gamma = nullptr,
                                                const float* xs = nullptr) {
    constexpr int E = Entry<D>::value;
    float sqa[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) sqa[b] = 0.f;
    constexpr int NX = (MODE == XM_SILU || MODE == XM_GAMMA2) ? 2 : 1;     // words per element
    const int tid = threadIdx.x;
    const int n_ent = ng * 32 * NB;
    // entries per thread per pass: every pass is one poll round trip (B = 8 stages 8x the entries)
    constexpr int XPT = NX == 2 ? (NB >= 8 ? 2 : 1) : (NB >= 8 ? 4 : 2);
    for (int t0 = tid; t0 < n_ent; t0 += NW * 32 * XPT) {
        unsigned long long v[XPT][NX][D];
        bool need[XPT];
#pragma unroll
        for (int u = 0; u < XPT; ++u) {
            const int t = t0 + u * NW * 32;
            const int b = t % NB;
            const int ss = (g_begin + t / (NB * 32)) * 32 + ((t / NB) & 31);
            need[u] = t < n_ent && b < B && ss < N_ss;
#pragma unroll
            for (int q = 0; q < NX; ++q)
#pragma unroll
                for (int e = 0; e < D; ++e) v[u][q][e] = 0;
        }
        // poll: reload every word of this thread until all are final (a
        // watchdog turns a lost producer into a kernel error, not a hang)
        bool done = false;
        const unsigned long long t_start = dev::globaltimer();
        for (int round = 0; !done; ++round) {
            done = true;
            if (dev::globaltimer() - t_start > 4000000000ull) __trap();
            if (round > 0 && backoff > 0) __nanosleep(backoff);
#pragma unroll
            for (int u = 0; u < XPT; ++u) {
                if (!need[u]) continue;
                const int t = t0 + u * NW * 32;
                const int b = t % NB;
                const int ss = (g_begin + t / (NB * 32)) * 32 + ((t / NB) & 31);
#pragma unroll
                for (int q = 0; q < NX; ++q) {
                    const unsigned long long* src = (q == 0 ? x : x2) + (size_t)b * F_in + (size_t)ss * D;
                    const unsigned long long want = (unsigned long long)(q == 0 ? ks : ks2);
#pragma unroll
                    for (int e = 0; e < D; ++e) {
                        if ((v[u][q][e] >> kCntShift) == want) continue;
                        if (sys)
                            asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v[u][q][e]) : "l"(src + e) : "memory");
                        else
                            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v[u][q][e]) : "l"(src + e) : "memory");
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < XPT; ++u)
#pragma unroll
                for (int q = 0; q < NX; ++q)
#pragma unroll
                    for (int e = 0; e < D; ++e)
                        if (need[u] && (v[u][q][e] >> kCntShift) != (unsigned long long)(q == 0 ? ks : ks2)) done = false;
        }
#pragma unroll
        for (int u = 0; u < XPT; ++u) {
            const int t = t0 + u * NW * 32;
            if (t >= n_ent) continue;
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            if (need[u]) {
                const int b = t % NB;
                const int ss = (g_begin + t / (NB * 32)) * 32 + ((t / NB) & 31);
#pragma unroll
                for (int e = 0; e < D; ++e) {
                    const long long val = (long long)(v[u][0][e] & kCntMask) - (long long)ks * kCntBias;
                    uint32_t h;
                    if (MODE == XM_WORDS) {
                        h = __half_as_ushort(__double2half((double)val * kAccInv));
                    } else if (MODE == XM_GAMMA || MODE == XM_GAMMA2) {
                        long long vs = val;
                        if (MODE == XM_GAMMA2)
                            vs += (long long)(v[u][NX - 1][e] & kCntMask) - (long long)ks2 * kCntBias;
                        const float f = (float)((double)vs * kAccInv);
#pragma unroll
                        for (int bb = 0; bb < NB; ++bb)
                            if (bb == b) sqa[bb] += f * f;
                        h = __half_as_ushort(__float2half_rn(f * __half2float(gamma[(size_t)ss * D + e])));
                    } else {
                        const long long val2 = (long long)(v[u][NX - 1][e] & kCntMask) - (long long)ks2 * kCntBias;
                        float g = (float)((double)val * kAccInv);
                        float uu = (float)((double)val2 * kAccInv);
                        if (xs) {
                            float sb = xs[0];
#pragma unroll
                            for (int bb = 1; bb < NB; ++bb)
                                if (bb == b) sb = xs[bb];
                            g *= sb;
                            uu *= sb;
                        }
                        h = __half_as_ushort(__float2half_rn(g / (1.0f + expf(-g)) * uu));
                    }
                    w[e >> 1] |= h << (16 * (e & 1));
                }
            }
            if (XF) {
                store_x_f32<D, NB>(s_x, t, w);
                continue;
            }
            uint32_t* dst = reinterpret_cast<uint32_t*>(s_x + (size_t)t * E);
#pragma unroll
            for (int q = 0; q < E / 4; ++q) dst[q] = w[q];
        }
    }
    if ((MODE == XM_GAMMA || MODE == XM_GAMMA2) && sq) {
        const int lane = tid & 31;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            float a = sqa[b];
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
            if (lane == 0) sq[(tid >> 5) * NB + b] = a;
        }
    }
}

// RMSNorm scale of the counted vector x [B][n] (ks contributions per word):
// scale[b] = 1 / sqrt(mean_i value_i^2 + eps), fp32 sums in a FIXED order
// (per-thread strided partials, warp butterfly, warps in order) so that every
// CTA computes bit-identical scales.  Polls every word (the whole vector
// must be final).  red: NW*8 floats of SMEM; scale: 8 floats of SMEM.
template <int NB, int NW>
__device__ __noinline__ void norm_scale(const unsigned long long* x, int ks, int n, int B, float eps, bool sys,
                                        float* red, float* scale) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NT = NW * 32;
    float acc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = 0.f;
    constexpr int U = 8;   // words in flight per thread
    const int total = B * n;
    for (int i0 = tid; i0 < total; i0 += NT * U) {
        unsigned long long v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = 0;
        bool done = false;
        const unsigned long long t_start = dev::globaltimer();
        while (!done) {
            done = true;
            if (dev::globaltimer() - t_start > 4000000000ull) __trap();
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * NT;
                if (i >= total || (v[u] >> kCntShift) == (unsigned long long)ks) continue;
                if (sys)
                    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v[u]) : "l"(x + i) : "memory");
                else
                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v[u]) : "l"(x + i) : "memory");
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 + u * NT < total && (v[u] >> kCntShift) != (unsigned long long)ks) done = false;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * NT;
            if (i >= total) continue;
            const float f = (float)((double)((long long)(v[u] & kCntMask) - (long long)ks * kCntBias) * kAccInv);
            const int b = i / n;
#pragma unroll
            for (int bb = 0; bb < NB; ++bb)
                if (bb == b) acc[bb] += f * f;
        }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        float a = acc[b];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
        if (lane == 0) red[warp * 8 + b] = a;
    }
    asm volatile("bar.sync 1, %0;" :: "n"(NT) : "memory");
    if (tid < NB) {
        float a = 0.f;
        for (int w = 0; w < NW; ++w) a += red[w * 8 + tid];
        scale[tid] = 1.0f / sqrtf(a / (float)n + eps);
    }
    asm volatile("bar.sync 1, %0;" :: "n"(NT) : "memory");
}

}  // namespace core
}  // namespace fasq
