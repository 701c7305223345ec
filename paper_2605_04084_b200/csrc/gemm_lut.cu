// gemm_lut.cu -- FASQ prefill GEMM, table-lookup variant (sm_100a).
//
// Alg. 3's math: for each token l and subspace ss a lookup table
// LUT_ss[k] = dot(X[l]_ss, T_cluster[ss][k]) over all K_s centroids,
// then Y[l][j] += LUT_ss[T_index[ss][j]].  The paper's design is output-
// stationary with a double-buffered 257-float LUT per (token, subspace); here
// one CTA (16 warps, 2 rows per thread) owns 1024 weight rows x MT = 6 tokens
// (3 token-pair LUT images = 192 KiB at C = 256: the per-group LUT build and
// index re-layout are amortised over 6 tokens), builds the LUTs of a whole
// 32-subspace group at once in SMEM, [C][32 subspaces] fp32 per token laid out
// like the GEMV codebook image, and every lane (= 4 weight rows, rotated
// subspace order) gathers conflict-free with the one-`prmt` address.  The
// group's index block is first re-laid in SMEM from the subspace-major HBM
// layout into row-rotated rows (byte p of row r = subspace (p + r) & 31).  The
// gathers are pure FADD on CUDA cores -- no tensor cores --
// which is why the EXPAND variant exists (gemm_tc.cu).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "fasq_internal.cuh"

namespace fasq {

namespace {

constexpr int LUT_MT = 6;          // tokens per CTA
constexpr int LUT_RPT = 2;         // weight rows per thread
constexpr int LUT_THREADS = 512;
constexpr int LUT_R = LUT_THREADS * LUT_RPT;   // 1024 rows per CTA

struct LutParams {
    const uint8_t* idx;       // [n_groups][F_out_pad/64][32][64] (fasq_internal.cuh)
    const uint8_t* cbimg;     // [n_groups][C][32][E], E = 4*EW bytes (d <= 2: 4, d = 4: 8, d = 8: 16)
    const __half* X;          // [M][F_in]
    void* Y;
    float* part;              // split-K (gridDim.z > 1): fp32 partials [z][M][F_out] (per-call workspace)
    int M, F_in, F_out, F_out_pad, n_groups, N_ss, C, d, y_f32;
};

// LUT SMEM: token pair tp = t>>1 occupies C*256 B; row k = [t even: 32 x f32][t odd: 32 x f32];
// then the row-rotated index block [LUT_R][32] bytes.
// EW = 32-bit words per codebook entry / x slice (1: d <= 2, 2: d = 4, 4: d = 8):
// LUT entry = dot(x_ss, c_k) accumulated word by word in the GEMV's order.
template <int EW>
__global__ void __launch_bounds__(LUT_THREADS, 1) k_gemm_lut(LutParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int C = p.C;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r_base = blockIdx.x * LUT_R;
    const int m0 = blockIdx.y * LUT_MT;
    const uint32_t lut_u = dev::smem_u32(smem);
    uint8_t* s_idx = smem + (size_t)(LUT_MT / 2) * C * 256;
    const int rot = lane;   // natural byte order of the row-rotated index layout
    uint32_t Lr[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) v |= (uint32_t)(((4 * w + j + rot) & 31) * 4) << (8 * j);
        Lr[w] = v;
    }
    float acc[LUT_RPT][LUT_MT];
#pragma unroll
    for (int q = 0; q < LUT_RPT; ++q)
#pragma unroll
        for (int t = 0; t < LUT_MT; ++t) acc[q][t] = 0.f;

    // split-K (short L, Alg. 3's split-K): blockIdx.z owns groups [g0, g1)
    const int g0 = (int)((long long)blockIdx.z * p.n_groups / gridDim.z);
    const int g1 = (int)((long long)(blockIdx.z + 1) * p.n_groups / gridDim.z);
    for (int g = g0; g < g1; ++g) {
        __syncthreads();   // previous group's gathers done
        // build: entry (t, k, sub) = sum_e x[t][sub*d+e] * c[sub][k][e]  (fp32, exact fp16 products)
        const uint32_t* cbg = reinterpret_cast<const uint32_t*>(p.cbimg + (size_t)g * C * 128 * EW);
        // this thread's subspace is fixed (LUT_THREADS is a multiple of 32): its
        // x slices for the MT tokens are loaded once per group
        const int sub = tid & 31, ss = g * 32 + sub;
        uint32_t xv[LUT_MT][EW];
#pragma unroll
        for (int t = 0; t < LUT_MT; ++t) {
            const int m = m0 + t;
#pragma unroll
            for (int q = 0; q < EW; ++q) xv[t][q] = 0;
            if (m < p.M && ss < p.N_ss) {
                const uint16_t* xs = reinterpret_cast<const uint16_t*>(p.X) + (size_t)m * p.F_in + (size_t)ss * p.d;
                if (EW == 1) {
                    xv[t][0] = p.d == 2 ? (uint32_t)xs[0] | ((uint32_t)xs[1] << 16) : (uint32_t)xs[0];
                } else {
#pragma unroll
                    for (int q = 0; q < EW; ++q) xv[t][q] = (uint32_t)xs[2 * q] | ((uint32_t)xs[2 * q + 1] << 16);
                }
            }
        }
#pragma unroll 4
        for (int e = tid; e < C * 32; e += LUT_THREADS) {
            const int k = e >> 5;
            uint32_t c[EW];
#pragma unroll
            for (int q = 0; q < EW; ++q) c[q] = cbg[(size_t)e * EW + q];
#pragma unroll
            for (int t = 0; t < LUT_MT; ++t) {
                float v = 0.f;
#pragma unroll
                for (int q = 0; q < EW; ++q) v = dev::fhfma2(c[q], xv[t][q], v);
                reinterpret_cast<float*>(smem)[((t >> 1) * C * 64) + k * 64 + (t & 1) * 32 + sub] = v;
            }
        }
        // index block re-layout: 16-row chunks of subspace s -> rotated rows
        for (int q = tid; q < (LUT_R / 16) * 32; q += LUT_THREADS) {
            const int sub = q & 31, ch = q >> 5;
            const int r0 = r_base + ch * 16;
            if (r0 >= p.F_out_pad) continue;
            const uint4 v = *reinterpret_cast<const uint4*>(p.idx + idx_offset(g, r0, sub, p.F_out_pad));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int rl = ch * 16 + j;
                s_idx[rl * 32 + ((sub - rl) & 31)] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < LUT_RPT; ++q) {
            const int rl = q * LUT_THREADS + warp * 32 + lane;
            const int row = r_base + rl;
            if (row >= p.F_out_pad) continue;
            const uint4* ip = reinterpret_cast<const uint4*>(s_idx + rl * 32);
            const uint4 v0 = ip[0], v1 = ip[1];
            const uint32_t iw[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
            for (int st = 0; st < 32; ++st) {
                const int j = st & 3;
                const uint32_t sel = (uint32_t)(4 + j) | ((uint32_t)j << 4) | ((uint32_t)(12 + j) << 8) |
                                     ((uint32_t)(12 + j) << 12);
                const uint32_t a = dev::prmt(iw[st >> 2], Lr[st >> 2], sel);
#pragma unroll
                for (int t = 0; t < LUT_MT; ++t)
                    acc[q][t] += __uint_as_float(dev::lds32(lut_u + (uint32_t)((t >> 1) * C * 256 + (t & 1) * 128) + a));
            }
        }
    }
#pragma unroll
    for (int q = 0; q < LUT_RPT; ++q) {
        const int row = r_base + q * LUT_THREADS + warp * 32 + lane;
        if (row >= p.F_out) continue;
#pragma unroll
        for (int t = 0; t < LUT_MT; ++t) {
            const int m = m0 + t;
            if (m >= p.M) continue;
            if (gridDim.z > 1) { p.part[((size_t)blockIdx.z * p.M + m) * p.F_out + row] = acc[q][t]; continue; }
            if (p.y_f32) reinterpret_cast<float*>(p.Y)[(size_t)m * p.F_out + row] = acc[q][t];
            else reinterpret_cast<__half*>(p.Y)[(size_t)m * p.F_out + row] = __float2half_rn(acc[q][t]);
        }
    }
}

// split-K merge: Y = sum over z = 0..ks-1 in fixed order (deterministic)
__global__ void k_lut_merge(const float* __restrict__ part, int ks, int64_t n, void* Y, int y_f32) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float v = 0.f;
    for (int z = 0; z < ks; ++z) v += __ldcs(part + (size_t)z * n + i);
    if (y_f32) reinterpret_cast<float*>(Y)[i] = v;
    else reinterpret_cast<__half*>(Y)[i] = __float2half_rn(v);
}

template <int EW>
fasq_status launch_lut(const LutParams& p, dim3 grid, size_t smem, cudaStream_t st) {
    static std::once_flag once;   // per instantiation
    static size_t lim = 0;
    std::call_once(once, [] { lim = set_max_dyn_smem(k_gemm_lut<EW>); });
    if (lim < smem) { set_error("gemm_lut: SMEM"); return FASQ_E_UNSUPPORTED; }
    k_gemm_lut<EW><<<grid, LUT_THREADS, smem, st>>>(p);
    return FASQ_OK;
}

}  // namespace

fasq_status gemm_lut_launch(const fasq_layer* L, const __half* X, int64_t M, void* Y, fasq_dtype yt,
                            cudaStream_t st) {

    if (M > (1ll << 30)) return FASQ_E_UNSUPPORTED;
    LutParams p{};
    p.idx = L->idx;
    p.cbimg = L->cbimg;
    p.X = X;
    p.Y = Y;
    p.M = (int)M;
    p.F_in = (int)L->F_in;
    p.F_out = (int)L->F_out;
    p.F_out_pad = L->F_out_pad;
    p.n_groups = L->n_groups;
    p.N_ss = L->N_ss;
    p.C = L->C;
    p.d = L->d;
    p.y_f32 = yt == FASQ_F32;
    const size_t smem = (size_t)(LUT_MT / 2) * L->C * 256 + (size_t)LUT_R * 32;
    dim3 grid((unsigned)((L->F_out_pad + LUT_R - 1) / LUT_R), (unsigned)((M + LUT_MT - 1) / LUT_MT));
    // short L: fewer (row, token) tiles than 2 waves of SMs -> split the groups
    // over gridDim.z (fp32 partials in a per-call workspace + a fixed-order merge)
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const long long tiles = (long long)grid.x * grid.y;
    int ks = 1;
    if (const char* e = getenv("FASQ_LUT_KSPLIT")) ks = atoi(e);
    else if (tiles < 2ll * sms) ks = (int)std::min<long long>(L->n_groups, (2ll * sms + tiles - 1) / tiles);
    ks = std::max(1, std::min(ks, L->n_groups));
    float* part = nullptr;
    const int64_t n = M * L->F_out;
    float* part_call = nullptr;
    if (ks > 1) {   // partials are overwritten: the stream's workspace, else a per-call one
        fasq_status a = stream_workspace(st, WS_GEMM_LUT, (size_t)ks * n * sizeof(float), reinterpret_cast<void**>(&part));
        if (a != FASQ_OK) return a;
        if (!part) {
            a = dev_alloc_t(&part_call, (size_t)ks * n * sizeof(float), st);
            if (a != FASQ_OK) return a;
            part = part_call;
        }
        grid.z = (unsigned)ks;
        p.part = part;
    }
    fasq_status s = L->d <= 2 ? launch_lut<1>(p, grid, smem, st)
                  : L->d == 4 ? launch_lut<2>(p, grid, smem, st) : launch_lut<4>(p, grid, smem, st);
    cudaError_t e = cudaGetLastError();
    if (s == FASQ_OK && e != cudaSuccess) s = cuda_fail(e, "k_gemm_lut");
    if (s == FASQ_OK && ks > 1) {
        k_lut_merge<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, ks, n, Y, yt == FASQ_F32);
        e = cudaGetLastError();
        if (e != cudaSuccess) s = cuda_fail(e, "k_lut_merge");
    }
    dev_free(part_call, st);
    if (s != FASQ_OK) return s;
    set_launch_count(ks > 1 ? 2 : 1);
    return FASQ_OK;
}

}  // namespace fasq
