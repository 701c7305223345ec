// pack.cu -- GPU k-means packer (Alg. 1), bit-exact with the CPU
// oracle for the same (d, C, group, seed, iters).
//
// Per codebook g (independent k-means problems -- Alg. 1's "parallel for",
// P:164), following DESIGN.md "Pack reading" step by step:
//   keys   : each point's d fp16 bit patterns (-0 -> +0), element 0 most
//            significant; segmented radix sort per codebook; unique set U.
//   init   : seeded partial Fisher-Yates over U with splitmix64
//            (state = seed ^ (g+1)*0x9E3779B97F4A7C15), m = min(C, |U|);
//            slots >= m copy slot 0.
//   Lloyd  : assign = argmin_k sum_e (p_e - c_ke)^2 with separately rounded
//            fp32 __fsub_rn/__fmul_rn/__fadd_rn (no FMA contraction), strict
//            '<' in ascending k; stop when the assignment is unchanged;
//            update = exact int64 sums of p*2^24 (integer atomics, order-
//            independent) and one fp64 divide; empty clusters keep c.
//   final  : c_hat = fp16_rn(c) (-0 -> +0), one more assign against c_hat.
// Every step is integer arithmetic or a fixed sequence of IEEE RN operations,
// so the bytes equal the oracle's (tests/test_gpu_pack.py).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "fasq_internal.cuh"

namespace fasq {

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint16_t canon16(uint16_t h) { return h == 0x8000u ? (uint16_t)0 : h; }

__device__ __forceinline__ uint64_t splitmix64_next(uint64_t& s) {
    s += kGolden;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_check_finite(const uint16_t* __restrict__ W, int64_t n, int* flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool bad = false;
    for (; i < n; i += stride) bad |= (W[i] & 0x7c00u) == 0x7c00u;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Points of codebook g: t = (ss - g*group)*F_out + j is W[j, ss*d : ss*d+d]
// (reading R1).  P[g*n + t][e] = canonical fp16 bits; key = d x 16 bits,
// element 0 most significant (hi: elements 0..3, lo: 4..7 for d = 8).
__global__ void k_points_keys(const uint16_t* __restrict__ W, int64_t F_out, int64_t F_in, int d, int group,
                              int64_t n, int64_t total, uint16_t* __restrict__ P, uint64_t* __restrict__ khi,
                              uint64_t* __restrict__ klo) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int64_t g = i / n, t = i % n;
    int64_t ss = g * group + t / F_out, j = t % F_out;
    const uint16_t* src = W + j * F_in + ss * d;
    uint64_t hi = 0, lo = 0;
    for (int e = 0; e < d; ++e) {
        uint16_t h = canon16(src[e]);
        P[i * d + e] = h;
        if (d <= 4) hi = (hi << 16) | h;
        else if (e < 4) hi = (hi << 16) | h;
        else lo = (lo << 16) | h;
    }
    khi[i] = hi;
    if (klo) klo[i] = lo;
}

__global__ void k_seg_offsets(int* off, int N_cb, int64_t n) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g <= N_cb) off[g] = (int)(g * n);
}

__global__ void k_unique_flags(const uint64_t* __restrict__ hi, const uint64_t* __restrict__ lo, int64_t n,
                               int64_t total, int* __restrict__ flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int f = (i % n == 0) || hi[i] != hi[i - 1] || (lo && lo[i] != lo[i - 1]);
    flag[i] = f;
}

__global__ void k_scatter_unique(const uint64_t* __restrict__ hi, const uint64_t* __restrict__ lo,
                                 const int* __restrict__ flag, const int* __restrict__ pos, int64_t total,
                                 uint64_t* __restrict__ Uhi, uint64_t* __restrict__ Ulo) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    if (flag[i]) {
        Uhi[pos[i]] = hi[i];
        if (lo) Ulo[pos[i]] = lo[i];
    }
}

__device__ __forceinline__ float key_elem(uint64_t hi, uint64_t lo, int d, int e) {
    uint16_t h;
    if (d <= 4) h = (uint16_t)(hi >> (16 * (d - 1 - e)));
    else h = e < 4 ? (uint16_t)(hi >> (16 * (3 - e))) : (uint16_t)(lo >> (16 * (7 - e)));
    return __half2float(__ushort_as_half(h));
}

// One thread per codebook: partial Fisher-Yates, init centroids (fp32).
__global__ void k_init(uint64_t* __restrict__ Uhi, uint64_t* __restrict__ Ulo, const int* __restrict__ pos,
                       const int* __restrict__ flag, int64_t n, int N_cb, int C, int d, uint64_t seed,
                       float* __restrict__ cent) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= N_cb) return;
    const int64_t s0 = pos[(int64_t)g * n];
    const int64_t last = (int64_t)(g + 1) * n - 1;
    const int64_t cnt = pos[last] + flag[last] - s0;
    const int64_t m = cnt < C ? cnt : C;
    uint64_t st = seed ^ ((uint64_t)(g + 1) * kGolden);
    for (int64_t i = 0; i < m; ++i) {
        uint64_t r = splitmix64_next(st);
        int64_t j = i + (int64_t)(r % (uint64_t)(cnt - i));
        uint64_t a = Uhi[s0 + i]; Uhi[s0 + i] = Uhi[s0 + j]; Uhi[s0 + j] = a;
        if (Ulo) { uint64_t b = Ulo[s0 + i]; Ulo[s0 + i] = Ulo[s0 + j]; Ulo[s0 + j] = b; }
    }
    for (int k = 0; k < C; ++k) {
        int64_t src = s0 + (k < m ? k : 0);
        uint64_t hi = Uhi[src], lo = Ulo ? Ulo[src] : 0;
        for (int e = 0; e < d; ++e) cent[((int64_t)g * C + k) * d + e] = key_elem(hi, lo, d, e);
    }
}

// argmin_k D(p, c_k): D = sum_e (p_e - c_ke)^2 left to right, separately
// rounded fp32 ops (never contracted), strict '<', ascending k.
template <int D>
__device__ __forceinline__ int nearest(const float* p, const float* __restrict__ sc, int C, float* bestD_out = nullptr) {
    int best = 0;
    float bestD = 0.f;
    for (int k = 0; k < C; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < D; ++e) {
            float dl = __fsub_rn(p[e], sc[k * D + e]);
            float sq = __fmul_rn(dl, dl);
            acc = (e == 0) ? sq : __fadd_rn(acc, sq);
        }
        if (k == 0 || acc < bestD) { bestD = acc; best = k; }
    }
    if (bestD_out) *bestD_out = bestD;
    return best;
}

// ---- packing variants (NEXT-4) ------------------------------------------------
// k-means++ (reading R17) in exact integer arithmetic, one CTA per
// codebook: q = fp16 value * 2^24 (exact int64), D2 = sum_e (dq)^2 as u128;
// centre 0 = point next() % n; then r = (next() << 64 | next()) mod total and
// the next centre is the smallest t whose inclusive prefix of dist exceeds r;
// total == 0: remaining slots copy centre 0.  Same splitmix64 stream as R3.
typedef unsigned __int128 u128;
constexpr int kPPThreads = 512;

template <int D>
__device__ __forceinline__ u128 d2_pts(const uint16_t* __restrict__ a, const uint16_t* __restrict__ b) {
    u128 s = 0;
#pragma unroll
    for (int e = 0; e < D; ++e) {
        const long long qa = (long long)__dmul_rn((double)__half2float(__ushort_as_half(a[e])), 16777216.0);
        const long long qb = (long long)__dmul_rn((double)__half2float(__ushort_as_half(b[e])), 16777216.0);
        const __int128 df = (__int128)qa - (__int128)qb;
        s += (u128)(df * df);
    }
    return s;
}

template <int D>
__global__ void __launch_bounds__(kPPThreads) k_kmeanspp(const uint16_t* __restrict__ P, int64_t n, int C,
                                                         uint64_t seed, u128* __restrict__ dist_all,
                                                         float* __restrict__ cent) {
    const int g = blockIdx.x, tid = threadIdx.x;
    const uint16_t* Pg = P + (size_t)g * n * D;
    u128* dist = dist_all + (size_t)g * n;
    __shared__ u128 s_sum[kPPThreads];
    __shared__ long long s_pick;
    __shared__ int s_stop;
    const int64_t per = (n + kPPThreads - 1) / kPPThreads;
    const int64_t t0 = min(n, per * tid), t1 = min(n, t0 + per);
    uint64_t st = seed ^ ((uint64_t)(g + 1) * kGolden);   // thread 0's stream
    if (tid == 0) s_pick = (long long)(splitmix64_next(st) % (uint64_t)n);
    __syncthreads();
    long long first = s_pick;
    for (int64_t t = t0; t < t1; ++t) dist[t] = d2_pts<D>(Pg + t * D, Pg + first * D);
    if (tid < D) cent[((size_t)g * C) * D + tid] = __half2float(__ushort_as_half(Pg[first * D + tid]));
    int k = 1;
    for (; k < C; ++k) {
        u128 cs = 0;
        for (int64_t t = t0; t < t1; ++t) cs += dist[t];
        s_sum[tid] = cs;
        __syncthreads();
        if (tid == 0) {
            u128 total = 0;
            for (int i = 0; i < kPPThreads; ++i) total += s_sum[i];
            s_stop = total == 0;
            if (total != 0) {
                const u128 hi = splitmix64_next(st), lo = splitmix64_next(st);
                u128 r = ((hi << 64) | lo) % total;
                int c = 0;
                while (r >= s_sum[c]) { r -= s_sum[c]; ++c; }   // chunk holding r (its sum > r)
                const int64_t c0 = min(n, per * c), c1 = min(n, c0 + per);
                long long pick = c1 - 1;
                u128 acc = 0;
                for (int64_t t = c0; t < c1; ++t) {
                    acc += dist[t];
                    if (acc > r) { pick = t; break; }
                }
                s_pick = pick;
            }
        }
        __syncthreads();
        if (s_stop) break;
        const long long pk = s_pick;
        for (int64_t t = t0; t < t1; ++t) {
            const u128 dd = d2_pts<D>(Pg + t * D, Pg + pk * D);
            if (dd < dist[t]) dist[t] = dd;
        }
        if (tid < D) cent[((size_t)g * C + k) * D + tid] = __half2float(__ushort_as_half(Pg[pk * D + tid]));
        __syncthreads();   // s_sum / s_pick reuse
    }
    __syncthreads();
    for (int q = k * D + tid; q < C * D; q += kPPThreads) cent[(size_t)g * C * D + q] = cent[(size_t)g * C * D + q % D];
}

constexpr int kAssignThreads = 256;

template <int D>
__global__ void __launch_bounds__(kAssignThreads) k_assign_accum(
    const uint16_t* __restrict__ P, const float* __restrict__ cent, int64_t n, int C, int it,
    uint16_t* __restrict__ asg, const uint16_t* __restrict__ prev, unsigned long long* __restrict__ S,
    unsigned long long* __restrict__ cnt, int* __restrict__ changed, const int* __restrict__ done,
    float* __restrict__ bestD) {
    const int g = blockIdx.y;
    if (done[g]) return;
    extern __shared__ __align__(16) uint8_t sm[];
    float* sc = reinterpret_cast<float*>(sm);                                    // C*D
    unsigned long long* sS = reinterpret_cast<unsigned long long*>(sm + ((C * D * 4 + 15) / 16) * 16);
    unsigned long long* sN = sS + C * D;
    for (int q = threadIdx.x; q < C * D; q += blockDim.x) {
        sc[q] = cent[(int64_t)g * C * D + q];
        sS[q] = 0ull;
    }
    for (int q = threadIdx.x; q < C; q += blockDim.x) sN[q] = 0ull;
    __syncthreads();
    bool chg = false;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = (int64_t)g * n + t;
        float p[D];
#pragma unroll
        for (int e = 0; e < D; ++e) p[e] = __half2float(__ushort_as_half(P[i * D + e]));
        float bd;
        const int a = nearest<D>(p, sc, C, &bd);
        if (bestD) bestD[i] = bd;
        asg[i] = (uint16_t)a;
        if (it > 1 && a != prev[i]) chg = true;
        atomicAdd(&sN[a], 1ull);
#pragma unroll
        for (int e = 0; e < D; ++e) {
            long long v = (long long)__dmul_rn((double)p[e], 16777216.0);   // exact
            atomicAdd(&sS[a * D + e], (unsigned long long)v);
        }
    }
    if (__syncthreads_or(chg) && threadIdx.x == 0) atomicOr(&changed[g], 1);
    for (int q = threadIdx.x; q < C * D; q += blockDim.x)
        if (sS[q]) atomicAdd(&S[(int64_t)g * C * D + q], sS[q]);
    for (int q = threadIdx.x; q < C; q += blockDim.x)
        if (sN[q]) atomicAdd(&cnt[(int64_t)g * C + q], sN[q]);
}

// One block per codebook: stop test, then c = fp32((fp64(S)/fp64(n)) * 2^-24).
// With bestD (empty = 1, reading R18): empty clusters, ascending
// k, are reseeded with the points farthest from their assigned centroid
// (this iteration's fp32 distance), ties -> lowest t, each point at most once.
__global__ void k_update(float* __restrict__ cent, unsigned long long* __restrict__ S,
                         unsigned long long* __restrict__ cnt, int* __restrict__ changed, int* __restrict__ done,
                         int* __restrict__ iters_run, int C, int d, int it, const float* __restrict__ bestD,
                         const uint16_t* __restrict__ P, int64_t n) {
    const int g = blockIdx.x;
    __shared__ int s_skip;
    __shared__ unsigned long long s_best;
    __shared__ long long s_taken[1024];   // <= C empty clusters (C <= 1024)
    __shared__ int s_ntaken;
    if (threadIdx.x == 0) {
        int sk = done[g];
        if (!sk) {
            iters_run[g] = it;
            if (it > 1 && !changed[g]) { done[g] = 1; sk = 1; }
        }
        s_skip = sk;
    }
    __syncthreads();
    if (s_skip) return;
    if (bestD) {
        if (threadIdx.x == 0) s_ntaken = 0;
        __syncthreads();
        for (int k = 0; k < C; ++k) {
            if (cnt[(int64_t)g * C + k] != 0ull) continue;   // block-uniform
            if (threadIdx.x == 0) s_best = 0ull;
            __syncthreads();
            // key: distance bits (>= 0: order-preserving) high, ~t low -> max = farthest, lowest t
            unsigned long long mine = 0ull;
            for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
                bool used = false;
                for (int q2 = 0; q2 < s_ntaken; ++q2) used |= s_taken[q2] == t;
                if (used) continue;
                const unsigned long long key = ((unsigned long long)__float_as_uint(bestD[(int64_t)g * n + t]) << 32) |
                                               (unsigned long long)(0xFFFFFFFFu - (unsigned)t);
                mine = max(mine, key);
            }
            atomicMax(&s_best, mine);
            __syncthreads();
            if (s_best != 0ull) {
                const long long t = (long long)(0xFFFFFFFFu - (unsigned)(s_best & 0xFFFFFFFFull));
                if (threadIdx.x < d)
                    cent[((int64_t)g * C + k) * d + threadIdx.x] =
                        __half2float(__ushort_as_half(P[((int64_t)g * n + t) * d + threadIdx.x]));
                if (threadIdx.x == 0) s_taken[s_ntaken++] = t;
            }
            __syncthreads();
        }
    }
    for (int q = threadIdx.x; q < C * d; q += blockDim.x) {
        const int k = q / d;
        const int64_t off = (int64_t)g * C * d + q;
        const long long nk = (long long)cnt[(int64_t)g * C + k];
        if (nk > 0) {
            double mean = __ddiv_rn(__ll2double_rn((long long)S[off]), __ll2double_rn(nk));
            cent[off] = __double2float_rn(__dmul_rn(mean, 1.0 / 16777216.0));
        }
        S[off] = 0ull;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < C; k += blockDim.x) cnt[(int64_t)g * C + k] = 0ull;
    if (threadIdx.x == 0) changed[g] = 0;
}

__global__ void k_finalize_cb(const float* __restrict__ cent, __half* __restrict__ cb, int64_t total) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= total) return;
    uint16_t h = __half_as_ushort(__float2half_rn(cent[q]));
    cb[q] = __ushort_as_half(canon16(h));
}

template <int D>
__global__ void __launch_bounds__(kAssignThreads) k_final_assign(const uint16_t* __restrict__ P,
                                                                 const __half* __restrict__ cb, int64_t n, int C,
                                                                 int group, int64_t F_out, uint16_t* __restrict__ idx) {
    const int g = blockIdx.y;
    extern __shared__ __align__(16) uint8_t sm[];
    float* sc = reinterpret_cast<float*>(sm);
    for (int q = threadIdx.x; q < C * D; q += blockDim.x) sc[q] = __half2float(cb[(int64_t)g * C * D + q]);
    __syncthreads();
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = (int64_t)g * n + t;
        float p[D];
#pragma unroll
        for (int e = 0; e < D; ++e) p[e] = __half2float(__ushort_as_half(P[i * D + e]));
        const int a = nearest<D>(p, sc, C);
        const int64_t ss = (int64_t)g * group + t / F_out, j = t % F_out;
        idx[ss * F_out + j] = (uint16_t)a;
    }
}

inline unsigned nb(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

template <int D>
fasq_status lloyd_and_finalize(const uint16_t* P, float* cent, int64_t n, int N_cb, int C, int group,
                               int64_t F_out, int iters, uint16_t* asg0, uint16_t* asg1, unsigned long long* S,
                               unsigned long long* cnt, int* changed, int* done, int* iters_run, __half* cb_out,
                               uint16_t* idx_out, cudaStream_t st, float* bestD, u128* ppdist, uint64_t seed) {
    if (ppdist) {   // k-means++ init replaces the distinct-sample init (reading R17)
        k_kmeanspp<D><<<N_cb, kPPThreads, 0, st>>>(P, n, C, seed, ppdist, cent);
        FASQ_CUDA_TRY(cudaGetLastError());
        add_launch_count(1);
    }
    const size_t smem = ((size_t)C * D * 4 + 15) / 16 * 16 + (size_t)C * D * 8 + (size_t)C * 8;
    const int chunks = (int)std::min<int64_t>((n + kAssignThreads - 1) / kAssignThreads, 64);
    dim3 grid(chunks, N_cb);
    for (int it = 1; it <= iters; ++it) {
        uint16_t* cur = (it & 1) ? asg1 : asg0;
        uint16_t* prv = (it & 1) ? asg0 : asg1;
        k_assign_accum<D><<<grid, kAssignThreads, smem, st>>>(P, cent, n, C, it, cur, prv, S, cnt, changed, done,
                                                              bestD);
        FASQ_CUDA_TRY(cudaGetLastError());
        k_update<<<N_cb, 256, 0, st>>>(cent, S, cnt, changed, done, iters_run, C, D, it, bestD, P, n);
        FASQ_CUDA_TRY(cudaGetLastError());
    }
    k_finalize_cb<<<nb((int64_t)N_cb * C * D, 256), 256, 0, st>>>(cent, cb_out, (int64_t)N_cb * C * D);
    FASQ_CUDA_TRY(cudaGetLastError());
    k_final_assign<D><<<grid, kAssignThreads, (size_t)C * D * 4, st>>>(P, cb_out, n, C, group, F_out, idx_out);
    FASQ_CUDA_TRY(cudaGetLastError());
    add_launch_count(2 * iters + 2);
    return FASQ_OK;
}

struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    template <class T>
    T* get(size_t count) {
        void* p = nullptr;
        if (dev_alloc(&p, count * sizeof(T) + 16, st) != FASQ_OK) return nullptr;
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~Scratch() {
        for (void* p : ptrs) dev_free(p, st);
    }
};

}  // namespace

fasq_status pack_run(const __half* W_, fasq_layer* L, const fasq_pack_params* prm, cudaStream_t st,
                     __half* cb_out, uint16_t* idx_out) {
    const uint16_t* W = reinterpret_cast<const uint16_t*>(W_);
    const int d = L->d, C = L->C, group = L->group, N_cb = L->N_cb;
    const int64_t F_out = L->F_out, F_in = L->F_in;
    const int64_t n = (int64_t)group * F_out;
    const int64_t total = n * N_cb;
    if (total > (int64_t)INT32_MAX) return FASQ_E_UNSUPPORTED;
    set_launch_count(0);
    Scratch sc(st);
    // (a1) non-finite check (one host sync)
    int* flag = sc.get<int>(1);
    if (!flag) return FASQ_E_OOM;
    FASQ_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
    k_check_finite<<<1184, 256, 0, st>>>(W, F_out * F_in, flag);
    FASQ_CUDA_TRY(cudaGetLastError());
    int hflag = 0;
    FASQ_CUDA_TRY(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    FASQ_CUDA_TRY(cudaStreamSynchronize(st));
    if (hflag) { set_error("fasq_pack: W holds inf/NaN"); return FASQ_E_NONFINITE; }

    const bool wide = d == 8;
    uint16_t* P = sc.get<uint16_t>((size_t)total * d);
    uint64_t* khi = sc.get<uint64_t>(total);
    uint64_t* klo = wide ? sc.get<uint64_t>(total) : nullptr;
    uint64_t* shi = sc.get<uint64_t>(total);
    uint64_t* slo = wide ? sc.get<uint64_t>(total) : nullptr;
    int* off = sc.get<int>(N_cb + 1);
    int* uflag = sc.get<int>(total);
    int* pos = sc.get<int>(total);
    float* cent = sc.get<float>((size_t)N_cb * C * d);
    uint16_t* asg0 = sc.get<uint16_t>(total);
    uint16_t* asg1 = sc.get<uint16_t>(total);
    unsigned long long* S = sc.get<unsigned long long>((size_t)N_cb * C * d);
    unsigned long long* cnt = sc.get<unsigned long long>((size_t)N_cb * C);
    int* changed = sc.get<int>(N_cb);
    int* done = sc.get<int>(N_cb);
    int* iters_run = sc.get<int>(N_cb);
    float* bestD = prm->empty == 1 ? sc.get<float>(total) : nullptr;
    u128* ppdist = prm->init == 1 ? sc.get<u128>(total) : nullptr;
    if ((prm->empty == 1 && !bestD) || (prm->init == 1 && !ppdist)) return FASQ_E_OOM;
    if (!P || !khi || !shi || !off || !uflag || !pos || !cent || !asg0 || !asg1 || !S || !cnt || !changed ||
        !done || !iters_run || (wide && (!klo || !slo)))
        return FASQ_E_OOM;
    FASQ_CUDA_TRY(cudaMemsetAsync(S, 0, (size_t)N_cb * C * d * 8, st));
    FASQ_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)N_cb * C * 8, st));
    FASQ_CUDA_TRY(cudaMemsetAsync(changed, 0, (size_t)N_cb * 4, st));
    FASQ_CUDA_TRY(cudaMemsetAsync(done, 0, (size_t)N_cb * 4, st));
    FASQ_CUDA_TRY(cudaMemsetAsync(iters_run, 0, (size_t)N_cb * 4, st));

    // (a2) keys, per-codebook sort, unique set, seeded init
    k_points_keys<<<nb(total, 256), 256, 0, st>>>(W, F_out, F_in, d, group, n, total, P, khi, klo);
    FASQ_CUDA_TRY(cudaGetLastError());
    k_seg_offsets<<<nb(N_cb + 1, 256), 256, 0, st>>>(off, N_cb, n);
    FASQ_CUDA_TRY(cudaGetLastError());
    const int end_bit = d <= 4 ? 16 * d : 64;
    if (!wide) {
        size_t tb = 0;
        FASQ_CUDA_TRY(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tb, khi, shi, (int)total, N_cb, off, off + 1,
                                                              0, end_bit, st));
        void* tmp = sc.get<uint8_t>(tb);
        if (!tmp) return FASQ_E_OOM;
        FASQ_CUDA_TRY(cub::DeviceSegmentedRadixSort::SortKeys(tmp, tb, khi, shi, (int)total, N_cb, off, off + 1, 0,
                                                              end_bit, st));
    } else {
        // LSD over the 128-bit key: stable sort by lo, then stable sort by hi
        size_t tb1 = 0, tb2 = 0;
        FASQ_CUDA_TRY(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tb1, klo, slo, khi, shi, (int)total, N_cb,
                                                               off, off + 1, 0, 64, st));
        FASQ_CUDA_TRY(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tb2, shi, khi, slo, klo, (int)total, N_cb,
                                                               off, off + 1, 0, 64, st));
        void* tmp = sc.get<uint8_t>(std::max(tb1, tb2));
        if (!tmp) return FASQ_E_OOM;
        FASQ_CUDA_TRY(cub::DeviceSegmentedRadixSort::SortPairs(tmp, tb1, klo, slo, khi, shi, (int)total, N_cb, off,
                                                               off + 1, 0, 64, st));
        // now (slo sorted, shi carried) -> sort by hi carrying lo: keys shi -> khi, values slo -> klo
        FASQ_CUDA_TRY(cub::DeviceSegmentedRadixSort::SortPairs(tmp, tb2, shi, khi, slo, klo, (int)total, N_cb, off,
                                                               off + 1, 0, 64, st));
        // sorted result is in (khi, klo); move to (shi, slo)
        FASQ_CUDA_TRY(cudaMemcpyAsync(shi, khi, (size_t)total * 8, cudaMemcpyDeviceToDevice, st));
        FASQ_CUDA_TRY(cudaMemcpyAsync(slo, klo, (size_t)total * 8, cudaMemcpyDeviceToDevice, st));
    }
    k_unique_flags<<<nb(total, 256), 256, 0, st>>>(shi, slo, n, total, uflag);
    FASQ_CUDA_TRY(cudaGetLastError());
    {
        size_t tb = 0;
        FASQ_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, uflag, pos, (int)total, st));
        void* tmp = sc.get<uint8_t>(tb);
        if (!tmp) return FASQ_E_OOM;
        FASQ_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, uflag, pos, (int)total, st));
    }
    // U (compacted) reuses the key buffers
    k_scatter_unique<<<nb(total, 256), 256, 0, st>>>(shi, slo, uflag, pos, total, khi, klo);
    FASQ_CUDA_TRY(cudaGetLastError());
    k_init<<<nb(N_cb, 64), 64, 0, st>>>(khi, klo, pos, uflag, n, N_cb, C, d, prm->seed, cent);
    FASQ_CUDA_TRY(cudaGetLastError());
    add_launch_count(8);

    // (a3) Lloyd + (a4) finalize
    switch (d) {
        case 1: return lloyd_and_finalize<1>(P, cent, n, N_cb, C, group, F_out, prm->iters, asg0, asg1, S, cnt,
                                             changed, done, iters_run, cb_out, idx_out, st, bestD,
                                             ppdist, prm->seed);
        case 2: return lloyd_and_finalize<2>(P, cent, n, N_cb, C, group, F_out, prm->iters, asg0, asg1, S, cnt,
                                             changed, done, iters_run, cb_out, idx_out, st, bestD,
                                             ppdist, prm->seed);
        case 4: return lloyd_and_finalize<4>(P, cent, n, N_cb, C, group, F_out, prm->iters, asg0, asg1, S, cnt,
                                             changed, done, iters_run, cb_out, idx_out, st, bestD,
                                             ppdist, prm->seed);
        case 8: return lloyd_and_finalize<8>(P, cent, n, N_cb, C, group, F_out, prm->iters, asg0, asg1, S, cnt,
                                             changed, done, iters_run, cb_out, idx_out, st, bestD,
                                             ppdist, prm->seed);
    }
    return FASQ_E_UNSUPPORTED;
}

}  // namespace fasq
