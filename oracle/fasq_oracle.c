/*
 * oracle/fasq_oracle.c -- FASQ CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct host implementation of what the FASQ hot path
 * computes (arXiv 2605.04084, /root/reference/PAPER.md, cited as P:<line>).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and
 * `bench.py --impl reference`) may load this library.  It shares NO code, header,
 * table or constant generator with the CUDA product path
 * (paper_2605_04084_b200/csrc); neither includes the other.
 *
 * What is here:
 *   fasq_ref_pack         Alg. 1: per-codebook k-means -> fp16
 *                         codebooks + uint8 indices, step by step as DESIGN.md
 *                         "Pack reading" fixes it.
 *   fasq_ref_pack_range_ex  the same with the SPEC's packing variants (NEXT-4):
 *                         exact-integer k-means++ init (reading R17) and
 *                         empty-cluster reseeding from the farthest point
 *                         (reading R18).
 *   fasq_ref_lloyd_fp32   the same Lloyd loop for ONE codebook, stopped before
 *                         finalisation (test hook for WCSS monotonicity).
 *   fasq_ref_pack16_range_ex / _reconstruct16 / _gemm_rows16   the same with
 *                         uint16 index tables for C <= 1024 (NEXT-2: Eq. 4's
 *                         ceil(log2 K_s)-bit indices; 2-512 /
 *                         2-1024 in Table 2); fasq_ref_index_bits
 *                         = ceil(log2 K_s).
 *   fasq_ref_pack_dim0_range / _reconstruct_dim0 / _gemm_rows_dim0   the
 *                         paper's dim = 0 partition (Eq. 2 first case; the
 *                         layout of its experiments): subspaces along
 *                         the OUTPUT axis, T_index [N_ss = F_out/d][F_in].
 *   fasq_ref_reconstruct  the naive reconstruction: W_hat[j][ss*d+e]
 *                         = T_cluster[cb(ss)][T_index[ss][j]][e].
 *   fasq_ref_gemm_rows    y[b][j] = sum_ss sum_e fp64(W_hat[j][ss*d+e]) *
 *                         fp64(x[b][ss*d+e]) -- reconstruct-then-multiply in
 *                         fp64 (the plain definition that Eq. 3, P:200-203,
 *                         reaches exactly), ascending (ss, e) summation order.
 *   fasq_ref_f32_to_f16 / fasq_ref_f16_to_f32   IEEE binary16 conversions.
 *   fasq_ref_splitmix64_next                     the PRNG of the init step.
 *
 * Precision contract: every pack step is integer arithmetic or a fixed sequence
 * of IEEE-754 round-to-nearest basic operations.  This file MUST be compiled
 * with -ffp-contract=off and without -ffast-math (oracle/build.py does this) so
 * that a*b+c is never fused.
 *
 * Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".  Every
 * function here is pinned; none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Status codes (same numeric meaning as the product ABI, declared here
 * independently; nothing is shared). */
#define REF_OK 0
#define REF_E_ARG (-1)
#define REF_E_NONDIVISIBLE (-2)
#define REF_E_CLUSTER_OVERFLOW (-3)
#define REF_E_NONFINITE (-4)
#define REF_E_UNSUPPORTED (-6)
#define REF_E_OOM (-8)

/* ------------------------------------------------------------------------ */
/* IEEE binary16 <-> binary32                                                */
/* ------------------------------------------------------------------------ */

/* binary16 -> binary32, exact (every binary16 value is a binary32 value). */
float fasq_ref_f16_to_f32(uint16_t h) {
    uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    uint32_t exp = ((uint32_t)h >> 10) & 0x1fu;
    uint32_t man = (uint32_t)h & 0x3ffu;
    uint32_t bits;
    if (exp == 0x1fu) {                 /* inf / nan */
        bits = sign | 0x7f800000u | (man << 13);
    } else if (exp != 0) {              /* normal */
        bits = sign | ((exp - 15u + 127u) << 23) | (man << 13);
    } else if (man == 0) {              /* +-0 */
        bits = sign;
    } else {                            /* subnormal: man * 2^-24, exact */
        float v = (float)man * 0x1p-24f; /* man < 2^10, product exact */
        memcpy(&bits, &v, 4);
        bits |= sign;
    }
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

/* binary32 -> binary16 with roundTiesToEven, including subnormals and
 * overflow to infinity.  NaN maps to a quiet NaN with the same sign. */
uint16_t fasq_ref_f32_to_f16(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t ax = x & 0x7fffffffu;
    if (ax > 0x7f800000u) return (uint16_t)(sign | 0x7e00u);  /* NaN */
    if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u); /* >= 65520 -> inf */
    if (ax >= 0x38800000u) {            /* result is a normal binary16 */
        uint32_t e = (ax >> 23) - 127u + 15u;
        uint32_t m = ax & 0x7fffffu;
        uint32_t h = (e << 10) | (m >> 13);
        uint32_t rem = m & 0x1fffu;
        if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h += 1u; /* may carry into exp: fine */
        return (uint16_t)(sign | h);
    }
    if (ax <= 0x33000000u) return (uint16_t)sign; /* |f| <= 2^-25: rounds to 0 (tie -> even 0) */
    /* subnormal result: round(|f| / 2^-24) to nearest even */
    uint32_t m = (ax & 0x7fffffu) | 0x800000u;   /* 24-bit significand */
    int e = (int)(ax >> 23) - 127;               /* -25 < e < -14 */
    int shift = -(e + 1);                        /* 14..24; value = m * 2^(e-23) = (m >> shift) units of 2^-24 */
    uint32_t h = m >> shift;
    uint32_t rem = m & ((1u << shift) - 1u);
    uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1u))) h += 1u;
    return (uint16_t)(sign | h);
}

void fasq_ref_f32_to_f16_array(const float* in, uint16_t* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = fasq_ref_f32_to_f16(in[i]);
}
void fasq_ref_f16_to_f32_array(const uint16_t* in, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = fasq_ref_f16_to_f32(in[i]);
}

/* ------------------------------------------------------------------------ */
/* splitmix64 (reading R3: the seeded init's PRNG)                 */
/* ------------------------------------------------------------------------ */
uint64_t fasq_ref_splitmix64_next(uint64_t* state) {
    *state += 0x9E3779B97F4A7C15ull;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------------ */
/* (a1) partition and validate -- Eq. 2, SPEC plan_config        */
/* ------------------------------------------------------------------------ */
/* cmax: 256 for uint8 indices (the kernels' "1 B index"), 1024 for the
 * uint16 entry points (Eq. 4: ceil(log2 K_s)-bit indices; Table 2's
 * 2-512 / 2-1024 design points, P:479-488 -- NEXT-2). */
static int validate_c(int64_t F_out, int64_t F_in, int32_t d, int32_t C, int32_t group, int32_t cmax) {
    if (F_out < 1 || F_in < 1 || d < 1 || C < 1 || group < 1) return REF_E_ARG;
    if (d != 1 && d != 2 && d != 4 && d != 8) return REF_E_UNSUPPORTED;
    if (C > cmax) return REF_E_UNSUPPORTED;
    if (F_in % d != 0) return REF_E_NONDIVISIBLE;
    int64_t N_ss = F_in / d;
    if (N_ss % group != 0) return REF_E_NONDIVISIBLE;
    int64_t n_pts = (int64_t)group * F_out;
    if ((int64_t)C > n_pts) return REF_E_CLUSTER_OVERFLOW;
    if (n_pts > (1ll << 23)) return REF_E_UNSUPPORTED;    /* int64 exact-sum bound, R5 */
    return REF_OK;
}
int fasq_ref_validate(int64_t F_out, int64_t F_in, int32_t d, int32_t C, int32_t group) {
    return validate_c(F_out, F_in, d, C, group, 256);
}
int fasq_ref_validate16(int64_t F_out, int64_t F_in, int32_t d, int32_t C, int32_t group) {
    return validate_c(F_out, F_in, d, C, group, 1024);
}

/* Eq. 4: bits of one index = ceil(log2 K_s), the smallest b with
 * 2^b >= K_s (0 for K_s = 1). */
int32_t fasq_ref_index_bits(int32_t C) {
    int32_t b = 0;
    while (((int64_t)1 << b) < (int64_t)C) ++b;
    return b;
}

/* ------------------------------------------------------------------------ */
/* Pack, one codebook (Alg. 1 body "(C, I) <- KMeans(W_ss, K_s)")     */
/* ------------------------------------------------------------------------ */

/* A point is d binary16 bit patterns with -0 mapped to +0 (reading R2). */
static uint16_t canon(uint16_t h) { return h == 0x8000u ? (uint16_t)0 : h; }

/* Lexicographic order of d-tuples of uint16, element 0 most significant. */
static int cmp_tuple(const uint16_t* a, const uint16_t* b, int d) {
    for (int e = 0; e < d; ++e) {
        if (a[e] < b[e]) return -1;
        if (a[e] > b[e]) return 1;
    }
    return 0;
}

/* Plain top-down merge sort of point ids by their key (qsort has no context
 * argument in C11). */
static void merge_sort_rows(const uint16_t* pts, int d, int64_t* idx, int64_t* tmp, int64_t n) {
    if (n < 2) return;
    int64_t h = n / 2;
    merge_sort_rows(pts, d, idx, tmp, h);
    merge_sort_rows(pts, d, idx + h, tmp, n - h);
    int64_t i = 0, j = h, k = 0;
    while (i < h && j < n) {
        if (cmp_tuple(pts + idx[j] * d, pts + idx[i] * d, d) < 0) tmp[k++] = idx[j++];
        else tmp[k++] = idx[i++];
    }
    while (i < h) tmp[k++] = idx[i++];
    while (j < n) tmp[k++] = idx[j++];
    memcpy(idx, tmp, (size_t)n * sizeof(int64_t));
}

/* Assign step: a_t = argmin_k D(p_t, c_k), D = sum_e (p_e - c_ke)^2 evaluated
 * left to right with separately rounded fp32 subtract, multiply and add;
 * strict '<' over ascending k so ties go to the lowest k (reading R7). */
static int32_t nearest_d(const float* p, const float* cent, int C, int d, float* bestD_out) {
    int32_t best = 0;
    float bestD = 0.0f;
    for (int k = 0; k < C; ++k) {
        float D = 0.0f;
        for (int e = 0; e < d; ++e) {
            float delta = p[e] - cent[(size_t)k * d + e];
            float sq = delta * delta;
            D = (e == 0) ? sq : D + sq;
        }
        if (k == 0 || D < bestD) { bestD = D; best = k; }
    }
    if (bestD_out) *bestD_out = bestD;
    return best;
}
static int32_t nearest(const float* p, const float* cent, int C, int d) { return nearest_d(p, cent, C, d, NULL); }

/* k-means++ initialisation (NEXT-4, reading R17) in
 * exact integer arithmetic so that any implementation reproduces it bit for
 * bit: coordinates q = fp16 value * 2^24 (exact int64), D2(t, u) = sum_e
 * (q_te - q_ue)^2 as an unsigned 128-bit integer.  The first centre is point
 * next() % n; then, while centres are missing, r = (next() << 64 | next()) mod
 * total with total = sum_t dist(t) (dist = D2 to the nearest chosen centre),
 * and the next centre is the smallest t whose inclusive prefix sum of dist
 * exceeds r (D^2 sampling).  total == 0 (every distinct point is a centre):
 * the remaining slots copy centre 0 (as reading R3's slots >= m).  The
 * splitmix64 state is seeded exactly as R3's.  chosen[k] = point id. */
typedef unsigned __int128 u128;
static u128 d2_int(const int64_t* q, int64_t t, int64_t u, int d) {
    u128 s = 0;
    for (int e = 0; e < d; ++e) {
        __int128 df = (__int128)q[t * d + e] - (__int128)q[u * d + e];
        s += (u128)(df * df);
    }
    return s;
}
static int kmeanspp(const uint16_t* pts, int64_t n, int d, int C, uint64_t seed, int64_t g, int64_t* chosen) {
    int64_t* q = (int64_t*)malloc((size_t)n * d * sizeof(int64_t));
    u128* dist = (u128*)malloc((size_t)n * sizeof(u128));
    if (!q || !dist) { free(q); free(dist); return -1; }
    for (int64_t t = 0; t < n * d; ++t) q[t] = (int64_t)((double)fasq_ref_f16_to_f32(pts[t]) * 16777216.0);
    uint64_t st = seed ^ ((uint64_t)(g + 1) * 0x9E3779B97F4A7C15ull);
    chosen[0] = (int64_t)(fasq_ref_splitmix64_next(&st) % (uint64_t)n);
    for (int64_t t = 0; t < n; ++t) dist[t] = d2_int(q, t, chosen[0], d);
    int k = 1;
    for (; k < C; ++k) {
        u128 total = 0;
        for (int64_t t = 0; t < n; ++t) total += dist[t];
        if (total == 0) break;
        u128 hi = fasq_ref_splitmix64_next(&st);
        u128 lo = fasq_ref_splitmix64_next(&st);
        u128 r = ((hi << 64) | lo) % total;
        u128 acc = 0;
        int64_t pick = n - 1;
        for (int64_t t = 0; t < n; ++t) {
            acc += dist[t];
            if (acc > r) { pick = t; break; }
        }
        chosen[k] = pick;
        for (int64_t t = 0; t < n; ++t) {
            u128 dd = d2_int(q, t, pick, d);
            if (dd < dist[t]) dist[t] = dd;
        }
    }
    for (; k < C; ++k) chosen[k] = chosen[0];
    free(q); free(dist);
    return 0;
}

/* Runs init + Lloyd for one codebook.  pts: n x d canonical fp16 bits.
 * cent (out): C x d fp32 centroids after the loop.  assign (out): the
 * assignment of the last assign pass.  Returns the number of assign passes
 * executed (0..iters), or <0 on allocation failure. */
static int lloyd_one(const uint16_t* pts, int64_t n, int d, int C, uint64_t seed, int64_t g,
                     int iters, float* cent, int32_t* assign, int init_mode, int empty_mode) {
    /* step 3: keys = the d fp16 patterns; U = sorted unique keys */
    int64_t* order = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t* tmp = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    float* pf = (float*)malloc((size_t)n * d * sizeof(float));
    int32_t* prev = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int64_t* S = (int64_t*)malloc((size_t)C * d * sizeof(int64_t));
    int64_t* cnt = (int64_t*)malloc((size_t)C * sizeof(int64_t));
    if (!order || !tmp || !pf || !prev || !S || !cnt) {
        free(order); free(tmp); free(pf); free(prev); free(S); free(cnt);
        return -1;
    }
    for (int64_t t = 0; t < n; ++t) order[t] = t;
    merge_sort_rows(pts, d, order, tmp, n);
    int64_t nU = 0; /* compact unique rows into order[0..nU) (each a representative point id) */
    for (int64_t t = 0; t < n; ++t) {
        if (nU == 0 || cmp_tuple(pts + order[t] * d, pts + order[nU - 1] * d, d) != 0)
            order[nU++] = order[t];
    }
    if (init_mode == 1) {
        /* k-means++ (reading R17) */
        if (kmeanspp(pts, n, d, C, seed, g, order) != 0) {
            free(order); free(tmp); free(pf); free(prev); free(S); free(cnt);
            return -1;
        }
        for (int k = 0; k < C; ++k)
            for (int e = 0; e < d; ++e) cent[(size_t)k * d + e] = fasq_ref_f16_to_f32(pts[order[k] * d + e]);
    } else {
    /* step 4: seeded partial Fisher-Yates over U, m = min(C, |U|) */
    int64_t m = (int64_t)C < nU ? (int64_t)C : nU;
    uint64_t st = seed ^ ((uint64_t)(g + 1) * 0x9E3779B97F4A7C15ull);
    for (int64_t i = 0; i < m; ++i) {
        uint64_t r = fasq_ref_splitmix64_next(&st);
        int64_t j = i + (int64_t)(r % (uint64_t)(nU - i));
        int64_t sw = order[i]; order[i] = order[j]; order[j] = sw;
    }
    for (int k = 0; k < C; ++k) {
        int64_t src = order[k < m ? k : 0];
        for (int e = 0; e < d; ++e) cent[(size_t)k * d + e] = fasq_ref_f16_to_f32(pts[src * d + e]);
    }
    }
    for (int64_t t = 0; t < n * d; ++t) pf[t] = fasq_ref_f16_to_f32(pts[t]);

    /* step 5: Lloyd */
    float* bestD = empty_mode == 1 ? (float*)malloc((size_t)(n > 0 ? n : 1) * sizeof(float)) : NULL;
    int64_t* taken = empty_mode == 1 ? (int64_t*)malloc((size_t)C * sizeof(int64_t)) : NULL;
    if (empty_mode == 1 && (!bestD || !taken)) {
        free(bestD); free(taken); free(order); free(tmp); free(pf); free(prev); free(S); free(cnt);
        return -1;
    }
    int ran = 0;
    for (int it = 1; it <= iters; ++it) {
        int changed = 0;
        for (int64_t t = 0; t < n; ++t) {
            int32_t a = nearest_d(pf + t * d, cent, C, d, bestD ? bestD + t : NULL);
            if (it > 1 && a != prev[t]) changed = 1;
            assign[t] = a;
        }
        ran = it;
        if (it > 1 && !changed) break;     /* assignments unchanged: fixed point */
        memcpy(prev, assign, (size_t)n * sizeof(int32_t));
        /* update: exact int64 fixed-point sums in units of 2^-24, one fp64 divide */
        memset(S, 0, (size_t)C * d * sizeof(int64_t));
        memset(cnt, 0, (size_t)C * sizeof(int64_t));
        for (int64_t t = 0; t < n; ++t) {
            int32_t a = assign[t];
            cnt[a] += 1;
            for (int e = 0; e < d; ++e)
                S[(size_t)a * d + e] += (int64_t)((double)pf[t * d + e] * 16777216.0);
        }
        if (empty_mode == 1) {
            /* reseed (reading R18): empty clusters, ascending k, take the
             * points farthest from their assigned centroid (this iteration's fp32
             * assignment distance), ties -> lowest t, each point at most once */
            int64_t ntaken = 0;
            for (int k = 0; k < C; ++k) {
                if (cnt[k] != 0) continue;
                int64_t best = -1;
                for (int64_t t = 0; t < n; ++t) {
                    int used = 0;
                    for (int64_t q2 = 0; q2 < ntaken; ++q2) used |= taken[q2] == t;
                    if (used) continue;
                    if (best < 0 || bestD[t] > bestD[best]) best = t;
                }
                if (best < 0) continue;
                taken[ntaken++] = best;
                for (int e = 0; e < d; ++e) cent[(size_t)k * d + e] = pf[best * d + e];
            }
        }
        for (int k = 0; k < C; ++k) {
            if (cnt[k] == 0) continue;       /* empty cluster: kept (R5) or reseeded above (R18) */
            for (int e = 0; e < d; ++e) {
                double mean = (double)S[(size_t)k * d + e] / (double)cnt[k];
                cent[(size_t)k * d + e] = (float)(mean * (1.0 / 16777216.0));
            }
        }
    }
    free(bestD); free(taken);
    free(order); free(tmp); free(pf); free(prev); free(S); free(cnt);
    return ran;
}

/* Gathers the points of codebook g (reading R1: point t = (ss - g*group)*F_out + j
 * is W[j, ss*d : ss*d+d]) into pts (n x d), canonicalising -0. */
static void gather_points(const uint16_t* W, int64_t F_out, int64_t F_in, int d, int group,
                          int64_t g, uint16_t* pts) {
    for (int64_t s = 0; s < group; ++s) {
        int64_t ss = g * group + s;
        for (int64_t j = 0; j < F_out; ++j) {
            int64_t t = s * F_out + j;
            for (int e = 0; e < d; ++e) pts[t * d + e] = canon(W[j * F_in + ss * d + e]);
        }
    }
}

/* Packs codebooks [g0, g1) of W (fp16 bits, [F_out][F_in] row major).
 * codebooks: [N_cb][C][d] fp16 bits (only rows g0..g1-1 written);
 * indices:   [N_ss][F_out] uint8 (only subspaces of codebooks g0..g1-1 written);
 * iters_run: optional [N_cb] number of assign passes executed.
 * Deterministic for any OpenMP thread count (codebooks are independent). */
/* idx8 (C <= 256) or idx16 (C <= 1024, NEXT-2): exactly one is non-NULL; the
 * arithmetic is the same for both, only the stored index width differs. */
static int pack_range_impl(const uint16_t* W, int64_t F_out, int64_t F_in, int32_t d, int32_t C,
                           int32_t group, uint64_t seed, int32_t iters, int32_t init_mode, int32_t empty_mode,
                           int64_t g0, int64_t g1, uint16_t* codebooks, uint8_t* idx8, uint16_t* idx16,
                           int32_t* iters_run) {
    if (init_mode < 0 || init_mode > 1 || empty_mode < 0 || empty_mode > 1) return REF_E_ARG;
    int st = validate_c(F_out, F_in, d, C, group, idx16 ? 1024 : 256);
    if (st != REF_OK) return st;
    if (iters < 0) return REF_E_ARG;
    int64_t N_ss = F_in / d, N_cb = N_ss / group;
    if (g0 < 0 || g1 > N_cb || g0 > g1) return REF_E_ARG;
    for (int64_t i = 0; i < F_out * F_in; ++i) {
        uint16_t h = W[i];
        if ((h & 0x7c00u) == 0x7c00u) return REF_E_NONFINITE;   /* inf / nan */
    }
    int64_t n = (int64_t)group * F_out;
    int fail = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t g = g0; g < g1; ++g) {
        uint16_t* pts = (uint16_t*)malloc((size_t)n * d * sizeof(uint16_t));
        float* cent = (float*)malloc((size_t)C * d * sizeof(float));
        float* centh = (float*)malloc((size_t)C * d * sizeof(float));
        int32_t* asg = (int32_t*)malloc((size_t)n * sizeof(int32_t));
        float* pf = (float*)malloc((size_t)d * sizeof(float));
        if (!pts || !cent || !centh || !asg || !pf) {
#pragma omp atomic write
            fail = 1;
        } else {
            gather_points(W, F_out, F_in, d, group, g, pts);
            int ran = lloyd_one(pts, n, d, C, seed, g, iters, cent, asg, init_mode, empty_mode);
            if (ran < 0) {
#pragma omp atomic write
                fail = 1;
            } else {
                if (iters_run) iters_run[g] = ran;
                /* step 6: finalize -- c_hat = fp16_rn(c) (-0 -> +0), then one more
                 * assign against fp32(c_hat) */
                for (int64_t q = 0; q < (int64_t)C * d; ++q) {
                    uint16_t h = canon(fasq_ref_f32_to_f16(cent[q]));
                    codebooks[g * C * d + q] = h;
                    centh[q] = fasq_ref_f16_to_f32(h);
                }
                for (int64_t s = 0; s < group; ++s) {
                    int64_t ss = g * group + s;
                    for (int64_t j = 0; j < F_out; ++j) {
                        int64_t t = s * F_out + j;
                        for (int e = 0; e < d; ++e) pf[e] = fasq_ref_f16_to_f32(pts[t * d + e]);
                        const int32_t a = nearest(pf, centh, C, d);
                        if (idx16) idx16[ss * F_out + j] = (uint16_t)a;
                        else idx8[ss * F_out + j] = (uint8_t)a;
                    }
                }
            }
        }
        free(pts); free(cent); free(centh); free(asg); free(pf);
    }
    return fail ? REF_E_OOM : REF_OK;
}

int fasq_ref_pack_range_ex(const uint16_t* W, int64_t F_out, int64_t F_in, int32_t d, int32_t C,
                           int32_t group, uint64_t seed, int32_t iters, int32_t init_mode, int32_t empty_mode,
                           int64_t g0, int64_t g1, uint16_t* codebooks, uint8_t* indices, int32_t* iters_run) {
    if (!indices) return REF_E_ARG;
    return pack_range_impl(W, F_out, F_in, d, C, group, seed, iters, init_mode, empty_mode, g0, g1, codebooks,
                           indices, NULL, iters_run);
}

/* The same with uint16 indices, C <= 1024 (NEXT-2: Eq. 4's ceil(log2 K_s)-bit
 * indices for K_s = 512 / 1024, Table 2). */
int fasq_ref_pack16_range_ex(const uint16_t* W, int64_t F_out, int64_t F_in, int32_t d, int32_t C,
                             int32_t group, uint64_t seed, int32_t iters, int32_t init_mode, int32_t empty_mode,
                             int64_t g0, int64_t g1, uint16_t* codebooks, uint16_t* indices, int32_t* iters_run) {
    if (!indices) return REF_E_ARG;
    return pack_range_impl(W, F_out, F_in, d, C, group, seed, iters, init_mode, empty_mode, g0, g1, codebooks,
                           NULL, indices, iters_run);
}

int fasq_ref_pack_range(const uint16_t* W, int64_t F_out, int64_t F_in, int32_t d, int32_t C,
                        int32_t group, uint64_t seed, int32_t iters, int64_t g0, int64_t g1,
                        uint16_t* codebooks, uint8_t* indices, int32_t* iters_run) {
    return fasq_ref_pack_range_ex(W, F_out, F_in, d, C, group, seed, iters, 0, 0, g0, g1, codebooks, indices,
                                  iters_run);
}

int fasq_ref_pack(const uint16_t* W, int64_t F_out, int64_t F_in, int32_t d, int32_t C,
                  int32_t group, uint64_t seed, int32_t iters, uint16_t* codebooks,
                  uint8_t* indices, int32_t* iters_run) {
    int st = fasq_ref_validate(F_out, F_in, d, C, group);
    if (st != REF_OK) return st;
    int64_t N_cb = (F_in / d) / group;
    return fasq_ref_pack_range(W, F_out, F_in, d, C, group, seed, iters, 0, N_cb, codebooks,
                               indices, iters_run);
}

/* ------------------------------------------------------------------------ */
/* dim = 0: subspaces along the OUTPUT axis (Eq. 2 first case;   */
/* the layout of the paper's experiments, P:444 -- NEXT-4)                  */
/* ------------------------------------------------------------------------ */
/* W in R^{F_out x F_in}; subspace ss = output rows [ss*d, ss*d + d), N_ss =
 * F_out/d; the datapoints are the F_in columns: point (ss, j) = (W[ss*d+0][j],
 * ..., W[ss*d+d-1][j]); T_index is [N_ss][F_in].  This is exactly the dim = 1
 * partition of W^T (its rows are W's columns), so the pack runs Alg. 1 on
 * the transposed matrix with the same arithmetic: point t = s*F_in + j of
 * codebook g is W^T[j, ss*d : ss*d+d] = W[ss*d : ss*d+d, j]. */
int fasq_ref_pack_dim0_range(const uint16_t* W, int64_t F_out, int64_t F_in, int32_t d, int32_t C,
                             int32_t group, uint64_t seed, int32_t iters, int32_t init_mode, int32_t empty_mode,
                             int64_t g0, int64_t g1, uint16_t* codebooks, uint8_t* indices, int32_t* iters_run) {
    if (!W || !indices || F_out < 1 || F_in < 1) return REF_E_ARG;
    uint16_t* WT = (uint16_t*)malloc((size_t)F_out * F_in * sizeof(uint16_t));
    if (!WT) return REF_E_OOM;
    for (int64_t o = 0; o < F_out; ++o)
        for (int64_t j = 0; j < F_in; ++j) WT[j * F_out + o] = W[o * F_in + j];
    int st = pack_range_impl(WT, F_in, F_out, d, C, group, seed, iters, init_mode, empty_mode, g0, g1, codebooks,
                             indices, NULL, iters_run);
    free(WT);
    return st;
}

/* W_hat[ss*d+e][j] = codebooks[ss/group][indices[ss][j]][e]  (fp16 bits), dim = 0 */
int fasq_ref_reconstruct_dim0(const uint16_t* codebooks, const uint8_t* indices, int64_t F_out, int64_t F_in,
                              int32_t d, int32_t C, int32_t group, uint16_t* W_hat) {
    if (F_out < 1 || F_in < 1 || d < 1 || C < 1 || group < 1) return REF_E_ARG;
    if (F_out % d) return REF_E_NONDIVISIBLE;
    int64_t N_ss = F_out / d;
    if (N_ss % group) return REF_E_NONDIVISIBLE;
    for (int64_t ss = 0; ss < N_ss; ++ss)
        for (int64_t j = 0; j < F_in; ++j) {
            int64_t k = indices[ss * F_in + j];
            if (k >= C) return REF_E_ARG;
            for (int e = 0; e < d; ++e)
                W_hat[(ss * d + e) * F_in + j] = codebooks[((ss / group) * C + k) * d + e];
        }
    return REF_OK;
}

/* Y[b][r] = sum over i ascending of fp64(W_hat[j0+r][i]) * fp64(X[b][i]) with
 * W_hat the dim = 0 reconstruction: the plain definition y = W_hat . x. */
int fasq_ref_gemm_rows_dim0(const uint16_t* codebooks, const uint8_t* indices, int64_t F_out, int64_t F_in,
                            int32_t d, int32_t C, int32_t group, const uint16_t* X, int64_t M, int64_t j0,
                            int64_t j1, double* Y) {
    if (F_out < 1 || F_in < 1 || d < 1 || C < 1 || group < 1 || M < 0) return REF_E_ARG;
    if (F_out % d) return REF_E_NONDIVISIBLE;
    if ((F_out / d) % group) return REF_E_NONDIVISIBLE;
    if (j0 < 0 || j1 > F_out || j0 > j1) return REF_E_ARG;
    int64_t R = j1 - j0;
    double* Wr = (double*)malloc((size_t)(R > 0 ? R : 1) * F_in * sizeof(double));
    double* Xd = (double*)malloc((size_t)(M > 0 ? M : 1) * F_in * sizeof(double));
    if (!Wr || !Xd) { free(Wr); free(Xd); return REF_E_OOM; }
    int bad = 0;
    for (int64_t r = 0; r < R; ++r) {
        const int64_t o = j0 + r, ss = o / d, e = o % d;
        for (int64_t i = 0; i < F_in; ++i) {
            int64_t k = indices[ss * F_in + i];
            if (k >= C) { bad = 1; k = 0; }
            Wr[r * F_in + i] = (double)fasq_ref_f16_to_f32(codebooks[((ss / group) * C + k) * d + e]);
        }
    }
    for (int64_t q = 0; q < M * F_in; ++q) Xd[q] = (double)fasq_ref_f16_to_f32(X[q]);
    if (bad) { free(Wr); free(Xd); return REF_E_ARG; }
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t b = 0; b < M; ++b)
        for (int64_t r = 0; r < R; ++r) {
            double acc = 0.0;
            for (int64_t i = 0; i < F_in; ++i) acc = acc + Wr[r * F_in + i] * Xd[b * F_in + i];
            Y[b * R + r] = acc;
        }
    free(Wr); free(Xd);
    return REF_OK;
}

/* Test hook: init + Lloyd for codebook g only, WITHOUT finalisation.
 * cent: [C][d] fp32; assign: [group*F_out].  Returns assign passes run. */
int fasq_ref_lloyd_fp32(const uint16_t* W, int64_t F_out, int64_t F_in, int32_t d, int32_t C,
                        int32_t group, uint64_t seed, int32_t iters, int64_t g, float* cent,
                        int32_t* assign) {
    int st = fasq_ref_validate16(F_out, F_in, d, C, group);   /* int32 assignment: any C <= 1024 */
    if (st != REF_OK) return st;
    int64_t n = (int64_t)group * F_out;
    uint16_t* pts = (uint16_t*)malloc((size_t)n * d * sizeof(uint16_t));
    if (!pts) return REF_E_OOM;
    gather_points(W, F_out, F_in, d, group, g, pts);
    int ran = lloyd_one(pts, n, d, C, seed, g, iters, cent, assign, 0, 0);
    free(pts);
    return ran < 0 ? REF_E_OOM : ran;
}

/* ------------------------------------------------------------------------ */
/* Product: reconstruct-then-multiply (P:195-196 naive path; Eq. 3) */
/* ------------------------------------------------------------------------ */

/* T_index[ss][j] from a uint8 (wide = 0) or uint16 (wide = 1) table */
static int64_t index_at(const void* indices, int wide, int64_t i) {
    return wide ? (int64_t)((const uint16_t*)indices)[i] : (int64_t)((const uint8_t*)indices)[i];
}

/* W_hat[j][ss*d+e] = codebooks[ss/group][indices[ss][j]][e]  (fp16 bits) */
static int reconstruct_impl(const uint16_t* codebooks, const void* indices, int wide, int64_t F_out,
                            int64_t F_in, int32_t d, int32_t C, int32_t group, uint16_t* W_hat) {
    if (F_out < 1 || F_in < 1 || d < 1 || C < 1 || group < 1) return REF_E_ARG;
    if (F_in % d) return REF_E_NONDIVISIBLE;
    int64_t N_ss = F_in / d;
    if (N_ss % group) return REF_E_NONDIVISIBLE;
    for (int64_t j = 0; j < F_out; ++j)
        for (int64_t ss = 0; ss < N_ss; ++ss) {
            int64_t k = index_at(indices, wide, ss * F_out + j);
            if (k >= C) return REF_E_ARG;
            for (int e = 0; e < d; ++e)
                W_hat[j * F_in + ss * d + e] = codebooks[((ss / group) * C + k) * d + e];
        }
    return REF_OK;
}
int fasq_ref_reconstruct(const uint16_t* codebooks, const uint8_t* indices, int64_t F_out,
                         int64_t F_in, int32_t d, int32_t C, int32_t group, uint16_t* W_hat) {
    return reconstruct_impl(codebooks, indices, 0, F_out, F_in, d, C, group, W_hat);
}
int fasq_ref_reconstruct16(const uint16_t* codebooks, const uint16_t* indices, int64_t F_out,
                           int64_t F_in, int32_t d, int32_t C, int32_t group, uint16_t* W_hat) {
    return reconstruct_impl(codebooks, indices, 1, F_out, F_in, d, C, group, W_hat);
}

/* Y[b][j - j0] = sum over (ss, e) ascending of fp64(W_hat[j][ss*d+e]) *
 * fp64(X[b][ss*d+e]) for rows j in [j0, j1) and b in [0, M).  fp16 x fp16
 * products are exact in fp64; only the running sum rounds.  Parallel over
 * (b, j) -- every output is computed independently in a fixed order. */
static int gemm_rows_impl(const uint16_t* codebooks, const void* indices, int wide, int64_t F_out,
                          int64_t F_in, int32_t d, int32_t C, int32_t group, const uint16_t* X,
                          int64_t M, int64_t j0, int64_t j1, double* Y) {
    if (F_out < 1 || F_in < 1 || d < 1 || C < 1 || group < 1 || M < 0) return REF_E_ARG;
    if (F_in % d) return REF_E_NONDIVISIBLE;
    int64_t N_ss = F_in / d;
    if (N_ss % group) return REF_E_NONDIVISIBLE;
    if (j0 < 0 || j1 > F_out || j0 > j1) return REF_E_ARG;
    int64_t R = j1 - j0;
    /* reconstruct the requested rows of W_hat (fp16 -> fp64, exact) */
    double* Wr = (double*)malloc((size_t)(R > 0 ? R : 1) * F_in * sizeof(double));
    double* Xd = (double*)malloc((size_t)(M > 0 ? M : 1) * F_in * sizeof(double));
    if (!Wr || !Xd) { free(Wr); free(Xd); return REF_E_OOM; }
    int bad = 0;
    for (int64_t r = 0; r < R; ++r)
        for (int64_t ss = 0; ss < N_ss; ++ss) {
            int64_t k = index_at(indices, wide, ss * F_out + (j0 + r));
            if (k >= C) bad = 1;
            for (int e = 0; e < d; ++e)
                Wr[r * F_in + ss * d + e] =
                    (double)fasq_ref_f16_to_f32(codebooks[((ss / group) * C + (k < C ? k : 0)) * d + e]);
        }
    for (int64_t q = 0; q < M * F_in; ++q) Xd[q] = (double)fasq_ref_f16_to_f32(X[q]);
    if (bad) { free(Wr); free(Xd); return REF_E_ARG; }
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t b = 0; b < M; ++b)
        for (int64_t r = 0; r < R; ++r) {
            double acc = 0.0;
            const double* w = Wr + r * F_in;
            const double* x = Xd + b * F_in;
            for (int64_t i = 0; i < F_in; ++i) acc = acc + w[i] * x[i];
            Y[b * R + r] = acc;
        }
    free(Wr); free(Xd);
    return REF_OK;
}
int fasq_ref_gemm_rows(const uint16_t* codebooks, const uint8_t* indices, int64_t F_out,
                       int64_t F_in, int32_t d, int32_t C, int32_t group, const uint16_t* X,
                       int64_t M, int64_t j0, int64_t j1, double* Y) {
    return gemm_rows_impl(codebooks, indices, 0, F_out, F_in, d, C, group, X, M, j0, j1, Y);
}
int fasq_ref_gemm_rows16(const uint16_t* codebooks, const uint16_t* indices, int64_t F_out,
                         int64_t F_in, int32_t d, int32_t C, int32_t group, const uint16_t* X,
                         int64_t M, int64_t j0, int64_t j1, double* Y) {
    return gemm_rows_impl(codebooks, indices, 1, F_out, F_in, d, C, group, X, M, j0, j1, Y);
}

int fasq_ref_gemm(const uint16_t* codebooks, const uint8_t* indices, int64_t F_out, int64_t F_in,
                  int32_t d, int32_t C, int32_t group, const uint16_t* X, int64_t M, double* Y) {
    return fasq_ref_gemm_rows(codebooks, indices, F_out, F_in, d, C, group, X, M, 0, F_out, Y);
}

int fasq_ref_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void fasq_ref_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
