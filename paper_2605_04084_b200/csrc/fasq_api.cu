// fasq_api.cu -- the extern "C" boundary of libfasq.so (include/fasq.h).
// Argument marshalling, validation, layer lifetime; all compute is in the
// kernels of layout.cu / gemv.cu / gemm_*.cu / pack.cu.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fasq_internal.cuh"

namespace fasq {

static thread_local std::string t_err;
static thread_local int t_launches = 0;

void set_error(const std::string& msg) { t_err = msg; }
fasq_status cuda_fail(cudaError_t e, const char* what) {
    t_err = std::string(what) + ": " + cudaGetErrorString(e);
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? FASQ_E_OOM : FASQ_E_CUDA;
}
void set_launch_count(int n) { t_launches = n; }
void add_launch_count(int n) { t_launches += n; }

static fasq_status check_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        set_error("no CUDA device available (FASQ has no CPU fallback)");
        return FASQ_E_CUDA;
    }
    return FASQ_OK;
}

static void destroy(fasq_layer* L) {
    if (!L) return;
    dev_free(L->idx, 0);
    dev_free(L->cbimg, 0);
    dev_free(L->cbmap, 0);
    dev_free(L->cb, 0);
    dev_free(L->cbimg_x, 0);
    dev_free(L->cbmap_x, 0);
    delete L;
}

}  // namespace fasq

using namespace fasq;

extern "C" {

int32_t fasq_abi_version(void) { return FASQ_ABI_VERSION; }

const char* fasq_status_string(fasq_status s) {
    switch (s) {
        case FASQ_OK: return "FASQ_OK";
        case FASQ_E_ARG: return "FASQ_E_ARG: invalid argument";
        case FASQ_E_NONDIVISIBLE: return "FASQ_E_NONDIVISIBLE: F_in % d or N_ss % group != 0";
        case FASQ_E_CLUSTER_OVERFLOW: return "FASQ_E_CLUSTER_OVERFLOW: C > points per codebook";
        case FASQ_E_NONFINITE: return "FASQ_E_NONFINITE: W holds inf/NaN";
        case FASQ_E_SHAPE: return "FASQ_E_SHAPE: operand shape mismatch";
        case FASQ_E_UNSUPPORTED: return "FASQ_E_UNSUPPORTED: parameter outside the supported range";
        case FASQ_E_CUDA: return "FASQ_E_CUDA: CUDA error";
        case FASQ_E_OOM: return "FASQ_E_OOM: device allocation failed";
        case FASQ_E_RANGE: return "FASQ_E_RANGE: a counted partial left its |v| < 2^18 range";
    }
    return "FASQ: unknown status";
}

const char* fasq_last_error_message(void) { return t_err.c_str(); }
int32_t fasq_last_launch_count(void) { return t_launches; }

fasq_status fasq_import_ex(const void* codebooks_dev, const void* indices_dev, int64_t F_out, int64_t F_in,
                           int32_t d, int32_t C, int32_t group, uint32_t layout, void* stream, fasq_layer** out) {
    if (!out) return FASQ_E_ARG;
    *out = nullptr;
    if (!codebooks_dev || !indices_dev) return FASQ_E_ARG;
    fasq_layer* L = new fasq_layer();
    fasq_status s = init_layer_shape(L, F_out, F_in, d, C, group, layout);
    if (s == FASQ_OK) s = check_device();
    if (s == FASQ_OK) s = alloc_layer_storage(L, (cudaStream_t)stream);
    if (s == FASQ_OK)
        s = build_physical_from_logical(L, static_cast<const __half*>(codebooks_dev), indices_dev,
                                        (cudaStream_t)stream);
    if (s != FASQ_OK) { destroy(L); return s; }
    set_launch_count(2);
    *out = L;
    return FASQ_OK;
}

fasq_status fasq_import(const void* codebooks_dev, const void* indices_dev, int64_t F_out, int64_t F_in,
                        int32_t d, int32_t C, int32_t group, void* stream, fasq_layer** out) {
    return fasq_import_ex(codebooks_dev, indices_dev, F_out, F_in, d, C, group, C > 256 ? FASQ_LAYOUT_PACKED : 0u,
                          stream, out);
}

fasq_status fasq_pack(const void* W_dev, int64_t F_out, int64_t F_in, const fasq_pack_params* prm,
                      void* stream, fasq_layer** out) {
    if (!out) return FASQ_E_ARG;
    *out = nullptr;
    if (!W_dev || !prm) return FASQ_E_ARG;
    if (prm->iters < 0 || prm->init < 0 || prm->init > 1 || prm->empty < 0 || prm->empty > 1) return FASQ_E_ARG;
    fasq_layer* L = new fasq_layer();
    const uint32_t layout = prm->layout | (prm->C > 256 ? FASQ_LAYOUT_PACKED : 0u);
    fasq_status s = init_layer_shape(L, F_out, F_in, prm->d, prm->C, prm->group, layout);
    // points per codebook: group x (datapoints = F_out rows, or F_in columns for dim = 0)
    const int64_t n_dp = L->dim0 ? F_in : F_out;
    if (s == FASQ_OK && (int64_t)prm->C > (int64_t)prm->group * n_dp) s = FASQ_E_CLUSTER_OVERFLOW;
    if (s == FASQ_OK && (int64_t)prm->group * n_dp > (1ll << 23)) s = FASQ_E_UNSUPPORTED;
    if (s == FASQ_OK) s = check_device();
    cudaStream_t st = (cudaStream_t)stream;
    if (s == FASQ_OK) s = alloc_layer_storage(L, st);
    uint16_t* idx_log = nullptr;   // the packer writes uint16 indices for every C
    uint8_t* idx8 = nullptr;
    __half* WT = nullptr;
    const int64_t nidx = (int64_t)L->N_ss * n_dp;
    if (s == FASQ_OK) s = dev_alloc_t(&idx_log, (size_t)nidx * 2, st);
    if (s == FASQ_OK && L->dim0) {
        // dim = 0 (Eq. 2 first case) is the dim = 1 partition of W^T: pack the
        // transposed matrix with the same kernels (exactly as the oracle does)
        s = dev_alloc_t(&WT, (size_t)F_out * F_in * 2, st);
        if (s == FASQ_OK) s = transpose_f16(static_cast<const __half*>(W_dev), WT, F_out, F_in, st);
        fasq_layer T{};
        T.F_out = F_in;
        T.F_in = F_out;
        T.d = L->d;
        T.C = L->C;
        T.group = L->group;
        T.N_ss = L->N_ss;
        T.N_cb = L->N_cb;
        if (s == FASQ_OK) s = pack_run(WT, &T, prm, st, L->cb, idx_log);
    } else if (s == FASQ_OK) {
        s = pack_run(static_cast<const __half*>(W_dev), L, prm, st, L->cb, idx_log);
    }
    if (s == FASQ_OK && L->idx_w == 1) {
        s = dev_alloc_t(&idx8, (size_t)nidx, st);
        if (s == FASQ_OK) s = idx16_to_8(idx_log, idx8, nidx, st);
    }
    if (s == FASQ_OK)
        s = build_physical_from_logical(L, L->cb, L->idx_w == 1 ? static_cast<const void*>(idx8) : idx_log, st);
    dev_free(idx_log, st);
    dev_free(idx8, st);
    dev_free(WT, st);
    if (s != FASQ_OK) { cudaStreamSynchronize(st); destroy(L); return s; }
    *out = L;
    return FASQ_OK;
}

fasq_status fasq_export(const fasq_layer* L, void* codebooks_dev, void* indices_dev, void* stream) {
    if (!L) return FASQ_E_ARG;
    fasq_status s = export_logical(L, static_cast<__half*>(codebooks_dev), indices_dev, (cudaStream_t)stream);
    if (s == FASQ_OK) set_launch_count(indices_dev ? 1 : 0);
    return s;
}

fasq_status fasq_shard_rows(const fasq_layer* L, int32_t rank, int32_t world, void* stream, fasq_layer** out) {
    if (!out) return FASQ_E_ARG;
    *out = nullptr;
    if (!L || world < 1 || rank < 0 || rank >= world) return FASQ_E_ARG;
    if (L->F_out % world) return FASQ_E_SHAPE;
    if (L->dim0) { set_error("shard_rows: dim = 0 layers are not row-sharded"); return FASQ_E_UNSUPPORTED; }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = L->F_out / world, row0 = rows * rank;
    // via the logical form: export -> slice rows -> import (any row0; the
    // physical rotation depends on r mod 32)
    uint8_t* full = nullptr;
    uint8_t* part = nullptr;
    fasq_status s = FASQ_OK;
    const size_t w = (size_t)L->idx_w;   // logical index element bytes
    s = dev_alloc_t(&full, (size_t)L->N_ss * L->F_out * w, st);
    if (s == FASQ_OK) s = dev_alloc_t(&part, (size_t)L->N_ss * rows * w, st);
    if (s == FASQ_OK) s = export_logical(L, nullptr, full, st);
    if (s == FASQ_OK) {
        cudaError_t e = cudaMemcpy2DAsync(part, (size_t)rows * w, full + row0 * w, (size_t)L->F_out * w,
                                          (size_t)rows * w, (size_t)L->N_ss, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) s = cuda_fail(e, "shard copy");
    }
    fasq_layer* S = nullptr;
    if (s == FASQ_OK) {
        S = new fasq_layer();
        s = init_layer_shape(S, rows, L->F_in, L->d, L->C, L->group, layer_layout(L));
        if (s == FASQ_OK) s = alloc_layer_storage(S, st);
        if (s == FASQ_OK) s = build_physical_from_logical(S, L->cb, part, st);
        if (s == FASQ_OK) S->row_offset = L->row_offset + (int32_t)row0;
    }
    dev_free(full, st);
    dev_free(part, st);
    if (s != FASQ_OK) { cudaStreamSynchronize(st); destroy(S); return s; }
    *out = S;
    return FASQ_OK;
}

fasq_status fasq_layer_info_get(const fasq_layer* L, fasq_layer_info* info) {
    if (!L || !info) return FASQ_E_ARG;
    std::memset(info, 0, sizeof(*info));
    info->F_out = L->F_out;
    info->F_in = L->F_in;
    info->d = L->d;
    info->C = L->C;
    info->group = L->group;
    info->N_ss = L->N_ss;
    info->N_cb = L->N_cb;
    info->row_offset = L->row_offset;
    int lg = 0;
    while ((1 << lg) < L->C) ++lg;
    info->index_bits = L->bits ? L->bits : 8;
    info->layout = layer_layout(L);
    // Eq. 4's index table: index_bits per (subspace, datapoint), rounded up to bytes
    info->index_bytes = ((int64_t)L->N_ss * (L->dim0 ? L->F_in : L->F_out) * info->index_bits + 7) / 8;
    info->codebook_bytes = L->cb_bytes;
    info->device_bytes = L->idx_bytes + L->cbimg_bytes + L->cb_bytes + (L->cbimg_x ? L->cbimg_bytes : 0);
    info->bits_per_weight = 8.0 * (double)(info->index_bytes + info->codebook_bytes) / ((double)L->F_out * L->F_in);
    info->eff_bits_W = (double)lg / L->d;
    return FASQ_OK;
}

fasq_status fasq_layer_distinct_centroids(const fasq_layer* L, int64_t* distinct, void* stream) {
    if (!L || !distinct) return FASQ_E_ARG;
    return count_distinct_centroids(L, distinct, (cudaStream_t)stream);
}

void fasq_free(fasq_layer* L) {
    if (!L) return;
    cudaDeviceSynchronize();
    destroy(L);
}

fasq_status fasq_gemv_ex(const fasq_layer* L, const void* x_dev, int32_t B, void* y_dev, fasq_dtype yt,
                         uint32_t flags, void* stream) {
    if (!L || !x_dev || !y_dev) return FASQ_E_ARG;
    if (B < 1) return FASQ_E_ARG;
    if (yt != FASQ_F16 && yt != FASQ_F32) return FASQ_E_ARG;
    if (B > 8) {   // beyond the CUDA-core decode kernels (P:410 dispatch)
        // B <= 128: the tcgen05 decode kernel (weights as the UMMA M operand); else the prefill GEMM
        if (B <= 128 && B >= gemv_tc_min_batch() && gemv_tc_supported(L, B) && !(flags & ~FASQ_FLAG_PDL))
            return gemv_tc_launch(L, static_cast<const __half*>(x_dev), B, y_dev, yt, flags, (cudaStream_t)stream);
        if (flags) return FASQ_E_UNSUPPORTED;
        return fasq_gemm(L, x_dev, B, y_dev, yt, FASQ_GEMM_AUTO, stream);
    }
    return gemv_launch(L, static_cast<const __half*>(x_dev), B, y_dev, yt, flags, (cudaStream_t)stream);
}

fasq_status fasq_gemv_grouped(const fasq_layer* const* layers, int32_t n, const void* x_dev, int32_t B,
                              void* const* ys_dev, fasq_dtype yt, const fasq_gemv_opts* opts, void* stream) {
    if (!layers || !x_dev || !ys_dev || n < 1) return FASQ_E_ARG;
    if (n > 4) return FASQ_E_UNSUPPORTED;
    for (int i = 0; i < n; ++i)
        if (!layers[i] || !ys_dev[i]) return FASQ_E_ARG;
    if (B < 1 || B > 8) return FASQ_E_UNSUPPORTED;
    if (yt != FASQ_F16 && yt != FASQ_F32 && yt != FASQ_ACC_I64) return FASQ_E_ARG;
    bool special = false;
    for (int i = 0; i < n; ++i) special = special || layers[i]->bits || layers[i]->dim0;
    if (special) {   // NEXT-2 packed / NEXT-4 dim = 0: one layer per launch, fp16 x, no chain options
        if (n != 1 || (opts && (opts->flags & FASQ_FLAG_X_ACC || opts->n_next || opts->zero_dev)))
            return FASQ_E_UNSUPPORTED;
        const uint32_t fl = opts ? opts->flags : 0u;
        if (layers[0]->dim0)
            return gemv_dim0_launch(layers[0], static_cast<const __half*>(x_dev), B, ys_dev[0], yt, fl,
                                    (cudaStream_t)stream);
        return gemv_packed_launch(layers[0], static_cast<const __half*>(x_dev), B, ys_dev[0], yt, fl,
                                  (cudaStream_t)stream);
    }
    GemvOpts o{};
    if (opts) {
        if (opts->n_next < 0 || opts->n_next > 4 || opts->zero_bytes < 0 || (opts->zero_bytes & 7)) return FASQ_E_ARG;
        o.flags = opts->flags;
        o.next = opts->next_layers;
        o.n_next = opts->next_layers ? opts->n_next : 0;
        o.zero_ptr = opts->zero_dev;
        o.zero_bytes = opts->zero_dev ? opts->zero_bytes : 0;
    }
    o.x_acc = (o.flags & FASQ_FLAG_X_ACC) ? 1 : 0;
    o.y_acc = yt == FASQ_ACC_I64;
    return gemv_grouped_launch2(layers, n, x_dev, B, ys_dev, yt == FASQ_ACC_I64 ? FASQ_F32 : yt, o,
                                (cudaStream_t)stream);
}

fasq_status fasq_acc_convert(const void* acc_dev, int64_t n, void* out_dev, fasq_dtype out_dtype, void* stream) {
    if (!acc_dev || !out_dev || n < 0) return FASQ_E_ARG;
    if (out_dtype != FASQ_F16 && out_dtype != FASQ_F32) return FASQ_E_ARG;
    return acc_convert_launch(acc_dev, n, out_dev, out_dtype, (cudaStream_t)stream);
}

fasq_status fasq_gemv(const fasq_layer* L, const void* x_dev, int32_t B, void* y_dev, fasq_dtype yt,
                      void* stream) {
    return fasq_gemv_ex(L, x_dev, B, y_dev, yt, 0u, stream);
}

fasq_status fasq_gemv_host(const fasq_layer* L, const void* x_host, int32_t B, void* y_host, fasq_dtype yt,
                           void* stream) {
    if (!L || !x_host || !y_host) return FASQ_E_ARG;
    if (B < 1 || B > 8) return FASQ_E_UNSUPPORTED;
    if (yt != FASQ_F16 && yt != FASQ_F32) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t xb = (size_t)B * L->F_in * 2, yb = (size_t)B * L->F_out * (yt == FASQ_F32 ? 4 : 2);
    void *xd = nullptr, *yd = nullptr;
    if (dev_alloc(&xd, xb, st) != FASQ_OK || dev_alloc(&yd, yb, st) != FASQ_OK) {
        dev_free(xd, st);
        return FASQ_E_OOM;
    }
    fasq_status s = FASQ_OK;
    cudaError_t e = cudaMemcpyAsync(xd, x_host, xb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) s = cuda_fail(e, "H2D x");
    int launches = 0;
    if (s == FASQ_OK) {
        s = gemv_launch(L, static_cast<const __half*>(xd), B, yd, yt, 0u, st);
        launches = t_launches;
    }
    if (s == FASQ_OK) {
        e = cudaMemcpyAsync(y_host, yd, yb, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = cuda_fail(e, "D2H y");
    }
    dev_free(xd, st);
    dev_free(yd, st);
    e = cudaStreamSynchronize(st);
    if (s == FASQ_OK && e != cudaSuccess) s = cuda_fail(e, "gemv_host sync");
    if (s == FASQ_OK) set_launch_count(launches);
    return s;
}

// measured crossover against EXPAND (profiles/r02/short_gemm_sweep.jsonl): M <= 128 on the
// 4096-row layers, M <= 96 on the 14336-row ones (more row tiles: EXPAND fills the SMs)
static int64_t gemm_short_max(const fasq_layer* L) {
    const char* e = getenv("FASQ_GEMM_TC_DECODE_MAX");
    if (e) return atoll(e);
    // measured crossovers against EXPAND's split-K (profiles/r02/short_gemm_sweep_v3.jsonl):
    // 4096 x 14336 and 1024 x 4096 <= 64, 4096^2 <= 32, 14336 x 4096 <= 16
    if (L->F_in > 8192 || L->F_out <= 2048) return 64;
    if (L->F_out > 8192) return 16;
    return 32;
}

fasq_status fasq_gemm(const fasq_layer* L, const void* X_dev, int64_t M, void* Y_dev, fasq_dtype yt,
                      fasq_gemm_algo algo, void* stream) {
    if (!L || !X_dev || !Y_dev) return FASQ_E_ARG;
    if (M < 1) return FASQ_E_ARG;
    if (yt != FASQ_F16 && yt != FASQ_F32) return FASQ_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const __half* X = static_cast<const __half*>(X_dev);
    if (L->bits || L->dim0) {
        // NEXT-2 packed indices / NEXT-4 dim = 0: no tensor-core / LUT prefill
        // kernel reads these layouts; the product runs as their GEMVs over
        // 8-token slices (correct for any M, not a prefill-speed path)
        if (algo != FASQ_GEMM_AUTO) return FASQ_E_UNSUPPORTED;
        const size_t yb = yt == FASQ_F32 ? 4 : 2;
        int launches = 0;
        for (int64_t m0 = 0; m0 < M; m0 += 8) {
            const int b = (int)std::min<int64_t>(8, M - m0);
            fasq_status s = gemv_launch(L, X + m0 * L->F_in, b,
                                        static_cast<uint8_t*>(Y_dev) + (size_t)m0 * L->F_out * yb, yt, 0u, st);
            if (s != FASQ_OK) return s;
            launches += t_launches;
        }
        set_launch_count(launches);
        return FASQ_OK;
    }
    switch (algo) {
        case FASQ_GEMM_LUT: return gemm_lut_launch(L, X, M, Y_dev, yt, st);
        case FASQ_GEMM_EXPAND_TC:
            if (!gemm_tc_supported(L, M)) return FASQ_E_UNSUPPORTED;
            return gemm_tc_launch(L, X, M, Y_dev, yt, st);
        case FASQ_GEMM_AUTO:
            // short L (M <= gemm_short_max: 32-96 by shape, FASQ_GEMM_TC_DECODE_MAX): the
            // tcgen05 decode kernel (weights as UMMA M, tokens as N); above it EXPAND
            if (M <= gemm_short_max(L) && gemv_tc_supported(L, (int)M))
                return gemv_tc_launch(L, X, (int)M, Y_dev, yt, 0u, st);
            if (gemm_tc_supported(L, M)) return gemm_tc_launch(L, X, M, Y_dev, yt, st);
            return gemm_lut_launch(L, X, M, Y_dev, yt, st);
    }
    return FASQ_E_ARG;
}

fasq_status fasq_gemm_grouped(const fasq_layer* const* layers, int32_t n, const void* X_dev, int64_t M,
                              void* const* Y_dev, fasq_dtype yt, fasq_gemm_algo algo, void* stream) {
    if (!layers || !Y_dev || !X_dev || n < 1 || M < 1) return FASQ_E_ARG;
    if (yt != FASQ_F16 && yt != FASQ_F32) return FASQ_E_ARG;
    for (int l = 0; l < n; ++l) {
        if (!layers[l] || !Y_dev[l]) return FASQ_E_ARG;
        if (layers[l]->F_in != layers[0]->F_in) return FASQ_E_SHAPE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    // one EXPAND launch when every layer would run EXPAND on its own
    bool one = n > 1 && (algo == FASQ_GEMM_AUTO || algo == FASQ_GEMM_EXPAND_TC) && gemm_tc_groupable(layers, n, M);
    if (one && algo == FASQ_GEMM_AUTO)
        for (int l = 0; l < n; ++l)
            if (M <= gemm_short_max(layers[l]) && gemv_tc_supported(layers[l], (int)M)) one = false;
    if (one) return gemm_tc_launch_grouped(layers, n, static_cast<const __half*>(X_dev), M, Y_dev, yt, st);
    int launches = 0;
    for (int l = 0; l < n; ++l) {
        const fasq_status s = fasq_gemm(layers[l], X_dev, M, Y_dev[l], yt, algo, stream);
        if (s != FASQ_OK) return s;
        launches += fasq_last_launch_count();
    }
    set_launch_count(launches);
    return FASQ_OK;
}

}  // extern "C"
