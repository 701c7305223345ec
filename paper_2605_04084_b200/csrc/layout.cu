// layout.cu -- logical <-> physical layout transforms for FASQ layers (sm_100a).
//
// Logical (ABI) layout: codebooks fp16 [N_cb][C][d], indices u8 [N_ss][F_out]
// (Alg. 1 outputs T_cluster / T_index).  Physical layout: see
// fasq_internal.cuh and DESIGN.md "Data layout in HBM".
#include <mutex>

#include "fasq_internal.cuh"

namespace fasq {

uint32_t layer_layout(const fasq_layer* L) {
    return (L->bits ? FASQ_LAYOUT_PACKED : 0u) | (L->dim0 ? FASQ_LAYOUT_DIM0 : 0u);
}

fasq_status init_layer_shape(fasq_layer* L, int64_t F_out, int64_t F_in, int32_t d, int32_t C,
                             int32_t group, uint32_t layout) {
    if (F_out < 1 || F_in < 1 || d < 1 || C < 1 || group < 1) return FASQ_E_ARG;
    if (layout & ~(FASQ_LAYOUT_PACKED | FASQ_LAYOUT_DIM0)) return FASQ_E_ARG;
    if (d != 1 && d != 2 && d != 4 && d != 8) return FASQ_E_UNSUPPORTED;
    if (layout & FASQ_LAYOUT_DIM0) {
        // NEXT-4: dim = 0 (Eq. 2 first case): subspaces over the OUTPUT rows
        if (layout & FASQ_LAYOUT_PACKED) return FASQ_E_UNSUPPORTED;
        if (C > 256) return FASQ_E_UNSUPPORTED;
        if (F_out % d) return FASQ_E_NONDIVISIBLE;
        const int64_t N_ss = F_out / d;
        if (N_ss % group) return FASQ_E_NONDIVISIBLE;
        if (F_in > (1ll << 24) || N_ss > (1ll << 24)) return FASQ_E_UNSUPPORTED;
        L->F_out = F_out;
        L->F_in = F_in;
        L->d = d;
        L->C = C;
        L->group = group;
        L->N_ss = (int32_t)N_ss;
        L->N_cb = (int32_t)(N_ss / group);
        L->dim0 = 1;
        L->K_pad = (int32_t)((F_in + 63) / 64 * 64);
        L->F_out_pad = (int32_t)((F_out + kRowBlock - 1) / kRowBlock * kRowBlock);
        L->n_groups = (int32_t)((N_ss + kGroupSubs - 1) / kGroupSubs);
        L->E = entry_bytes(d);
        L->idx_w = 1;
        L->idx_bytes = (int64_t)L->n_groups * L->K_pad * kGroupSubs;
        L->cbimg_bytes = (int64_t)L->n_groups * C * kGroupSubs * L->E;
        L->cb_bytes = (int64_t)L->N_cb * C * d * 2;
        return FASQ_OK;
    }
    const int32_t packed = (layout & FASQ_LAYOUT_PACKED) ? 1 : 0;
    if (C > 1024 || (C > 256 && !packed)) return FASQ_E_UNSUPPORTED;
    // packed layers (NEXT-2): d = 2, the sub-vector size of every Table 2 point
    // (2-128 ... 2-1024); the GEMV stages one group's codebook image
    // (C x 32 x 4 B <= 128 KiB) per SMEM slot
    if (packed && (d != 2 || C < 2)) return FASQ_E_UNSUPPORTED;
    if (F_in % d) return FASQ_E_NONDIVISIBLE;
    int64_t N_ss = F_in / d;
    if (N_ss % group) return FASQ_E_NONDIVISIBLE;
    if (F_out > (1ll << 24) || N_ss > (1ll << 24)) return FASQ_E_UNSUPPORTED;
    L->F_out = F_out;
    L->F_in = F_in;
    L->d = d;
    L->C = C;
    L->group = group;
    L->N_ss = (int32_t)N_ss;
    L->N_cb = (int32_t)(N_ss / group);
    L->F_out_pad = (int32_t)((F_out + kRowBlock - 1) / kRowBlock * kRowBlock);
    L->n_groups = (int32_t)((N_ss + kGroupSubs - 1) / kGroupSubs);
    L->E = entry_bytes(d);
    L->idx_w = C > 256 ? 2 : 1;
    if (packed) {
        int b = 1;
        while ((1 << b) < C) ++b;   // ceil(log2 C), >= 1
        L->bits = b;
        L->seg = 8 * b;             // 64 codes x b bits
        L->idx_bytes = (int64_t)L->n_groups * (L->F_out_pad / kRowBlock) * kGroupSubs * L->seg;
    } else {
        L->idx_bytes = (int64_t)L->n_groups * L->F_out_pad * kGroupSubs;
    }
    L->cbimg_bytes = (int64_t)L->n_groups * C * kGroupSubs * L->E;
    L->cb_bytes = (int64_t)L->N_cb * C * d * 2;
    return FASQ_OK;
}

// Pair tensor map {32 words, n_groups, C} over a codebook image with strides
// {C*128, 128} B: a box {32, 2, C} at group g lands in SMEM as the codebook
// PAIR [C][g, g+1][32 words].
static fasq_status encode_pair_map(const uint8_t* img, const fasq_layer* L, void** map_out, cudaStream_t st) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return FASQ_E_CUDA; }
    CUtensorMap m;
    cuuint64_t gdim[3] = {32, (cuuint64_t)L->n_groups, (cuuint64_t)L->C};
    cuuint64_t gstr[2] = {(cuuint64_t)L->C * 128, 128};
    cuuint32_t box[3] = {32, 2, (cuuint32_t)L->C};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint8_t*>(img), gdim, gstr, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        set_error("codebook pair tensor map: encode failed");
        return FASQ_E_CUDA;
    }
    fasq_status s = dev_alloc(map_out, sizeof(CUtensorMap), st);
    if (s != FASQ_OK) return s;
    FASQ_CUDA_TRY(cudaMemcpyAsync(*map_out, &m, sizeof(m), cudaMemcpyHostToDevice, st));
    FASQ_CUDA_TRY(cudaStreamSynchronize(st));   // m is a host local
    return FASQ_OK;
}

fasq_status alloc_layer_storage(fasq_layer* L, cudaStream_t st) {
    FASQ_CUDA_TRY(cudaGetDevice(&L->device));
    // through the library allocator (alloc.cu), in stream order on the creation stream
    fasq_status s = dev_alloc_t(&L->idx, (size_t)L->idx_bytes, st);
    if (s == FASQ_OK) s = dev_alloc_t(&L->cbimg, (size_t)L->cbimg_bytes, st);
    if (s == FASQ_OK) s = dev_alloc_t(&L->cb, (size_t)L->cb_bytes, st);
    if (s != FASQ_OK) return s;
    if (L->E == 4 && L->bits == 0) {
        // codebook PAIR tensor map (the map only depends on the cbimg pointer and
        // shape, so it is encoded now and stays valid for the layer's lifetime)
        s = encode_pair_map(L->cbimg, L, &L->cbmap, st);
        if (s != FASQ_OK) return s;
    }
    return FASQ_OK;
}

// One thread per (group g, 16-row chunk, subspace s): 16 output bytes.
__global__ void k_idx_logical_to_phys(const uint8_t* __restrict__ idx_log, uint8_t* __restrict__ phys,
                                      int F_out, int F_out_pad, int N_ss, int n_groups) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n_chunks = (int64_t)F_out_pad / 16;
    if (t >= (int64_t)n_groups * n_chunks * kGroupSubs) return;
    const int s = (int)(t % kGroupSubs);
    const int64_t ch = (t / kGroupSubs) % n_chunks;
    const int64_t g = t / (kGroupSubs * n_chunks);
    const int64_t ss = g * kGroupSubs + s;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    for (int j = 0; j < 16; ++j) {
        const int64_t r = ch * 16 + j;
        const uint32_t v = (ss < N_ss && r < F_out) ? idx_log[ss * F_out + r] : 0u;
        w[j >> 2] |= v << (8 * (j & 3));
    }
    *reinterpret_cast<uint4*>(phys + idx_offset(g, ch * 16, s, F_out_pad)) = make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void k_idx_phys_to_logical(const uint8_t* __restrict__ phys, uint8_t* __restrict__ idx_log,
                                      int F_out, int F_out_pad, int N_ss, int n_groups) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n_chunks = (int64_t)F_out_pad / 16;
    if (t >= (int64_t)n_groups * n_chunks * kGroupSubs) return;
    const int s = (int)(t % kGroupSubs);
    const int64_t ch = (t / kGroupSubs) % n_chunks;
    const int64_t g = t / (kGroupSubs * n_chunks);
    const int64_t ss = g * kGroupSubs + s;
    if (ss >= N_ss) return;
    const uint4 v = *reinterpret_cast<const uint4*>(phys + idx_offset(g, ch * 16, s, F_out_pad));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    for (int j = 0; j < 16; ++j) {
        const int64_t r = ch * 16 + j;
        if (r < F_out) idx_log[ss * F_out + r] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
    }
}

// Packed layout (NEXT-2): one thread per (group g, 64-row block, subspace s)
// segment = the LSB-first bitstream of the 64 rows' codes.  Codes >= C (a
// caller error) raise *bad.
template <class IT>
__global__ void k_idx_logical_to_packed(const IT* __restrict__ idx_log, uint8_t* __restrict__ phys, int F_out,
                                        int F_out_pad, int N_ss, int n_groups, int C, int bits,
                                        int* __restrict__ bad) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nblk = F_out_pad / kRowBlock;
    if (t >= (int64_t)n_groups * nblk * kGroupSubs) return;
    const int s = (int)(t % kGroupSubs);
    const int64_t blk = (t / kGroupSubs) % nblk;
    const int64_t g = t / (kGroupSubs * nblk);
    const int64_t ss = g * kGroupSubs + s;
    uint32_t w[20];
    for (int i = 0; i < 2 * bits; ++i) w[i] = 0u;
    for (int r = 0; r < kRowBlock; ++r) {
        const int64_t row = blk * kRowBlock + r;
        uint32_t v = (ss < N_ss && row < F_out) ? (uint32_t)idx_log[ss * F_out + row] : 0u;
        if (v >= (uint32_t)C) { atomicOr(bad, 1); v = 0u; }
        const int p = r * bits;
        w[p >> 5] |= v << (p & 31);
        if ((p & 31) + bits > 32) w[(p >> 5) + 1] |= v >> (32 - (p & 31));
    }
    uint32_t* dst = reinterpret_cast<uint32_t*>(phys + t * (8 * bits));
    for (int i = 0; i < 2 * bits; ++i) dst[i] = w[i];
}

template <class IT>
__global__ void k_idx_packed_to_logical(const uint8_t* __restrict__ phys, IT* __restrict__ idx_log, int F_out,
                                        int F_out_pad, int N_ss, int n_groups, int bits) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nblk = F_out_pad / kRowBlock;
    if (t >= (int64_t)n_groups * nblk * kGroupSubs) return;
    const int s = (int)(t % kGroupSubs);
    const int64_t blk = (t / kGroupSubs) % nblk;
    const int64_t g = t / (kGroupSubs * nblk);
    const int64_t ss = g * kGroupSubs + s;
    if (ss >= N_ss) return;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(phys + t * (8 * bits));
    const uint32_t mask = (1u << bits) - 1u;
    for (int r = 0; r < kRowBlock; ++r) {
        const int64_t row = blk * kRowBlock + r;
        if (row >= F_out) break;
        const int p = r * bits;
        uint32_t v = src[p >> 5] >> (p & 31);
        if ((p & 31) + bits > 32) v |= src[(p >> 5) + 1] << (32 - (p & 31));
        idx_log[ss * F_out + row] = (IT)(v & mask);
    }
}

// dim = 0 layout: one thread per (group g, 16-column block, subspace s): 16 bytes
// (columns >= F_in and subspaces >= N_ss hold 0).
__global__ void k_idx_dim0_to_phys(const uint8_t* __restrict__ idx_log, uint8_t* __restrict__ phys, int F_in,
                                   int K_pad, int N_ss, int n_groups) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nb = K_pad / 16;
    if (t >= (int64_t)n_groups * nb * kGroupSubs) return;
    const int s = (int)(t % kGroupSubs);
    const int64_t jb = (t / kGroupSubs) % nb;
    const int64_t g = t / (kGroupSubs * nb);
    const int64_t ss = g * kGroupSubs + s;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    for (int q = 0; q < 16; ++q) {
        const int64_t j = jb * 16 + q;
        const uint32_t v = (ss < N_ss && j < F_in) ? idx_log[ss * F_in + j] : 0u;
        w[q >> 2] |= v << (8 * (q & 3));
    }
    *reinterpret_cast<uint4*>(phys + t * 16) = make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void k_idx_dim0_to_logical(const uint8_t* __restrict__ phys, uint8_t* __restrict__ idx_log, int F_in,
                                      int K_pad, int N_ss, int n_groups) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nb = K_pad / 16;
    if (t >= (int64_t)n_groups * nb * kGroupSubs) return;
    const int s = (int)(t % kGroupSubs);
    const int64_t jb = (t / kGroupSubs) % nb;
    const int64_t g = t / (kGroupSubs * nb);
    const int64_t ss = g * kGroupSubs + s;
    if (ss >= N_ss) return;
    for (int q = 0; q < 16; ++q) {
        const int64_t j = jb * 16 + q;
        if (j < F_in) idx_log[ss * F_in + j] = phys[t * 16 + q];
    }
}

// 32 x 32 tiles through SMEM (coalesced both ways)
__global__ void k_transpose_f16(const __half* __restrict__ in, __half* __restrict__ out, int64_t rows, int64_t cols) {
    __shared__ __half tile[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
    }
}

fasq_status transpose_f16(const __half* in, __half* out, int64_t rows, int64_t cols, cudaStream_t st) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    k_transpose_f16<<<grid, dim3(32, 8), 0, st>>>(in, out, rows, cols);
    FASQ_CUDA_TRY(cudaGetLastError());
    return FASQ_OK;
}

// uint8 logical -> the byte layout, from a uint16 logical table (GPU pack output)
__global__ void k_idx16_to_8(const uint16_t* __restrict__ a, uint8_t* __restrict__ b, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = (uint8_t)a[i];
}

// One thread per (group g, k, lane): entry of E bytes.
__global__ void k_build_cbimg(const __half* __restrict__ cb, uint8_t* __restrict__ img, int C, int d,
                              int group, int N_ss, int n_groups, int E) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)n_groups * C * kGroupSubs;
    if (t >= total) return;
    int lane = (int)(t % kGroupSubs);
    int k = (int)((t / kGroupSubs) % C);
    int g = (int)(t / ((int64_t)kGroupSubs * C));
    int ss = g * kGroupSubs + lane;
    uint16_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = 0;
    if (ss < N_ss) {
        const uint16_t* src = reinterpret_cast<const uint16_t*>(cb) + ((int64_t)(ss / group) * C + k) * d;
        for (int e = 0; e < d; ++e) v[e] = src[e];
    }
    uint16_t* dst = reinterpret_cast<uint16_t*>(img + t * E);
    for (int e = 0; e < E / 2; ++e) dst[e] = v[e];
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// cbimg_x: word s of k-row k of every group moves to position s ^ ((k & 7) << 2).
__global__ void k_build_cbimg_x(const uint32_t* __restrict__ img, uint32_t* __restrict__ img_x, int C,
                                int64_t total) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int s = (int)(t % kGroupSubs);
    const int64_t row = t / kGroupSubs;          // g * C + k
    const int k = (int)(row % C);
    img_x[row * kGroupSubs + (s ^ ((k & 7) << 2))] = img[t];
}

fasq_status ensure_cbimg_x(const fasq_layer* Lc, cudaStream_t st) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    fasq_layer* L = const_cast<fasq_layer*>(Lc);   // a derived cache; the PQ data stays immutable
    if (L->cbimg_x) return FASQ_OK;
    if (L->d != 2 || L->E != 4 || L->bits || L->dim0) return FASQ_E_UNSUPPORTED;
    uint8_t* img = nullptr;
    fasq_status s = dev_alloc_t(&img, (size_t)L->cbimg_bytes, st);
    if (s != FASQ_OK) return s;
    const int64_t total = (int64_t)L->n_groups * L->C * kGroupSubs;
    k_build_cbimg_x<<<nblk(total, 256), 256, 0, st>>>(reinterpret_cast<const uint32_t*>(L->cbimg),
                                                       reinterpret_cast<uint32_t*>(img), L->C, total);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { dev_free(img, st); return cuda_fail(e, "k_build_cbimg_x"); }
    void* map = nullptr;
    s = encode_pair_map(img, L, &map, st);
    if (s != FASQ_OK) { dev_free(img, st); return s; }
    L->cbimg_x = img;
    L->cbmap_x = map;
    return FASQ_OK;
}

fasq_status build_physical_from_logical(fasq_layer* L, const __half* cb_logical, const void* idx_logical,
                                        cudaStream_t st) {
    if (cb_logical != L->cb)
        FASQ_CUDA_TRY(cudaMemcpyAsync(L->cb, cb_logical, (size_t)L->cb_bytes, cudaMemcpyDeviceToDevice, st));
    if (L->dim0) {
        const int64_t n = (int64_t)L->n_groups * (L->K_pad / 16) * kGroupSubs;
        k_idx_dim0_to_phys<<<nblk(n, 256), 256, 0, st>>>(static_cast<const uint8_t*>(idx_logical), L->idx,
                                                         (int)L->F_in, L->K_pad, L->N_ss, L->n_groups);
        FASQ_CUDA_TRY(cudaGetLastError());
        return build_cbimg(L, st);
    }
    if (L->bits == 0) {
        int64_t n = (int64_t)L->n_groups * (L->F_out_pad / 16) * kGroupSubs;
        k_idx_logical_to_phys<<<nblk(n, 256), 256, 0, st>>>(static_cast<const uint8_t*>(idx_logical), L->idx,
                                                             (int)L->F_out, L->F_out_pad, L->N_ss, L->n_groups);
        FASQ_CUDA_TRY(cudaGetLastError());
        return build_cbimg(L, st);
    }
    // packed (NEXT-2): codes >= C are rejected (checked here, one small D2H)
    int* bad = nullptr;
    fasq_status s = dev_alloc_t(&bad, sizeof(int), st);
    if (s != FASQ_OK) return s;
    int h = 0;
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), st);
    const int64_t n = (int64_t)L->n_groups * (L->F_out_pad / kRowBlock) * kGroupSubs;
    if (e == cudaSuccess) {
        if (L->idx_w == 2)
            k_idx_logical_to_packed<uint16_t><<<nblk(n, 128), 128, 0, st>>>(
                static_cast<const uint16_t*>(idx_logical), L->idx, (int)L->F_out, L->F_out_pad, L->N_ss,
                L->n_groups, L->C, L->bits, bad);
        else
            k_idx_logical_to_packed<uint8_t><<<nblk(n, 128), 128, 0, st>>>(
                static_cast<const uint8_t*>(idx_logical), L->idx, (int)L->F_out, L->F_out_pad, L->N_ss,
                L->n_groups, L->C, L->bits, bad);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    dev_free(bad, st);
    if (e != cudaSuccess) return cuda_fail(e, "packed index layout");
    if (h) { set_error("import: an index is >= C"); return FASQ_E_ARG; }
    return build_cbimg(L, st);
}

fasq_status idx16_to_8(const uint16_t* a, uint8_t* b, int64_t n, cudaStream_t st) {
    k_idx16_to_8<<<nblk(n, 256), 256, 0, st>>>(a, b, n);
    FASQ_CUDA_TRY(cudaGetLastError());
    return FASQ_OK;
}

fasq_status build_cbimg(fasq_layer* L, cudaStream_t st) {
    int64_t n = (int64_t)L->n_groups * L->C * kGroupSubs;
    k_build_cbimg<<<nblk(n, 256), 256, 0, st>>>(L->cb, L->cbimg, L->C, L->d, L->group, L->N_ss, L->n_groups,
                                                 L->E);
    FASQ_CUDA_TRY(cudaGetLastError());
    return FASQ_OK;
}

fasq_status export_logical(const fasq_layer* L, __half* cb_out, void* idx_out_, cudaStream_t st) {
    if (cb_out)
        FASQ_CUDA_TRY(cudaMemcpyAsync(cb_out, L->cb, (size_t)L->cb_bytes, cudaMemcpyDeviceToDevice, st));
    if (idx_out_ && L->dim0) {
        const int64_t n = (int64_t)L->n_groups * (L->K_pad / 16) * kGroupSubs;
        k_idx_dim0_to_logical<<<nblk(n, 256), 256, 0, st>>>(L->idx, static_cast<uint8_t*>(idx_out_), (int)L->F_in,
                                                            L->K_pad, L->N_ss, L->n_groups);
        FASQ_CUDA_TRY(cudaGetLastError());
        return FASQ_OK;
    }
    if (idx_out_ && L->bits) {
        const int64_t n = (int64_t)L->n_groups * (L->F_out_pad / kRowBlock) * kGroupSubs;
        if (L->idx_w == 2)
            k_idx_packed_to_logical<uint16_t><<<nblk(n, 128), 128, 0, st>>>(
                L->idx, static_cast<uint16_t*>(idx_out_), (int)L->F_out, L->F_out_pad, L->N_ss, L->n_groups, L->bits);
        else
            k_idx_packed_to_logical<uint8_t><<<nblk(n, 128), 128, 0, st>>>(
                L->idx, static_cast<uint8_t*>(idx_out_), (int)L->F_out, L->F_out_pad, L->N_ss, L->n_groups, L->bits);
        FASQ_CUDA_TRY(cudaGetLastError());
        return FASQ_OK;
    }
    uint8_t* idx_out = static_cast<uint8_t*>(idx_out_);
    if (idx_out) {
        int64_t n = (int64_t)L->n_groups * (L->F_out_pad / 16) * kGroupSubs;
        k_idx_phys_to_logical<<<nblk(n, 256), 256, 0, st>>>(L->idx, idx_out, (int)L->F_out, L->F_out_pad,
                                                             L->N_ss, L->n_groups);
        FASQ_CUDA_TRY(cudaGetLastError());
    }
    return FASQ_OK;
}

// Distinct fp16 centroids per codebook (P:241 dedup): one thread per
// codebook, entry k counts if no k' < k has identical bits (O(C^2 d)).
__global__ void k_count_distinct(const uint16_t* __restrict__ cb, int N_cb, int C, int d,
                                 unsigned long long* __restrict__ total) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= N_cb) return;
    const uint16_t* c = cb + (size_t)g * C * d;
    unsigned n = 0;
    for (int k = 0; k < C; ++k) {
        bool dup = false;
        for (int k2 = 0; k2 < k && !dup; ++k2) {
            bool eq = true;
            for (int e = 0; e < d; ++e) eq &= c[k * d + e] == c[k2 * d + e];
            dup = eq;
        }
        n += dup ? 0u : 1u;
    }
    atomicAdd(total, (unsigned long long)n);
}

fasq_status count_distinct_centroids(const fasq_layer* L, int64_t* distinct, cudaStream_t st) {
    unsigned long long* t = nullptr;
    fasq_status s = dev_alloc_t(&t, sizeof(unsigned long long), st);
    if (s != FASQ_OK) return s;
    unsigned long long h = 0;
    cudaError_t e = cudaMemsetAsync(t, 0, sizeof(h), st);
    if (e == cudaSuccess) {
        k_count_distinct<<<nblk(L->N_cb, 128), 128, 0, st>>>(reinterpret_cast<const uint16_t*>(L->cb), L->N_cb,
                                                             L->C, L->d, t);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, t, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    dev_free(t, st);
    if (e != cudaSuccess) return cuda_fail(e, "count_distinct_centroids");
    *distinct = (int64_t)h;
    set_launch_count(1);
    return FASQ_OK;
}

}  // namespace fasq
