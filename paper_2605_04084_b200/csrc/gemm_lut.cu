// gemm_lut.cu -- placeholder
#include "fasq_internal.cuh"
namespace fasq {
fasq_status gemm_lut_launch(const fasq_layer*, const __half*, int64_t, void*, fasq_dtype, cudaStream_t) {
    return FASQ_E_UNSUPPORTED;
}
}  // namespace fasq
