// gemm_tc.cu -- placeholder
#include "fasq_internal.cuh"
namespace fasq {
bool gemm_tc_supported(const fasq_layer*, int64_t) { return false; }
fasq_status gemm_tc_launch(const fasq_layer*, const __half*, int64_t, void*, fasq_dtype, cudaStream_t) {
    return FASQ_E_UNSUPPORTED;
}
}  // namespace fasq
