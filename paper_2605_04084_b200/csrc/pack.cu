// pack.cu -- GPU k-means packer (placeholder until the bit-exact packer lands).
#include "fasq_internal.cuh"
namespace fasq {
fasq_status pack_run(const __half*, fasq_layer*, const fasq_pack_params*, cudaStream_t, __half*, uint8_t*) {
    set_error("fasq_pack: GPU packer not built yet");
    return FASQ_E_UNSUPPORTED;
}
}  // namespace fasq
