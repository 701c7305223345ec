// chain_k8.cu -- k_chain instances for batch width NB = 8 (chain_kernel.cuh).
#include "chain_kernel.cuh"

namespace fasq {
namespace chainimpl {
FASQ_CHAIN_DISPATCH_DEF(8)
}  // namespace chainimpl
}  // namespace fasq
