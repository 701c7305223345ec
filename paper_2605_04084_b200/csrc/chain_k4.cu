// chain_k4.cu -- k_chain instances for batch width NB = 4 (chain_kernel.cuh).
#include "chain_kernel.cuh"

namespace fasq {
namespace chainimpl {
FASQ_CHAIN_DISPATCH_DEF(4)
}  // namespace chainimpl
}  // namespace fasq
