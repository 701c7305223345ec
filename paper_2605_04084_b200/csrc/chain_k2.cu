// chain_k2.cu -- k_chain instances for batch width NB = 2 (chain_kernel.cuh).
#include "chain_kernel.cuh"

namespace fasq {
namespace chainimpl {
FASQ_CHAIN_DISPATCH_DEF(2)
}  // namespace chainimpl
}  // namespace fasq
