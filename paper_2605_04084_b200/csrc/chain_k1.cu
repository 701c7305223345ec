// chain_k1.cu -- k_chain instances for batch width NB = 1 (chain_kernel.cuh).
#include "chain_kernel.cuh"

namespace fasq {
namespace chainimpl {
FASQ_CHAIN_DISPATCH_DEF(1)
}  // namespace chainimpl
}  // namespace fasq
