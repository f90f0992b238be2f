// fw1d_pfw_huge.cu -- very large (n or m > 16384) instantiations of the batched 1-D FW /
// OT kernel (pairwise FW): one CTA of FW_THREADS_BIG threads per problem,
// per-problem arrays in the workspace, per-thread arrays past the register
// budget in local memory (a correctness path).  Own translation unit: these
// instantiations compile in parallel with the rest.
#define UOT_FW_BIG_TU
#include "fw1d_kernel.cuh"

namespace uot {
namespace fwk {
UOT_FW_HUGE(, true)
}  // namespace fwk
}  // namespace uot
