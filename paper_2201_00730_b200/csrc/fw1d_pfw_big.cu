// fw1d_pfw_big.cu -- large-problem (n or m > 4096) instantiations of the batched 1-D
// FW / OT kernel (pairwise FW): one CTA of FW_THREADS_BIG threads per
// problem, per-problem arrays in the workspace (fw1d_kernel.cuh).  A separate
// translation unit so these instantiations compile in parallel.
#define UOT_FW_BIG_TU
#include "fw1d_kernel.cuh"

namespace uot {
namespace fwk {
UOT_FW_BIG(, true)
}  // namespace fwk
}  // namespace uot
