// fw1d_pfw_giant.cu -- pairwise-FW instantiations of the rolled-loop kernel for
// n or m > 32768 (see fw1d_giant.cu).
#define UOT_FW_BIG_TU
#include "fw1d_kernel.cuh"

namespace uot {
namespace fwk {
UOT_FW_GIANT(, true)
}  // namespace fwk
}  // namespace uot
