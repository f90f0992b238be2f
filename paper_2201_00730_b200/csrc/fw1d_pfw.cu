// fw1d_pfw.cu -- pairwise Frank-Wolfe instantiation of the 1-D FW kernel
// (src/fw.py:255-357; see pfw_step in fw1d_kernel.cuh).
#include "fw1d_kernel.cuh"

namespace uot {
namespace fwk {

int launch_fw_pairwise(const FwArgs& a, int batch, cudaStream_t st) {
  return launch_fw_impl<true>(a, batch, st);
}

}  // namespace fwk
}  // namespace uot
