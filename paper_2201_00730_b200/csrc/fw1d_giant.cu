// fw1d_giant.cu -- n or m > 32768 (up to 262144 per side) instantiations of the
// batched 1-D FW / OT kernel: 64 / 128 / 256 atoms per thread and side at
// FW_THREADS_BIG threads, the per-atom loops rolled and the per-thread arrays in
// local memory -- a correctness path that keeps the boundary free of a size cap
// at the sizes the reference handles in minutes (src/ot1d.py:112-172 has none).
#define UOT_FW_BIG_TU
#include "fw1d_kernel.cuh"

namespace uot {
namespace fwk {
UOT_FW_GIANT(, false)
}  // namespace fwk
}  // namespace uot
