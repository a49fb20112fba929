// Instantiation unit: gather kernels for d = 3, double arithmetic, polynomial taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_3d_p(int m) { return kernel_for<3, double, true, kMaxM3>(m); }
}  // namespace bnfft
