// Instantiation unit: gather kernels for d = 2, double arithmetic, polynomial taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_2d_p(int m) { return kernel_for<2, double, true, kMaxM2>(m); }
}  // namespace bnfft
