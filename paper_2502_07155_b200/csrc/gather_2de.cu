// Instantiation unit: gather kernels for d = 2, double arithmetic, exact taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_2d_e(int m) { return kernel_for<2, double, false, kMaxM2>(m); }
}  // namespace bnfft
