// Instantiation unit: gather kernels for d = 3, double arithmetic, exact taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_3d_e(int m) { return kernel_for<3, double, false, kMaxM3>(m); }
}  // namespace bnfft
