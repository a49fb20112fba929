// Instantiation unit: gather kernels for d = 3, double arithmetic.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_3d(int m) { return kernel_for<3, double, kMaxM3>(m); }
}  // namespace bnfft
