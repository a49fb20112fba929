// Instantiation unit: gather kernels for d = 2, double arithmetic.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_2d(int m) { return kernel_for<2, double, kMaxM2>(m); }
}  // namespace bnfft
