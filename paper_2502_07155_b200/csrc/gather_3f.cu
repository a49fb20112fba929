// Instantiation unit: gather kernels for d = 3, float arithmetic.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_3f(int m) { return kernel_for<3, float, kMaxM3>(m); }
}  // namespace bnfft
