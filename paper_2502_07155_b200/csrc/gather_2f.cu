// Instantiation unit: gather kernels for d = 2, float arithmetic.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_2f(int m) { return kernel_for<2, float, kMaxM2>(m); }
}  // namespace bnfft
