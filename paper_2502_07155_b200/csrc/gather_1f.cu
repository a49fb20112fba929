// Instantiation unit: gather kernels for d = 1, float arithmetic.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_1f(int m) { return kernel_for<1, float, kMaxM1>(m); }
}  // namespace bnfft
