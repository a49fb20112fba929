// Instantiation unit: gather kernels for d = 1, double arithmetic.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_1d(int m) { return kernel_for<1, double, kMaxM1>(m); }
}  // namespace bnfft
