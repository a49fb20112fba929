// Instantiation unit: gather kernels for d = 1, float arithmetic, polynomial taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_1f_p(int m) { return kernel_for<1, float, true, kMaxM1>(m); }
}  // namespace bnfft
