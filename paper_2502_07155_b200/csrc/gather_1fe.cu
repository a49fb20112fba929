// Instantiation unit: gather kernels for d = 1, float arithmetic, exact taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_1f_e(int m) { return kernel_for<1, float, false, kMaxM1>(m); }
}  // namespace bnfft
