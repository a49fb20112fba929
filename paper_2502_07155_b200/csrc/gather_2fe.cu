// Instantiation unit: gather kernels for d = 2, float arithmetic, exact taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_2f_e(int m) { return kernel_for<2, float, false, kMaxM2>(m); }
}  // namespace bnfft
