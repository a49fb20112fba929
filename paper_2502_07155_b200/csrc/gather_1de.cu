// Instantiation unit: gather kernels for d = 1, double arithmetic, exact taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_1d_e(int m) { return kernel_for<1, double, false, kMaxM1>(m); }
}  // namespace bnfft
