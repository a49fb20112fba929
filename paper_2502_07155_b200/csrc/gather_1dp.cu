// Instantiation unit: gather kernels for d = 1, double arithmetic, polynomial taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_1d_p(int m) { return kernel_for<1, double, true, kMaxM1>(m); }
}  // namespace bnfft
