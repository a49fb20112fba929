// Instantiation unit: gather kernels for d = 2, float arithmetic, polynomial taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_2f_p(int m) { return kernel_for<2, float, true, kMaxM2>(m); }
}  // namespace bnfft
