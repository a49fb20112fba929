// Instantiation unit: gather kernels for d = 3, float arithmetic, exact taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_3f_e(int m) { return kernel_for<3, float, false, kMaxM3>(m); }
const void* gather3c_kernel_e() { return (const void*)gather3c_kernel<false>; }
}  // namespace bnfft
