// Instantiation unit: gather kernels for d = 3, float arithmetic, polynomial taps.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_3f_p(int m) { return kernel_for<3, float, true, kMaxM3>(m); }
const void* gather3c_kernel_p() { return (const void*)gather3c_kernel<true>; }
}  // namespace bnfft
