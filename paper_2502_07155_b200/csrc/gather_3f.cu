// Dispatch for d = 3, float: polynomial-tap or exact-tap kernels.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_3f_p(int m);
const void* gather_kernel_3f_e(int m);
const void* gather_kernel_3f(int m, bool poly) { return poly ? gather_kernel_3f_p(m) : gather_kernel_3f_e(m); }
}  // namespace bnfft
