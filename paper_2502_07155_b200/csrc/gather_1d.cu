// Dispatch for d = 1, double: polynomial-tap or exact-tap kernels.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_1d_p(int m);
const void* gather_kernel_1d_e(int m);
const void* gather_kernel_1d(int m, bool poly) { return poly ? gather_kernel_1d_p(m) : gather_kernel_1d_e(m); }
}  // namespace bnfft
