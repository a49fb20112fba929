// Dispatch for d = 3, double: polynomial-tap or exact-tap kernels.
#include "gather_impl.cuh"

namespace bnfft {
const void* gather_kernel_3d_p(int m);
const void* gather_kernel_3d_e(int m);
const void* gather_kernel_3d(int m, bool poly) { return poly ? gather_kernel_3d_p(m) : gather_kernel_3d_e(m); }
}  // namespace bnfft
