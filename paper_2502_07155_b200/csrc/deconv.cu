// Row a3, Algorithm 2 step 1: theta^(k) = f^(k)/psi^(k) on I_M, 0 on
// I_L \ I_M, written as the cuFFT input X[k mod L] = f^(k) prod_t q(k_t) with
// q(k) = (-1)^k / (L psi^_1(k)).  The (-1)^{sum k_t} factor makes the unnormalised inverse DFT
// of step 2 return theta_l at the centred index l + L/2 (reading A9); 1/L per dimension is the
// 1/|I_L| of eq. def_theta (A8).  Only the M^d entries of I_M are written: the rest of
// the out-of-place FFT input was zeroed at plan creation and cuFFT C2C never writes its input.
#include "bnfft_internal.h"

namespace bnfft {

template <typename C, typename R>
__global__ void deconv_kernel(const C* __restrict__ fhat, C* __restrict__ X,
                              const double* __restrict__ q, int d, int64_t M, int64_t L,
                              int64_t Md, int64_t Ld, int64_t total) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = idx / Md;
    int64_t r = idx - b * Md;
    int64_t it[3];
    for (int t = d - 1; t >= 0; --t) {
      it[t] = r % M;
      r /= M;
    }
    double qq = 1.0;
    int64_t flat = 0;
    for (int t = 0; t < d; ++t) {
      qq *= q[it[t]];
      int64_t k = it[t] - M / 2;
      int64_t pk = k < 0 ? k + L : k;
      flat = flat * L + pk;
    }
    C v = fhat[idx];
    R s = (R)qq;
    v.x *= s;
    v.y *= s;
    X[b * Ld + flat] = v;
  }
}

cudaError_t launch_deconv(bnfft_plan_s* p, const void* fhat) {
  int64_t total = p->Md * p->opts.batch;
  if (total == 0) return cudaSuccess;
  int64_t blocks = std::min<int64_t>((total + 255) / 256, 148LL * 32);
  if (p->c128)
    deconv_kernel<double2, double><<<(unsigned)blocks, 256, 0, p->stream>>>(
        (const double2*)fhat, (double2*)p->d_fft_in, p->d_q, p->opts.d, p->opts.M, p->L, p->Md,
        p->Ld, total);
  else
    deconv_kernel<float2, float><<<(unsigned)blocks, 256, 0, p->stream>>>(
        (const float2*)fhat, (float2*)p->d_fft_in, p->d_q, p->opts.d, p->opts.M, p->L, p->Md,
        p->Ld, total);
  p->launches++;
  return cudaGetLastError();
}

}  // namespace bnfft
