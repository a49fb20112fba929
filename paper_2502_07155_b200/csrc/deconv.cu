// Row a3, Algorithm 2 step 1: theta^(k) = f^(k)/psi^(k) on I_M, 0 on
// I_L \ I_M, written as the cuFFT input X[k mod L] = f^(k) prod_t q(k_t) with
// q(k) = (-1)^k / (L psi^_1(k)).  The (-1)^{sum k_t} factor makes the unnormalised inverse DFT
// of step 2 return theta_l at the centred index l + L/2 (reading A9); 1/L per dimension is the
// 1/|I_L| of eq. def_theta (A8).  Only the M^d entries of I_M are written: the rest of
// the out-of-place FFT input was zeroed at plan creation and cuFFT C2C never writes its input.
#include "bnfft_internal.h"

namespace bnfft {

// L0: modulus of the first index (L; M for the pruned 3-D transform's compact plane buffer, whose
// plane k_1 mod M holds k_1 in I_M).
template <typename C, typename R>
__global__ void deconv_kernel(const C* __restrict__ fhat, C* __restrict__ X,
                              const double* __restrict__ q, int d, int64_t M, int64_t L,
                              int64_t Md, int64_t Ld, int64_t total, int64_t L0) {
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
      int64_t pk = k < 0 ? k + (t == 0 ? L0 : L) : k;
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
  int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 32);
  void* X = p->pfft3 ? p->d_fft_p : p->d_fft_in;
  const int64_t L0 = p->pfft3 ? p->opts.M : p->L;
  if (p->c128)
    deconv_kernel<double2, double><<<(unsigned)blocks, 256, 0, p->stream>>>(
        (const double2*)fhat, (double2*)X, p->d_q, p->opts.d, p->opts.M, p->L, p->Md,
        p->Ld, total, L0);
  else
    deconv_kernel<float2, float><<<(unsigned)blocks, 256, 0, p->stream>>>(
        (const float2*)fhat, (float2*)X, p->d_q, p->opts.d, p->opts.M, p->L, p->Md,
        p->Ld, total, L0);
  p->launches++;
  return cudaGetLastError();
}

}  // namespace bnfft

namespace bnfft {

// BNFFT_DIST_SLAB step 1 for one rank's k_1 chunk [k0_lo, k0_hi) (d = 3, batch 1): the same products
// as deconv_kernel, written to out[k_1 - k0_lo][k_2 mod L][k_3 mod L] (the input of the rank's 2-D
// FFTs over (k_2, k_3)); entries outside I_M stay zero from plan creation.
template <typename C, typename R>
__global__ void deconv_slab_kernel(const C* __restrict__ fhat, C* __restrict__ X, const double* __restrict__ q,
                                   int64_t M, int64_t L, int64_t k0_lo, int64_t total) {
  const int64_t MM = M * M;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = idx / MM;                 // chunk-local k_1 index
    const int64_t r = idx - i0 * MM;
    const int64_t i1 = r / M, i2 = r - (r / M) * M;
    const int64_t c0 = k0_lo + M / 2 + i0;       // centred index of k_1
    const int64_t k1 = i1 - M / 2, k2 = i2 - M / 2;
    const double qq = q[c0] * q[i1] * q[i2];
    C v = fhat[c0 * MM + r];
    const R s = (R)qq;
    v.x *= s;
    v.y *= s;
    X[(i0 * L + (k1 < 0 ? k1 + L : k1)) * L + (k2 < 0 ? k2 + L : k2)] = v;
  }
}

cudaError_t launch_deconv_slab(bnfft_plan_s* p, const void* fhat, void* out, int64_t k0_lo, int64_t k0_hi) {
  const int64_t total = (k0_hi - k0_lo) * p->opts.M * p->opts.M;
  if (total <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 32);
  if (p->c128)
    deconv_slab_kernel<double2, double><<<(unsigned)blocks, 256, 0, p->stream>>>(
        (const double2*)fhat, (double2*)out, p->d_q, p->opts.M, p->L, k0_lo, total);
  else
    deconv_slab_kernel<float2, float><<<(unsigned)blocks, 256, 0, p->stream>>>(
        (const float2*)fhat, (float2*)out, p->d_q, p->opts.M, p->L, k0_lo, total);
  p->launches++;
  return cudaGetLastError();
}

}  // namespace bnfft
