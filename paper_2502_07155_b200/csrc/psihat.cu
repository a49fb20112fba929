// Algorithm 2 step 0(a): psi^_1(k), k in I_M, on the device.
//
// psi^(v) = int psi(t) e^{-2 pi i v t} dt with psi even and supported on
// [-m/L, m/L], so psi^(v) = 2 int_0^{m/L} psi(t) cos(2 pi v t) dt.  Reading A4:
// t = (m/L) sin(theta), theta in [0, pi/2], then kQuadN-point Gauss-Legendre (nodes/weights
// from the host, Newton iteration in plan.cu).  In grid units tau = L t = m sin(theta):
//   psi^(k) = 2 sum_q W_q (m/L) cos(theta_q) sinc(pi tau_q) phi(tau_q/L) cos(2 pi k tau_q / L).
// Also writes q(k) = (-1)^k / (L psi^_1(k)), which folds D_psihat's 1/|I_L| (A8) and the
// centring shift of the grid (A9) into one factor per dimension.
#include "bnfft_internal.h"

namespace bnfft {

__global__ void psihat_kernel(const double* __restrict__ gl, double* __restrict__ psihat,
                              double* __restrict__ q, int64_t M, int64_t L, WinParams wp) {
  __shared__ double g[kQuadN];
  __shared__ double tq[kQuadN];
  if (threadIdx.x < kQuadN) {
    double theta = gl[threadIdx.x];
    double w = gl[kQuadN + threadIdx.x];
    double s, c;
    sincos(theta, &s, &c);
    double tau = wp.m * s;
    double sinc = sinpi(tau) / (M_PI * tau);   // tau > 0 at interior GL nodes
    g[threadIdx.x] = w * (double(wp.m) / double(L)) * c * sinc * phi_tau_d(tau, wp);
    tq[threadIdx.x] = tau;
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    double k = double(i - M / 2);
    double acc = 0.0;
#pragma unroll 8
    for (int j = 0; j < kQuadN; ++j) acc += g[j] * cospi(2.0 * k * tq[j] / double(L));
    double ph = 2.0 * acc;
    psihat[i] = ph;
    int64_t ki = i - M / 2;
    double sgn = (ki & 1) ? -1.0 : 1.0;
    q[i] = sgn / (double(L) * ph);
  }
}

// flatness max_k |L psi^(k) - 1| and min_k |psi^(k)| / |psi^(0)| (vanishing check)
__global__ void psihat_check_kernel(const double* __restrict__ psihat, int64_t M, int64_t L,
                                    double* __restrict__ out) {
  __shared__ double smax[256], smin[256];
  double mx = 0.0, mn = 1e300;
  double p0 = fabs(psihat[M / 2]);
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    double v = psihat[i];
    mx = fmax(mx, fabs(double(L) * v - 1.0));
    mn = fmin(mn, fabs(v) / p0);
  }
  smax[threadIdx.x] = mx;
  smin[threadIdx.x] = mn;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = smax[0];
    out[1] = smin[0];
  }
}

cudaError_t launch_psihat(bnfft_plan_s* p) {
  int64_t M = p->opts.M;
  int blocks = (int)std::min<int64_t>((M + 255) / 256, 148 * 8);
  psihat_kernel<<<blocks, 256, 0, p->stream>>>(p->d_gl, p->d_psihat, p->d_q, M, p->L, p->wp);
  psihat_check_kernel<<<1, 256, 0, p->stream>>>(p->d_psihat, M, p->L, p->d_flat);
  p->launches += 2;
  return cudaGetLastError();
}

}  // namespace bnfft
