// Algorithm 2 step 0(a): psi^_1(k), k in I_M, on the device, plus the
// plan-time tap polynomials of the gather (row a6).  With BNFFT_ALG1 the same kernels compute
// Algorithm 1's phi^_1(k) and fit the taps of the window phi (no sinc factor).
//
// psi^(v) = int psi(t) e^{-2 pi i v t} dt with psi even and supported on
// [-m/L, m/L], so psi^(v) = 2 int_0^{m/L} psi(t) cos(2 pi v t) dt.  Reading A4:
// t = (m/L) sin(theta), theta in [0, pi/2], then kQuadN-point Gauss-Legendre (nodes/weights
// from the host, Newton iteration in plan.cu).  In grid units tau = L t = m sin(theta):
//   psi^(k) = 2 sum_q g_q cos(2 pi k tau_q / L),  g_q = W_q (m/L) cos(theta_q) sinc(pi tau_q) phi(tau_q/L).
// psi^ is even, so only k = 0..M/2 are summed; each thread takes kRun consecutive k and advances
// e^{2 pi i k tau_q/L} by one complex multiplication per k (sincospi once per run).
// Also writes q(k) = (-1)^k / (L psi^_1(k)), which folds D_psihat's 1/|I_L| (A8) and the
// centring shift of the grid (A9) into one factor per dimension, and reduces the flatness
// max_k |L psi^(k) - 1| and min_k |psi^(k)|/|psi^(0)| with integer atomics on the
// IEEE bit patterns of non-negative doubles (order-preserving, deterministic).
#include "bnfft_internal.h"

namespace bnfft {

constexpr int kRun = 8;

__global__ void __launch_bounds__(256) psihat_kernel(const double* __restrict__ gl,
                                                     double* __restrict__ psihat,
                                                     double* __restrict__ q, int64_t M, int64_t L,
                                                     WinParams wp,
                                                     unsigned long long* __restrict__ flat) {
  __shared__ double g[kQuadN], tq[kQuadN], cs[kQuadN], sn[kQuadN];
  __shared__ double p0;
  if (threadIdx.x < kQuadN) {
    double theta = gl[threadIdx.x];
    double w = gl[kQuadN + threadIdx.x];
    double s, c;
    sincos(theta, &s, &c);
    double tau = wp.m * s;
    // tau > 0 at interior GL nodes; Algorithm 1 transforms the window itself (phi^)
    double sinc = wp.alg1 ? 1.0 : sinpi(tau) / (M_PI * tau);
    g[threadIdx.x] = w * (double(wp.m) / double(L)) * c * sinc * phi_tau_d(tau, wp);
    tq[threadIdx.x] = tau;
    double ss, cc;
    sincospi(2.0 * tau / double(L), &ss, &cc);   // one step e^{2 pi i tau/L}
    cs[threadIdx.x] = cc;
    sn[threadIdx.x] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int j = 0; j < kQuadN; ++j) a += g[j];
    p0 = 2.0 * a;
  }
  __syncthreads();
  const int64_t half = M / 2;                      // k = 0..half
  const int64_t nrun = (half + 1 + kRun - 1) / kRun;
  double fmax_loc = 0.0, rmin_loc = 1e300;
  // two lanes per run: lane parity h sums quadrature nodes j = h, h+2, ...; the pair combines with
  // one shuffle (fixed order: even-lane partial + odd-lane partial)
  const int h = threadIdx.x & 1;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  // the loop bound is warp-uniform (the pair shuffle needs all 32 lanes); lanes past nrun compute a
  // dummy run and store nothing
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t wbase = (gtid >> 5) << 4;          // first run of this warp (16 runs per warp)
  for (int64_t rw = wbase; rw < nrun; rw += nthreads >> 1) {
    const int64_t r = rw + ((threadIdx.x & 31) >> 1);
    const bool live = r < nrun;
    const int64_t k0 = (live ? r : 0) * kRun;
    double acc[kRun];
#pragma unroll
    for (int t = 0; t < kRun; ++t) acc[t] = 0.0;
    for (int j = h; j < kQuadN; j += 2) {
      double zs, zc;
      sincospi(2.0 * double(k0) * tq[j] / double(L), &zs, &zc);
      const double ws = sn[j], wc = cs[j], gj = g[j];
#pragma unroll
      for (int t = 0; t < kRun; ++t) {
        acc[t] = fma(gj, zc, acc[t]);
        double nc = zc * wc - zs * ws;
        double ns = fma(zs, wc, zc * ws);
        zc = nc;
        zs = ns;
      }
    }
#pragma unroll
    for (int t = 0; t < kRun; ++t) {
      const double other = __shfl_xor_sync(0xffffffffu, acc[t], 1);
      acc[t] = h ? other + acc[t] : acc[t] + other;
    }
    if (h || !live) continue;
#pragma unroll
    for (int t = 0; t < kRun; ++t) {
      const int64_t k = k0 + t;
      if (k > half) break;
      const double ph = 2.0 * acc[t];
      const double sgn = (k & 1) ? -1.0 : 1.0;
      const double qq = sgn / (double(L) * ph);
      // centred table index i = k + M/2 holds psi^(k); evenness gives psi^(-k)
      if (k < half) {
        psihat[half + k] = ph;
        q[half + k] = qq;
      }
      if (k >= 1) {
        psihat[half - k] = ph;
        q[half - k] = qq;
      }
      // I_M contains -M/2 (= -half) but not +M/2; psi^(half) = psi^(-half) by evenness
      fmax_loc = fmax(fmax_loc, fabs(double(L) * ph - 1.0));
      rmin_loc = fmin(rmin_loc, fabs(ph) / fabs(p0));
    }
  }
  // block reduce, then one atomic per block
  __shared__ double rmax[256], rmn[256];
  rmax[threadIdx.x] = fmax_loc;
  rmn[threadIdx.x] = rmin_loc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rmax[threadIdx.x] = fmax(rmax[threadIdx.x], rmax[threadIdx.x + s]);
      rmn[threadIdx.x] = fmin(rmn[threadIdx.x], rmn[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicMax(&flat[0], (unsigned long long)__double_as_longlong(rmax[0]));
    atomicMin(&flat[1], (unsigned long long)__double_as_longlong(rmn[0]));
  }
}

cudaError_t launch_psihat(bnfft_plan_s* p) {
  int64_t M = p->opts.M;
  int64_t nrun = (M / 2 + 1 + kRun - 1) / kRun;
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((2 * nrun + 255) / 256, (int64_t)sm_count() * 8));
  unsigned long long init[2] = {0ull, 0x7fefffffffffffffull};   // 0.0, DBL_MAX
  cudaError_t e = cudaMemcpyAsync(p->d_flat, init, sizeof(init), cudaMemcpyHostToDevice, p->stream);
  if (e != cudaSuccess) return e;
  psihat_kernel<<<blocks, 256, 0, p->stream>>>(p->d_gl, p->d_psihat, p->d_q, M, p->L, p->wp,
                                              (unsigned long long*)p->d_flat);
  p->launches += 1;
  return cudaGetLastError();
}

// psi^_1 (phi^_1 for Algorithm 1) at arbitrary frequencies v[i] (bnfft_kernel_hat).
__global__ void kernel_hat_kernel(const double* __restrict__ gl, const double* __restrict__ v,
                                  double* __restrict__ out, int64_t n, int64_t L, WinParams wp) {
  __shared__ double g[kQuadN], tq[kQuadN];
  if (threadIdx.x < kQuadN) {
    double theta = gl[threadIdx.x];
    double w = gl[kQuadN + threadIdx.x];
    double s, c;
    sincos(theta, &s, &c);
    double tau = wp.m * s;
    double sinc = wp.alg1 ? 1.0 : sinpi(tau) / (M_PI * tau);
    g[threadIdx.x] = w * (double(wp.m) / double(L)) * c * sinc * phi_tau_d(tau, wp);
    tq[threadIdx.x] = tau;
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < kQuadN; ++j) acc += g[j] * cospi(2.0 * v[i] * tq[j] / double(L));
    out[i] = 2.0 * acc;
  }
}

cudaError_t launch_kernel_hat(bnfft_plan_s* p, const double* v_dev, double* out_dev, int64_t n) {
  if (n <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
  kernel_hat_kernel<<<blocks, 256, 0, p->stream>>>(p->d_gl, v_dev, out_dev, n, p->L, p->wp);
  p->launches++;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ tap polynomials (plan time)
// Exact tap value w_i(u) = psi(u + m-1-i) (grid units) divided by the sinh edge factor.
__device__ double tap_exact_d(int i, double u, int m, const WinParams& wp, bool edge_sqrt,
                              bool divide_edge) {
  const double tau = u + double(m - 1 - i);
  const double sinc = (tau == 0.0 || wp.alg1) ? 1.0 : sinpi(tau) / (M_PI * tau);
  double v = sinc * phi_tau_d(tau, wp);
  if (edge_sqrt && divide_edge && (i == 0 || i == 2 * m - 1)) {
    // sinh edge taps: v = sinc * sinh(beta r)/sinh(beta) with r = sqrt(1-(tau/m)^2);
    // the fitted part is sinc * (sinh(beta r)/r) / sinh(beta)  (entire in r^2).
    const double t = tau / m;
    const double r = sqrt(fmax((1.0 - t) * (1.0 + t), 0.0));
    const double shr = (r > 1e-8) ? sinh(wp.beta * r) / r : wp.beta * (1.0 + wp.beta * wp.beta * r * r / 6.0);
    v = sinc * shr * wp.inv_norm;
  }
  return v;
}

// One thread per tap: Chebyshev interpolation at NC points of x = 2u - 1, converted to monomials.
__global__ void tapfit_kernel(int T, int NC, WinParams wp, int edge_sqrt, double* __restrict__ coef) {
  const int i = threadIdx.x;
  if (i >= T) return;
  const int m = T / 2;
  double v[32], c[32], tk[32], tkm1[32], a[32];
  for (int j = 0; j < NC; ++j) {
    const double xj = cospi((j + 0.5) / NC);
    v[j] = tap_exact_d(i, 0.5 * (xj + 1.0), m, wp, edge_sqrt, true);
  }
  for (int k = 0; k < NC; ++k) {
    double s = 0.0;
    for (int j = 0; j < NC; ++j) s += v[j] * cospi(k * (j + 0.5) / NC);
    c[k] = s * 2.0 / NC;
  }
  c[0] *= 0.5;
  for (int k = 0; k < NC; ++k) a[k] = tk[k] = tkm1[k] = 0.0;
  tkm1[0] = 1.0;     // T_0
  tk[1] = 1.0;       // T_1
  a[0] = c[0];
  if (NC > 1) a[1] += c[1];
  for (int k = 2; k < NC; ++k) {
    // T_k = 2 x T_{k-1} - T_{k-2}
    double tn[32];
    tn[0] = -tkm1[0];
    for (int e = 1; e < NC; ++e) tn[e] = 2.0 * tk[e - 1] - tkm1[e];
    for (int e = 0; e < NC; ++e) {
      tkm1[e] = tk[e];
      tk[e] = tn[e];
      a[e] += c[k] * tn[e];
    }
  }
  for (int k = 0; k < NC; ++k) coef[i * NC + k] = a[k];
}

// Max |poly - exact| over 1025 points of u in [0,1] per tap, evaluated in the gather's
// precision (float when fp32 != 0).  Result: err[i].
__global__ void tapcheck_kernel(int T, int NC, WinParams wp, int edge_sqrt, int fp32,
                                const double* __restrict__ coef, double* __restrict__ err) {
  const int i = blockIdx.x;
  const int m = T / 2;
  __shared__ double red[256];
  double e = 0.0;
  for (int j = threadIdx.x; j <= 1024; j += blockDim.x) {
    const double u = j / 1024.0;
    if (u == 0.0 || u == 1.0) continue;   // Kronecker branch in the gather
    const double ex = tap_exact_d(i, u, m, wp, edge_sqrt, false);
    // the gather stores taps i < m only and evaluates tap 2m-1-i as P_i(-x) (mirror symmetry)
    const int ii = i < m ? i : T - 1 - i;
    const double sgn = i < m ? 1.0 : -1.0;
    double ap;
    if (fp32) {
      const float xf = (float)(2.0 * u - 1.0);
      const float yf = xf * xf;
      float e = (float)coef[ii * NC + NC - 2], o = (float)coef[ii * NC + NC - 1];
      for (int k = NC / 2 - 2; k >= 0; --k) {
        e = fmaf(e, yf, (float)coef[ii * NC + 2 * k]);
        o = fmaf(o, yf, (float)coef[ii * NC + 2 * k + 1]);
      }
      float h = fmaf((float)sgn * xf, o, e);
      float uf = (float)u;
      if (edge_sqrt && i == 0) h *= sqrtf((1.0f - uf) * (float(2 * m - 1) + uf)) * (1.0f / m);
      if (edge_sqrt && i == T - 1) h *= sqrtf(uf * (float(2 * m) - uf)) * (1.0f / m);
      ap = h;
    } else {
      const double x = 2.0 * u - 1.0;
      const double y = x * x;
      double e = coef[ii * NC + NC - 2], o = coef[ii * NC + NC - 1];
      for (int k = NC / 2 - 2; k >= 0; --k) {
        e = fma(e, y, coef[ii * NC + 2 * k]);
        o = fma(o, y, coef[ii * NC + 2 * k + 1]);
      }
      double h = fma(sgn * x, o, e);
      if (edge_sqrt && i == 0) h *= sqrt((1.0 - u) * (double(2 * m - 1) + u)) / m;
      if (edge_sqrt && i == T - 1) h *= sqrt(u * (double(2 * m) - u)) / m;
      ap = h;
    }
    e = fmax(e, fabs(ap - ex));
  }
  red[threadIdx.x] = e;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) err[i] = red[0];
}

cudaError_t launch_tapfit(bnfft_plan_s* p, int NC, double* d_coef, double* d_err) {
  const int T = 2 * p->opts.m;
  const int edge = p->opts.window == BNFFT_SINH ? 1 : 0;
  tapfit_kernel<<<1, 32, 0, p->stream>>>(T, NC, p->wp, edge, d_coef);
  tapcheck_kernel<<<T, 256, 0, p->stream>>>(T, NC, p->wp, edge, p->c128 ? 0 : 1, d_coef, d_err);
  p->launches += 2;
  return cudaGetLastError();
}

}  // namespace bnfft
