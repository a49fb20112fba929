// Row a6, Algorithm 2 step 3: the short sums
//     f_j = sum_{l in J_{L,m}(x_j) cap I_L} theta_l psi(x_j - l/L),
// psi(x) = sinc(L pi x) phi(x) (eq. sinc_reg), tensor product over dimensions (A3).
//
// With c_t = floor(L x_t) and u_t = L x_t - c_t in [0,1), the 2m taps per dimension are
// l_t = c_t - m + 1 + i, i = 0..2m-1 (reading A6: the (2m+1)-th member of J at integer L x_t has
// psi = 0), at offsets tau = L x_t - l_t = u_t + (m-1-i).  sinc(pi tau) = (-1)^{m-1-i}
// sin(pi u)/(pi tau): one sinpi per node and dimension (SURVEY §8(a) "per-node tap evaluation").
// u == 0 (a grid node) is the Kronecker case of the interpolation property: the
// weight of tap i = m-1 is exactly 1 and all others exactly 0, so f_j == theta_{c} bitwise.
//
// Work decomposition: nodes are sorted by bin (row a1); CTA k owns sorted nodes
// [256k, 256k+256).  For every bin segment in its chunk the CTA stages the bin's grid
// neighbourhood (bin + (m-1, m) halo, zero outside I_L = reading A5 zero extension) into shared
// memory, then each thread contracts its node's (2m)^d taps from shared memory in a fixed order
// (bitwise reproducible) and writes f to the user position perm[i].
#pragma once
#include <algorithm>

#include "bnfft_internal.h"

namespace bnfft {

template <typename R> struct CT;
template <> struct CT<float> { using C = float2; };
template <> struct CT<double> { using C = double2; };

struct GatherParams {
  const double* xs;
  const uint32_t* perm;
  const uint32_t* bin_start;
  const void* grid;
  void* out;
  int64_t n, L, Ld;
  double Lf;
  int batch, bt;
  int log2W[3];
  int64_t nb[3];
  int box[3];
  int box_elems;
  WinParams wp;
};

__device__ __forceinline__ double sinpi_r(double u) { return sinpi(u); }
__device__ __forceinline__ float sinpi_r(float u) { return sinpif(u); }
__device__ __forceinline__ double phi_r(double tau, const WinParams& w) { return phi_tau_d(tau, w); }
__device__ __forceinline__ float phi_r(float tau, const WinParams& w) { return phi_tau_f(tau, w); }
template <typename R> __device__ __forceinline__ R pi_r();
template <> __device__ __forceinline__ double pi_r<double>() { return 3.141592653589793; }
template <> __device__ __forceinline__ float pi_r<float>() { return 3.14159265f; }

// Per-dimension node state: u in working precision, s = sin(pi u), and the Kronecker tap
// (-1 if none) for u == 0 (tap m-1) or u rounded to 1 (tap m).
template <typename R>
struct DimState {
  R u, s;
  int hit;
};

template <int T, typename R>
__device__ __forceinline__ DimState<R> dim_state(double u_d) {
  constexpr int m = T / 2;
  DimState<R> st;
  st.u = (R)u_d;
  st.hit = -1;
  if (st.u == R(0)) st.hit = m - 1;
  else if (st.u == R(1)) st.hit = m;
  st.s = sinpi_r(st.u);
  return st;
}

template <int T, typename R>
__device__ __forceinline__ R tap_weight(const DimState<R>& st, int i, const WinParams& wp) {
  constexpr int m = T / 2;
  if (st.hit >= 0) return i == st.hit ? R(1) : R(0);
  const int j = m - 1 - i;
  const R tau = st.u + (R)j;
  const R sg = (j & 1) ? -st.s : st.s;
  return sg / (pi_r<R>() * tau) * phi_r(tau, wp);
}

template <typename C> __device__ __forceinline__ C czero();
template <> __device__ __forceinline__ float2 czero<float2>() { return make_float2(0.f, 0.f); }
template <> __device__ __forceinline__ double2 czero<double2>() { return make_double2(0.0, 0.0); }

template <int D, int T, typename R>
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(GatherParams p) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* box = reinterpret_cast<C*>(smem_raw);
  __shared__ uint32_t sh_key[kGatherThreads];
  constexpr int m = T / 2;

  const int64_t i0 = (int64_t)blockIdx.x * kGatherThreads;
  const int64_t i1 = min(i0 + (int64_t)kGatherThreads, p.n);
  const int64_t i = i0 + threadIdx.x;
  const bool active = i < i1;

  DimState<R> st[D];
  R w[D][T];     // weights of dims 1..D-1 (dim 0 for D == 1, 2); D == 3 recomputes dim 0
  int off[D];
  uint32_t key = 0, dst = 0;
  if (active) {
    dst = p.perm[i];
#pragma unroll
    for (int t = 0; t < D; ++t) {
      double xv = p.xs[i * D + t];
      double Lx = __dmul_rn(p.Lf, xv);
      double fl = floor(Lx);
      double u = Lx - fl;
      int64_t c = (int64_t)fl + p.L / 2;
      if (c > p.L - 1) { c = p.L - 1; u = 1.0; }   // fl(L x) == L/2 (non-power-of-2 L)
      int64_t bt = c >> p.log2W[t];
      key = key * (uint32_t)p.nb[t] + (uint32_t)bt;
      off[t] = (int)(c - (bt << p.log2W[t]));
      st[t] = dim_state<T, R>(u);
      if (D < 3 || t > 0) {
#pragma unroll
        for (int k = 0; k < T; ++k) w[t][k] = tap_weight<T, R>(st[t], k, p.wp);
      }
    }
  }
  sh_key[threadIdx.x] = key;
  __syncthreads();

  const C* __restrict__ grid = (const C*)p.grid;
  C* __restrict__ out = (C*)p.out;
  int64_t s = i0;
  while (s < i1) {
    const uint32_t b = sh_key[s - i0];
    const int64_t e = min(i1, (int64_t)p.bin_start[b + 1]);
    int64_t org[3] = {0, 0, 0};
    {
      uint32_t rem = b;
      for (int t = D - 1; t >= 0; --t) {
        int64_t bt = rem % (uint32_t)p.nb[t];
        rem /= (uint32_t)p.nb[t];
        org[t] = (bt << p.log2W[t]) - (m - 1);
      }
    }
    const bool mine = active && i >= s && i < e;
    for (int b0 = 0; b0 < p.batch; b0 += p.bt) {
      const int nbt = min(p.bt, p.batch - b0);
      __syncthreads();
      const int total = nbt * p.box_elems;
      for (int idx = threadIdx.x; idx < total; idx += kGatherThreads) {
        int bb = idx / p.box_elems;
        int r = idx - bb * p.box_elems;
        int q[3];
#pragma unroll
        for (int t = D - 1; t >= 0; --t) {
          q[t] = r % p.box[t];
          r /= p.box[t];
        }
        bool ok = true;
        int64_t flat = 0;
#pragma unroll
        for (int t = 0; t < D; ++t) {
          int64_t pt = org[t] + q[t];
          ok = ok && pt >= 0 && pt < p.L;
          flat = flat * p.L + pt;
        }
        box[idx] = ok ? grid[(int64_t)(b0 + bb) * p.Ld + flat] : czero<C>();
      }
      __syncthreads();
      if (mine) {
        for (int bb = 0; bb < nbt; ++bb) {
          const C* bx = box + bb * p.box_elems;
          R ax = 0, ay = 0;
          if (D == 1) {
#pragma unroll
            for (int k = 0; k < T; ++k) {
              C g = bx[off[0] + k];
              ax += w[0][k] * g.x;
              ay += w[0][k] * g.y;
            }
          } else if (D == 2) {
#pragma unroll
            for (int a = 0; a < T; ++a) {
              const C* row = bx + (off[0] + a) * p.box[1] + off[1];
              R rx = 0, ry = 0;
#pragma unroll
              for (int k = 0; k < T; ++k) {
                C g = row[k];
                rx += w[1][k] * g.x;
                ry += w[1][k] * g.y;
              }
              ax += w[0][a] * rx;
              ay += w[0][a] * ry;
            }
          } else {
#pragma unroll 1
            for (int a = 0; a < T; ++a) {
              const R wa = tap_weight<T, R>(st[0], a, p.wp);
              const C* plane = bx + (off[0] + a) * p.box[1] * p.box[2];
              R px = 0, py = 0;
#pragma unroll
              for (int bq = 0; bq < T; ++bq) {
                const C* row = plane + (off[1] + bq) * p.box[2] + off[2];
                R rx = 0, ry = 0;
#pragma unroll
                for (int k = 0; k < T; ++k) {
                  C g = row[k];
                  rx += w[2][k] * g.x;
                  ry += w[2][k] * g.y;
                }
                px += w[1][bq] * rx;
                py += w[1][bq] * ry;
              }
              ax += wa * px;
              ay += wa * py;
            }
          }
          C res;
          res.x = ax;
          res.y = ay;
          out[(int64_t)(b0 + bb) * p.n + dst] = res;
        }
      }
    }
    s = e;
  }
}

template <int D, typename R, int MM>
static const void* kernel_for(int m) {
  if (m == MM) return (const void*)gather_kernel<D, 2 * MM, R>;
  if constexpr (MM > 1) return kernel_for<D, R, MM - 1>(m);
  return nullptr;
}

constexpr int kMaxM1 = 16, kMaxM2 = 12, kMaxM3 = 8;

// one translation unit per (D, precision) instantiates its kernels (parallel build)
const void* gather_kernel_1f(int m);
const void* gather_kernel_1d(int m);
const void* gather_kernel_2f(int m);
const void* gather_kernel_2d(int m);
const void* gather_kernel_3f(int m);
const void* gather_kernel_3d(int m);

}  // namespace bnfft
