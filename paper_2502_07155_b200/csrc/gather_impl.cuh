// Row a6, Algorithm 2 step 3: the short sums
//     f_j = sum_{l in J_{L,m}(x_j) cap I_L} theta_l psi(x_j - l/L),
// psi(x) = sinc(L pi x) phi(x) (eq. sinc_reg), tensor product over dimensions (A3).
//
// With c_t = floor(L x_t) and u_t = L x_t - c_t in [0,1), the 2m taps per dimension are
// l_t = c_t - m + 1 + i, i = 0..2m-1 (reading A6: the (2m+1)-th member of J at integer L x_t has
// psi = 0), at offsets tau = L x_t - l_t = u_t + (m-1-i).  u == 0 (a grid node) is the Kronecker
// case of the interpolation property: tap m-1 is exactly 1 and all others exactly 0,
// so f_j == theta_c bitwise.
//
// Tap values (POLY = true, the default): w_i(u) = psi(u + m-1-i) is, per tap, a smooth function of
// u on [0,1]; the plan fits it (tapfit kernel, FP64 Chebyshev interpolation) by a degree-P
// polynomial in x = 2u-1 (P = 9 for complex64, 17 for complex128; fit error ~1e-8 / ~1e-14, checked
// at plan time).  For the sinh window the two edge taps carry the sqrt(1-(tau/m)^2) branch point
// of eq. varphisinh at |tau| = m; there w_i = P_i(x) * sqrt(1-(tau/m)^2) with P_i analytic.  The
// coefficients travel as kernel parameters, so every Horner step is one FFMA/DFMA with a
// constant-bank operand.  POLY = false evaluates sinc * phi directly (fallback for shapes whose fit
// fails the plan-time check).
//
// Work decomposition: nodes are sorted by (user block, bin) (row a1).  CTA k owns sorted nodes
// [256k, 256k+256).  The chunk's maximal runs of equal bin ("segments") are found by a block scan;
// up to `smax` segments per round have their grid neighbourhood (bin + (m-1, m) halo, zero outside
// I_L = reading A5 zero extension) staged into shared memory; every thread then contracts its
// node's (2m)^d taps from its segment's box in a fixed order (bitwise reproducible) and writes f
// to the user position perm[i].
#pragma once
#include <algorithm>

#include "bnfft_internal.h"

namespace bnfft {

template <typename R> struct CT;
template <> struct CT<float> { using C = float2; };
template <> struct CT<double> { using C = double2; };

template <typename R> struct PolyN;
template <> struct PolyN<float> { static constexpr int NC = 10; };   // degree 9
template <> struct PolyN<double> { static constexpr int NC = 18; };  // degree 17

constexpr int kMaxTaps = 32;

template <typename R>
struct GatherParams {
  const double* xs;
  const uint32_t* perm;
  const void* grid;
  void* out;
  int64_t n, L, Ld;
  double Lf;
  int batch, bt, smax;
  int log2W[3];
  int64_t nb[3];
  int box[3];
  int box_elems;
  int edge_sqrt;          // sinh window: edge taps carry sqrt(1-(tau/m)^2)
  R inv_m;
  int boxcap;             // d = 1 kernel: staged-box capacity in complex elements
  WinParams wp;
  alignas(16) R coef[PolyN<R>::NC][kMaxTaps];   // degree-major: coef[k][i] of tap i
};

__device__ __forceinline__ double sinpi_r(double u) { return sinpi(u); }
__device__ __forceinline__ float sinpi_r(float u) { return sinpif(u); }
__device__ __forceinline__ double phi_r(double tau, const WinParams& w) { return phi_tau_d(tau, w); }
__device__ __forceinline__ float phi_r(float tau, const WinParams& w) { return phi_tau_f(tau, w); }
__device__ __forceinline__ double sqrt_r(double v) { return sqrt(v); }
__device__ __forceinline__ float sqrt_r(float v) { return sqrtf(v); }
template <typename R> __device__ __forceinline__ R pi_r();
template <> __device__ __forceinline__ double pi_r<double>() { return 3.141592653589793; }
template <> __device__ __forceinline__ float pi_r<float>() { return 3.14159265f; }

// Per-dimension node state.
template <typename R>
struct DimState {
  R u, x, s;   // u, x = 2u-1, s = sin(pi u) (exact path) ; hit = Kronecker tap or -1
  R sq0, sq1;  // sinh edge factors sqrt(1-(tau/m)^2) for taps 0 and 2m-1
  int hit;
};

template <int T, typename R, bool POLY>
__device__ __forceinline__ DimState<R> dim_state(double u_d, const GatherParams<R>& p) {
  constexpr int m = T / 2;
  DimState<R> st;
  st.u = (R)u_d;
  st.x = (R)(2.0 * u_d - 1.0);
  st.hit = -1;
  if (st.u == R(0)) st.hit = m - 1;
  else if (st.u == R(1)) st.hit = m;
  if (POLY) {
    st.s = 0;
    if (p.edge_sqrt) {
      const R a = R(1) - st.u;   // tap 0: tau = m-1+u, 1-(tau/m)^2 = (1-u)(2m-1+u)/m^2
      st.sq0 = sqrt_r(a * (R(2 * m - 1) + st.u)) * p.inv_m;
      st.sq1 = sqrt_r(st.u * (R(2 * m) - st.u)) * p.inv_m;   // tap 2m-1: tau = u-m
    } else {
      st.sq0 = st.sq1 = R(1);
    }
  } else {
    st.s = sinpi_r(st.u);
    st.sq0 = st.sq1 = R(1);
  }
  return st;
}

template <int T, typename R, bool POLY>
__device__ __forceinline__ R tap_weight(const DimState<R>& st, int i, const GatherParams<R>& p) {
  constexpr int m = T / 2;
  constexpr int NC = PolyN<R>::NC;
  if (st.hit >= 0) return i == st.hit ? R(1) : R(0);
  if (POLY) {
    R h = p.coef[NC - 1][i];
#pragma unroll
    for (int k = NC - 2; k >= 0; --k) h = fma(h, st.x, p.coef[k][i]);
    if (i == 0) h *= st.sq0;
    if (i == T - 1) h *= st.sq1;
    return h;
  } else {
    const int j = m - 1 - i;
    const R tau = st.u + (R)j;
    const R sg = (j & 1) ? -st.s : st.s;
    return sg / (pi_r<R>() * tau) * phi_r(tau, p.wp);
  }
}

// All T taps of one dimension.  POLY: Horner in x = 2u-1; the float path evaluates tap pairs with
// packed FFMA2 (sm_100 fma.rn.f32x2), the coefficient pair coming from the kernel parameters.
template <int T, bool POLY>
__device__ __forceinline__ void all_taps(const DimState<float>& st, const GatherParams<float>& p,
                                         float (&w)[T]) {
  if (!POLY || st.hit >= 0) {
#pragma unroll
    for (int k = 0; k < T; ++k) w[k] = tap_weight<T, float, POLY>(st, k, p);
    return;
  }
  constexpr int NC = PolyN<float>::NC;
  const float2 xx = make_float2(st.x, st.x);
#pragma unroll
  for (int j = 0; j < T / 2; ++j) {
    float2 h = reinterpret_cast<const float2*>(p.coef[NC - 1])[j];
#pragma unroll
    for (int k = NC - 2; k >= 0; --k) h = __ffma2_rn(h, xx, reinterpret_cast<const float2*>(p.coef[k])[j]);
    w[2 * j] = h.x;
    w[2 * j + 1] = h.y;
  }
  w[0] *= st.sq0;
  w[T - 1] *= st.sq1;
}

template <int T, bool POLY>
__device__ __forceinline__ void all_taps(const DimState<double>& st, const GatherParams<double>& p,
                                         double (&w)[T]) {
#pragma unroll
  for (int k = 0; k < T; ++k) w[k] = tap_weight<T, double, POLY>(st, k, p);
}

// acc += w * g  (complex g, real w)
__device__ __forceinline__ void cmac(float2& acc, float w, float2 g) {
  acc = __ffma2_rn(make_float2(w, w), g, acc);
}
__device__ __forceinline__ void cmac(double2& acc, double w, double2 g) {
  acc.x = fma(w, g.x, acc.x);
  acc.y = fma(w, g.y, acc.y);
}

template <typename C> __device__ __forceinline__ C czero();
template <> __device__ __forceinline__ float2 czero<float2>() { return make_float2(0.f, 0.f); }
template <> __device__ __forceinline__ double2 czero<double2>() { return make_double2(0.0, 0.0); }

template <int D, int T, typename R, bool POLY>
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const __grid_constant__ GatherParams<R> p) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* box = reinterpret_cast<C*>(smem_raw);
  __shared__ uint32_t sh_key[kGatherThreads];
  __shared__ uint32_t sh_seg_key[kGatherThreads];
  __shared__ int sh_warp[kGatherThreads / 32];
  constexpr int m = T / 2;
  constexpr bool kW0Reg = (D < 3) || (T <= 8);   // keep dim-0 weights in registers

  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * kGatherThreads;
  const int64_t i1 = min(i0 + (int64_t)kGatherThreads, p.n);
  const int64_t i = i0 + tid;
  const bool active = i < i1;

  DimState<R> st[D];
  R w[D][T];
  int off[D];
  uint32_t key = 0xffffffffu, dst = 0;
  if (active) {
    dst = p.perm[i];
#pragma unroll
    for (int t = 0; t < D; ++t) {
      double xv = p.xs[i * D + t];
      double Lx = __dmul_rn(p.Lf, xv);
      double fl = floor(Lx);
      double u = Lx - fl;
      int64_t c = (int64_t)fl + p.L / 2;
      if (c > p.L - 1) { c = p.L - 1; u = 1.0; }   // fl(L x) == L/2 (defensive)
      int64_t bt = c >> p.log2W[t];
      key = (t == 0 ? 0u : key * (uint32_t)p.nb[t]) + (uint32_t)bt;
      off[t] = (int)(c - (bt << p.log2W[t]));
      st[t] = dim_state<T, R, POLY>(u, p);
      if (t > 0 || kW0Reg) all_taps<T, POLY>(st[t], p, w[t]);
    }
  }
  // ---- segments: maximal runs of equal bin inside the chunk (block scan of run starts)
  sh_key[tid] = key;
  __syncthreads();
  const bool start = active && (tid == 0 || sh_key[tid - 1] != key);
  const unsigned ball = __ballot_sync(0xffffffffu, start);
  const int lane = tid & 31, wid = tid >> 5;
  if (lane == 0) sh_warp[wid] = __popc(ball);
  __syncthreads();
  int seg_base = 0, nseg = 0;
#pragma unroll
  for (int w2 = 0; w2 < kGatherThreads / 32; ++w2) {
    int c = sh_warp[w2];
    if (w2 < wid) seg_base += c;
    nseg += c;
  }
  const int my_seg_incl = seg_base + __popc(ball & ((2u << lane) - 1u));   // segments started <= me
  const int my_seg = my_seg_incl - 1;
  if (start) sh_seg_key[my_seg] = key;
  __syncthreads();

  const C* __restrict__ grid = (const C*)p.grid;
  C* __restrict__ out = (C*)p.out;
  const int smax = p.smax;
  for (int s0 = 0; s0 < nseg; s0 += smax) {
    const int ns = min(smax, nseg - s0);
    const bool mine = active && my_seg >= s0 && my_seg < s0 + ns;
    for (int b0 = 0; b0 < p.batch; b0 += p.bt) {
      const int nbt = min(p.bt, p.batch - b0);
      __syncthreads();
      // ---- stage ns boxes x nbt spectra
      const int per_seg = nbt * p.box_elems;
      const int total = ns * per_seg;
      for (int idx = tid; idx < total; idx += kGatherThreads) {
        const int sg = idx / per_seg;
        int r = idx - sg * per_seg;
        const int bb = r / p.box_elems;
        r -= bb * p.box_elems;
        uint32_t rem = sh_seg_key[s0 + sg];
        int64_t org[3];
#pragma unroll
        for (int t = D - 1; t >= 0; --t) {
          int64_t btc = rem % (uint32_t)p.nb[t];
          rem /= (uint32_t)p.nb[t];
          org[t] = (btc << p.log2W[t]) - (m - 1);
        }
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
        box[idx] = ok ? __ldg(&grid[(int64_t)(b0 + bb) * p.Ld + flat]) : czero<C>();
      }
      __syncthreads();
      if (mine) {
        const C* bseg = box + (my_seg - s0) * per_seg;
        for (int bb = 0; bb < nbt; ++bb) {
          const C* bx = bseg + bb * p.box_elems;
          R ax = 0, ay = 0;
          if (D == 1) {
            const C* row = bx + off[0];
            C acc = czero<C>();
#pragma unroll
            for (int k = 0; k < T; ++k) cmac(acc, w[0][k], row[k]);
            ax = acc.x;
            ay = acc.y;
          } else if (D == 2) {
#pragma unroll
            for (int a = 0; a < T; ++a) {
              const C* row = bx + (off[0] + a) * p.box[1] + off[1];
              C racc = czero<C>();
#pragma unroll
              for (int k = 0; k < T; ++k) cmac(racc, w[1][k], row[k]);
              ax = fma(w[0][a], racc.x, ax);
              ay = fma(w[0][a], racc.y, ay);
            }
          } else {
            auto plane_sum = [&](int a, R wa) {
              const C* plane = bx + (off[0] + a) * p.box[1] * p.box[2];
              R px = 0, py = 0;
#pragma unroll
              for (int bq = 0; bq < T; ++bq) {
                const C* row = plane + (off[1] + bq) * p.box[2] + off[2];
                C racc = czero<C>();
#pragma unroll
                for (int k = 0; k < T; ++k) cmac(racc, w[2][k], row[k]);
                px = fma(w[1][bq], racc.x, px);
                py = fma(w[1][bq], racc.y, py);
              }
              ax = fma(wa, px, ax);
              ay = fma(wa, py, ay);
            };
            if constexpr (kW0Reg) {
#pragma unroll
              for (int a = 0; a < T; ++a) plane_sum(a, w[0][a]);
            } else {
#pragma unroll 1
              for (int a = 0; a < T; ++a) plane_sum(a, tap_weight<T, R, POLY>(st[0], a, p));
            }
          }
          C res;
          res.x = ax;
          res.y = ay;
          out[(int64_t)(b0 + bb) * p.n + dst] = res;
        }
      }
    }
  }
}

// d = 1 gather.  CTA k owns sorted nodes [k*256*NPT, (k+1)*256*NPT) (thread t takes
// k*256*NPT + j*256 + t, j < NPT: coalesced loads).  The nodes are sorted by bin inside user
// blocks, so the chunk's cells span a short range [cmin, cmax]: the grid window
// [cmin-m+1, cmax+m] (zero outside I_L) is staged once into shared memory with contiguous loads.
// If the window exceeds the box capacity (sparse node sets) the taps are read straight from
// global memory through L1 instead.
constexpr int kNPT1 = 4;

template <int T, typename R, bool POLY>
__global__ void __launch_bounds__(kGatherThreads) gather1_kernel(const __grid_constant__ GatherParams<R> p) {
  using C = typename CT<R>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* box = reinterpret_cast<C*>(smem_raw);
  __shared__ int s_min[kGatherThreads / 32], s_max[kGatherThreads / 32];
  constexpr int m = T / 2;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kGatherThreads * kNPT1;
  int cell[kNPT1];
  double uu[kNPT1];
  uint32_t dst[kNPT1];
  int cmin = 0x7fffffff, cmax = -1;
#pragma unroll
  for (int j = 0; j < kNPT1; ++j) {
    const int64_t i = base + j * kGatherThreads + tid;
    cell[j] = -1;
    if (i < p.n) {
      dst[j] = __ldg(&p.perm[i]);
      const double Lx = __dmul_rn(p.Lf, __ldg(&p.xs[i]));
      const double fl = floor(Lx);
      double u = Lx - fl;
      int64_t c = (int64_t)fl + p.L / 2;
      if (c > p.L - 1) { c = p.L - 1; u = 1.0; }
      cell[j] = (int)c;
      uu[j] = u;
      cmin = min(cmin, (int)c);
      cmax = max(cmax, (int)c);
    }
  }
  cmin = __reduce_min_sync(0xffffffffu, cmin);
  cmax = __reduce_max_sync(0xffffffffu, cmax);
  if (lane == 0) {
    s_min[wid] = cmin;
    s_max[wid] = cmax;
  }
  __syncthreads();
#pragma unroll
  for (int w2 = 0; w2 < kGatherThreads / 32; ++w2) {
    cmin = min(cmin, s_min[w2]);
    cmax = max(cmax, s_max[w2]);
  }
  const int64_t lo = (int64_t)cmin - (m - 1);
  const int nbox = cmax - cmin + T;
  const C* __restrict__ grid = (const C*)p.grid;
  C* __restrict__ out = (C*)p.out;
  const int nbt_cap = p.boxcap / nbox;            // spectra per staged slice (0: not staged)
  const int step = nbt_cap > 0 ? min(nbt_cap, p.batch) : p.batch;
  for (int b0 = 0; b0 < p.batch; b0 += step) {
    const int nbt = min(step, p.batch - b0);
    if (nbt_cap > 0) {
      if (b0 > 0) __syncthreads();
      for (int bb = 0; bb < nbt; ++bb) {
        const C* src = grid + (int64_t)(b0 + bb) * p.Ld;
        for (int q = tid; q < nbox; q += kGatherThreads) {
          const int64_t pos = lo + q;
          box[bb * nbox + q] = (pos >= 0 && pos < p.L) ? __ldg(&src[pos]) : czero<C>();
        }
      }
      __syncthreads();
    }
#pragma unroll 1
    for (int j = 0; j < kNPT1; ++j) {
      if (cell[j] < 0) continue;
      const DimState<R> st = dim_state<T, R, POLY>(uu[j], p);
      R w[T];
      all_taps<T, POLY>(st, p, w);
      for (int bb = 0; bb < nbt; ++bb) {
        C acc = czero<C>();
        if (nbt_cap > 0) {
          const C* row = box + bb * nbox + (cell[j] - cmin);
#pragma unroll
          for (int k = 0; k < T; ++k) cmac(acc, w[k], row[k]);
        } else {
          const C* src = grid + (int64_t)(b0 + bb) * p.Ld;
          const int64_t l0 = (int64_t)cell[j] - (m - 1);
          if (l0 >= 0 && l0 + T <= p.L) {
#pragma unroll
            for (int k = 0; k < T; ++k) cmac(acc, w[k], __ldg(&src[l0 + k]));
          } else {
#pragma unroll
            for (int k = 0; k < T; ++k) {
              const int64_t pos = l0 + k;
              if (pos >= 0 && pos < p.L) cmac(acc, w[k], __ldg(&src[pos]));
            }
          }
        }
        out[(int64_t)(b0 + bb) * p.n + dst[j]] = acc;
      }
    }
  }
}

template <int D, typename R, bool POLY, int MM>
static const void* kernel_for(int m) {
  if (m == MM) {
    if constexpr (D == 1) return (const void*)gather1_kernel<2 * MM, R, POLY>;
    else return (const void*)gather_kernel<D, 2 * MM, R, POLY>;
  }
  if constexpr (MM > 1) return kernel_for<D, R, POLY, MM - 1>(m);
  return nullptr;
}

constexpr int kMaxM1 = 16, kMaxM2 = 12, kMaxM3 = 8;

// one translation unit per (D, precision, tap mode) instantiates its kernels (parallel build)
const void* gather_kernel_1f(int m, bool poly);
const void* gather_kernel_1d(int m, bool poly);
const void* gather_kernel_2f(int m, bool poly);
const void* gather_kernel_2d(int m, bool poly);
const void* gather_kernel_3f(int m, bool poly);
const void* gather_kernel_3d(int m, bool poly);

}  // namespace bnfft
