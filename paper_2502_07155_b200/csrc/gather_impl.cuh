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
#include <cuda.h>

#include <algorithm>

#include "bnfft_internal.h"

namespace bnfft {

template <typename R> struct CT;
template <> struct CT<float> { using C = float2; };
template <> struct CT<double> { using C = double2; };

template <typename R> struct PolyN;
template <> struct PolyN<float> { static constexpr int NC = 10; };   // degree 9
template <> struct PolyN<double> { static constexpr int NC = 18; };  // degree 17
// Mirror symmetry: psi is even, so w_{2m-1-i}(u) = w_i(1-u), i.e. P_{2m-1-i}(x) = P_i(-x).  Only
// taps i < m are stored, split into even/odd parts P_i(x) = E_i(x^2) + x O_i(x^2); one Horner pass
// in y = x^2 over the pair (E_i, O_i) then gives both w_i = E + xO and w_{2m-1-i} = E - xO.
template <typename R> struct PolyH { static constexpr int NH = PolyN<R>::NC / 2; };

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
  int xs_user;            // xs in user order: node i of the sorted order is xs[perm[i]]
  R* pre_w;               // BNFFT_PRECOMPUTE_PSI: tap weights [n][2m] of the sorted nodes (or null)
  const uint32_t* key_start;   // binned kernel: first sorted position of each (user block, bin)
  int64_t nkeys;
  int tbox[3];            // binned kernel: TMA box extents per dim (dim 0 slowest), innermost padded
  int nslice;             // batch slices per unit (bt spectra each)
  int bufstride;          // binned kernel: elements between the staging buffers (128-B aligned)
  int nbuf;               // binned kernel: staging buffers (2 or 3), released by mbarrier
  int morton_bits;        // d = 3 cooperative kernel: bits per bin coordinate of the Z-order walk
  int64_t nkeys_morton;   // user blocks x 8^morton_bits
  int sorted_out;         // BNFFT_SORTED_OUTPUT: f written at the sorted position i, not at perm[i]
  int l2_hint;            // d = 3 y-sweep kernel: bit 0 outputs stored evict-first, bit 1 grid boxes evict-last
  WinParams wp;
  alignas(16) R ceo[PolyH<R>::NH][kMaxTaps / 2][2];   // [k][i][0] = E_i coeff k, [k][i][1] = O_i
};

__device__ __forceinline__ double sinpi_r(double u) { return sinpi(u); }
__device__ __forceinline__ float sinpi_r(float u) { return sinpif(u); }
__device__ __forceinline__ double phi_r(double tau, const WinParams& w) { return phi_tau_d(tau, w); }
__device__ __forceinline__ float phi_r(float tau, const WinParams& w) { return phi_tau_f(tau, w); }
__device__ __forceinline__ double sqrt_r(double v) { return sqrt(v); }
// complex64 edge factors: MUFU reciprocal square root times v (~2 ulp; taps need ~1e-7 absolute),
// v >= 0 (v == 0 only for Kronecker nodes, which do not use the factor)
__device__ __forceinline__ float sqrt_r(float v) {
  // v * rsqrt(v) with one MUFU op: the argument is clamped to a normal float, so the approximate,
  // flush-to-zero form needs no denormal fix-up (error ~1 ulp, below the complex64 tap-fit error)
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(v, 1e-30f)));
  return v * r;
}
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
  if constexpr (sizeof(R) == 4) st.x = fmaf(2.0f, st.u, -1.0f);   // complex64: from the rounded u
  else st.x = (R)(2.0 * u_d - 1.0);
  st.hit = (st.u == R(0)) ? m - 1 : ((st.u == R(1)) ? m : -1);
  if (p.wp.alg1) st.hit = -1;   // Algorithm 1: phi(l/L) is no Kronecker delta
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
  if (st.hit >= 0) return i == st.hit ? R(1) : R(0);
  if (POLY) {
    constexpr int NH = PolyH<R>::NH;
    const int ii = i < m ? i : T - 1 - i;
    const R xs = i < m ? st.x : -st.x;
    const R y = st.x * st.x;
    R e = p.ceo[NH - 1][ii][0], o = p.ceo[NH - 1][ii][1];
#pragma unroll
    for (int k = NH - 2; k >= 0; --k) {
      e = fma(e, y, p.ceo[k][ii][0]);
      o = fma(o, y, p.ceo[k][ii][1]);
    }
    R h = fma(xs, o, e);
    if (i == 0) h *= st.sq0;
    if (i == T - 1) h *= st.sq1;
    return h;
  } else {
    const int j = m - 1 - i;
    const R tau = st.u + (R)j;
    if (p.wp.alg1) return phi_r(tau, p.wp);          // Algorithm 1: the window itself
    const R sg = (j & 1) ? -st.s : st.s;
    return sg / (pi_r<R>() * tau) * phi_r(tau, p.wp);
  }
}

// All T taps of one dimension.  POLY: one Horner pass in y = x^2 over the (E_i, O_i) pairs of the
// m stored taps, packed FFMA2 (sm_100 fma.rn.f32x2) for float with the coefficient pair taken from
// the kernel parameters; then w_i = E + xO and w_{2m-1-i} = E - xO.
template <int T, bool POLY>
__device__ __forceinline__ void all_taps(const DimState<float>& st, const GatherParams<float>& p,
                                         float (&w)[T]) {
  if (!POLY || st.hit >= 0) {
#pragma unroll
    for (int k = 0; k < T; ++k) w[k] = tap_weight<T, float, POLY>(st, k, p);
    return;
  }
  constexpr int NH = PolyH<float>::NH;
  constexpr int m = T / 2;
  const float y = st.x * st.x;
  const float2 yy = make_float2(y, y);
  const float2 xm = make_float2(st.x, -st.x);
#pragma unroll
  for (int i = 0; i < m; ++i) {
    float2 h = *reinterpret_cast<const float2*>(p.ceo[NH - 1][i]);
#pragma unroll
    for (int k = NH - 2; k >= 0; --k) h = __ffma2_rn(h, yy, *reinterpret_cast<const float2*>(p.ceo[k][i]));
    const float2 r = __ffma2_rn(xm, make_float2(h.y, h.y), make_float2(h.x, h.x));
    w[i] = r.x;
    w[T - 1 - i] = r.y;
  }
  w[0] *= st.sq0;
  w[T - 1] *= st.sq1;
}

template <int T, bool POLY>
__device__ __forceinline__ void all_taps(const DimState<double>& st, const GatherParams<double>& p,
                                         double (&w)[T]) {
  if (!POLY || st.hit >= 0) {
#pragma unroll
    for (int k = 0; k < T; ++k) w[k] = tap_weight<T, double, POLY>(st, k, p);
    return;
  }
  constexpr int NH = PolyH<double>::NH;
  constexpr int m = T / 2;
  const double y = st.x * st.x;
#pragma unroll
  for (int i = 0; i < m; ++i) {
    double e = p.ceo[NH - 1][i][0], o = p.ceo[NH - 1][i][1];
#pragma unroll
    for (int k = NH - 2; k >= 0; --k) {
      e = fma(e, y, p.ceo[k][i][0]);
      o = fma(o, y, p.ceo[k][i][1]);
    }
    w[i] = fma(st.x, o, e);
    w[T - 1 - i] = fma(-st.x, o, e);
  }
  w[0] *= st.sq0;
  w[T - 1] *= st.sq1;
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
    const int64_t src = p.xs_user ? (int64_t)dst : i;
#pragma unroll
    for (int t = 0; t < D; ++t) {
      double xv = p.xs[src * D + t];
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
          out[(int64_t)(b0 + bb) * p.n + (p.sorted_out ? i : (int64_t)dst)] = res;
        }
      }
    }
  }
}

// d = 1 gather: persistent CTAs, TMA bulk-copy staging, software pipeline.
//
// Chunk k = sorted nodes [k*CH, (k+1)*CH), CH = 256*NPT (thread t takes k*CH + j*256 + t).  Nodes
// are sorted by bin inside user blocks, so a chunk's cells span a short range [cmin, cmax]; its grid
// window [cmin-m+1, cmax+m] is one contiguous range of theta, staged into shared memory by a single
// cp.async.bulk (TMA, completion on an mbarrier); parts outside I_L are zero-filled (reading A5).
// Per CTA iteration (chunk k): the window of chunk k+G is issued (its node data arrived during the
// previous iteration), the node data of chunk k+2G is loaded into registers, then chunk k is
// computed from its window, so both the node loads and the window copy overlap compute.  Windows
// larger than the buffer (sparse node sets) fall back to direct global loads for that chunk.
template <typename R> struct NPT1 { static constexpr int v = sizeof(R) == 4 ? 4 : 2; };

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <typename R, int NPT>
struct NodeSet1 {
  double x[NPT];
  uint32_t dst[NPT];
};

template <typename R, int NPT>
__device__ __forceinline__ void load_nodes1(const GatherParams<R>& p, int64_t chunk, NodeSet1<R, NPT>& ns) {
  const int64_t base = chunk * (int64_t)kGatherThreads * NPT + threadIdx.x;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int64_t i = base + j * kGatherThreads;
    if (i < p.n) {
      ns.dst[j] = __ldg(&p.perm[i]);
      ns.x[j] = __ldg(&p.xs[p.xs_user ? (int64_t)ns.dst[j] : i]);
    } else {
      ns.x[j] = 2.0;   // marks an inactive slot (valid nodes lie in [-1/2, 1/2))
      ns.dst[j] = 0;
    }
  }
}

// cell c in [0, L) and u in [0, 1]; returns false for inactive slots.
__device__ __forceinline__ bool node_cell(double xv, double Lf, int64_t L, int& c, double& u) {
  if (xv > 1.0) return false;
  const double Lx = __dmul_rn(Lf, xv);
  const double fl = floor(Lx);
  u = Lx - fl;
  const int L32 = (int)L;                  // L < 2^31
  int cc = __double2int_rz(fl) + (L32 >> 1);
  u = (cc > L32 - 1) ? 1.0 : u;            // fl(L x) == L/2 (defensive)
  c = min(cc, L32 - 1);
  return true;
}

struct Window1 {
  int64_t lo;      // grid index of buffer element 0 (16-byte aligned)
  int nbox;        // elements in the window
  int staged;      // 1: in shared memory, 0: read from global
};

// Block-wide cell range of a chunk -> window; thread 0 issues the bulk copy, all threads zero-fill
// the parts outside [0, L).  Contains one __syncthreads.
template <int T, typename R, int NPT>
__device__ __forceinline__ Window1 issue_window1(const GatherParams<R>& p, const NodeSet1<R, NPT>& ns,
                                                 typename CT<R>::C* buf, uint64_t* bar, int* s_red) {
  using C = typename CT<R>::C;
  constexpr int m = T / 2;
  constexpr int kAl = 16 / sizeof(C);   // elements per 16 bytes
  int cmin = 0x7fffffff, cmax = -1;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    int c;
    double u;
    if (node_cell(ns.x[j], p.Lf, p.L, c, u)) {
      cmin = min(cmin, c);
      cmax = max(cmax, c);
    }
  }
  cmin = __reduce_min_sync(0xffffffffu, cmin);
  cmax = __reduce_max_sync(0xffffffffu, cmax);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_red[wid] = cmin;
    s_red[8 + wid] = cmax;
  }
  __syncthreads();
#pragma unroll
  for (int w2 = 0; w2 < kGatherThreads / 32; ++w2) {
    cmin = min(cmin, s_red[w2]);
    cmax = max(cmax, s_red[8 + w2]);
  }
  Window1 win;
  int64_t lo = (int64_t)cmin - (m - 1);
  lo -= ((lo % kAl) + kAl) % kAl;                       // align down (lo may be negative)
  int64_t hi = (int64_t)cmax + m + 1;                   // exclusive
  hi += (kAl - (hi - lo) % kAl) % kAl;
  win.lo = lo;
  win.nbox = (int)(hi - lo);
  win.staged = win.nbox <= p.boxcap;
  if (win.staged) {
    const int64_t g0 = lo > 0 ? lo : (int64_t)0, g1 = hi < p.L ? hi : p.L;
    const bool periodic = p.wp.alg1 != 0;     // Algorithm 1: periodic index set (eq. indexset_x)
    if (threadIdx.x == 0) {
      const int64_t wlo = periodic ? (g0 - lo) : 0, whi = periodic ? (hi - g1) : 0;
      const uint32_t bytes = (uint32_t)((g1 - g0 + wlo + whi) * (int64_t)sizeof(C));
      mbar_expect_tx(bar, bytes);
      if (g1 > g0) tma_bulk_g2s(buf + (g0 - lo), (const C*)p.grid + g0, (uint32_t)((g1 - g0) * sizeof(C)), bar);
      if (wlo) tma_bulk_g2s(buf, (const C*)p.grid + (lo + p.L), (uint32_t)(wlo * sizeof(C)), bar);
      if (whi) tma_bulk_g2s(buf + (g1 - lo), (const C*)p.grid, (uint32_t)(whi * sizeof(C)), bar);
    }
    if (!periodic) {
      // zero extension outside I_L (generic stores, disjoint from the TMA range)
      for (int64_t q = threadIdx.x; q < g0 - lo; q += kGatherThreads) buf[q] = czero<C>();
      for (int64_t q = (g1 - lo) + threadIdx.x; q < hi - lo; q += kGatherThreads) buf[q] = czero<C>();
    }
  }
  return win;
}

// row stride of the precomputed weight table: 2m rounded up to 16 bytes (vector loads)
template <int T, typename R>
struct PreStride {
  static constexpr int V = 16 / (int)sizeof(R);
  static constexpr int v = (T + V - 1) / V * V;
};

template <int T, typename R, bool POLY, bool PRE = false>
__global__ void __launch_bounds__(kGatherThreads) gather1_kernel(const __grid_constant__ GatherParams<R> p) {
  using C = typename CT<R>::C;
  constexpr int NPT = NPT1<R>::v;
  constexpr int m = T / 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* buf0 = reinterpret_cast<C*>(smem_raw);
  C* buf1 = buf0 + p.boxcap;
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ int s_red[16];
  const int64_t CH = (int64_t)kGatherThreads * NPT;
  const int64_t nchunks = (p.n + CH - 1) / CH;
  const int64_t G = gridDim.x;
  int64_t k = blockIdx.x;
  if (k >= nchunks) return;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const C* __restrict__ grid = (const C*)p.grid;
  C* __restrict__ out = (C*)p.out;

  NodeSet1<R, NPT> cur, nxt;
  load_nodes1<R, NPT>(p, k, cur);
  Window1 wcur = issue_window1<T, R, NPT>(p, cur, buf0, &bars[0], s_red);
  if (k + G < nchunks) load_nodes1<R, NPT>(p, k + G, nxt);
  uint32_t phases = 0u;   // bit b: parity of the next completion of bars[b]
  for (int it = 0; k < nchunks; ++it, k += G) {
    const int b = it & 1;
    C* bcur = b ? buf1 : buf0;
    // (1) window of chunk k+G into the other buffer (its previous user, chunk k-G, finished before
    //     the barrier inside issue_window1)
    Window1 wnxt{0, 0, 0};
    if (k + G < nchunks) wnxt = issue_window1<T, R, NPT>(p, nxt, b ? buf0 : buf1, &bars[b ^ 1], s_red);
    else __syncthreads();   // zero-fill of the current window visible to all threads
    // (2) node data of chunk k+2G into registers (in flight during the compute below)
    NodeSet1<R, NPT> nn;
    if (k + 2 * G < nchunks) load_nodes1<R, NPT>(p, k + 2 * G, nn);
    // (3) compute chunk k
    if (wcur.staged) {
      mbar_wait(&bars[b], (phases >> b) & 1u);
      phases ^= 1u << b;
    }
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      int c;
      double u;
      if (!node_cell(cur.x[j], p.Lf, p.L, c, u)) continue;
      R w[T];
      if constexpr (PRE) {   // Algorithm 2 step 0(b): weights precomputed by set_nodes
        const int64_t i = k * (int64_t)kGatherThreads * NPT + j * kGatherThreads + threadIdx.x;
        const R* src = p.pre_w + i * PreStride<T, R>::v;
#pragma unroll
        for (int q = 0; q < T; q += 16 / (int)sizeof(R)) {
          if constexpr (sizeof(R) == 4) {
            const float4 v4 = __ldg(reinterpret_cast<const float4*>(src + q));
            w[q] = v4.x; w[q + 1] = v4.y;
            if (q + 2 < T) { w[q + 2] = v4.z; w[q + 3] = v4.w; }
          } else {
            const double2 v2 = __ldg(reinterpret_cast<const double2*>(src + q));
            w[q] = v2.x; w[q + 1] = v2.y;
          }
        }
      } else {
        const DimState<R> st = dim_state<T, R, POLY>(u, p);
        all_taps<T, POLY>(st, p, w);
      }
      C acc = czero<C>();
      if (wcur.staged) {
        const C* row = bcur + (c - (m - 1) - wcur.lo);
#pragma unroll
        for (int kk = 0; kk < T; ++kk) cmac(acc, w[kk], row[kk]);
      } else {
        const int64_t l0 = (int64_t)c - (m - 1);
#pragma unroll
        for (int kk = 0; kk < T; ++kk) {
          int64_t pos = l0 + kk;
          if (p.wp.alg1) pos = pos < 0 ? pos + p.L : (pos >= p.L ? pos - p.L : pos);
          if (pos >= 0 && pos < p.L) cmac(acc, w[kk], __ldg(&grid[pos]));
        }
      }
      out[p.sorted_out ? k * (int64_t)kGatherThreads * NPT + j * kGatherThreads + threadIdx.x : (int64_t)cur.dst[j]] = acc;
    }
    cur = nxt;
    nxt = nn;
    wcur = wnxt;
  }
}

// ---- d = 1, batch 1, large grids (plan.d1_binned): bins of W = 2^bin_log2 cells, so the sort key
// (user block, bin) is a single radix digit.  Work item = one key: its nodes [key_start[k],
// key_start[k+1]) and the fixed window [bin*W - m + 1, bin*W + W + m) (16-byte aligned; zero outside
// I_L, reading A5, or wrapped for Algorithm 1).  Persistent CTAs take keys k = blockIdx.x + j*gridDim;
// the window of the CTA's next key is in flight (TMA bulk copy, mbarrier) while the current key's
// nodes are contracted, 256 * NPT at a time with the next batch's node data prefetched into registers.
template <typename R, int NPT, int NT>
__device__ __forceinline__ void load_nodes_range(const GatherParams<R>& p, int64_t base, int64_t end,
                                                 NodeSet1<R, NPT>& ns) {
  if (p.xs_user) {   // user-order node copy: x[perm[i]] (dependent loads)
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int64_t i = base + j * NT + threadIdx.x;
      ns.dst[j] = i < end ? __ldg(&p.perm[i]) : 0u;
      ns.x[j] = i < end ? __ldg(&p.xs[ns.dst[j]]) : 2.0;   // 2.0: inactive slot
    }
  } else {            // sorted node copy: independent streaming loads
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int64_t i = base + j * NT + threadIdx.x;
      ns.dst[j] = i < end ? __ldg(&p.perm[i]) : 0u;
      ns.x[j] = i < end ? __ldg(&p.xs[i]) : 2.0;
    }
  }
}

template <typename R>
__device__ __forceinline__ int64_t bin_window_lo(const GatherParams<R>& p, int64_t bin, int m) {
  constexpr int EPV = 16 / (int)sizeof(typename CT<R>::C);
  int64_t lo = (bin << p.log2W[0]) - (m - 1);
  lo -= ((lo % EPV) + EPV) % EPV;
  return lo;
}

// Thread 0 only: window of key k into buf -- zero extension outside I_L (reading A5; generic stores
// published by the expect_tx arrive that follows them) or wrapped copies (Algorithm 1), then the TMA
// bulk copies completing on bar.
template <typename R>
__device__ __forceinline__ void issue_bin_window(const GatherParams<R>& p, int64_t k, int m,
                                                 typename CT<R>::C* buf, uint64_t* bar) {
  using C = typename CT<R>::C;
  const int64_t lo = bin_window_lo(p, k % p.nb[0], m);
  const int64_t hi = lo + p.boxcap;
  const int64_t g0 = lo > 0 ? lo : (int64_t)0, g1 = hi < p.L ? hi : p.L;
  const bool periodic = p.wp.alg1 != 0;
  const int64_t wlo = periodic ? (g0 - lo) : 0, whi = periodic ? (hi - g1) : 0;
  if (!periodic) {
    for (int64_t q = 0; q < g0 - lo; ++q) buf[q] = czero<C>();
    for (int64_t q = g1 - lo; q < hi - lo; ++q) buf[q] = czero<C>();
  }
  mbar_expect_tx(bar, (uint32_t)((g1 - g0 + wlo + whi) * (int64_t)sizeof(C)));
  if (g1 > g0) tma_bulk_g2s(buf + (g0 - lo), (const C*)p.grid + g0, (uint32_t)((g1 - g0) * sizeof(C)), bar);
  if (wlo) tma_bulk_g2s(buf, (const C*)p.grid + (lo + p.L), (uint32_t)(wlo * sizeof(C)), bar);
  if (whi) tma_bulk_g2s(buf + (g1 - lo), (const C*)p.grid, (uint32_t)(whi * sizeof(C)), bar);
}

constexpr int kGather1bThreads = 512;
constexpr int kGather1bBufs = 3;   // window buffers: the issuer needs only the key before last released

template <int T, typename R, bool POLY>
__global__ void __launch_bounds__(kGather1bThreads, 2) gather1b_kernel(const __grid_constant__ GatherParams<R> p) {
  using C = typename CT<R>::C;
  constexpr int NPT = NPT1<R>::v;
  constexpr int m = T / 2;
  constexpr int NT = kGather1bThreads;
  constexpr int NB = kGather1bBufs;
  constexpr int64_t CHN = (int64_t)NT * NPT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* bufs = reinterpret_cast<C*>(smem_raw);
  __shared__ __align__(8) uint64_t full[NB], empty[NB];
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NT);
    }
    fence_mbar_init();
  }
  __syncthreads();
  C* __restrict__ out = (C*)p.out;
  const int64_t G = gridDim.x, k0 = blockIdx.x;
  auto nonempty = [&](int64_t k) { return __ldg(&p.key_start[k + 1]) > __ldg(&p.key_start[k]); };
  // prologue: windows of the first NB-1 keys
  if (threadIdx.x == 0) {
    for (int t = 0; t < NB - 1; ++t) {
      const int64_t k = k0 + t * G;
      if (k < p.nkeys && nonempty(k)) issue_bin_window<R>(p, k, m, bufs + t * p.boxcap, &full[t]);
    }
  }
  int64_t s0 = 0, s1 = 0;
  NodeSet1<R, NPT> cur, nxt;
  if (k0 < p.nkeys) {
    s0 = __ldg(&p.key_start[k0]);
    s1 = __ldg(&p.key_start[k0 + 1]);
    load_nodes_range<R, NPT, NT>(p, s0, s1, cur);
  }
  uint32_t fph = 0u;   // parity of the next completion of full[b]
  for (int t = 0; k0 + t * G < p.nkeys; ++t) {
    const int64_t k = k0 + t * G;
    const int b = t % NB;
    // window of key t+NB-1 into the buffer of key t-1 (thread 0 waits until every thread released it)
    if (threadIdx.x == 0) {
      const int64_t kn = k + (NB - 1) * G;
      if (kn < p.nkeys && nonempty(kn)) {
        const int bn = (t + NB - 1) % NB;
        if (t >= 1) mbar_wait(&empty[bn], (uint32_t)((t - 1) / NB) & 1u);
        issue_bin_window<R>(p, kn, m, bufs + bn * p.boxcap, &full[bn]);
      }
    }
    // first chunk of the next key in flight while this key is contracted
    int64_t s0n = 0, s1n = 0;
    if (k + G < p.nkeys) {
      s0n = __ldg(&p.key_start[k + G]);
      s1n = __ldg(&p.key_start[k + G + 1]);
      load_nodes_range<R, NPT, NT>(p, s0n, s1n, nxt);
    }
    if (s1 > s0) {
      mbar_wait(&full[b], (fph >> b) & 1u);
      fph ^= 1u << b;
      const C* bcur = bufs + b * p.boxcap;
      const int64_t lo = bin_window_lo(p, k % p.nb[0], m);
      for (int64_t base = s0; base < s1; base += CHN) {
        if (base > s0) load_nodes_range<R, NPT, NT>(p, base, s1, cur);   // tail chunks (rare)
#pragma unroll
        for (int j = 0; j < NPT; ++j) {
          int c;
          double u;
          if (!node_cell(cur.x[j], p.Lf, p.L, c, u)) continue;
          const DimState<R> st = dim_state<T, R, POLY>(u, p);
          R w[T];
          all_taps<T, POLY>(st, p, w);
          C acc = czero<C>();
          const C* row = bcur + (c - (m - 1) - lo);
#pragma unroll
          for (int kk = 0; kk < T; ++kk) cmac(acc, w[kk], row[kk]);
          out[p.sorted_out ? base + j * NT + threadIdx.x : (int64_t)cur.dst[j]] = acc;
        }
      }
    }
    mbar_arrive(&empty[b]);   // this thread is done with buffer b
    cur = nxt;
    s0 = s0n;
    s1 = s1n;
  }
}

// D == 1: the pipelined window kernel (batch == 1) or, for batched d = 1 plans, the generic
// segment kernel (returned for m + 100); m + 200: the step 0(b) weight kernel, m + 300: the window
// kernel reading those weights.
// d = 2, 3 gather: persistent CTAs over the sort keys (user block, bin), TMA tensor staging.
//
// Work item = (key u, batch slice s).  The bin's grid neighbourhood (bin + (m-1, m) halo) is one box
// of the theta tensor; cp.async.bulk.tensor copies it into shared memory with out-of-bound elements
// zero-filled by the TMA unit (zero extension outside I_L, reading A5).  Items are double-buffered:
// the box of the CTA's next item is in flight while the current one is contracted.  The nodes of
// the key are processed 256 at a time; each thread evaluates its node's tap polynomials (all dims)
// and contracts the (2m)^d taps from shared memory in a fixed order.
__device__ __forceinline__ void tma_load_box(const CUtensorMap* tm, void* dst, uint64_t* bar, int rank,
                                             const int* c) {
  const uint32_t d = smem_u32(dst), b = smem_u32(bar);
  const uint64_t t = reinterpret_cast<uint64_t>(tm);
  if (rank == 2)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(d), "l"(t), "r"(b), "r"(c[0]), "r"(c[1]) : "memory");
  else if (rank == 3)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(d), "l"(t), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory");
  else if (rank == 4)
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
        ::"r"(d), "l"(t), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
        ::"r"(d), "l"(t), "r"(b), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
}

// Issue the box of item (u, s) (thread 0 only).  The tensor map lives in global memory (written once
// at plan creation).  Tensor coordinates are innermost first; complex128
// adds an innermost dimension of 2 doubles; batch is the outermost dimension.
template <int D, typename R>
__device__ __forceinline__ void issue_box(const GatherParams<R>& p, const CUtensorMap* tm, int64_t u, int sl,
                                          void* dst, uint64_t* bar, uint32_t bytes) {
  int64_t nbins = 1;
#pragma unroll
  for (int t = 0; t < D; ++t) nbins *= p.nb[t];
  uint32_t rem = (uint32_t)(u % nbins);
  int org[3];
#pragma unroll
  for (int t = D - 1; t >= 0; --t) {
    const uint32_t bt = rem % (uint32_t)p.nb[t];
    rem /= (uint32_t)p.nb[t];
    org[t] = (int)((int64_t)bt << p.log2W[t]) - (p.wp.m - 1);
  }
  // the innermost box start must be 16-byte aligned: complex64 boxes start at an even z (the box
  // is one element wider than the halo needs; the kernel adds the shift back)
  if (sizeof(R) == 4) org[D - 1] &= ~1;
  int c[5];
  int r = 0;
  if (sizeof(R) == 8) c[r++] = 0;                // complex128: re/im pair
#pragma unroll
  for (int t = D - 1; t >= 0; --t) c[r++] = org[t];
  if (p.batch > 1) c[r++] = sl * p.bt;
  mbar_expect_tx(bar, bytes);
  tma_load_box(tm, dst, bar, r, c);
}

constexpr int kMaxBoxBufs = 6;

template <int D, int T, typename R, bool POLY>
__global__ void __launch_bounds__(kGatherThreads) gatherN_kernel(const __grid_constant__ GatherParams<R> p,
                                                                 const CUtensorMap* __restrict__ tmap) {
  using C = typename CT<R>::C;
  constexpr int m = T / 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxBoxBufs], empty[kMaxBoxBufs];
  __shared__ int64_t s_u[kMaxBoxBufs];   // item (key) staged in each buffer, -1: end of the CTA's items
  __shared__ int s_sl[kMaxBoxBufs];
  const int BZ = p.tbox[D - 1];                      // innermost (padded) extent
  const int BY = D == 3 ? p.tbox[1] : 1;
  const int box_elems = p.box_elems;                 // per spectrum (with padding)
  const uint32_t buf_elems = (uint32_t)box_elems * p.bt;
  C* const buf0 = reinterpret_cast<C*>(smem_raw);
  const uint32_t bytes = buf_elems * (uint32_t)sizeof(C);
  const int64_t G = gridDim.x;
  const int nsl = p.nslice;
  const int NB = p.nbuf;
  C* __restrict__ out = (C*)p.out;

  // The CTA's item sequence: keys u = blockIdx.x + j*G (non-empty ones), slices 0..nsl-1 each.
  // Item i uses buffer i % NB.  Thread 0 walks the sequence and stages item i + NB - 1 (descriptor in
  // s_u / s_sl, box by TMA) once every thread has released item i - 1, the previous user of that
  // buffer; so NB - 1 boxes are in flight while an item is contracted (small items: deep ring).
  int64_t wu = blockIdx.x;   // thread 0's walk position
  int wsl = 0;
  auto next_key = [&](int64_t u) -> int64_t {
    while (u < p.nkeys && __ldg(&p.key_start[u + 1]) == __ldg(&p.key_start[u])) u += G;
    return u;
  };
  auto stage = [&](int bq) {   // thread 0: the next item of the walk into buffer bq (or the end mark)
    if (wu < p.nkeys) {
      s_u[bq] = wu;
      s_sl[bq] = wsl;
      issue_box<D, R>(p, tmap, wu, wsl, buf0 + bq * p.bufstride, &full[bq], bytes);
      if (++wsl == nsl) {
        wsl = 0;
        wu = next_key(wu + G);
      }
    } else {
      s_u[bq] = -1;
      mbar_arrive(&full[bq]);   // completes the phase: waiters read the end mark
    }
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < NB; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], blockDim.x);
    }
    fence_mbar_init();
    wu = next_key(wu);
    for (int q = 0; q < NB - 1; ++q) stage(q);
  }
  __syncthreads();
  for (int it = 0;; ++it) {
    const int b = it % NB;
    if (threadIdx.x == 0) {
      const int bn = (it + NB - 1) % NB;
      if (it >= 1 && NB > 2) mbar_wait(&empty[bn], (uint32_t)((it - 1) / NB) & 1u);
      stage(bn);   // NB == 2: the CTA barrier at the end of item it-1 released the buffer
    }
    mbar_wait(&full[b], (uint32_t)(it / NB) & 1u);
    const int64_t u = s_u[b];
    if (u < 0) break;
    const int sl = s_sl[b];
    const C* box = buf0 + b * p.bufstride;
    // bin origin (cells) of key u
    int64_t nbins = 1;
#pragma unroll
    for (int t = 0; t < D; ++t) nbins *= p.nb[t];
    uint32_t rem = (uint32_t)(u % nbins);
    int bo[3];
#pragma unroll
    for (int t = D - 1; t >= 0; --t) {
      const uint32_t bt = rem % (uint32_t)p.nb[t];
      rem /= (uint32_t)p.nb[t];
      bo[t] = (int)(bt << p.log2W[t]);
    }
    const int64_t i_beg = __ldg(&p.key_start[u]), i_end = __ldg(&p.key_start[u + 1]);
    const int nbt = min(p.bt, p.batch - sl * p.bt);
    for (int64_t i = i_beg + threadIdx.x; i < i_end; i += blockDim.x) {
      const uint32_t dst = __ldg(&p.perm[i]);
      const int64_t src = p.xs_user ? (int64_t)dst : i;
      int off[3];
      R w[D][T];
#pragma unroll
      for (int t = 0; t < D; ++t) {
        const double Lx = __dmul_rn(p.Lf, __ldg(&p.xs[src * D + t]));
        const double fl = floor(Lx);
        double uu = Lx - fl;
        int64_t c = (int64_t)fl + p.L / 2;
        if (c > p.L - 1) { c = p.L - 1; uu = 1.0; }
        off[t] = (int)c - bo[t];
        if (sizeof(R) == 4 && t == D - 1) off[t] += (bo[t] - (m - 1)) & 1;   // even-aligned box start
        const DimState<R> st = dim_state<T, R, POLY>(uu, p);
        all_taps<T, POLY>(st, p, w[t]);
      }
      for (int bb = 0; bb < nbt; ++bb) {
        const C* bx = box + bb * box_elems;
        C acc = czero<C>();
        if (D == 2) {
#pragma unroll
          for (int a = 0; a < T; ++a) {
            const C* row = bx + (off[0] + a) * BZ + off[1];
            C racc = czero<C>();
#pragma unroll
            for (int k = 0; k < T; ++k) cmac(racc, w[1][k], row[k]);
            cmac(acc, w[0][a], racc);
          }
        } else {
#pragma unroll 1
          for (int a = 0; a < T; ++a) {
            const C* plane = bx + (off[0] + a) * BY * BZ;
            C pacc = czero<C>();
#pragma unroll
            for (int bq = 0; bq < T; ++bq) {
              const C* row = plane + (off[1] + bq) * BZ + off[2];
              C racc = czero<C>();
#pragma unroll
              for (int k = 0; k < T; ++k) cmac(racc, w[2][k], row[k]);
              cmac(pacc, w[1][bq], racc);
            }
            R wa = w[0][0];
#pragma unroll
            for (int q = 1; q < T; ++q) wa = (a == q) ? w[0][q] : wa;
            cmac(acc, wa, pacc);
          }
        }
        out[(int64_t)(sl * p.bt + bb) * p.n + (p.sorted_out ? i : (int64_t)dst)] = acc;
      }
    }
    // buffer b is refilled NB-1 items later: handed back per thread by mbarrier, or (two large
    // batched boxes) by a CTA barrier, which measured faster there (cfg5)
    if (NB > 2) mbar_arrive(&empty[b]);
    else __syncthreads();
  }
}

// Morton (Z-order) index v -> row-major bin key (or -1 when the decoded bin lies outside the bin
// grid, which is padded to powers of two for the interleaving); user block = v >> 3*mbits.
__device__ __forceinline__ int64_t morton_key3(int64_t v, const GatherParams<float>& p) {
  const int mb = p.morton_bits;
  const int64_t blk = v >> (3 * mb);
  uint32_t c[3] = {0u, 0u, 0u};
  uint32_t vv = (uint32_t)(v & ((1ll << (3 * mb)) - 1));
  for (int bit = 0; bit < mb; ++bit) {
    c[2] |= ((vv >> (3 * bit)) & 1u) << bit;
    c[1] |= ((vv >> (3 * bit + 1)) & 1u) << bit;
    c[0] |= ((vv >> (3 * bit + 2)) & 1u) << bit;
  }
  if (c[0] >= (uint32_t)p.nb[0] || c[1] >= (uint32_t)p.nb[1] || c[2] >= (uint32_t)p.nb[2]) return -1;
  const int64_t nbins = p.nb[0] * p.nb[1] * p.nb[2];
  return blk * nbins + ((int64_t)c[0] * p.nb[1] + c[1]) * p.nb[2] + c[2];
}

// d = 3, m = 4, complex64, batch 1: half-warp-cooperative contraction (TMA staging as gatherN).
//
// With one node per thread, the 32 lanes of a warp read 32 unrelated rows of the box: random
// 8-byte shared-memory accesses with ~4-way bank conflicts.  Here each half-warp contracts one
// node: lane (r, c) = ((lane >> 3) & 1, lane & 7) reads z index c of rows b = 2k + r, k < 4, of every
// x-plane.  The box rows hold kRow3 = 24 elements (192 B; bins are 8 x 8 x 16 cells, so 16 + 2m = 24
// is exactly the halo extent), which puts rows b and b+1 16 banks apart: each half-warp phase of an
// LDS.64 reads two conflict-free 64-byte rows, 2 wavefronts per instruction (the minimum).  Lanes
// first prepare 32 nodes (cells, the 24 tap weights) into a per-warp stash; then the half-warps
// contract the stashed nodes pairwise and reduce over their 16 lanes with shuffles.
constexpr int kRow3 = 24;

template <bool POLY>
__global__ void __launch_bounds__(kGatherThreads) gather3c_kernel(const __grid_constant__ GatherParams<float> p,
                                                                  const CUtensorMap* __restrict__ tmap) {
  using C = float2;
  constexpr int T = 8, m = 4, D = 3;
  constexpr int kW = kGatherThreads / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[1];
  // per stashed node: x weights [0,8), y weights split by parity [8,16) = (w_y[0], w_y[2], w_y[4],
  // w_y[6], w_y[1], ...), z weights [16,24); offsets + destination as one int4
  __shared__ __align__(16) float s_w[kW][32][3 * T];
  __shared__ __align__(16) int4 s_od[kW][32];
  const int BZ = kRow3, BY = p.tbox[1];
  const int box_elems = p.box_elems;
  const uint32_t bytes = (uint32_t)box_elems * (uint32_t)sizeof(C);
  C* const box = reinterpret_cast<C*>(smem_raw);
  const int64_t G = gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int hw = lane >> 4, rr = (lane >> 3) & 1, cz = lane & 7;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    fence_mbar_init();
  }
  __syncthreads();
  C* __restrict__ out = (C*)p.out;
  uint32_t phase = 0u;
  // keys visited in Morton (Z) order of the bin coordinates, so that the bins in flight at one time
  // form a compact 3-D block and their halos are served from L2
  const int64_t nvirt = p.nkeys_morton;
  for (int64_t v = blockIdx.x; v < nvirt; v += G) {
    const int64_t u = morton_key3(v, p);
    if (u < 0) continue;
    const int64_t i_beg = __ldg(&p.key_start[u]), i_end = __ldg(&p.key_start[u + 1]);
    if (i_beg == i_end) continue;
    if (threadIdx.x == 0) issue_box<D, float>(p, tmap, u, 0, box, &bars[0], bytes);
    // bin origin (cells)
    const int64_t nbins = p.nb[0] * p.nb[1] * p.nb[2];
    uint32_t rem = (uint32_t)(u % nbins);
    int bo[3];
#pragma unroll
    for (int t = D - 1; t >= 0; --t) {
      const uint32_t btc = rem % (uint32_t)p.nb[t];
      rem /= (uint32_t)p.nb[t];
      bo[t] = (int)(btc << p.log2W[t]);
    }
    const int zshift = (bo[2] - (m - 1)) & 1;      // even-aligned box start (issue_box)
    bool waited = false;
    for (int64_t g0 = i_beg + (int64_t)wid * 32; g0 < i_end; g0 += kGatherThreads) {
      // ---- stash: lane prepares node g0 + lane (overlaps the TMA of the box)
      const int nn = (int)min((int64_t)32, i_end - g0);
      if (lane < nn) {
        const int64_t i = g0 + lane;
        const uint32_t dst = __ldg(&p.perm[i]);
        const int64_t src = p.xs_user ? (int64_t)dst : i;
        int od[3];
#pragma unroll
        for (int t = 0; t < D; ++t) {
          const double Lx = __dmul_rn(p.Lf, __ldg(&p.xs[src * D + t]));
          const double fl = floor(Lx);
          double uu = Lx - fl;
          int64_t c = (int64_t)fl + p.L / 2;
          if (c > p.L - 1) { c = p.L - 1; uu = 1.0; }
          int o = (int)c - bo[t];
          if (t == D - 1) o += zshift;
          od[t] = o;
          const DimState<float> st = dim_state<T, float, POLY>(uu, p);
          float w[T];
          all_taps<T, POLY>(st, p, w);
          float4* sw = reinterpret_cast<float4*>(&s_w[wid][lane][t * T]);
          if (t == 1) {
            sw[0] = make_float4(w[0], w[2], w[4], w[6]);
            sw[1] = make_float4(w[1], w[3], w[5], w[7]);
          } else {
            sw[0] = make_float4(w[0], w[1], w[2], w[3]);
            sw[1] = make_float4(w[4], w[5], w[6], w[7]);
          }
        }
        s_od[wid][lane] = make_int4(od[0], od[1], od[2], p.sorted_out ? (int)i : (int)dst);
      }
      __syncwarp();
      if (!waited) {
        mbar_wait(&bars[0], phase);
        waited = true;
      }
      // ---- contract stashed nodes two at a time (half-warp hw takes node q + hw)
      for (int q0 = 0; q0 < nn; q0 += 2) {
        const int q = min(q0 + hw, nn - 1);
        const int4 od = s_od[wid][q];
        const float4 wx0 = *reinterpret_cast<const float4*>(&s_w[wid][q][0]);
        const float4 wx1 = *reinterpret_cast<const float4*>(&s_w[wid][q][4]);
        const float4 wy = *reinterpret_cast<const float4*>(&s_w[wid][q][T + 4 * rr]);
        const float wxa[T] = {wx0.x, wx0.y, wx0.z, wx0.w, wx1.x, wx1.y, wx1.z, wx1.w};
        const float wyk[T / 2] = {wy.x, wy.y, wy.z, wy.w};
        const C* bx = box + ((od.x * BY + od.y + rr) * BZ + od.z + cz);
        C acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < T; ++a) {
          const C* pl = bx + a * BY * BZ;
          C t = make_float2(0.f, 0.f);
#pragma unroll
          for (int k = 0; k < T / 2; ++k) cmac(t, wyk[k], pl[2 * k * BZ]);
          cmac(acc, wxa[a], t);
        }
        const float wz = s_w[wid][q][2 * T + cz];
        acc = __fmul2_rn(make_float2(wz, wz), acc);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        }
        if ((lane & 15) == 0 && q0 + hw < nn) out[(uint32_t)od.w] = acc;
      }
      __syncwarp();
    }
    if (!waited) mbar_wait(&bars[0], phase);   // warps without nodes still consume the phase
    phase ^= 1u;
    __syncthreads();   // box free before the next item's TMA
  }
}

// Algorithm 2 step 0(b), d = 1: the 2m weights psi(x_j - l/L) of every sorted node, stored
// [n][2m] for the gather (BNFFT_PRECOMPUTE_PSI).
template <int T, typename R, bool POLY>
__global__ void __launch_bounds__(kGatherThreads) prepsi1_kernel(const __grid_constant__ GatherParams<R> p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t dst = __ldg(&p.perm[i]);
    int c = 0;
    double u = 0.0;
    node_cell(__ldg(&p.xs[p.xs_user ? (int64_t)dst : i]), p.Lf, p.L, c, u);
    const DimState<R> st = dim_state<T, R, POLY>(u, p);
    R w[T];
    all_taps<T, POLY>(st, p, w);
    R* o = p.pre_w + i * PreStride<T, R>::v;
#pragma unroll
    for (int k = 0; k < T; ++k) o[k] = w[k];
  }
}

template <int D, typename R, bool POLY, int MM>
static const void* kernel_for(int m) {
  if (m == MM) {
    if constexpr (D == 1) return (const void*)gather1_kernel<2 * MM, R, POLY>;
    else return (const void*)gatherN_kernel<D, 2 * MM, R, POLY>;
  }
  if constexpr (D == 1) {
    if (m == MM + 100) return (const void*)gather_kernel<1, 2 * MM, R, POLY>;
    if (m == MM + 200) return (const void*)prepsi1_kernel<2 * MM, R, POLY>;
    if (m == MM + 300) return (const void*)gather1_kernel<2 * MM, R, POLY, true>;
    if (m == MM + 400) return (const void*)gather1b_kernel<2 * MM, R, POLY>;
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
