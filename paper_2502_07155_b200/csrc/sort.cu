// Row a1: node preprocessing (set_nodes).  Validation + bin keys (K1), stable LSD radix sort of
// (key, user index) pairs (K2), sorted node copy and bin offsets (K3).  Hand-written, deterministic:
// no atomics decide any position, so the permutation is bit-identical to a stable argsort of
// the keys (reading A14: ties broken by the original index).
//
// Cell of a node (P:467-474 with reading A6): c_t = floor(L x_t), the grid point with l_t <= L x_t;
// stored shifted to [0, L) as c_t + L/2.  L*x_t is one IEEE double product (__dmul_rn, never
// contracted into an FMA).
#include <algorithm>

#include "bnfft_internal.h"

namespace bnfft {

struct KeyParams {
  int d;
  int64_t L;
  double Lf;
  int log2W[3];
  int64_t nb[3];
  int strict;
  double box_lo, box_hi;
  int colbits;       // rec3 plans: minor key digit = c_1 mod 2^colbits (the y column inside the bin)
};

enum { BAD_NOT_FINITE = 1, BAD_RANGE = 2, BAD_BOX = 3 };

struct SegLayout {
  int64_t tpb;      // tiles per user block
  int64_t ntiles;
};
__device__ __forceinline__ int64_t hist_index(const SegLayout& sl, int64_t tile, int dg, int ndig) {
  const int64_t blk = tile / sl.tpb;
  const int64_t tib = tile - blk * sl.tpb;
  const int64_t tin = min(sl.tpb, sl.ntiles - blk * sl.tpb);
  return blk * sl.tpb * ndig + (int64_t)dg * tin + tib;
}

// rec3 plans: the minor key digit below the x-line bin.  colbits == 4 (gather3y): the y column c_1 mod 16;
// colbits == 5 (gather3q): (half of the bin's z extent, y column) = ((c_2 >> 2) & 1) << 4 | c_1 mod 16.
__device__ __forceinline__ uint32_t minor_digit(uint32_t cy, uint32_t cz, int colbits) {
  return colbits == 5 ? ((((cz >> 2) & 1u) << 4) | (cy & 15u)) : (cy & ((1u << colbits) - 1u));
}

// K1: validate + key.  bad = min over nodes of (index << 4 | code).  Each thread handles a pair of
// consecutive nodes with 16-byte loads/stores (2*D doubles, 2 keys).
// The common case in one pass: all coordinates in [-1/2, 1/2) (NaN fails the comparison) and, with
// STRICT_DOMAIN, inside the closed feasible box; the caller falls back to node_key for the error code.
template <int D>
__device__ __forceinline__ bool node_key_fast(const double* xv, const KeyParams& kp, uint32_t& key) {
  bool ok = true;
  key = 0;
  uint32_t cy = 0, cz = 0;
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const double v = xv[t];
    ok &= (v >= -0.5) & (v < 0.5);
    if (kp.strict) ok &= (v >= kp.box_lo) & (v <= kp.box_hi);
    const double Lx = __dmul_rn(kp.Lf, v);
    int c = __double2int_rz(floor(Lx)) + (int)(kp.L >> 1);
    c = min(c, (int)kp.L - 1);
    key = key * (uint32_t)kp.nb[t] + ((uint32_t)c >> kp.log2W[t]);
    if (t == 1) cy = (uint32_t)c;
    if (t == 2) cz = (uint32_t)c;
  }
  if (D >= 2 && kp.colbits) key = (key << kp.colbits) | minor_digit(cy, cz, kp.colbits);
  if (!ok) key = 0;
  return ok;
}

template <int D>
__device__ __forceinline__ uint32_t node_key(const double* xv, const KeyParams& kp, int& code) {
  uint32_t key = 0, cy = 0, cz = 0;
  bool nonfinite = false, range = false, box = false;
#pragma unroll
  for (int t = 0; t < D; ++t) {
    const double v = xv[t];
    if (!isfinite(v)) { nonfinite = true; continue; }
    if (!(v >= -0.5 && v < 0.5)) { range = true; continue; }
    if (kp.strict && !(v >= kp.box_lo && v <= kp.box_hi)) box = true;
    const double Lx = __dmul_rn(kp.Lf, v);
    int c = __double2int_rz(floor(Lx)) + (int)(kp.L >> 1);
    c = min(c, (int)kp.L - 1);         // fl(L x) == L/2 for x < 1/2 (defensive)
    key = key * (uint32_t)kp.nb[t] + ((uint32_t)c >> kp.log2W[t]);
    if (t == 1) cy = (uint32_t)c;
    if (t == 2) cz = (uint32_t)c;
  }
  if (D >= 2 && kp.colbits) key = (key << kp.colbits) | minor_digit(cy, cz, kp.colbits);
  code = nonfinite ? BAD_NOT_FINITE : range ? BAD_RANGE : box ? BAD_BOX : 0;
  return code ? 0u : key;
}

// rec3 plans (y-sweep gather, d = 3): the node's record for the gather, computed here once in user
// order -- u_t = L x_t - floor(L x_t) rounded to float (the complex64 path's u, reading A11), and
// the cell's position in its 1 x 16 x 8 x-line bin ((c_y & 15) << 3 | (c_z & 7)); clamped cells
// (fl(L x) == L/2) take u = 1 as in every gather.
__device__ __forceinline__ float4 node_rec3(const double* xv, const KeyParams& kp) {
  float u[3];
  int c[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const double Lx = __dmul_rn(kp.Lf, xv[t]);
    const double fl = floor(Lx);
    double w = Lx - fl;
    int ci = __double2int_rz(fl) + (int)(kp.L >> 1);
    if (ci > (int)kp.L - 1) {
      ci = (int)kp.L - 1;
      w = 1.0;
    }
    u[t] = (float)w;
    c[t] = ci;
  }
  // cell position in the bin: (column << 3 | z offset) for gather3y; (minor digit << 2 | z offset inside
  // the half) for gather3q
  const uint32_t md = kp.colbits == 5 ? ((minor_digit((uint32_t)c[1], (uint32_t)c[2], 5) << 2) | (uint32_t)(c[2] & 3))
                                      : (uint32_t)(((c[1] & 15) << 3) | (c[2] & 7));
  return make_float4(u[0], u[1], u[2], __uint_as_float(md));
}

template <int D>
__global__ void keys_kernel(const double* __restrict__ x, int64_t n, KeyParams kp,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                            unsigned long long* __restrict__ bad, double* __restrict__ xcopy,
                            int aligned16, float4* __restrict__ rec) {
  // xcopy != nullptr: user-order node copy (d <= 2 user-blocked plans: the gather reads xcopy[perm[i]]
  // inside an L2-resident user block; or no radix pass: the identity permutation).
  // vals (identity permutation) is only written when no radix pass will run; the first pass
  // generates v = index itself.  aligned16 == 0 (x not 16-byte aligned): scalar loads.
  const int64_t npair = (n + 1) / 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npair;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = 2 * q;
    double xv[2 * D];
    const bool full = i + 1 < n;
    if (full && aligned16) {
      const double2* src = reinterpret_cast<const double2*>(x + i * D);
#pragma unroll
      for (int h = 0; h < D; ++h) {
        const double2 v = __ldg(&src[h]);
        xv[2 * h] = v.x;
        xv[2 * h + 1] = v.y;
      }
      if (xcopy) {
        double2* dstc = reinterpret_cast<double2*>(xcopy + i * D);
#pragma unroll
        for (int h = 0; h < D; ++h) dstc[h] = make_double2(xv[2 * h], xv[2 * h + 1]);
      }
    } else {
#pragma unroll
      for (int t = 0; t < 2 * D; ++t) {
        const bool in = t < D || full;
        xv[t] = in ? x[i * D + t] : 0.0;
        if (xcopy && in) xcopy[i * D + t] = xv[t];
      }
    }
    int c0 = 0, c1 = 0;
    const uint32_t k0 = node_key<D>(xv, kp, c0);
    const uint32_t k1 = full ? node_key<D>(xv + D, kp, c1) : 0u;
    if (c0) atomicMin(bad, ((unsigned long long)i << 4) | (unsigned long long)c0);
    if (c1) atomicMin(bad, ((unsigned long long)(i + 1) << 4) | (unsigned long long)c1);
    if (D == 3 && rec) {
      rec[i] = node_rec3(xv, kp);
      if (full) rec[i + 1] = node_rec3(xv + D, kp);
    }
    if (full) {
      reinterpret_cast<uint2*>(keys)[q] = make_uint2(k0, k1);
      if (vals) reinterpret_cast<uint2*>(vals)[q] = make_uint2((uint32_t)i, (uint32_t)(i + 1));
    } else {
      keys[i] = k0;
      if (vals) vals[i] = (uint32_t)i;
    }
  }
}

// K1 + K2a of the first radix pass: one CTA per sort tile (kSortTile nodes, kSortItems/2 node pairs
// per thread) validates, keys and copies its nodes as keys_kernel does and also counts the tile's
// first-pass digits (shared-memory integer counts: order-free) into the block-major histogram.
template <int D>
__global__ void __launch_bounds__(kSortThreads) keys_hist_kernel(
    const double* __restrict__ x, int64_t n, KeyParams kp, uint32_t* __restrict__ keys,
    unsigned long long* __restrict__ bad, double* __restrict__ xcopy, int aligned16, int bits,
    uint32_t* __restrict__ hist, SegLayout sl, float4* __restrict__ rec) {
  // rec (rec3 plans, D = 3): the nodes' 16-B gather records in user order (node_rec3)
  __shared__ uint32_t cnt[1 << kMaxDigitBits];
  const int ndig = 1 << bits;
  const uint32_t mask = ndig - 1;
  for (int dgt = threadIdx.x; dgt < ndig; dgt += blockDim.x) cnt[dgt] = 0;
  __syncthreads();
  const int64_t q0 = (int64_t)blockIdx.x * (kSortTile / 2);
  constexpr int NP = kSortItems / 2;
  double xv[NP][2 * D];
  // all loads first (independent, in flight together)
#pragma unroll
  for (int jj = 0; jj < NP; ++jj) {
    const int64_t i = 2 * (q0 + jj * kSortThreads + threadIdx.x);
    const bool full = i + 1 < n;
    if (full && aligned16) {
      const double2* src = reinterpret_cast<const double2*>(x + i * D);
#pragma unroll
      for (int h = 0; h < D; ++h) {
        const double2 v = __ldg(&src[h]);
        xv[jj][2 * h] = v.x;
        xv[jj][2 * h + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int t = 0; t < 2 * D; ++t) {
        const bool in = i < n && (t < D || full);
        xv[jj][t] = in ? __ldg(&x[i * D + t]) : 0.0;
      }
    }
  }
#pragma unroll
  for (int jj = 0; jj < NP; ++jj) {
    const int64_t q = q0 + jj * kSortThreads + threadIdx.x;
    const int64_t i = 2 * q;
    if (i >= n) continue;
    const bool full = i + 1 < n;
    if (xcopy) {
      if (full && aligned16) {
        double2* dstc = reinterpret_cast<double2*>(xcopy + i * D);
#pragma unroll
        for (int h = 0; h < D; ++h) dstc[h] = make_double2(xv[jj][2 * h], xv[jj][2 * h + 1]);
      } else {
#pragma unroll
        for (int t = 0; t < 2 * D; ++t)
          if (t < D || full) xcopy[i * D + t] = xv[jj][t];
      }
    }
    uint32_t k0, k1 = 0u;
    const bool ok0 = node_key_fast<D>(xv[jj], kp, k0);
    const bool ok1 = !full || node_key_fast<D>(xv[jj] + D, kp, k1);
    if (!(ok0 && ok1)) {   // rare: error codes of the offending nodes
      int c0 = 0, c1 = 0;
      node_key<D>(xv[jj], kp, c0);
      if (full) node_key<D>(xv[jj] + D, kp, c1);
      if (c0) atomicMin(bad, ((unsigned long long)i << 4) | (unsigned long long)c0);
      if (c1) atomicMin(bad, ((unsigned long long)(i + 1) << 4) | (unsigned long long)c1);
    }
    if (D == 3 && rec) {
      rec[i] = node_rec3(xv[jj], kp);
      if (full) rec[i + 1] = node_rec3(xv[jj] + D, kp);
    }
    atomicAdd(&cnt[k0 & mask], 1u);
    if (full) atomicAdd(&cnt[k1 & mask], 1u);
    if (keys) {   // null: the one-pass d = 1 scatter recomputes the keys from x
      if (full) reinterpret_cast<uint2*>(keys)[q] = make_uint2(k0, k1);
      else keys[i] = k0;
    }
  }
  __syncthreads();
  for (int dgt = threadIdx.x; dgt < ndig; dgt += blockDim.x)
    hist[hist_index(sl, blockIdx.x, dgt, ndig)] = cnt[dgt];
}

// Sort key = (user block, bin): the input is in user order, so the user-block part of the key is
// already sorted; the radix passes run over the bin digits only, with the per-tile histograms laid
// out block-major so that the scan never moves an element across a user block:
//   hist[blk*tpb*ndig + dg*tiles_in(blk) + tile_in_blk]      (scan order = (blk, digit, tile)).
// K2a: per-tile digit histogram.
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(
    const uint32_t* __restrict__ keys, int64_t n, int shift, int bits,
    uint32_t* __restrict__ hist, SegLayout sl) {
  __shared__ uint32_t cnt[1 << kMaxDigitBits];
  const int ndig = 1 << bits;
  const uint32_t mask = ndig - 1;
  for (int dgt = threadIdx.x; dgt < ndig; dgt += blockDim.x) cnt[dgt] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  uint32_t kk[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    int64_t idx = base + j * kSortThreads + threadIdx.x;
    kk[j] = idx < n ? __ldg(&keys[idx]) : 0xffffffffu;
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j)   // integer counts: order-free
    if (kk[j] != 0xffffffffu) atomicAdd(&cnt[(kk[j] >> shift) & mask], 1u);
  __syncthreads();
  for (int dgt = threadIdx.x; dgt < ndig; dgt += blockDim.x)
    hist[hist_index(sl, blockIdx.x, dgt, ndig)] = cnt[dgt];
}

// Exclusive scan of a uint32 array (3 phases).  Block = 256 threads x 16 items = 4096.
constexpr int kScanItems = 16;
constexpr int kScanBlock = 256 * kScanItems;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < 8 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < 8) warp_sums[lane] = s;
  }
  __syncthreads();
  uint32_t before = (w > 0 ? warp_sums[w - 1] : 0) + x - v;
  *total = warp_sums[7];
  __syncthreads();
  return before;
}

// kScanItems consecutive entries from base (a multiple of kScanItems): 16-byte loads when complete
__device__ __forceinline__ void load_items(const uint32_t* __restrict__ in, int64_t base, int64_t n,
                                           uint32_t (&v)[kScanItems]) {
  if (base + kScanItems <= n) {
    const uint4* src = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
    for (int j = 0; j < kScanItems / 4; ++j) {
      const uint4 q = src[j];
      v[4 * j] = q.x;
      v[4 * j + 1] = q.y;
      v[4 * j + 2] = q.z;
      v[4 * j + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) v[j] = (base + j < n) ? in[base + j] : 0u;
  }
}

__global__ void __launch_bounds__(256) scan_reduce_kernel(const uint32_t* __restrict__ in,
                                                          int64_t n, uint32_t* __restrict__ part) {
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  load_items(in, base, n, v);
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) s += v[j];
  uint32_t tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256) scan_part_kernel(uint32_t* __restrict__ part, int64_t np) {
  // single block; sequential over chunks of 256*kScanItems
  uint32_t carry = 0;
  for (int64_t c0 = 0; c0 < np; c0 += kScanBlock) {
    const int64_t base = c0 + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      v[j] = (base + j < np) ? part[base + j] : 0;
      s += v[j];
    }
    uint32_t tot;
    uint32_t run = carry + block_excl_scan(s, &tot);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      if (base + j < np) part[base + j] = run;
      run += v[j];
    }
    carry += tot;
  }
}

__global__ void __launch_bounds__(256) scan_down_kernel(const uint32_t* __restrict__ in, int64_t n,
                                                        const uint32_t* __restrict__ part,
                                                        uint32_t* __restrict__ out) {
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  load_items(in, base, n, v);
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) s += v[j];
  uint32_t tot;
  uint32_t run = part[blockIdx.x] + block_excl_scan(s, &tot);
  uint32_t o[kScanItems];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    o[j] = run;
    run += v[j];
  }
  if (base + kScanItems <= n) {   // 16-byte stores (base is a multiple of 16 elements)
    uint4* dst = reinterpret_cast<uint4*>(out + base);
#pragma unroll
    for (int j = 0; j < kScanItems / 4; ++j) dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
      if (base + j < n) out[base + j] = o[j];
  }
}

// Lanes of the warp holding the same digit (including the caller), by intersecting one ballot per
// digit bit (cheaper than MATCH.ANY); invalid lanes (tile tail) form their own group.
// Every lane executes every ballot (no early exit: the full-mask ballots need all 32 lanes).
template <int BITS>
__device__ __forceinline__ uint32_t peers_by_ballot(uint32_t dg, bool valid) {
  const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
  uint32_t peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const uint32_t bit = (dg >> b) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, bit);
    peers &= ~(bal ^ (0u - bit));          // bit ? bal : ~bal
  }
  return valid ? (peers & vmask) : ~vmask;
}

// K2b: stable scatter.  Warp w of the CTA owns tile elements [w*256, (w+1)*256), visited in
// 8 rounds of 32 consecutive elements; ranks within the warp come from warp-private digit
// counters (match_any groups equal digits in a round, lower lanes first), ranks across warps
// from an exclusive prefix over the warp counters, ranks across tiles from the scanned
// histogram.  Element order inside the tile is therefore preserved.  The tile is first reordered
// by digit in shared memory and then written out in digit runs (coalesced stores).
// vin == nullptr: values are the element indices (first pass; identity permutation).
#ifndef SCATTER_MIN_CTAS
#define SCATTER_MIN_CTAS 3   // 40 registers: 3 CTAs (48 warps) per SM; measured 1.70 -> 1.64 ms per cfg4 sort
#endif
template <int BITS>
__global__ void __launch_bounds__(kSortThreads, SCATTER_MIN_CTAS) radix_scatter_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
    uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n, int shift,
    const uint32_t* __restrict__ hist_scan, SegLayout sl, const double* __restrict__ xin,
    double* __restrict__ xsout, int d) {
  // last pass only (xsout != nullptr): also writes the sorted node copy xs[pos] = x[perm[pos]];
  // the random reads of x stay inside one L2-resident user block for d <= 2.
  constexpr int bits = BITS;
  constexpr int kWarps = kSortThreads / 32;
  constexpr int kPerWarp = kSortTile / kWarps;
  __shared__ uint32_t wcnt[kWarps][1 << kMaxDigitBits];
  __shared__ uint32_t gbase[1 << kMaxDigitBits];
  __shared__ uint32_t tstart[1 << kMaxDigitBits];
  extern __shared__ uint32_t sdyn[];      // skey[kSortTile], sval[kSortTile]
  uint32_t* skey = sdyn;
  uint32_t* sval = sdyn + kSortTile;
  __shared__ uint32_t wsum[kWarps];
  const int ndig = 1 << bits;
  const uint32_t mask = ndig - 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * ndig; i += kSortThreads) wcnt[i >> BITS][i & (ndig - 1)] = 0;
  {
    const int64_t h0 = hist_index(sl, blockIdx.x, 0, ndig);
    const int64_t hs = hist_index(sl, blockIdx.x, 1, ndig) - h0;   // stride between digits
    for (int dgt = threadIdx.x; dgt < ndig; dgt += blockDim.x) gbase[dgt] = hist_scan[h0 + dgt * hs];
  }
  __syncthreads();
  const int64_t tbase = (int64_t)blockIdx.x * kSortTile;
  const int tile_n = (int)min((int64_t)kSortTile, n - tbase);
  const uint32_t* __restrict__ kt = kin + tbase;          // tile-relative 32-bit indexing
  const uint32_t* __restrict__ vt = vin ? vin + tbase : nullptr;
  const int wbase = w * kPerWarp;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t k[kSortItems], v[kSortItems], r[kSortItems];
  // all loads first (independent, in flight together), then the ranking rounds
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int li = wbase + j * 32 + lane;
    const bool valid = li < tile_n;
    k[j] = valid ? __ldg(&kt[li]) : 0u;
    v[j] = valid ? (vt ? __ldg(&vt[li]) : (uint32_t)(tbase + li)) : 0u;
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const bool valid = wbase + j * 32 + lane < tile_n;
    const uint32_t dg = valid ? ((k[j] >> shift) & mask) : 0xffffffffu;
    const uint32_t peers = peers_by_ballot<BITS>(dg, valid);
    const uint32_t cnt = valid ? wcnt[w][dg] : 0u;
    r[j] = cnt + __popc(peers & lt_mask);
    __syncwarp();
    // every lane of the group stores the same new count (no leader election needed)
    if (valid) wcnt[w][dg] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over warps, tile count
  uint32_t tcount = 0;
  const int dg0 = threadIdx.x;   // ndig <= 256 <= blockDim
  if (dg0 < ndig) {
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
      uint32_t t = wcnt[ww][dg0];
      wcnt[ww][dg0] = tcount;
      tcount += t;
    }
  }
  // exclusive scan of tcount over digits (block scan)
  uint32_t x = tcount;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (dg0 < ndig) {
    uint32_t before = 0;
    for (int ww = 0; ww < w; ++ww) before += wsum[ww];
    tstart[dg0] = before + x - tcount;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    if (wbase + j * 32 + lane < tile_n) {
      uint32_t dg = (k[j] >> shift) & mask;
      uint32_t lpos = tstart[dg] + wcnt[w][dg] + r[j];
      skey[lpos] = k[j];
      sval[lpos] = v[j];
    }
  }
  __syncthreads();
  for (int li = threadIdx.x; li < tile_n; li += kSortThreads) {
    uint32_t kk = skey[li];
    uint32_t dg = (kk >> shift) & mask;
    uint32_t pos = gbase[dg] + (uint32_t)li - tstart[dg];
    if (kout) kout[pos] = kk;   // null: sorted keys not needed (one-pass sort, offsets from the histogram)
    const uint32_t vv = sval[li];
    vout[pos] = vv;
    if (xsout) {
      if (d == 2)   // 16-B records (rec3): one vector load per node
        reinterpret_cast<double2*>(xsout)[pos] = __ldg(reinterpret_cast<const double2*>(xin) + vv);
      else
        for (int t = 0; t < d; ++t) xsout[(int64_t)pos * d + t] = __ldg(&xin[(int64_t)vv * d + t]);
    }
  }
}

// K3: key offsets over the full sort key (user block, bin): key'(i) = (i >> ub_log2) * nbins +
// (skey[i] >> colbits) (sorted position i lies in user block i >> ub_log2); key_start[b] = first sorted
// position with key' >= b.  Four sorted keys per thread (16-byte loads) plus the preceding one.
__device__ __forceinline__ int64_t full_key(const uint32_t* skeys, int64_t i, int ub_log2, int64_t nbins,
                                            int colbits, uint32_t sk) {
  (void)skeys;
  return (i >> ub_log2) * nbins + (int64_t)(sk >> colbits);
}

__global__ void build_kernel(const double* __restrict__ x, const uint32_t* __restrict__ perm,
                             const uint32_t* __restrict__ skeys, double* __restrict__ xs,
                             uint32_t* __restrict__ key_start, int64_t n, int d, int64_t nbins,
                             int ub_log2, int64_t nkeys, int colbits) {
  (void)x;
  (void)perm;
  (void)xs;
  (void)d;
  const int64_t nq = (n + 4) / 4;   // groups of 4 positions covering [0, n]
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nq; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 4 * g;
    uint32_t k4[4];
    if (i0 + 4 <= n && (((uintptr_t)(skeys + i0)) & 15) == 0) {
      const uint4 q = *reinterpret_cast<const uint4*>(skeys + i0);
      k4[0] = q.x;
      k4[1] = q.y;
      k4[2] = q.z;
      k4[3] = q.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) k4[j] = i0 + j < n ? skeys[i0 + j] : 0u;
    }
    int64_t kprev = i0 == 0 ? -1 : full_key(skeys, i0 - 1, ub_log2, nbins, colbits, skeys[i0 - 1]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t i = i0 + j;
      if (i > n) break;
      const int64_t kcur = i == n ? nkeys : full_key(skeys, i, ub_log2, nbins, colbits, k4[j]);
      for (int64_t b = kprev + 1; b <= kcur; ++b) key_start[b] = (uint32_t)i;
      kprev = kcur;
    }
  }
}

static int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sm_count() * 32));
}

// K2b for d = 1 one-pass plans (d1_binned): the keys are recomputed from x (exactly as K1 computed
// the histogram's), ranked stably per tile like radix_scatter_kernel, and the tile is reordered in
// shared memory together with its node coordinates, so one pass writes both the permutation and the
// sorted node copy in digit runs (the gather then streams x instead of gathering it).
template <int BITS>
__global__ void __launch_bounds__(kSortThreads, 3) radix1x_scatter_kernel(
    const double* __restrict__ x, int64_t n, KeyParams kp, const uint32_t* __restrict__ hist_scan,
    SegLayout sl, uint32_t* __restrict__ perm_out, double* __restrict__ xs_out) {
  constexpr int kWarps = kSortThreads / 32;
  constexpr int kPerWarp = kSortTile / kWarps;
  constexpr int ndig = 1 << BITS;
  constexpr uint32_t mask = ndig - 1;
  __shared__ uint16_t wcnt[kWarps][ndig];   // counts <= kSortTile fit 16 bits (keeps 3 CTAs/SM)
  __shared__ uint32_t gbase[ndig];
  __shared__ uint32_t tstart[ndig];
  __shared__ uint32_t wsum[kWarps];
  extern __shared__ __align__(16) unsigned char dyn1x[];
  double* sx = reinterpret_cast<double*>(dyn1x);                     // [kSortTile], tile order
  uint16_t* sidx = reinterpret_cast<uint16_t*>(sx + kSortTile);      // [kSortTile], sorted slot -> tile index
  uint16_t* sdig = sidx + kSortTile;                                 // [kSortTile], sorted slot -> digit
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * ndig; i += kSortThreads) wcnt[i / ndig][i % ndig] = 0;
  {
    const int64_t h0 = hist_index(sl, blockIdx.x, 0, ndig);
    const int64_t hs = hist_index(sl, blockIdx.x, 1, ndig) - h0;
    for (int dgt = threadIdx.x; dgt < ndig; dgt += blockDim.x) gbase[dgt] = hist_scan[h0 + dgt * hs];
  }
  const int64_t tbase = (int64_t)blockIdx.x * kSortTile;
  const int tile_n = (int)min((int64_t)kSortTile, n - tbase);
  const int wbase = w * kPerWarp;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t k[kSortItems], r[kSortItems];
  double xv[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {   // all loads first (in flight together)
    const int li = wbase + j * 32 + lane;
    xv[j] = li < tile_n ? __ldg(&x[tbase + li]) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int li = wbase + j * 32 + lane;
    if (li < tile_n) {
      sx[li] = xv[j];
      uint32_t kk;
      node_key_fast<1>(&xv[j], kp, kk);
      k[j] = kk & mask;
    } else {
      k[j] = 0u;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const bool valid = wbase + j * 32 + lane < tile_n;
    const uint32_t dg = valid ? k[j] : 0xffffffffu;
    const uint32_t peers = peers_by_ballot<BITS>(dg, valid);
    const uint32_t cnt = valid ? wcnt[w][dg] : 0u;
    r[j] = cnt + __popc(peers & lt_mask);
    __syncwarp();
    if (valid) wcnt[w][dg] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  uint32_t tcount = 0;
  const int dg0 = threadIdx.x;
  if (dg0 < ndig) {
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
      uint32_t t = wcnt[ww][dg0];
      wcnt[ww][dg0] = tcount;
      tcount += t;
    }
  }
  uint32_t xs = tcount;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, xs, o);
    if (lane >= o) xs += y;
  }
  if (lane == 31) wsum[w] = xs;
  __syncthreads();
  if (dg0 < ndig) {
    uint32_t before = 0;
    for (int ww = 0; ww < w; ++ww) before += wsum[ww];
    tstart[dg0] = before + xs - tcount;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int li = wbase + j * 32 + lane;
    if (li < tile_n) {
      const uint32_t dg = k[j];
      const uint32_t lpos = tstart[dg] + wcnt[w][dg] + r[j];
      sidx[lpos] = (uint16_t)li;
      sdig[lpos] = (uint16_t)dg;
    }
  }
  __syncthreads();
  for (int li = threadIdx.x; li < tile_n; li += kSortThreads) {
    const uint32_t dg = sdig[li];
    const uint32_t pos = gbase[dg] + (uint32_t)li - tstart[dg];
    const uint32_t src = sidx[li];
    perm_out[pos] = (uint32_t)(tbase + src);
    xs_out[pos] = sx[src];
  }
}

static KeyParams key_params(const bnfft_plan_s* p) {
  KeyParams kp;
  kp.d = p->opts.d;
  kp.L = p->L;
  kp.Lf = (double)p->L;
  for (int t = 0; t < 3; ++t) {
    kp.log2W[t] = p->bin_log2[t];
    kp.nb[t] = p->nb_dim[t];
  }
  kp.strict = (p->opts.flags & BNFFT_STRICT_DOMAIN) ? 1 : 0;
  kp.box_lo = -0.5 + (double)p->opts.m / (double)p->L;
  kp.box_hi = 0.5 - (double)p->opts.m / (double)p->L;
  kp.colbits = p->col_bits;
  return kp;
}

constexpr int kRadix1xSmem = kSortTile * (int)(sizeof(double) + 2 * sizeof(uint16_t));

cudaError_t launch_keys(bnfft_plan_s* p, const double* x, int64_t n) {
  const KeyParams kp = key_params(p);
  cudaError_t e = cudaMemsetAsync(p->d_bad, 0xff, sizeof(unsigned long long), p->stream);
  if (e != cudaSuccess) return e;
  if (n > 0 && p->sort_passes > 0 && (p->opts.d <= 2 || p->rec3)) {   // first-pass histogram fused
    SegLayout sl;
    sl.ntiles = (n + kSortTile - 1) / kSortTile;
    sl.tpb = std::min<int64_t>(sl.ntiles, (int64_t)1 << std::max(0, p->ub_log2 - kSortTileLog2));
    const int b0 = std::min(p->digit_bits, p->key_bits);
    auto kfn = p->opts.d == 1 ? keys_hist_kernel<1> : p->opts.d == 2 ? keys_hist_kernel<2> : keys_hist_kernel<3>;
    kfn<<<(unsigned)sl.ntiles, kSortThreads, 0, p->stream>>>(x, n, kp, p->d1_binned ? nullptr : p->d_k0, p->d_bad,
                                                              p->xs_user ? p->d_xs : nullptr,
                                                              ((uintptr_t)x & 15) == 0 ? 1 : 0, b0, p->d_hist, sl,
                                                              p->rec3 ? (float4*)p->d_rec_user : nullptr);
    p->launches++;
  } else if (n > 0) {
    auto kfn = p->opts.d == 1 ? keys_kernel<1> : p->opts.d == 2 ? keys_kernel<2> : keys_kernel<3>;
    kfn<<<grid_for((n + 1) / 2, 256), 256, 0, p->stream>>>(x, n, kp, p->d_k0,
                                                           p->sort_passes ? nullptr : p->d_v0, p->d_bad,
                                                           (p->xs_user || !p->sort_passes) ? p->d_xs : nullptr,
                                                           ((uintptr_t)x & 15) == 0 ? 1 : 0,
                                                           p->rec3 ? (float4*)p->d_rec_user : nullptr);
    p->launches++;
  }
  return cudaGetLastError();
}

static cudaError_t exclusive_scan(bnfft_plan_s* p, const uint32_t* in, uint32_t* out, int64_t n) {
  int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  scan_reduce_kernel<<<(unsigned)nb, 256, 0, p->stream>>>(in, n, p->d_scan_part);
  scan_part_kernel<<<1, 256, 0, p->stream>>>(p->d_scan_part, nb);
  scan_down_kernel<<<(unsigned)nb, 256, 0, p->stream>>>(in, n, p->d_scan_part, out);
  p->launches += 3;
  return cudaGetLastError();
}

typedef void (*ScatterFn)(const uint32_t*, const uint32_t*, uint32_t*, uint32_t*, int64_t, int,
                          const uint32_t*, SegLayout, const double*, double*, int);
static ScatterFn scatter_for(int bits) {
  switch (bits) {
    case 1: return radix_scatter_kernel<1>;
    case 2: return radix_scatter_kernel<2>;
    case 3: return radix_scatter_kernel<3>;
    case 4: return radix_scatter_kernel<4>;
    case 5: return radix_scatter_kernel<5>;
    case 6: return radix_scatter_kernel<6>;
    case 7: return radix_scatter_kernel<7>;
    case 8: return radix_scatter_kernel<8>;
    default: return radix_scatter_kernel<9>;
  }
}

cudaError_t sort_prepare() {
  for (int b = 1; b <= kMaxDigitBits; ++b) {
    cudaError_t e = cudaFuncSetAttribute(scatter_for(b), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         2 * kSortTile * (int)sizeof(uint32_t));
    if (e != cudaSuccess) return e;
  }
  for (auto fn : {radix1x_scatter_kernel<7>, radix1x_scatter_kernel<8>, radix1x_scatter_kernel<9>}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kRadix1xSmem);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_sort(bnfft_plan_s* p, const double* x, int64_t n) {
  if (p->d1_binned && p->sort_passes == 1 && n > 0) {   // histogram from keys_hist_kernel
    SegLayout sl;
    sl.ntiles = (n + kSortTile - 1) / kSortTile;
    sl.tpb = std::min<int64_t>(sl.ntiles, (int64_t)1 << std::max(0, p->ub_log2 - kSortTileLog2));
    const int64_t nh = ((int64_t)1 << p->key_bits) * sl.ntiles;
    cudaError_t e = exclusive_scan(p, p->d_hist, p->d_hist, nh);
    if (e != cudaSuccess) return e;
    KeyParams kp = key_params(p);
    auto fn = p->key_bits >= 9 ? radix1x_scatter_kernel<9> : p->key_bits == 8 ? radix1x_scatter_kernel<8>
                                                                                : radix1x_scatter_kernel<7>;
    fn<<<(unsigned)sl.ntiles, kSortThreads, kRadix1xSmem, p->stream>>>(x, n, kp, p->d_hist, sl, p->d_v1, p->d_xs);
    p->launches++;
    p->d_skeys = nullptr;
    p->d_perm = p->d_v1;
    return cudaGetLastError();
  }
  uint32_t *kin = p->d_k0, *vin = nullptr, *kout = p->d_k1, *vout = p->d_v1;
  if (n > 0 && p->sort_passes > 0) {
    SegLayout sl;
    sl.ntiles = (n + kSortTile - 1) / kSortTile;
    sl.tpb = std::min<int64_t>(sl.ntiles, (int64_t)1 << std::max(0, p->ub_log2 - kSortTileLog2));
    int bits = p->digit_bits;
    for (int pass = 0; pass < p->sort_passes; ++pass) {
      int shift = pass * bits;
      int b = std::min(bits, p->key_bits - shift);
      int64_t nh = ((int64_t)1 << b) * sl.ntiles;
      if (pass > 0 || !(p->opts.d <= 2 || p->rec3)) {   // pass 0: counted by keys_hist_kernel
        radix_hist_kernel<<<(unsigned)sl.ntiles, kSortThreads, 0, p->stream>>>(kin, n, shift, b,
                                                                               p->d_hist, sl);
        p->launches++;
      }
      cudaError_t e = exclusive_scan(p, p->d_hist, p->d_hist, nh);
      if (e != cudaSuccess) return e;
      const bool last = pass == p->sort_passes - 1;
      // last pass: the sorted node copy xs (d doubles per node); none for rec3 plans, whose gather
      // reads the keys kernel's user-order records through the permutation (those random reads
      // overlap the gather's arithmetic instead of costing a bandwidth-bound pass here)
      scatter_for(b)<<<(unsigned)sl.ntiles, kSortThreads, 2 * kSortTile * sizeof(uint32_t), p->stream>>>(
          kin, vin, (last && p->sort_passes == 1) ? nullptr : kout, vout, n, shift, p->d_hist, sl, x,
          (last && !p->xs_user && !p->rec3) ? p->d_xs : nullptr, p->opts.d);
      p->launches++;
      std::swap(kin, kout);
      if (!vin) {
        vin = vout;
        vout = p->d_v0;
      } else {
        std::swap(vin, vout);
      }
    }
    p->d_skeys = kin;
    p->d_perm = vin;
  } else {
    p->d_skeys = p->d_k0;
    p->d_perm = p->d_v0;   // identity written by keys_kernel
  }
  return cudaGetLastError();
}

// Key offsets of a one-pass sort straight from the scanned digit histogram: with the whole key as
// the digit, the first sorted position of key (block, bin) is the scanned count of the block's first
// tile for digit `bin` (digit-major layout inside a block, hist_index).
__global__ void offsets_from_hist_kernel(const uint32_t* __restrict__ hist_scan, SegLayout sl, int ndig,
                                         int64_t nbins, int64_t nkeys, int64_t n,
                                         uint32_t* __restrict__ key_start, int colbits) {
  // colbits: the digit is (bin, minor digit); a bin starts at its minor digit 0
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= nkeys;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (k == nkeys) {
      key_start[k] = (uint32_t)n;
    } else {
      const int64_t blk = k / nbins;
      const int dg = (int)(k - blk * nbins);
      key_start[k] = hist_scan[hist_index(sl, blk * sl.tpb, dg << colbits, ndig)];
    }
  }
}

cudaError_t launch_build(bnfft_plan_s* p, const double* x, int64_t n) {
  if (p->sort_passes == 1 && n > 0) {
    SegLayout sl;
    sl.ntiles = (n + kSortTile - 1) / kSortTile;
    sl.tpb = std::min<int64_t>(sl.ntiles, (int64_t)1 << std::max(0, p->ub_log2 - kSortTileLog2));
    offsets_from_hist_kernel<<<grid_for(p->nkeys + 1, 256), 256, 0, p->stream>>>(
        p->d_hist, sl, 1 << p->digit_bits, p->nbins, p->nkeys, n, p->d_bin_start, p->col_bits);
    p->launches++;
    return cudaGetLastError();
  }
  build_kernel<<<grid_for((n + 4) / 4, 256), 256, 0, p->stream>>>(x, p->d_perm, p->d_skeys,
                                                            nullptr,   // xs comes from the sort
                                                            p->d_bin_start, n, p->opts.d,
                                                            p->nbins, p->ub_log2, p->nkeys, p->col_bits);
  p->launches++;
  return cudaGetLastError();
}

}  // namespace bnfft
