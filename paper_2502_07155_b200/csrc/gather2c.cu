// Row a6 for d = 2, complex64, batch 1, m <= 7 (BASELINE cfg3): quarter-warp-cooperative box gather.
//
// Step 3 of Algorithm 2 for d = 2: f_j = sum_a w0[a] sum_b w1[b] theta[c0-m+1+a, c1-m+1+b]
// (A3, taps A6).  gatherN_kernel gives one node to one thread; the 32 lanes of a warp then read 32
// unrelated box rows with 8-byte loads, and the random bank conflicts (2.8 wavefronts per load on
// cfg3) make the shared-memory pipe the wall.  Here
//   * phase 1 (one node per lane): cell, the 2 x 2m tap weights (exactly gatherN's arithmetic), into
//     a per-warp stash record: header (box byte offset of the window's first aligned column pair,
//     destination), w0[a], and the column weights by aligned pair position q = column - (first
//     column & ~1): cw[q] = w1[q - par], 0 outside the window (par = parity of the first column);
//   * phase 2 (one node per quarter-warp, up to 8 nodes per quarter and batch): lane l reads the aligned
//     column pair 2l, 2l + 1 of each of the 2m window rows with one 16-byte load -- the 8 lanes of a
//     quarter-warp read one contiguous 128-byte span, and a 128-bit shared load is served per
//     quarter-warp, so every load is one conflict-free wavefront -- contracts it with its two column
//     weights and the row weight, and three shuffles add the 8 lanes (fixed order: bitwise
//     reproducible; zero weights outside the window contribute exact zeros).
// Items (bins of 16 x 16 cells), TMA box ring and mbarrier hand-off are gatherN_kernel's.  Lanes whose
// pair lies beyond the window read the window's first pair with zero weights; the pair straddling
// the window's end may read one element past a box row (the next row, or the zeroed pad behind the
// box), also with a zero weight.
#include <cuda.h>

#include "gather_impl.cuh"

namespace bnfft {
namespace g2c {
constexpr int RECW = 36;   // words per stash record: hdr[4] | w0[16] | cw[16]  (144 B: conflict-free 16-B stores)
constexpr int PADB = 128;  // zeroed bytes behind each box buffer
}  // namespace g2c

size_t gather2c_stash_bytes(int threads) { return (size_t)(threads / 32) * 32 * g2c::RECW * 4; }
int gather2c_pad_bytes() { return g2c::PADB; }
int gather2c_max_m() { return 7; }

template <int T, bool POLY>
__global__ void __launch_bounds__(kGatherThreads, 3) gather2c_kernel(const __grid_constant__ GatherParams<float> p,
                                                                  const CUtensorMap* __restrict__ tmap) {
  using namespace g2c;
  using C = float2;
  constexpr int m = T / 2;
  static_assert(T >= 2 && T <= 14, "2m + 1 aligned column pairs fit a quarter-warp");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxBoxBufs], empty[kMaxBoxBufs];
  const int BZ = p.tbox[1];              // box row length (elements, even)
  const int box_elems = p.box_elems;
  C* const buf0 = reinterpret_cast<C*>(smem_raw);
  const uint32_t bytes = (uint32_t)box_elems * (uint32_t)sizeof(C);
  const int64_t G = gridDim.x;
  const int NB = p.nbuf;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int l = lane & 7, qw = lane >> 3;
  float* const stash = reinterpret_cast<float*>(smem_raw + (size_t)NB * p.bufstride * sizeof(C)) + wid * 32 * RECW;
  C* __restrict__ out = (C*)p.out;

  // zero the pad behind each box (TMA writes box bytes only)
  for (int q = 0; q < NB; ++q)
    for (int k = threadIdx.x; k < PADB / 8; k += blockDim.x) buf0[(size_t)q * p.bufstride + box_elems + k] = make_float2(0.f, 0.f);

  // Items: the non-empty keys blockIdx.x + j G.  Thread 0 stages their boxes NB - 1 items ahead (ring and
  // mbarrier hand-off as gatherN_kernel); every thread also walks the sequence itself, one item ahead,
  // and each warp loads the node data (permutation entry, coordinates) of its next batch -- in the
  // same item, else the next item's first -- during the current batch: no global-memory latency
  // between an item's box and its contraction, or between the batches of a large item.
  // (Measured slower on cfg3 and removed: claiming keys from a global counter, and splitting the
  // clustered centre's 4000-node bins into chunks that idle CTAs pick up -- the claim latency sits in
  // thread 0's staging path.)
  struct Item {
    int64_t u;          // key, or -1 past the CTA's last item
    uint32_t ib, ie;    // its sorted node range
  };
  auto item_from = [&](int64_t u) -> Item {   // first non-empty key of the walk at or after u
    while (u < p.nkeys) {
      const uint32_t ib = __ldg(&p.key_start[u]), ie = __ldg(&p.key_start[u + 1]);
      if (ie > ib) return Item{u, ib, ie};
      u += G;
    }
    return Item{-1, 0u, 0u};
  };
  Item ws = Item{-1, 0u, 0u};   // thread 0: staging position
  auto stage = [&](int bq) {
    if (ws.u >= 0) {
      issue_box<2, float>(p, tmap, ws.u, 0, buf0 + (size_t)bq * p.bufstride, &full[bq], bytes);
      ws = item_from(ws.u + G);
    }
  };
  struct NodeData {
    uint32_t dst;
    double2 x;
  };
  auto fetch_at = [&](int64_t i0, int64_t ie, NodeData& nd) {   // node i0 + lane of a batch
    const int64_t i = i0 + lane;
    if (i < ie) {
      nd.dst = __ldg(&p.perm[i]);
      nd.x = __ldg(reinterpret_cast<const double2*>(p.xs) + (p.xs_user ? (int64_t)nd.dst : i));
    }
  };
  auto fetch = [&](const Item& t, NodeData& nd) {   // node t.ib + 32 wid + lane (the warp's first batch)
    const uint32_t i = t.ib + (uint32_t)(32 * wid + lane);
    if (t.u >= 0 && i < t.ie) {
      nd.dst = __ldg(&p.perm[i]);
      nd.x = __ldg(reinterpret_cast<const double2*>(p.xs) + (p.xs_user ? nd.dst : i));
    }
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < NB; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], blockDim.x);
    }
    fence_mbar_init();
    ws = item_from(blockIdx.x);
    for (int q = 0; q < NB - 1; ++q) stage(q);
  }
  __syncthreads();
  const int64_t nbins = p.nb[0] * p.nb[1];
  Item cur = item_from(blockIdx.x);
  Item nxt = cur.u >= 0 ? item_from(cur.u + G) : cur;
  NodeData nd_cur, nd_nxt;
  nd_cur.dst = 0;
  nd_cur.x = make_double2(0.0, 0.0);
  nd_nxt = nd_cur;
  fetch(cur, nd_cur);
  for (int it = 0; cur.u >= 0; ++it) {
    const int b = it % NB;
    if (threadIdx.x == 0) {
      const int bn = (it + NB - 1) % NB;
      if (it >= 1) mbar_wait(&empty[bn], (uint32_t)((it - 1) / NB) & 1u);
      stage(bn);
    }
    const Item nn = nxt.u >= 0 ? item_from(nxt.u + G) : nxt;   // (its offsets are used next iteration)
    mbar_wait(&full[b], (uint32_t)(it / NB) & 1u);
    const int64_t u = cur.u;
    const uint32_t box_s = smem_u32(buf0 + (size_t)b * p.bufstride);
    const uint32_t rem = (uint32_t)(u % nbins);
    const int bo0 = (int)((rem / (uint32_t)p.nb[1]) << p.log2W[0]);
    const int bo1 = (int)((rem % (uint32_t)p.nb[1]) << p.log2W[1]);
    const int shift1 = (bo1 - (m - 1)) & 1;   // even-aligned box start (issue_box)
    const int64_t i_beg = cur.ib, i_end = cur.ie;
    if (i_beg + 32 * wid >= i_end) fetch(nxt, nd_cur);   // no batch for this warp in this item
    for (int64_t i0 = i_beg + 32 * wid; i0 < i_end; i0 += 32 * nwarps) {
      const int nbn = (int)min((int64_t)32, i_end - i0);
      // the warp's next batch (in this item, else the first one of the next item): in flight meanwhile
      if (i0 + 32 * nwarps < i_end) fetch_at(i0 + 32 * nwarps, i_end, nd_nxt);
      else fetch(nxt, nd_nxt);
      // ---- phase 1: lane = node i0 + lane
      if (lane < nbn) {
        const int64_t i = i0 + lane;
        const uint32_t dst = nd_cur.dst;
        const double2 xv = nd_cur.x;
        int off[2];
        float w[2][T];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const double Lx = __dmul_rn(p.Lf, t == 0 ? xv.x : xv.y);
          const double fl = floor(Lx);
          double uu = Lx - fl;
          int64_t c = (int64_t)fl + p.L / 2;
          if (c > p.L - 1) { c = p.L - 1; uu = 1.0; }
          off[t] = (int)c - (t == 0 ? bo0 : bo1);
          const DimState<float> st = dim_state<T, float, POLY>(uu, p);
          all_taps<T, POLY>(st, p, w[t]);
        }
        off[1] += shift1;
        const bool par = (off[1] & 1) != 0;
        float* r = stash + lane * RECW;
        reinterpret_cast<uint4*>(r)[0] =
            make_uint4((uint32_t)((off[0] * BZ + (off[1] & ~1)) * 8), p.sorted_out ? (uint32_t)i : dst, 0u, 0u);
        float a16[16], c16[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          a16[q] = q < T ? w[0][q < T ? q : 0] : 0.0f;
          const float e = q < T ? w[1][q < T ? q : 0] : 0.0f;                         // par == 0: w1[q]
          const float o = (q >= 1 && q - 1 < T) ? w[1][(q >= 1 && q - 1 < T) ? q - 1 : 0] : 0.0f;   // par == 1: w1[q - 1]
          c16[q] = par ? o : e;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          reinterpret_cast<float4*>(r)[1 + q] = make_float4(a16[4 * q], a16[4 * q + 1], a16[4 * q + 2], a16[4 * q + 3]);
          reinterpret_cast<float4*>(r)[5 + q] = make_float4(c16[4 * q], c16[4 * q + 1], c16[4 * q + 2], c16[4 * q + 3]);
        }
      }
      __syncwarp();
      // ---- phase 2: quarter-warp qw contracts nodes qw, qw + 4, ...
#pragma unroll 4
      for (int j0 = 0; j0 < nbn; j0 += 4) {   // (warp-uniform trip count: the shuffles below are full-warp)
        const bool live = j0 + qw < nbn;
        const int j = live ? j0 + qw : nbn - 1;
        const float* r = stash + j * RECW;
        const uint4 hdr = reinterpret_cast<const uint4*>(r)[0];
        const float2 cw = reinterpret_cast<const float2*>(r + 20)[l];
        float w0[16];
#pragma unroll
        for (int q = 0; q < (T + 3) / 4; ++q) {
          const float4 v = reinterpret_cast<const float4*>(r + 4)[q];
          w0[4 * q] = v.x;
          w0[4 * q + 1] = v.y;
          w0[4 * q + 2] = v.z;
          w0[4 * q + 3] = v.w;
        }
        // lanes beyond the window's last pair (weights zero) re-read the first pair
        const uint32_t a0 = box_s + hdr.x + (uint32_t)((l <= T / 2) ? l : 0) * 16u;
        float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int a = 0; a < T; ++a) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(a0 + (uint32_t)(a * BZ * 8)));
          float2 rr = __fmul2_rn(make_float2(cw.x, cw.x), make_float2(v.x, v.y));
          cmac(rr, cw.y, make_float2(v.z, v.w));
          if (a & 1) cmac(acc1, w0[a], rr);
          else cmac(acc0, w0[a], rr);
        }
        float2 f = __fadd2_rn(acc0, acc1);
        f = __fadd2_rn(f, make_float2(__shfl_xor_sync(0xffffffffu, f.x, 1), __shfl_xor_sync(0xffffffffu, f.y, 1)));
        f = __fadd2_rn(f, make_float2(__shfl_xor_sync(0xffffffffu, f.x, 2), __shfl_xor_sync(0xffffffffu, f.y, 2)));
        f = __fadd2_rn(f, make_float2(__shfl_xor_sync(0xffffffffu, f.x, 4), __shfl_xor_sync(0xffffffffu, f.y, 4)));
        if (l == 0 && live) out[hdr.y] = f;
      }
      __syncwarp();   // stash free for the next batch
      nd_cur = nd_nxt;
    }
    mbar_arrive(&empty[b]);
    cur = nxt;
    nxt = nn;
  }
}

template <bool POLY>
static const void* g2c_ptr(int m) {
  switch (m) {
    case 1: return (const void*)gather2c_kernel<2, POLY>;
    case 2: return (const void*)gather2c_kernel<4, POLY>;
    case 3: return (const void*)gather2c_kernel<6, POLY>;
    case 4: return (const void*)gather2c_kernel<8, POLY>;
    case 5: return (const void*)gather2c_kernel<10, POLY>;
    case 6: return (const void*)gather2c_kernel<12, POLY>;
    case 7: return (const void*)gather2c_kernel<14, POLY>;
  }
  return nullptr;
}

const void* gather2c_kernel_ptr(int m, bool poly) { return poly ? g2c_ptr<true>(m) : g2c_ptr<false>(m); }

}  // namespace bnfft
