// Row a6 for d = 3, m = 4, complex64, batch 1 (BASELINE cfg4): the z-sweep gather.
//
// Step 3 of Algorithm 2, f_j = sum_l theta_l prod_t w_t(l_t), evaluated as the separable
// contraction f_j = sum_a wx[a] sum_b wy[b] sum_c wz[c] theta[cx-3+a, cy-3+b, cz-3+c] (reading A3,
// taps A6).  One node needs 8 x 8 x 8 grid values; at cfg4 density (0.5 nodes per cell) each grid
// value is shared by 256 nodes, so the kernel is organised to reuse grid values from registers
// instead of re-reading shared memory per node (gather3c, its predecessor, read all 512 values of
// every node from shared memory and was bound by the shared-memory pipe):
//
//   * a CTA owns one bin (8 x 8 x 16 cells, the sort's bin, row a1); its grid neighbourhood
//     (15 x 15 x 26 complex64, zero outside I_L = reading A5) is staged by TMA, double-buffered;
//   * stash phase: every thread takes one or two of the bin's nodes, evaluates the 24 tap weights
//     (tap polynomials, R1) and files them in shared memory in column order -- a counting sort by
//     cell inside the bin (column (x, y) major, z minor), so a column's nodes are contiguous and
//     sorted by z;
//   * sweep phase: a warp takes one column (x, y) of the bin.  Lane (a, bq) = (lane & 7, lane >> 3)
//     holds the two grid rows (x-3+a, y-3+bq) and (x-3+a, y+1+bq) along z in registers and walks z
//     from the bottom of the bin to the top: at step z the rows' window [z-3, z+4] is in registers
//     (static indices -- the sweep is unrolled) and every node of cell (x, y, z) costs each lane
//     two 8-tap z-dots (FFMA2) and one complex MAC per row; a node's 32 lane partials are summed by
//     two shuffle levels and an 8-way shared-memory reduction.  A column's ~8 nodes share each row
//     load, cutting shared-memory wavefronts per node from ~42 (gather3c) to ~24.
//
// The per-node arithmetic does not depend on the order in which nodes are filed or processed (fixed
// tap order, fixed lane-to-row map, fixed shuffle/reduction tree), so results are bitwise
// reproducible and independent of the in-cell order the counting sort produces.
#include <cuda.h>

#include "gather_impl.cuh"

namespace bnfft {
namespace g3s {

constexpr int NT = 512, NW = NT / 32;
constexpr int T = 8;                   // 2m taps per dimension, m = 4
constexpr int RS = 26;                 // box z extent = row stride: 2*RS words = 4 * odd -> rows of
                                       // lanes a = 0..7 fall in distinct 16-B bank groups (LDS.128)
constexpr int BXY = 15;                // box x, y extents (8 cells + 2m - 1)
constexpr int BOX = BXY * BXY * RS;    // complex64 elements per box
constexpr int BOXB = (BOX * 8 + 127) / 128 * 128;
constexpr int CAP = 640;               // nodes per stash chunk (bins with more nodes are chunked)
constexpr int NPT = (CAP + NT - 1) / NT;
constexpr int REC = 28;                // words per stash record: wz[8] wx[8] wy[8] dst pad (16-B rows)
constexpr int CELLS = 1024;            // 8 x 8 x 16 cells per bin: (x, y) column major, z minor
constexpr int NCOL = 64;
constexpr int RB = 16;                 // nodes per reduction batch per warp
constexpr int RW = 36;                 // words per node in the reduction buffer (16 complex + pad)
constexpr int OFF_REC = 2 * BOXB;
constexpr int OFF_RED = OFF_REC + (CAP + 1) * REC * 4;   // record CAP: readable dummy (prefetch)
constexpr int OFF_CS = OFF_RED + NW * RB * RW * 4;
constexpr int SMEM = OFF_CS + (CELLS + 8) * 4;

}  // namespace g3s

size_t gather3s_smem() { return (size_t)g3s::SMEM; }
int gather3s_threads() { return g3s::NT; }
int gather3s_row_stride() { return g3s::RS; }

struct Node3 {
  double x[3];
  uint32_t dst;
};

// every third bit of x (Morton de-interleave, up to 10 bits)
__device__ __forceinline__ uint32_t compact3(uint32_t x) {
  x &= 0x09249249u;
  x = (x ^ (x >> 2)) & 0x030c30c3u;
  x = (x ^ (x >> 4)) & 0x0300f00fu;
  x = (x ^ (x >> 8)) & 0xff0000ffu;
  x = (x ^ (x >> 16)) & 0x000003ffu;
  return x;
}

// the CTA's next non-empty bin at Morton index >= v (stride G): {v, key, first node, end node};
// v = nvirt when there is none.  Called by one thread.
__device__ __forceinline__ void walk_bins(const GatherParams<float>& p, int64_t v, int64_t G, int64_t nvirt,
                                          int64_t* out) {
  const int mb = p.morton_bits;
  const int64_t nbins = p.nb[0] * p.nb[1] * p.nb[2];
  for (; v < nvirt; v += G) {
    const int64_t blk = v >> (3 * mb);
    const uint32_t vv = (uint32_t)(v & ((1ll << (3 * mb)) - 1));
    const uint32_t c2 = compact3(vv), c1 = compact3(vv >> 1), c0 = compact3(vv >> 2);
    if (c0 >= (uint32_t)p.nb[0] || c1 >= (uint32_t)p.nb[1] || c2 >= (uint32_t)p.nb[2]) continue;
    const int64_t u = blk * nbins + ((int64_t)c0 * p.nb[1] + c1) * p.nb[2] + c2;
    const int64_t b0 = __ldg(&p.key_start[u]), b1 = __ldg(&p.key_start[u + 1]);
    if (b1 > b0) {
      out[0] = v;
      out[1] = u;
      out[2] = b0;
      out[3] = b1;
      return;
    }
  }
  out[0] = nvirt;
  out[1] = out[2] = out[3] = 0;
}

template <bool POLY>
__global__ void __launch_bounds__(g3s::NT, 1) gather3s_kernel(const __grid_constant__ GatherParams<float> p,
                                                              const CUtensorMap* __restrict__ tmap) {
  using namespace g3s;
  extern __shared__ __align__(1024) unsigned char g3s_smem[];   // TMA destinations: 128-B aligned
  __shared__ __align__(8) uint64_t full[2];
  __shared__ int s_gctr;
  __shared__ uint32_t s_wsum[NW];
  __shared__ int64_t s_ring[3][4];     // bins: current, next, the one after (thread 0 walks ahead)
  float2* const boxes = reinterpret_cast<float2*>(g3s_smem);
  float* const rec = reinterpret_cast<float*>(g3s_smem + OFF_REC);
  float* const red = reinterpret_cast<float*>(g3s_smem + OFF_RED);
  uint32_t* const cs = reinterpret_cast<uint32_t*>(g3s_smem + OFF_CS);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int la = lane & 7, lbq = lane >> 3;
  float2* __restrict__ out = (float2*)p.out;
  const int64_t G = gridDim.x;
  const int64_t nvirt = p.nkeys_morton;
  const int64_t nbins = p.nb[0] * p.nb[1] * p.nb[2];
  const uint32_t bytes = (uint32_t)(BOX * sizeof(float2));
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
    walk_bins(p, blockIdx.x, G, nvirt, s_ring[0]);
    walk_bins(p, s_ring[0][0] + G, G, nvirt, s_ring[1]);
    if (s_ring[0][0] < nvirt) issue_box<3, float>(p, tmap, s_ring[0][1], 0, boxes, &full[0], bytes);
  }
  __syncthreads();
  if (s_ring[0][0] >= nvirt) return;

  auto load_nodes = [&](int64_t base, int64_t end, Node3 (&nd)[NPT]) {
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
      const int64_t i = base + tid + (int64_t)j * NT;
      if (j * NT + tid < CAP && i < end) {
        const uint32_t pj = __ldg(&p.perm[i]);
        nd[j].dst = p.sorted_out ? (uint32_t)i : pj;   // output position (BNFFT_SORTED_OUTPUT: sorted)
        const int64_t src = p.xs_user ? (int64_t)pj : i;
        nd[j].x[0] = __ldg(&p.xs[src * 3 + 0]);
        nd[j].x[1] = __ldg(&p.xs[src * 3 + 1]);
        nd[j].x[2] = __ldg(&p.xs[src * 3 + 2]);
      } else {
        nd[j].x[0] = 2.0;   // inactive slot (valid nodes lie in [-1/2, 1/2))
      }
    }
  };
  Node3 nd[NPT];
  load_nodes(s_ring[0][2], min(s_ring[0][3], s_ring[0][2] + CAP), nd);
  uint32_t phases = 0u;   // bit b: parity of the next completion of full[b]

  for (int it = 0;; ++it) {
    const int b = it & 1;
    const int64_t* cur = s_ring[it % 3];
    const int64_t* nxt = s_ring[(it + 1) % 3];
    const int64_t u = cur[1], i_beg = cur[2], i_end = cur[3];
    const bool has_nxt = nxt[0] < nvirt;
    const int64_t n_beg = nxt[2], n_end = nxt[3];
    if (cur[0] >= nvirt) break;
    const float2* box = boxes + (size_t)b * (BOXB / sizeof(float2));
    // the next bin's box into the other buffer (last read before the previous barrier)
    if (tid == 0 && has_nxt)
      issue_box<3, float>(p, tmap, nxt[1], 0, boxes + (size_t)(b ^ 1) * (BOXB / sizeof(float2)), &full[b ^ 1], bytes);
    // bin origin (cells)
    int bo[3];
    {
      uint32_t rem = (uint32_t)(u % nbins);
#pragma unroll
      for (int t = 2; t >= 0; --t) {
        const uint32_t btc = rem % (uint32_t)p.nb[t];
        rem /= (uint32_t)p.nb[t];
        bo[t] = (int)(btc << p.log2W[t]);
      }
    }
    bool waited = false;
    for (int64_t base = i_beg; base < i_end; base += CAP) {
      const int64_t cend = min(i_end, base + CAP);
      // ---------------- stash phase: cells, in-bin counting sort, tap weights
      for (int c = tid; c < CELLS + 8; c += NT) cs[c] = 0u;
      if (tid == 0) s_gctr = 0;
      __syncthreads();
      // thread 0 walks to the bin after next (its slot was last read at the top of the previous
      // iteration); the key_start loads complete while this bin is processed
      if (tid == 32 && base == i_beg) {
        if (has_nxt) walk_bins(p, nxt[0] + G, G, nvirt, s_ring[(it + 2) % 3]);
        else s_ring[(it + 2) % 3][0] = nvirt;
      }
      int key[NPT], rank[NPT];
      float uu[NPT][3];
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        key[j] = -1;
        if (nd[j].x[0] > 1.0) continue;
        int o[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const double Lx = __dmul_rn(p.Lf, nd[j].x[t]);
          const double fl = floor(Lx);
          double w = Lx - fl;
          int c = __double2int_rz(fl) + (int)(p.L >> 1);
          if (c > (int)p.L - 1) { c = (int)p.L - 1; w = 1.0; }   // fl(L x) == L/2 (defensive)
          o[t] = c - bo[t];
          uu[j][t] = (float)w;
        }
        key[j] = ((o[0] << 3) + o[1]) * 16 + o[2];
        rank[j] = (int)atomicAdd(&cs[key[j]], 1u);
      }
      __syncthreads();
      // exclusive scan of the 1024 cell counts (2 per thread), cs[1024] = total
      {
        const uint32_t c0 = cs[2 * tid], c1 = cs[2 * tid + 1];
        uint32_t s = c0 + c1, incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[wid] = incl;
        __syncthreads();
        uint32_t wbase = 0, tot = 0;
#pragma unroll
        for (int w2 = 0; w2 < NW; ++w2) {
          const uint32_t ws = s_wsum[w2];
          wbase += (w2 < wid) ? ws : 0u;
          tot += ws;
        }
        const uint32_t ex = wbase + incl - s;
        cs[2 * tid] = ex;
        cs[2 * tid + 1] = ex + c0;
        if (tid == 0) cs[CELLS] = tot;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        if (key[j] < 0) continue;
        float* r = rec + (cs[key[j]] + (uint32_t)rank[j]) * REC;
        float w[T];
        // x taps
        all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[j][0], p), p, w);
        reinterpret_cast<float4*>(r + 8)[0] = make_float4(w[0], w[1], w[2], w[3]);
        reinterpret_cast<float4*>(r + 8)[1] = make_float4(w[4], w[5], w[6], w[7]);
        // y taps, stored [bq][k] = wy[bq + 4k]
        all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[j][1], p), p, w);
        reinterpret_cast<float4*>(r + 16)[0] = make_float4(w[0], w[4], w[1], w[5]);
        reinterpret_cast<float4*>(r + 16)[1] = make_float4(w[2], w[6], w[3], w[7]);
        // z taps
        all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[j][2], p), p, w);
        reinterpret_cast<float4*>(r)[0] = make_float4(w[0], w[1], w[2], w[3]);
        reinterpret_cast<float4*>(r)[1] = make_float4(w[4], w[5], w[6], w[7]);
        reinterpret_cast<uint32_t*>(r)[24] = nd[j].dst;
      }
      // prefetch the next chunk's (or next bin's) nodes; they arrive during the sweep
      if (cend < i_end) load_nodes(cend, min(i_end, cend + CAP), nd);
      else if (has_nxt) load_nodes(n_beg, min(n_end, n_beg + CAP), nd);
      __syncthreads();
      if (!waited) {
        mbar_wait(&full[b], (phases >> b) & 1u);
        phases ^= 1u << b;
        waited = true;
      }
      // ---------------- sweep phase: warps take columns dynamically
      float* const rw = red + wid * (RB * RW);
      // sum of the 16 stored partials of the batch's first cnt nodes -> f (slot of entry k in word 32)
      auto flush = [&](int cnt) {
        __syncwarp();
        if (lane < cnt) {
          const float* ent = rw + lane * RW;
          const float4* e4 = reinterpret_cast<const float4*>(ent);
          float2 sa = make_float2(0.f, 0.f), sb2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 v4 = e4[q];
            sa = __fadd2_rn(sa, make_float2(v4.x, v4.y));
            sb2 = __fadd2_rn(sb2, make_float2(v4.z, v4.w));
          }
          const uint32_t slot = __float_as_uint(ent[32]);
          const uint32_t dst = reinterpret_cast<const uint32_t*>(rec)[slot * REC + 24];
          out[dst] = __fadd2_rn(sa, sb2);
        }
        __syncwarp();
      };
      int nst = 0;   // partials stored in this warp's batch (batches span columns)
      for (;;) {
        int g = 0;
        if (lane == 0) g = atomicAdd(&s_gctr, 1);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= NCOL) break;
        uint32_t cz[20];
        {
          const uint4* c4 = reinterpret_cast<const uint4*>(cs + g * 16);
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            const uint4 t4 = c4[q];
            cz[4 * q] = t4.x;
            cz[4 * q + 1] = t4.y;
            cz[4 * q + 2] = t4.z;
            cz[4 * q + 3] = t4.w;
          }
        }
        if (cz[0] == cz[16]) continue;
        const int ox = g >> 3, oy = g & 7;
        const float4* r0 = reinterpret_cast<const float4*>(box + ((ox + la) * BXY + oy + lbq) * RS);
        const float4* r1 = r0 + 2 * RS;   // rows b + 4: 4 * RS complex64 = 2 * RS float4
        float2 R0[24], R1[24];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          const float4 a4 = r0[q], b4 = r1[q];
          R0[2 * q] = make_float2(a4.x, a4.y);
          R0[2 * q + 1] = make_float2(a4.z, a4.w);
          R1[2 * q] = make_float2(b4.x, b4.y);
          R1[2 * q + 1] = make_float2(b4.z, b4.w);
        }
        uint32_t s = cz[0];
        const float* rp = rec + s * REC;
#pragma unroll
        for (int z = 0; z < 16; ++z) {
          if ((z & 1) == 0 && z / 2 + 5 < 12) {   // element pair z/2+5 (z + 10, z + 11)
            const int q = z / 2 + 5;
            const float4 a4 = r0[q], b4 = r1[q];
            R0[2 * q] = make_float2(a4.x, a4.y);
            R0[2 * q + 1] = make_float2(a4.z, a4.w);
            R1[2 * q] = make_float2(b4.x, b4.y);
            R1[2 * q + 1] = make_float2(b4.z, b4.w);
          }
          const uint32_t e = cz[z + 1];
          for (; s < e; ++s, rp += REC) {
            const float4 wz0 = reinterpret_cast<const float4*>(rp)[0];
            const float4 wz1 = reinterpret_cast<const float4*>(rp)[1];
            const float wxa = rp[8 + la];
            const float2 wyb = reinterpret_cast<const float2*>(rp + 16)[lbq];
            const float wzc[T] = {wz0.x, wz0.y, wz0.z, wz0.w, wz1.x, wz1.y, wz1.z, wz1.w};
            float2 d0 = make_float2(0.f, 0.f), d1 = d0;
#pragma unroll
            for (int c = 0; c < T; ++c) {
              cmac(d0, wzc[c], R0[z + 1 + c]);
              cmac(d1, wzc[c], R1[z + 1 + c]);
            }
            float2 acc = __fmul2_rn(make_float2(wxa * wyb.x, wxa * wyb.x), d0);
            cmac(acc, wxa * wyb.y, d1);
            float2 q;
            q.x = __shfl_xor_sync(0xffffffffu, acc.x, 16);
            q.y = __shfl_xor_sync(0xffffffffu, acc.y, 16);
            float* ent = rw + nst * RW;
            if (lane < 16) reinterpret_cast<float2*>(ent)[lane] = __fadd2_rn(acc, q);
            if (lane == 16) ent[32] = __uint_as_float(s);
            if (++nst == RB) {
              flush(RB);
              nst = 0;
            }
          }
        }
      }
      if (nst) flush(nst);
      nst = 0;
      __syncthreads();   // records and counts free for the next chunk
    }
    if (!waited) {       // (never: a non-empty bin has a chunk) keep the barrier phases consistent
      mbar_wait(&full[b], (phases >> b) & 1u);
      phases ^= 1u << b;
    }
  }
}

const void* gather3s_kernel_ptr(bool poly) {
  return poly ? (const void*)gather3s_kernel<true> : (const void*)gather3s_kernel<false>;
}

}  // namespace bnfft
