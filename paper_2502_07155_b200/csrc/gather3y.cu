// Row a6 for d = 3, m = 4, complex64, batch 1 (BASELINE cfg4): the y-sweep gather (default).
//
// Step 3 of Algorithm 2, f_j = sum_l theta_l prod_t w_t(l_t), as the separable contraction
//     f_j = sum_a wx[a] sum_b wy[b] sum_c wz[c] theta[cx-3+a, cy-3+b, cz-3+c]          (A3, taps A6)
// One node needs 8 x 8 x 8 grid values; at cfg4 density (0.5 nodes per cell) each grid value is
// shared by 256 nodes.  Reading all 512 values of every node from shared memory (gather3c) makes the
// shared-memory pipe the wall (4 KiB per node).  Here grid rows live in registers and are reused by
// every node of a 16-column x-line:
//
//   * sort (row a1): the key of a node is its x-line bin (cells cx x [16 by, 16 by + 16) x
//     [8 bz, 8 bz + 8), bins of 1 x 16 x 8 cells) with the y column c_y mod 16 as a minor digit, so
//     an x-line's nodes arrive in column order; the keys kernel writes a 16-B record per node in
//     user order (u_x, u_y, u_z as float, column and z offset; rec3), read here through the
//     permutation one batch ahead of use;
//   * a CTA of 16 warps = two teams of 8; an item = the 8 x-lines cx = 8X..8X+7 of one (by, bz),
//     warp w of a team contracts x-line 8X + w; items alternate between the teams and their grid
//     neighbourhoods (15 x 23 x 18 complex64, zero outside I_L = reading A5 zero extension) are
//     staged by TMA in a ring of three box buffers, so the next item's box is in flight while both
//     teams compute (mbarrier per buffer; the last warp of a team to release a box loads the item
//     three ahead into it);
//   * lane (a, q) = (lane & 7, lane >> 3) holds two grid rows along z (16 values each) of x-plane
//     cx-3+a: the rows r (box y index) of the current 8-row window with r mod 8 = q (slot 0) and
//     q + 4 (slot 1).  Moving the window from column y to y+1 drops row y and loads row y+8 into the
//     same (q, slot), so one 8-lane group loads one row per column step: grid data costs ~3 shared-
//     memory wavefronts per node instead of 32 (gather3c);
//   * per batch of 32 nodes each lane evaluates one node's 24 tap weights (tap polynomials, R1) into
//     a shared-memory record; per node the warp reads the record (z weights broadcast, y weights
//     pre-rotated to the lane groups), each lane forms two 8-tap z-dots from its registers (the
//     node's z offset selects the register window: a warp-uniform switch), contracts its two rows
//     with wy, the 4 row lanes of each x-plane are summed by two shuffles, and after the batch each
//     lane finishes one node's x contraction (sum_a wx[a] P_a) and stores it.
//
// The per-node arithmetic is independent of the order in which nodes are visited (fixed tap order,
// fixed lane-to-row map, fixed shuffle tree), so results are bitwise reproducible and equal for any
// permutation of the node set.
#include <cuda.h>

#include <vector>

#include "gather_impl.cuh"

namespace bnfft {
namespace g3y {

constexpr int NW = 16, NT = NW * 32;       // two teams of 8 warps; warp w of a team: x-line 8X + w
constexpr int NBUF = 3;                    // box ring: the teams' current items and the next one
constexpr int T = 8;                       // 2m taps per dimension, m = 4
constexpr int BX = 15, BY = 23, BZ = 18;   // box extents: 8 + 7, 16 + 7, 8 + 8 (+2: x-plane stride of
                                           // 23*18*8 B = 112 mod 128 -> conflict-free row loads)
constexpr int BOX = BX * BY * BZ;          // complex64 elements
constexpr int BOXB = (BOX * 8 + 127) / 128 * 128;
constexpr int REC = 24;                    // words per record: wz[8] | wy pairs[8] | wx[8]
constexpr int GN = 8;                      // nodes per reduction group
constexpr int OFF_REC = NBUF * BOXB;                           // float [NW][32][REC]
constexpr int OFF_PART = OFF_REC + NW * 32 * REC * 4;          // float2 [NW][GN][32]: lane partials
constexpr int OFF_MD = OFF_PART + NW * GN * 32 * 8;            // uint8 [NW][32]: (column << 3) | z offset
constexpr int SMEM = OFF_MD + NW * 32 + 32;   // (+32: md reads run one pair past a batch)
static_assert(OFF_REC % 16 == 0 && OFF_PART % 16 == 0, "16-B aligned records and partials");
static_assert(SMEM + 256 <= 227 * 1024, "shared memory per CTA");

}  // namespace g3y

size_t gather3y_smem() { return (size_t)g3y::SMEM; }
int gather3y_threads() { return g3y::NT; }
void gather3y_box(int* ext) {
  ext[0] = g3y::BX;
  ext[1] = g3y::BY;
  ext[2] = g3y::BZ;
}

// Items: groups of 8 x-lines (X, by, bz), visited in a Morton order with unequal bit counts per
// dimension (dense for power-of-two grids: every virtual index is a real item).  Item k of a CTA is
// the virtual index blockIdx.x + k * gridDim.x, so consecutive CTAs work on neighbouring items and
// their boxes' halos are served from L2.  The decoded items come from a plan-time table (one word per
// virtual index: X | Y << 10 | Z << 20, kG3yHole for holes), written by gather3y_item_table.
constexpr uint32_t kG3yHole = 0xffffffffu;

void gather3y_item_table(int64_t nX, int64_t nY, int64_t nZ, std::vector<uint32_t>& tab) {
  int bx = 0, byb = 0, bzb = 0;
  while (((int64_t)1 << bx) < nX) ++bx;
  while (((int64_t)1 << byb) < nY) ++byb;
  while (((int64_t)1 << bzb) < nZ) ++bzb;
  const int64_t nvirt = (int64_t)1 << (bx + byb + bzb);
  tab.assign((size_t)nvirt, kG3yHole);
  for (int64_t v = 0; v < nvirt; ++v) {
    int64_t X = 0, Y = 0, Z = 0;
    int bit = 0;
    for (int l = 0; l < 30; ++l) {
      if (l < bzb) { Z |= ((v >> bit) & 1) << l; ++bit; }
      if (l < byb) { Y |= ((v >> bit) & 1) << l; ++bit; }
      if (l < bx) { X |= ((v >> bit) & 1) << l; ++bit; }
    }
    if (X < nX && Y < nY && Z < nZ) tab[(size_t)v] = (uint32_t)(X | (Y << 10) | (Z << 20));
  }
}

// Load the item `it` (table word) into box buffer b, or complete the buffer's phase without data for
// a hole of the virtual index space (one thread).
__device__ __forceinline__ void g3y_produce(const CUtensorMap* tm, uint32_t it, float2* box, uint64_t* bar) {
  if (it == kG3yHole) {
    mbar_arrive(bar);
    return;
  }
  const int X = (int)(it & 1023u), Y = (int)((it >> 10) & 1023u), Z = (int)(it >> 20);
  const int c[3] = {Z * 8 - 4,    // z (innermost): even start (16-B aligned rows), one extra element
                    Y * 16 - 3,   // y
                    X * 8 - 3};   // x
  mbar_expect_tx(bar, (uint32_t)(g3y::BOX * sizeof(float2)));
  tma_load_box(tm, box, bar, 3, c);
}

// Phase B, load part: the permutation entry and the keys kernel's 16-B user-order record (rec3) of
// sorted node s0 + lane (issued one batch ahead: the random record read overlaps a batch of nodes).
__device__ __forceinline__ void g3y_fetch(const GatherParams<float>& p, uint32_t s0, uint32_t e, int lane,
                                          float4& c4, uint32_t& pj) {
  const uint32_t i = s0 + (uint32_t)lane;
  if (i < e) {
    pj = __ldg(&p.perm[i]);
#ifdef G3Y_ABL_SEQREC
    c4 = __ldg(reinterpret_cast<const float4*>(p.xs) + i);
#else
    c4 = __ldg(reinterpret_cast<const float4*>(p.xs) + pj);
#endif
  }
}

// The 8 taps of a node in one dimension (tap polynomials, R1; the same operations and order as
// all_taps): the Horner chains of the even/odd parts run on FFMA2 and share the coefficient operands.
// Kronecker nodes (u == 0 or 1) are fixed up by g3y_kron (exact 0/1 taps).
__device__ __forceinline__ void g3y_taps1(const GatherParams<float>& p, const float u, float (&w)[8]) {
  constexpr int m = 4, NH = PolyH<float>::NH;
  const float x = fmaf(2.0f, u, -1.0f);
  const float y = x * x;
  const float2 yy = make_float2(y, y), xm = make_float2(x, -x);
#pragma unroll
  for (int i = 0; i < m; ++i) {
    float2 h = *reinterpret_cast<const float2*>(p.ceo[NH - 1][i]);
#pragma unroll
    for (int k = NH - 2; k >= 0; --k) h = __ffma2_rn(h, yy, *reinterpret_cast<const float2*>(p.ceo[k][i]));
    const float2 r = __ffma2_rn(xm, make_float2(h.y, h.y), make_float2(h.x, h.x));
    w[i] = r.x;
    w[2 * m - 1 - i] = r.y;
  }
  if (p.edge_sqrt) {   // sinh window: the edge taps' sqrt(1 - (tau/m)^2) factors (dim_state)
    w[0] *= sqrt_r((1.0f - u) * ((float)(2 * m - 1) + u)) * p.inv_m;
    w[2 * m - 1] *= sqrt_r(u * ((float)(2 * m) - u)) * p.inv_m;
  }
}

// Kronecker node (interpolation property): exact 0/1 taps, by selects
__device__ __forceinline__ void g3y_kron(const float u, float (&w)[8]) {
  constexpr int m = 4;
  const bool h0 = u == 0.0f, h1 = u == 1.0f;
#pragma unroll
  for (int i = 0; i < 2 * m; ++i) w[i] = (h0 | h1) ? ((h0 ? i == m - 1 : i == m) ? 1.0f : 0.0f) : w[i];
}

// Phase B: records of sorted nodes [s0, min(s0 + 32, e)) (lane k: node s0 + k; the sort key's minor
// digit puts an x-line's nodes in y-column order): the 24 tap weights (tap polynomials, R1), the y
// weights as the pairs each row-lane group needs at the node's column, and the byte (column, z
// offset).  All lanes evaluate taps (idle lanes on u = 1/2) so that the rare Kronecker fix-up is a warp
// vote; idle lanes write a record at the last node's cell (the node loop runs in pairs and may touch
// one of them; its value is never stored).  Returns the lane's destination index.
template <bool POLY>
__device__ __forceinline__ uint32_t g3y_phase_b(const GatherParams<float>& p, uint32_t s0, uint32_t e, float* rec,
                                                uint8_t* mdb, int lane, const float4 c4, const uint32_t pj) {
  constexpr int T = g3y::T;
  const uint32_t i = s0 + (uint32_t)lane;
  const bool act = i < e;
  float w[3][T];
  const float uu[3] = {act ? c4.x : 0.5f, act ? c4.y : 0.5f, act ? c4.z : 0.5f};
  if (POLY) {
#ifdef G3Y_ABL_NOTAPS
    for (int t = 0; t < 3; ++t)
      for (int q = 0; q < T; ++q) w[t][q] = uu[0] * (float)(q + t);
#else
#pragma unroll
    for (int t = 0; t < 3; ++t) g3y_taps1(p, uu[t], w[t]);
    bool kr = false;
#pragma unroll
    for (int t = 0; t < 3; ++t) kr |= (uu[t] == 0.0f) | (uu[t] == 1.0f);
    if (__any_sync(0xffffffffu, kr)) {
#pragma unroll
      for (int t = 0; t < 3; ++t) g3y_kron(uu[t], w[t]);
    }
#endif
  } else {
    all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[0], p), p, w[0]);
    all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[1], p), p, w[1]);
    all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[2], p), p, w[2]);
  }
  uint32_t md = __float_as_uint(c4.w);
  md = __shfl_sync(0xffffffffu, md, act ? lane : (int)(e - 1u - s0));
  const int col = (int)(md >> 3);
  float* r = rec + lane * g3y::REC;
  reinterpret_cast<float4*>(r)[2] = make_float4(w[1][0], w[1][1], w[1][2], w[1][3]);
  reinterpret_cast<float4*>(r)[3] = make_float4(w[1][4], w[1][5], w[1][6], w[1][7]);
  // row-lane group q holds window rows b = (q - col) & 7 and b ^ 4: pairs (wy[b], wy[b ^ 4])
  float yq[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int b = (q - col) & 7;
    yq[2 * q] = r[8 + b];
    yq[2 * q + 1] = r[8 + (b ^ 4)];
  }
  reinterpret_cast<float4*>(r)[2] = make_float4(yq[0], yq[1], yq[2], yq[3]);
  reinterpret_cast<float4*>(r)[3] = make_float4(yq[4], yq[5], yq[6], yq[7]);
  reinterpret_cast<float4*>(r)[0] = make_float4(w[2][0], w[2][1], w[2][2], w[2][3]);
  reinterpret_cast<float4*>(r)[1] = make_float4(w[2][4], w[2][5], w[2][6], w[2][7]);
  reinterpret_cast<float4*>(r)[4] = make_float4(w[0][0], w[0][1], w[0][2], w[0][3]);
  reinterpret_cast<float4*>(r)[5] = make_float4(w[0][4], w[0][5], w[0][6], w[0][7]);
  mdb[lane] = (uint8_t)md;
  __syncwarp();
  return p.sorted_out ? i : pj;
}

// Shared-memory accesses of the node loop by 32-bit shared address (kept in registers; volatile asm
// so that the loads stay where they are written: the loop is latency-bound and the load placement is
// its schedule).
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}

// the lane's z values 1..15 of the box row at shared address a into a slot (value 0 of a row is never
// a tap: z offsets start at box index 1)
__device__ __forceinline__ void g3y_load_row(uint32_t a, float2 (&R)[16]) {
  R[1] = lds64(a + 8);
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    const float4 v = lds128(a + 16 * k);
    R[2 * k] = make_float2(v.x, v.y);
    R[2 * k + 1] = make_float2(v.z, v.w);
  }
}
// the same under a lane predicate (no divergent branch: the window advance of one lane group)
__device__ __forceinline__ void g3y_load_row_if(uint32_t a, int pred, float2 (&R)[16]) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.s32 p, %15, 0;\n"
      "@p ld.shared.v2.f32 {%0, %1}, [%14+8];\n"
      "@p ld.shared.v4.f32 {%2, %3, %4, %5}, [%14+16];\n"
      "@p ld.shared.v4.f32 {%6, %7, %8, %9}, [%14+32];\n"
      "@p ld.shared.v4.f32 {%10, %11, %12, %13}, [%14+48];\n}"
      : "+f"(R[1].x), "+f"(R[1].y), "+f"(R[2].x), "+f"(R[2].y), "+f"(R[3].x), "+f"(R[3].y), "+f"(R[4].x),
        "+f"(R[4].y), "+f"(R[5].x), "+f"(R[5].y), "+f"(R[6].x), "+f"(R[6].y), "+f"(R[7].x), "+f"(R[7].y)
      : "r"(a), "r"(pred));
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.s32 p, %17, 0;\n"
      "@p ld.shared.v4.f32 {%0, %1, %2, %3}, [%16+64];\n"
      "@p ld.shared.v4.f32 {%4, %5, %6, %7}, [%16+80];\n"
      "@p ld.shared.v4.f32 {%8, %9, %10, %11}, [%16+96];\n"
      "@p ld.shared.v4.f32 {%12, %13, %14, %15}, [%16+112];\n}"
      : "+f"(R[8].x), "+f"(R[8].y), "+f"(R[9].x), "+f"(R[9].y), "+f"(R[10].x), "+f"(R[10].y), "+f"(R[11].x),
        "+f"(R[11].y), "+f"(R[12].x), "+f"(R[12].y), "+f"(R[13].x), "+f"(R[13].y), "+f"(R[14].x), "+f"(R[14].y),
        "+f"(R[15].x), "+f"(R[15].y)
      : "r"(a), "r"(pred));
}

// z-dots of both slots for a node with z offset OZ (taps at box z index OZ + 1 + c); two partial
// sums per slot (even / odd taps) for instruction-level parallelism, added in a fixed order
template <int OZ>
__device__ __forceinline__ void g3y_zdot(const float2 (&R0)[16], const float2 (&R1)[16], const float4& wa,
                                         const float4& wb, float2& d0, float2& d1) {
  const float wz[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#ifdef G3Y_ONE_CHAIN
  d0 = __fmul2_rn(make_float2(wz[0], wz[0]), R0[OZ + 1]);
  d1 = __fmul2_rn(make_float2(wz[0], wz[0]), R1[OZ + 1]);
#pragma unroll
  for (int c = 1; c < 8; ++c) {
    cmac(d0, wz[c], R0[OZ + 1 + c]);
    cmac(d1, wz[c], R1[OZ + 1 + c]);
  }
#else
  float2 e0 = make_float2(0.f, 0.f), o0 = e0, e1 = e0, o1 = e0;
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    cmac(e0, wz[c], R0[OZ + 1 + c]);
    cmac(e1, wz[c], R1[OZ + 1 + c]);
    cmac(o0, wz[c + 1], R0[OZ + 2 + c]);
    cmac(o1, wz[c + 1], R1[OZ + 2 + c]);
  }
  d0 = __fadd2_rn(e0, o0);
  d1 = __fadd2_rn(e1, o1);
#endif
}

__device__ __forceinline__ void g3y_wait(uint64_t* bar, uint32_t parity) {
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

// Work distribution: slots s = 0, 1, 2, ... of a CTA are the x-lines (item s >> 3, x-line s & 7),
// claimed in order by whichever warp is free (shared-memory counter), so a slow x-line does not hold
// up the other warps of its item; a warp claims its next slot while it works on the current one and
// prefetches that slot's key offsets and first record batch.  Item k's box lives in ring buffer k % 3:
// the warp completing the item's eighth x-line loads item k + 3 into it.  (No deadlock: the oldest
// unfinished item's box is always loaded, and every warp holding one of its slots works on it.)
template <bool POLY>
__global__ void __launch_bounds__(g3y::NT, 1) gather3y_kernel(const __grid_constant__ GatherParams<float> p,
                                                              const CUtensorMap* __restrict__ tmap) {
  using namespace g3y;
  extern __shared__ __align__(128) unsigned char g3y_smem[];   // TMA destinations: 128-B aligned
  __shared__ __align__(8) uint64_t full[NBUF];
  __shared__ int s_done[NBUF];
  __shared__ volatile int s_tag[NBUF];   // item whose box buffer b holds or is loading
  __shared__ uint32_t s_next;             // slot counter
  float2* const boxes = reinterpret_cast<float2*>(g3y_smem);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int la = lane & 7, lq = lane >> 3;
  float* const rec = reinterpret_cast<float*>(g3y_smem + OFF_REC) + wid * 32 * REC;
  float2* const part = reinterpret_cast<float2*>(g3y_smem + OFF_PART) + wid * GN * 32;
  uint8_t* const mdb = g3y_smem + OFF_MD + wid * 32;
  float2* __restrict__ out = (float2*)p.out;
  const uint32_t G = gridDim.x;
  const uint32_t nvirt = (uint32_t)p.nkeys_morton;
  const uint32_t* __restrict__ items = reinterpret_cast<const uint32_t*>(tmap + 1);   // gather3y_item_table

  if (tid == 0) {
    s_next = 0;
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&full[b], 1);
      s_done[b] = 0;
    }
    fence_mbar_init();
    for (int b = 0; b < NBUF; ++b) {
      s_tag[b] = b;
      const uint32_t v = blockIdx.x + (uint32_t)b * G;
      if (v < nvirt) g3y_produce(tmap, __ldg(&items[v]), boxes + (size_t)b * (BOXB / 8), &full[b]);
    }
  }
  __syncthreads();

  // claim the next slot; its item k (or ~0u past the CTA's last item), x-line w and node range
  struct Slot {
    uint32_t k, b0, e0;
    int w;
  };
  auto claim = [&]() {
    Slot s;
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(&s_next, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    s.k = c >> 3;
    s.w = (int)(c & 7u);
    s.b0 = s.e0 = 0;
    const uint32_t v = blockIdx.x + s.k * G;
    if (v >= nvirt) {
      s.k = ~0u;
      return s;
    }
    const uint32_t it = __ldg(&items[v]);
    if (it == kG3yHole) return s;
    const int X = (int)(it & 1023u), Y = (int)((it >> 10) & 1023u), Z = (int)(it >> 20);
    const int cx = X * 8 + s.w;
    if (cx >= (int)p.L) return s;
    const int64_t key = ((int64_t)cx * p.nb[1] + Y) * p.nb[2] + Z;
    s.b0 = __ldg(&p.key_start[key]);
    s.e0 = __ldg(&p.key_start[key + 1]);
    return s;
  };
  // The first batch of a slot's nodes (permutation entries and records) is fetched during the
  // previous slot's last batch, and the next slot's key offsets at the start of the current one, so
  // no global-memory latency is exposed at slot boundaries.
  Slot cur = claim();
  Slot nxt = claim();
  float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t pj = 0;
  if (cur.b0 < cur.e0) g3y_fetch(p, cur.b0, cur.e0, lane, c4, pj);
  while (cur.k != ~0u) {
    const uint32_t k = cur.k;
    const int b = (int)(k % NBUF);
    const uint32_t nb0 = cur.b0, ne = cur.e0;
    const float2* box = boxes + (size_t)b * (BOXB / 8);
    const int xa = cur.w + la;       // box x index of the lane's rows
    uint32_t dst = 0;
    if (nb0 < ne) dst = g3y_phase_b<POLY>(p, nb0, ne, rec, mdb, lane, c4, pj);   // overlaps the box's TMA
    else if (nxt.b0 < nxt.e0) g3y_fetch(p, nxt.b0, nxt.e0, lane, c4, pj);
    while (s_tag[b] != (int)k) {
    }
    g3y_wait(&full[b], (k / NBUF) & 1u);
    if (nb0 < ne) {
      // ---- sweep: nodes in column order; the row window starts at the first node's column
      float2 R0[16], R1[16];
      const uint32_t rec_s = smem_u32(rec), mdb_s = smem_u32(mdb);
      // the lane's x-plane of the box (rows of 144 B)
      uint32_t row_s = smem_u32(box) + (uint32_t)(xa * (BY * BZ * 8));
      int lqo = lq;   // (opaque copies: kept in registers instead of being recomputed in the loop)
      asm volatile("" : "+r"(row_s), "+r"(lqo));
      int ycur = (int)(lds8(mdb_s) >> 3);
      g3y_load_row(row_s + (uint32_t)(ycur + ((lq - ycur) & 7)) * (BZ * 8), R0);
      g3y_load_row(row_s + (uint32_t)(ycur + ((lq + 4 - ycur) & 7)) * (BZ * 8), R1);
      for (uint32_t s0 = nb0;;) {
        const int nq = (int)min(32u, ne - s0);
        if (s0 + 32 < ne) g3y_fetch(p, s0 + 32, ne, lane, c4, pj);   // next batch, in flight meanwhile
        else if (nxt.b0 < nxt.e0) g3y_fetch(p, nxt.b0, nxt.e0, lane, c4, pj);   // the next slot's first batch
        auto advance = [&](int col) {
          if (ycur < col) {
#pragma unroll 1
            do {   // window [ycur, ycur + 8) -> [ycur + 1, ycur + 9): row ycur + 8
              const int rn = ycur + 8;
              const uint32_t a = row_s + (uint32_t)rn * (BZ * 8);
              const int mine = lqo == (rn & 3);
              if (rn & 4) g3y_load_row_if(a, mine, R1);
              else g3y_load_row_if(a, mine, R0);
            } while (++ycur < col);
          }
        };
        auto zdot = [&](uint32_t oz, const float4& wa, const float4& wb, float2& d0, float2& d1) {
          switch (oz) {
            case 0: g3y_zdot<0>(R0, R1, wa, wb, d0, d1); break;
            case 1: g3y_zdot<1>(R0, R1, wa, wb, d0, d1); break;
            case 2: g3y_zdot<2>(R0, R1, wa, wb, d0, d1); break;
            case 3: g3y_zdot<3>(R0, R1, wa, wb, d0, d1); break;
            case 4: g3y_zdot<4>(R0, R1, wa, wb, d0, d1); break;
            case 5: g3y_zdot<5>(R0, R1, wa, wb, d0, d1); break;
            case 6: g3y_zdot<6>(R0, R1, wa, wb, d0, d1); break;
            default: g3y_zdot<7>(R0, R1, wa, wb, d0, d1); break;
          }
        };
        // Nodes run in pairs, groups of GN.  Per node: window advance to its column, the lane's two
        // z-dots, their y contraction; the lane's share (x-plane a, row lanes q) goes to row j of the
        // group's partial buffer.  Records are loaded ahead of use: the pair's second node during the
        // first one's z-dots, the next pair's first node during the second one's.  After each group
        // lane (n, h) = (lane >> 2, lane & 3) contracts node n's partials of x-planes 2h, 2h + 1 (all
        // four row-lane groups) with wx, two shuffles add the four h, lanes h = 0 store (fixed
        // order: bitwise reproducible).
        uint32_t r_s = rec_s, ry_s = rec_s + 32 + 8 * lq, mq_s = mdb_s;   // running: record, y pair, md
        uint32_t mdA = lds8(mq_s);
        float4 waA = lds128(r_s), wbA = lds128(r_s + 16);
        float2 wyA = lds64(ry_s);
        for (int g0 = 0; g0 < nq; g0 += GN) {
          uint32_t pp = smem_u32(part) + 8 * lane;
          const uint32_t pe = pp + 256 * min(GN, (nq - g0 + 1) & ~1);
#pragma unroll 1
          do {
            float2 d0, d1, t;
            advance((int)(mdA >> 3));
            zdot(mdA & 7u, waA, wbA, d0, d1);
            const uint32_t mdB = lds8(mq_s + 1);
            const float4 waB = lds128(r_s + 4 * REC), wbB = lds128(r_s + 4 * REC + 16);
            const float2 wyB = lds64(ry_s + 4 * REC);
            t = __fmul2_rn(make_float2(wyA.x, wyA.x), d0);
            cmac(t, wyA.y, d1);
            sts64(pp, t);
            advance((int)(mdB >> 3));
            zdot(mdB & 7u, waB, wbB, d0, d1);
            mdA = lds8(mq_s + 2);          // (past the batch: unused)
            waA = lds128(r_s + 8 * REC);
            wbA = lds128(r_s + 8 * REC + 16);
            wyA = lds64(ry_s + 8 * REC);
            t = __fmul2_rn(make_float2(wyB.x, wyB.x), d0);
            cmac(t, wyB.y, d1);
            sts64(pp + 256, t);
            pp += 512;
            r_s += 8 * REC;
            ry_s += 8 * REC;
            mq_s += 2;
          } while (pp != pe);
          __syncwarp();
          {
            const int n = lane >> 2, h = lane & 3;
            const float2 wx = lds64(rec_s + (uint32_t)((g0 + n) * (4 * REC) + 64 + 8 * h));
            const uint32_t pr = smem_u32(part) + (uint32_t)(n * 256 + h * 16);
            float2 f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 v = lds128(pr + 64 * i);
              if (i == 0) f = __fmul2_rn(make_float2(wx.x, wx.x), make_float2(v.x, v.y));
              else cmac(f, wx.x, make_float2(v.x, v.y));
              cmac(f, wx.y, make_float2(v.z, v.w));
            }
            f = __fadd2_rn(f, make_float2(__shfl_xor_sync(0xffffffffu, f.x, 1), __shfl_xor_sync(0xffffffffu, f.y, 1)));
            f = __fadd2_rn(f, make_float2(__shfl_xor_sync(0xffffffffu, f.x, 2), __shfl_xor_sync(0xffffffffu, f.y, 2)));
            const uint32_t d = __shfl_sync(0xffffffffu, dst, g0 + n);
            if (h == 0 && g0 + n < nq) out[d] = f;
          }
          __syncwarp();   // partial buffer free for the next group
        }
        s0 += 32;
        if (s0 >= ne) break;
        dst = g3y_phase_b<POLY>(p, s0, ne, rec, mdb, lane, c4, pj);
      }
    }
    // ---- release box buffer b; the warp completing the item's eighth x-line loads item k + NBUF
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const int old = atomicAdd(&s_done[b], 1);
      if (old == 7) {
        s_done[b] = 0;
        const uint32_t kn = k + NBUF;
        const uint32_t vn = blockIdx.x + kn * G;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        s_tag[b] = (int)kn;
        __threadfence_block();
        if (vn < nvirt) g3y_produce(tmap, __ldg(&items[vn]), boxes + (size_t)b * (BOXB / 8), &full[b]);
      }
    }
    cur = nxt;
    if (cur.k != ~0u) nxt = claim();
  }
}

// ---------------------------------------------------------------------------------------------
// gather3q: the y-sweep with half-height rows and no z dispatch.
//
// gather3y's node loop spends a third of its instructions on warp-uniform control flow: the 8-way
// dispatch on the node's z offset (a register window cannot be indexed dynamically) and the window
// advance.  Here the sort's minor digit is (z half, column): an x-line's nodes arrive as two column
// sweeps, one per half of the bin's z extent (cells 8 bz + 4 h .. + 3).  A lane's rows then hold only
// the 12 z values of the half (box z index 4 h .. 4 h + 11), and the node's z offset dz in 0..3 is
// folded into its weights: the record stores wz12[k] = wz[k - 1 - dz] (0 outside the 8 taps), so every
// node runs the same straight-line 11-tap z-dots (22 FFMA2 instead of 16, no branches, 48 row
// registers instead of 64).  Everything else (items, boxes, TMA ring, slots, tap phase, reduction) is
// gather3y's; the x reduction runs per group of 4 nodes so that the 28-word records fit.
namespace g3q {

constexpr int NW = g3y::NW, NT = NW * 32, NBUF = g3y::NBUF, T = 8;
constexpr int BY = g3y::BY, BZ = g3y::BZ, BOXB = g3y::BOXB;   // gather3y's box
constexpr int RZ = 12;                     // z values per register row
constexpr int REC = 28;                    // words per record: wz12[12] | wy pairs[8] | wx[8]  (112 B: the
                                           // 16-B slots of 8 consecutive lanes' records are distinct)
constexpr int GN = 4;                      // nodes per reduction group
constexpr int OFF_REC = NBUF * BOXB;                           // float [NW][32][REC]
constexpr int OFF_PART = OFF_REC + NW * 32 * REC * 4;          // float2 [NW][GN][32]: lane partials
constexpr int OFF_MD = OFF_PART + NW * GN * 32 * 8;            // uint8 [NW][32]: (z half, column) << 2 | dz
constexpr int SMEM = OFF_MD + NW * 32 + 32;   // (+32: md reads run one pair past a batch)
static_assert(OFF_REC % 16 == 0 && OFF_PART % 16 == 0, "16-B aligned records and partials");
static_assert(SMEM + 128 <= 227 * 1024, "shared memory per CTA");

}  // namespace g3q

size_t gather3q_smem() { return (size_t)g3q::SMEM; }

// Phase B of gather3q (cf. g3y_phase_b): record of node s0 + lane.
template <bool POLY>
__device__ __forceinline__ uint32_t g3q_phase_b(const GatherParams<float>& p, uint32_t s0, uint32_t e, float* rec,
                                                uint8_t* mdb, int lane, const float4 c4, const uint32_t pj) {
  constexpr int T = g3q::T;
  const uint32_t i = s0 + (uint32_t)lane;
  const bool act = i < e;
  float w[3][T];
  const float uu[3] = {act ? c4.x : 0.5f, act ? c4.y : 0.5f, act ? c4.z : 0.5f};
  if (POLY) {
#pragma unroll
    for (int t = 0; t < 3; ++t) g3y_taps1(p, uu[t], w[t]);
    bool kr = false;
#pragma unroll
    for (int t = 0; t < 3; ++t) kr |= (uu[t] == 0.0f) | (uu[t] == 1.0f);
    if (__any_sync(0xffffffffu, kr)) {
#pragma unroll
      for (int t = 0; t < 3; ++t) g3y_kron(uu[t], w[t]);
    }
  } else {
    all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[0], p), p, w[0]);
    all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[1], p), p, w[1]);
    all_taps<T, POLY>(dim_state<T, float, POLY>((double)uu[2], p), p, w[2]);
  }
  uint32_t md = __float_as_uint(c4.w);
  md = __shfl_sync(0xffffffffu, md, act ? lane : (int)(e - 1u - s0));   // idle lanes: the last node's cell
  const int col = (int)((md >> 2) & 15u);
  const bool d1 = (md & 1u) != 0, d2 = (md & 2u) != 0;
  float* r = rec + lane * g3q::REC;
  // z weights by row position k (box z index 4 h + k): wz12[k] = wz[k - 1 - dz], by selects
  float z12[g3q::RZ];
#pragma unroll
  for (int k = 0; k < g3q::RZ; ++k) {
    const float a0 = (k - 1 >= 0 && k - 1 < T) ? w[2][(k - 1 >= 0 && k - 1 < T) ? k - 1 : 0] : 0.0f;
    const float a1 = (k - 2 >= 0 && k - 2 < T) ? w[2][(k - 2 >= 0 && k - 2 < T) ? k - 2 : 0] : 0.0f;
    const float a2 = (k - 3 >= 0 && k - 3 < T) ? w[2][(k - 3 >= 0 && k - 3 < T) ? k - 3 : 0] : 0.0f;
    const float a3 = (k - 4 >= 0 && k - 4 < T) ? w[2][(k - 4 >= 0 && k - 4 < T) ? k - 4 : 0] : 0.0f;
    const float s01 = d1 ? a1 : a0, s23 = d1 ? a3 : a2;
    z12[k] = d2 ? s23 : s01;
  }
  reinterpret_cast<float4*>(r)[3] = make_float4(w[1][0], w[1][1], w[1][2], w[1][3]);
  reinterpret_cast<float4*>(r)[4] = make_float4(w[1][4], w[1][5], w[1][6], w[1][7]);
  // row-lane group q holds window rows b = (q - col) & 7 and b ^ 4: pairs (wy[b], wy[b ^ 4])
  float yq[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int b = (q - col) & 7;
    yq[2 * q] = r[12 + b];
    yq[2 * q + 1] = r[12 + (b ^ 4)];
  }
  reinterpret_cast<float4*>(r)[3] = make_float4(yq[0], yq[1], yq[2], yq[3]);
  reinterpret_cast<float4*>(r)[4] = make_float4(yq[4], yq[5], yq[6], yq[7]);
  reinterpret_cast<float4*>(r)[0] = make_float4(z12[0], z12[1], z12[2], z12[3]);
  reinterpret_cast<float4*>(r)[1] = make_float4(z12[4], z12[5], z12[6], z12[7]);
  reinterpret_cast<float4*>(r)[2] = make_float4(z12[8], z12[9], z12[10], z12[11]);
  reinterpret_cast<float4*>(r)[5] = make_float4(w[0][0], w[0][1], w[0][2], w[0][3]);
  reinterpret_cast<float4*>(r)[6] = make_float4(w[0][4], w[0][5], w[0][6], w[0][7]);
  mdb[lane] = (uint8_t)md;
  __syncwarp();
  return p.sorted_out ? i : pj;
}

// the lane's 12 z values of the box row at shared address a (16-B aligned) into a slot
__device__ __forceinline__ void g3q_load_row(uint32_t a, float2 (&R)[g3q::RZ]) {
#pragma unroll
  for (int k = 0; k < g3q::RZ / 2; ++k) {
    const float4 v = lds128(a + 16 * k);
    R[2 * k] = make_float2(v.x, v.y);
    R[2 * k + 1] = make_float2(v.z, v.w);
  }
}
// the same under a lane predicate (no divergent branch: the window advance of one lane group)
__device__ __forceinline__ void g3q_load_row_if(uint32_t a, int pred, float2 (&R)[g3q::RZ]) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.s32 p, %13, 0;\n"
      "@p ld.shared.v4.f32 {%0, %1, %2, %3}, [%12];\n"
      "@p ld.shared.v4.f32 {%4, %5, %6, %7}, [%12+16];\n"
      "@p ld.shared.v4.f32 {%8, %9, %10, %11}, [%12+32];\n}"
      : "+f"(R[0].x), "+f"(R[0].y), "+f"(R[1].x), "+f"(R[1].y), "+f"(R[2].x), "+f"(R[2].y), "+f"(R[3].x),
        "+f"(R[3].y), "+f"(R[4].x), "+f"(R[4].y), "+f"(R[5].x), "+f"(R[5].y)
      : "r"(a), "r"(pred));
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.s32 p, %13, 0;\n"
      "@p ld.shared.v4.f32 {%0, %1, %2, %3}, [%12+48];\n"
      "@p ld.shared.v4.f32 {%4, %5, %6, %7}, [%12+64];\n"
      "@p ld.shared.v4.f32 {%8, %9, %10, %11}, [%12+80];\n}"
      : "+f"(R[6].x), "+f"(R[6].y), "+f"(R[7].x), "+f"(R[7].y), "+f"(R[8].x), "+f"(R[8].y), "+f"(R[9].x),
        "+f"(R[9].y), "+f"(R[10].x), "+f"(R[10].y), "+f"(R[11].x), "+f"(R[11].y)
      : "r"(a), "r"(pred));
}

// z-dots of both slots: positions 1..11 of the rows against wz12 (position 0 is never a tap); two
// partial sums per slot (odd / even positions), added in a fixed order
__device__ __forceinline__ void g3q_zdot(const float2 (&R0)[g3q::RZ], const float2 (&R1)[g3q::RZ], const float4& wa,
                                         const float4& wb, const float4& wc, float2& d0, float2& d1) {
  const float wz[12] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w, wc.x, wc.y, wc.z, wc.w};
  float2 e0 = __fmul2_rn(make_float2(wz[1], wz[1]), R0[1]), e1 = __fmul2_rn(make_float2(wz[1], wz[1]), R1[1]);
  float2 o0 = __fmul2_rn(make_float2(wz[2], wz[2]), R0[2]), o1 = __fmul2_rn(make_float2(wz[2], wz[2]), R1[2]);
#pragma unroll
  for (int k = 3; k < 11; k += 2) {
    cmac(e0, wz[k], R0[k]);
    cmac(e1, wz[k], R1[k]);
    cmac(o0, wz[k + 1], R0[k + 1]);
    cmac(o1, wz[k + 1], R1[k + 1]);
  }
  cmac(e0, wz[11], R0[11]);
  cmac(e1, wz[11], R1[11]);
  d0 = __fadd2_rn(e0, o0);
  d1 = __fadd2_rn(e1, o1);
}

template <bool POLY>
__global__ void __launch_bounds__(g3q::NT, 1) gather3q_kernel(const __grid_constant__ GatherParams<float> p,
                                                              const CUtensorMap* __restrict__ tmap) {
  using namespace g3q;
  extern __shared__ __align__(128) unsigned char g3q_smem[];   // TMA destinations: 128-B aligned
  __shared__ __align__(8) uint64_t full[NBUF];
  __shared__ int s_done[NBUF];
  __shared__ volatile int s_tag[NBUF];   // item whose box buffer b holds or is loading
  __shared__ uint32_t s_next;             // slot counter
  float2* const boxes = reinterpret_cast<float2*>(g3q_smem);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int la = lane & 7, lq = lane >> 3;
  float* const rec = reinterpret_cast<float*>(g3q_smem + OFF_REC) + wid * 32 * REC;
  float2* const part = reinterpret_cast<float2*>(g3q_smem + OFF_PART) + wid * GN * 32;
  uint8_t* const mdb = g3q_smem + OFF_MD + wid * 32;
  float2* __restrict__ out = (float2*)p.out;
  const uint32_t G = gridDim.x;
  const uint32_t nvirt = (uint32_t)p.nkeys_morton;
  const uint32_t* __restrict__ items = reinterpret_cast<const uint32_t*>(tmap + 1);   // gather3y_item_table

  if (tid == 0) {
    s_next = 0;
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&full[b], 1);
      s_done[b] = 0;
    }
    fence_mbar_init();
    for (int b = 0; b < NBUF; ++b) {
      s_tag[b] = b;
      const uint32_t v = blockIdx.x + (uint32_t)b * G;
      if (v < nvirt) g3y_produce(tmap, __ldg(&items[v]), boxes + (size_t)b * (BOXB / 8), &full[b]);
    }
  }
  __syncthreads();

  // slots: as gather3y_kernel
  struct Slot {
    uint32_t k, b0, e0;
    int w;
  };
  auto claim = [&]() {
    Slot s;
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(&s_next, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    s.k = c >> 3;
    s.w = (int)(c & 7u);
    s.b0 = s.e0 = 0;
    const uint32_t v = blockIdx.x + s.k * G;
    if (v >= nvirt) {
      s.k = ~0u;
      return s;
    }
    const uint32_t it = __ldg(&items[v]);
    if (it == kG3yHole) return s;
    const int X = (int)(it & 1023u), Y = (int)((it >> 10) & 1023u), Z = (int)(it >> 20);
    const int cx = X * 8 + s.w;
    if (cx >= (int)p.L) return s;
    const int64_t key = ((int64_t)cx * p.nb[1] + Y) * p.nb[2] + Z;
    s.b0 = __ldg(&p.key_start[key]);
    s.e0 = __ldg(&p.key_start[key + 1]);
    return s;
  };
  Slot cur = claim();
  Slot nxt = claim();
  float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t pj = 0;
  if (cur.b0 < cur.e0) g3y_fetch(p, cur.b0, cur.e0, lane, c4, pj);
  while (cur.k != ~0u) {
    const uint32_t k = cur.k;
    const int b = (int)(k % NBUF);
    const uint32_t nb0 = cur.b0, ne = cur.e0;
    const float2* box = boxes + (size_t)b * (BOXB / 8);
    const int xa = cur.w + la;       // box x index of the lane's rows
    uint32_t dst = 0;
    if (nb0 < ne) dst = g3q_phase_b<POLY>(p, nb0, ne, rec, mdb, lane, c4, pj);   // overlaps the box's TMA
    else if (nxt.b0 < nxt.e0) g3y_fetch(p, nxt.b0, nxt.e0, lane, c4, pj);
    while (s_tag[b] != (int)k) {
    }
    g3y_wait(&full[b], (k / NBUF) & 1u);
    if (nb0 < ne) {
      // ---- two column sweeps (z halves); the window position is vcur = z half << 4 | first row
      float2 R0[RZ], R1[RZ];
      const uint32_t rec_s = smem_u32(rec), mdb_s = smem_u32(mdb), part_s = smem_u32(part);
      uint32_t row_s = smem_u32(box) + (uint32_t)(xa * (BY * BZ * 8));   // the lane's x-plane (rows of 144 B)
      int lqo = lq;   // (opaque copies: kept in registers instead of being recomputed in the loop)
      asm volatile("" : "+r"(row_s), "+r"(lqo));
      int vcur;
      auto restart = [&](int v) {   // window rows y .. y + 7 of z half v >> 4
        const int y = v & 15;
        const uint32_t a = row_s + (uint32_t)(v >> 4) * 32u;
        g3q_load_row(a + (uint32_t)(y + ((lqo - y) & 7)) * (BZ * 8), R0);
        g3q_load_row(a + (uint32_t)(y + ((lqo + 4 - y) & 7)) * (BZ * 8), R1);
        vcur = v;
      };
      restart((int)(lds8(mdb_s) >> 2));
      for (uint32_t s0 = nb0;;) {
        const int nq = (int)min(32u, ne - s0);
        if (s0 + 32 < ne) g3y_fetch(p, s0 + 32, ne, lane, c4, pj);   // next batch, in flight meanwhile
        else if (nxt.b0 < nxt.e0) g3y_fetch(p, nxt.b0, nxt.e0, lane, c4, pj);   // the next slot's first batch
        auto advance = [&](int v) {
          if (vcur < v) {
            if ((v ^ vcur) & 16) {
              restart(v);
            } else {
#pragma unroll 1
              do {   // window [y, y + 8) -> [y + 1, y + 9): row y + 8
                const int rn = (vcur & 15) + 8;
                const uint32_t a = row_s + (uint32_t)(vcur >> 4) * 32u + (uint32_t)rn * (BZ * 8);
                const int mine = lqo == (rn & 3);
                if (rn & 4) g3q_load_row_if(a, mine, R1);
                else g3q_load_row_if(a, mine, R0);
              } while (++vcur < v);
            }
          }
        };
        // Nodes run in pairs, groups of GN (cf. gather3y_kernel): window advance, the lane's two
        // z-dots, their y contraction, the lane's share to row j of the group's partial buffer; the
        // pair's second record is loaded during the first node's z-dots, the next pair's first during
        // the second's.  After each group lane (n, h) = (lane >> 3, lane & 7) contracts node n's
        // partials of x-planes 2 (h & 3), 2 (h & 3) + 1 of row-lane groups 2 (h >> 2), 2 (h >> 2) + 1
        // with wx, three shuffles add the eight h, lanes h = 0 store (fixed order).
        uint32_t r_s = rec_s, ry_s = rec_s + 48 + 8 * lq, mq_s = mdb_s;   // running: record, y pair, md
        uint32_t mdA = lds8(mq_s);
        float4 waA = lds128(r_s), wbA = lds128(r_s + 16), wcA = lds128(r_s + 32);
        float2 wyA = lds64(ry_s);
        for (int g0 = 0; g0 < nq; g0 += GN) {
          uint32_t pp = part_s + 8 * lane;
          const uint32_t pe = pp + 256 * min(GN, (nq - g0 + 1) & ~1);
#pragma unroll 1
          do {
            float2 d0, d1, t;
            advance((int)(mdA >> 2));
            g3q_zdot(R0, R1, waA, wbA, wcA, d0, d1);
            const uint32_t mdB = lds8(mq_s + 1);
            const float4 waB = lds128(r_s + 4 * REC), wbB = lds128(r_s + 4 * REC + 16),
                         wcB = lds128(r_s + 4 * REC + 32);
            const float2 wyB = lds64(ry_s + 4 * REC);
            t = __fmul2_rn(make_float2(wyA.x, wyA.x), d0);
            cmac(t, wyA.y, d1);
            sts64(pp, t);
            advance((int)(mdB >> 2));
            g3q_zdot(R0, R1, waB, wbB, wcB, d0, d1);
            mdA = lds8(mq_s + 2);          // (past the batch: unused)
            waA = lds128(r_s + 8 * REC);
            wbA = lds128(r_s + 8 * REC + 16);
            wcA = lds128(r_s + 8 * REC + 32);
            wyA = lds64(ry_s + 8 * REC);
            t = __fmul2_rn(make_float2(wyB.x, wyB.x), d0);
            cmac(t, wyB.y, d1);
            sts64(pp + 256, t);
            pp += 512;
            r_s += 8 * REC;
            ry_s += 8 * REC;
            mq_s += 2;
          } while (pp != pe);
          __syncwarp();
          {
            const int n = lane >> 3, h = lane & 7, hp = h & 3, qh = h >> 2;
            const float2 wx = lds64(rec_s + (uint32_t)((g0 + n) * (4 * REC) + 80 + 8 * hp));
            const uint32_t pr = part_s + (uint32_t)(n * 256 + qh * 128 + hp * 16);
            const float4 v0 = lds128(pr), v1 = lds128(pr + 64);
            float2 f = __fmul2_rn(make_float2(wx.x, wx.x), make_float2(v0.x, v0.y));
            cmac(f, wx.y, make_float2(v0.z, v0.w));
            cmac(f, wx.x, make_float2(v1.x, v1.y));
            cmac(f, wx.y, make_float2(v1.z, v1.w));
            f = __fadd2_rn(f, make_float2(__shfl_xor_sync(0xffffffffu, f.x, 1), __shfl_xor_sync(0xffffffffu, f.y, 1)));
            f = __fadd2_rn(f, make_float2(__shfl_xor_sync(0xffffffffu, f.x, 2), __shfl_xor_sync(0xffffffffu, f.y, 2)));
            f = __fadd2_rn(f, make_float2(__shfl_xor_sync(0xffffffffu, f.x, 4), __shfl_xor_sync(0xffffffffu, f.y, 4)));
            const uint32_t d = __shfl_sync(0xffffffffu, dst, (g0 + n) & 31);
            if (h == 0 && g0 + n < nq) out[d] = f;
          }
          __syncwarp();   // partial buffer free for the next group
        }
        s0 += 32;
        if (s0 >= ne) break;
        dst = g3q_phase_b<POLY>(p, s0, ne, rec, mdb, lane, c4, pj);
      }
    }
    // ---- release box buffer b; the warp completing the item's eighth x-line loads item k + NBUF
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const int old = atomicAdd(&s_done[b], 1);
      if (old == 7) {
        s_done[b] = 0;
        const uint32_t kn = k + NBUF;
        const uint32_t vn = blockIdx.x + kn * G;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        s_tag[b] = (int)kn;
        __threadfence_block();
        if (vn < nvirt) g3y_produce(tmap, __ldg(&items[vn]), boxes + (size_t)b * (BOXB / 8), &full[b]);
      }
    }
    cur = nxt;
    if (cur.k != ~0u) nxt = claim();
  }
}

const void* gather3q_kernel_ptr(bool poly) {
  return poly ? (const void*)gather3q_kernel<true> : (const void*)gather3q_kernel<false>;
}

const void* gather3y_kernel_ptr(bool poly) {
  return poly ? (const void*)gather3y_kernel<true> : (const void*)gather3y_kernel<false>;
}

}  // namespace bnfft
