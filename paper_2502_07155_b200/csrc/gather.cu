// Row a6 gather: host-side dispatch and launch (kernels in gather_impl.cuh).
#include <cuda.h>

#include <cstring>
#include <vector>

#include "gather_impl.cuh"

namespace bnfft {

const void* gather3c_kernel_p();
const void* gather3c_kernel_e();
const void* gather3s_kernel_ptr(bool poly);
size_t gather3s_smem();
int gather3s_threads();
int gather3s_row_stride();
const void* gather3y_kernel_ptr(bool poly);
size_t gather3y_smem();
int gather3y_threads();
void gather3y_box(int* ext);
const void* gather3q_kernel_ptr(bool poly);
const void* gather2c_kernel_ptr(int m, bool poly);
size_t gather2c_stash_bytes(int threads);
int gather2c_pad_bytes();
int gather2c_max_m();
size_t gather3q_smem();
void gather3y_item_table(int64_t nX, int64_t nY, int64_t nZ, std::vector<uint32_t>& tab);

// d = 3, m = 4, complex64, batch 1: a specialised kernel chosen at plan creation (p->g3_kind) -- the
// y-sweep kernel gather3y (gather3y.cu, x-line bins of 1 x 16 x 8 cells) by default; the half-warp
// kernel gather3c (BNFFT_GATHER3C) and the z-sweep kernel gather3s (BNFFT_GATHER3S, gather3s.cu) on
// bins of 8 x 8 x 16 cells (measured slower on cfg4: DESIGN.md §8)
static bool use_coop3(const bnfft_plan_s* p) {
  return p->opts.d == 3 && p->opts.m == 4 && !p->c128 && p->opts.batch == 1;
}
static bool use_sweep3(const bnfft_plan_s* p) { return use_coop3(p) && p->g3_kind == 2; }
static bool use_ysweep3(const bnfft_plan_s* p) { return use_coop3(p) && (p->g3_kind == 0 || p->g3_kind == 3); }
static const void* coop3_kernel(const bnfft_plan_s* p) {
  if (p->g3_kind == 0) return gather3y_kernel_ptr(p->tap_poly);
  if (p->g3_kind == 3) return gather3q_kernel_ptr(p->tap_poly);
  if (p->g3_kind == 2) return gather3s_kernel_ptr(p->tap_poly);
  return p->tap_poly ? gather3c_kernel_p() : gather3c_kernel_e();
}

// d = 2, complex64, batch 1, m <= 7: the quarter-warp-cooperative box kernel (gather2c.cu) unless
// BNFFT_GATHER2N selects the thread-per-node kernel gatherN (chosen at plan creation: p->g2_coop)
static bool use_coop2(const bnfft_plan_s* p) { return p->g2_coop; }

static const void* select_kernel(int d, int m, bool c128, bool poly, bool batched = false, bool pre = false,
                                bool binned = false) {
  if (d == 1 && pre && !batched) return c128 ? gather_kernel_1d(m + 300, poly) : gather_kernel_1f(m + 300, poly);
  if (d == 1 && binned && !batched) return c128 ? gather_kernel_1d(m + 400, poly) : gather_kernel_1f(m + 400, poly);
  if (d == 3 && m == 4 && !c128 && !batched)
    return getenv("BNFFT_GATHER3S") ? gather3s_kernel_ptr(poly) : (poly ? gather3c_kernel_p() : gather3c_kernel_e());
  if (d == 1 && batched) return c128 ? gather_kernel_1d(m + 100, poly) : gather_kernel_1f(m + 100, poly);
  if (d == 1) return c128 ? gather_kernel_1d(m, poly) : gather_kernel_1f(m, poly);
  if (d == 2) return c128 ? gather_kernel_2d(m, poly) : gather_kernel_2f(m, poly);
  if (d == 3) return c128 ? gather_kernel_3d(m, poly) : gather_kernel_3f(m, poly);
  return nullptr;
}

int gather_supported(int d, int m) {
  if (m < 1) return 0;
  if (d == 1) return m <= kMaxM1;
  if (d == 2) return m <= kMaxM2;
  if (d == 3) return m <= kMaxM3;
  return 0;
}

size_t gather_box_elems(const bnfft_plan_s* p) {
  size_t e = 1;
  for (int t = 0; t < p->opts.d; ++t) e *= (size_t)((1 << p->bin_log2[t]) + 2 * p->opts.m - 1);
  return e;
}

// Dynamic shared memory for staged boxes; the kernel also uses ~2 KB of static shared memory, and
// the sum must stay under the 48 KB default (the attribute is raised only for single large boxes).
static size_t smem_budget() { return 40u << 10; }

// ---- d = 2, 3: TMA tensor map over theta and the binned persistent kernel
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static cudaError_t gatherN_prepare(bnfft_plan_s* p, const void* fn) {
  const int d = p->opts.d, T = 2 * p->opts.m;
  // box extents per dim (dim 0 slowest); the innermost extent is padded to 16 bytes for TMA
  int ext[3];
  for (int t = 0; t < d; ++t) ext[t] = (1 << p->bin_log2[t]) + T - 1;
  if (!p->c128) ext[d - 1] = (1 << p->bin_log2[d - 1]) + T;   // even start shift + 16-B multiple
  if (use_coop3(p)) ext[d - 1] = use_sweep3(p) ? gather3s_row_stride() : kRow3;   // conflict-free rows
  if (use_ysweep3(p)) gather3y_box(ext);
  size_t box_elems = 1;
  for (int t = 0; t < d; ++t) box_elems *= (size_t)ext[t];
  const size_t per = box_elems * p->csize;
  const size_t budget = 48u << 10;              // bytes per staging buffer
  int bt = (int)std::max<size_t>(1, std::min<size_t>((size_t)p->opts.batch, budget / per));
  if (bt > 256) bt = 256;
  const size_t buf_bytes = (per * bt + (use_coop2(p) ? (size_t)gather2c_pad_bytes() : 0) + 127) & ~(size_t)127;
  // coop kernel: one box buffer, more CTAs per SM; gatherN: a ring of up to kMaxBoxBufs buffers
  // (mbarrier-released, see gatherN_kernel) within 100 KB (at least two)
  int nbuf = 1;
  if (!use_coop3(p)) {
    nbuf = 3 * buf_bytes <= ((size_t)100 << 10) ? 3 : 2;
    if (const char* s = getenv("BNFFT_BOX_BUFS")) nbuf = std::max(2, std::min(kMaxBoxBufs, atoi(s)));   // tuning knob
  }
  if (use_coop2(p) && !getenv("BNFFT_BOX_BUFS")) nbuf = 2;   // measured best with 64-thread CTAs (cfg3)
  p->gather_nbuf = nbuf;
  p->gather_bt = bt;
  p->gather_nslice = (p->opts.batch + bt - 1) / bt;
  p->gather_box_elems = (int)box_elems;
  p->gather_bufstride = (int)(buf_bytes / p->csize);
  for (int t = 0; t < 3; ++t) p->gather_tbox[t] = t < d ? ext[t] : 1;
  p->gather_smem = use_sweep3(p) ? gather3s_smem() : use_ysweep3(p) ? (p->g3_kind == 3 ? gather3q_smem() : gather3y_smem()) : nbuf * buf_bytes;
  p->gather_threads = use_sweep3(p) ? gather3s_threads() : use_ysweep3(p) ? gather3y_threads() : kGatherThreads;
  if (use_coop2(p)) {   // small CTAs: a uniform cfg3 item (~64 nodes) is one batch per warp (knob: 64..256)
    p->gather_threads = 64;
    if (const char* s = getenv("BNFFT_GATHER2C_THREADS")) p->gather_threads = std::max(32, std::min(256, atoi(s) / 32 * 32));
    p->gather_smem += gather2c_stash_bytes(p->gather_threads);
  }
  // tuning knob: 128-thread box CTAs (measured equal to 256 on cfg3: the kernel is latency-bound on
  // the node loads and box hand-offs, not on idle threads of sparse bins)
  if (!use_coop3(p) && !use_coop2(p))
    if (const char* s = getenv("BNFFT_GATHERN_THREADS")) p->gather_threads = std::max(32, std::min(256, atoi(s) / 32 * 32));
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->gather_smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, nsm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, p->gather_threads, p->gather_smem);
  if (e != cudaSuccess) return e;
  p->gather_grid1 = (int64_t)std::max(1, per_sm) * nsm;

  // tensor map (innermost first): [re/im (c128)], z, y, (x), (batch)
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fp) return e != cudaSuccess ? e : cudaErrorNotSupported;
  cuuint64_t gdim[5], gstr[4];
  cuuint32_t box[5], estr[5];
  int r = 0;
  cuuint64_t stride = 8;
  if (p->c128) {
    gdim[r] = 2;
    box[r] = 2;
    ++r;
    stride = 16;
  }
  for (int t = d - 1; t >= 0; --t) {
    gdim[r] = (cuuint64_t)p->L;
    box[r] = (cuuint32_t)ext[t];
    ++r;
  }
  if (p->opts.batch > 1) {
    gdim[r] = (cuuint64_t)p->opts.batch;
    box[r] = (cuuint32_t)bt;
    ++r;
  }
  // byte strides of dims 1..r-1
  {
    int k = 0;
    cuuint64_t s = 8;                 // element = one double
    if (p->c128) { gstr[k++] = 16; s = 16; }
    (void)stride;
    cuuint64_t acc = s;
    for (int t = 0; t < d - 1; ++t) { acc *= (cuuint64_t)p->L; gstr[k++] = acc; }
    if (p->opts.batch > 1) gstr[k++] = (cuuint64_t)p->Ld * p->csize;
  }
  for (int i = 0; i < r; ++i) estr[i] = 1;
  CUresult cr = ((EncodeTiledFn)fp)(&p->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)r, p->d_grid, gdim, gstr,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  // y-sweep plans: the decoded item table (gather3y_item_table) follows the tensor map in the same
  // allocation (the kernel reads it at tmap + 1)
  std::vector<uint32_t> items;
  if (use_ysweep3(p)) gather3y_item_table((p->L + 7) >> 3, p->nb_dim[1], p->nb_dim[2], items);
  if (!p->d_tmap) {
    e = cudaMalloc((void**)&p->d_tmap, sizeof(CUtensorMap) + items.size() * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
  }
  e = cudaMemcpyAsync(p->d_tmap, &p->tmap, sizeof(CUtensorMap), cudaMemcpyHostToDevice, p->stream);
  if (e != cudaSuccess) return e;
  if (!items.empty()) {
    e = cudaMemcpyAsync(p->d_tmap + 1, items.data(), items.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                        p->stream);
    if (e != cudaSuccess) return e;
  }
  return cudaStreamSynchronize(p->stream);
}
constexpr int kMaxSegPerRound = 32;

cudaError_t gather_prepare(bnfft_plan_s* p) {
  const void* fn = select_kernel(p->opts.d, p->opts.m, p->c128, p->tap_poly, p->opts.batch > 1,
                                 (p->opts.flags & BNFFT_PRECOMPUTE_PSI) != 0, p->d1_binned);
  if (use_coop3(p)) fn = coop3_kernel(p);
  if (use_coop2(p)) fn = gather2c_kernel_ptr(p->opts.m, p->tap_poly);
  if (!fn) return cudaErrorInvalidValue;
  if (p->d1_binned) {
    // one window per bin (bin + halo, 16-byte aligned), double-buffered; persistent grid by occupancy
    int cap = (1 << p->bin_log2[0]) + 2 * p->opts.m + 2;
    cap += cap & 1;
    p->gather_box_cap = cap;
    p->gather_smem = (size_t)kGather1bBufs * cap * p->csize;
    p->gather_bt = 1;
    p->gather_smax = 1;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->gather_smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0, nsm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGather1bThreads, p->gather_smem);
    if (e != cudaSuccess) return e;
    if (const char* s = getenv("BNFFT_GATHER1_CTAS_PER_SM")) {   // tuning knob
      const int v = atoi(s);
      if (v >= 1 && v < per_sm) per_sm = v;
    }
    p->gather_grid1 = (int64_t)std::max(1, per_sm) * nsm;
    return cudaSuccess;
  }
  if (p->opts.d == 1 && p->opts.batch == 1) {
    // two contiguous windows (double buffer) of 12 KB each; persistent grid sized by occupancy
    // window: chunk cells (~256*NPT at density 1) + one bin + halo, capped at 40 KB per buffer
    p->gather_box_cap = (int)(std::min<size_t>(40u << 10, std::max<size_t>(12u << 10,
                        ((size_t)2048 + ((size_t)1 << p->bin_log2[0])) * p->csize)) / p->csize);
    p->gather_smem = 2 * (size_t)p->gather_box_cap * p->csize;
    p->gather_bt = 1;
    p->gather_smax = 1;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->gather_smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0, nsm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGatherThreads, p->gather_smem);
    if (e != cudaSuccess) return e;
    if (const char* s = getenv("BNFFT_GATHER1_CTAS_PER_SM")) {   // tuning knob
      const int v = atoi(s);
      if (v >= 1 && v < per_sm) per_sm = v;
    }
    p->gather_grid1 = (int64_t)std::max(1, per_sm) * nsm;
    return cudaSuccess;
  }
  if (p->opts.d >= 2) return gatherN_prepare(p, fn);
  size_t per = gather_box_elems(p) * p->csize;
  int bt = (int)std::max<size_t>(1, std::min<size_t>((size_t)p->opts.batch, smem_budget() / per));
  p->gather_bt = bt;
  int smax = (int)std::max<size_t>(1, std::min<size_t>(kMaxSegPerRound, smem_budget() / (per * bt)));
  p->gather_smax = smax;
  p->gather_smem = per * bt * smax;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(p->gather_smem, 1));
  if (e != cudaSuccess) return e;
  return cudaSuccess;
}

template <typename R>
static cudaError_t launch_gather_t(bnfft_plan_s* p, void* out, const void* fn, bool prepsi = false) {
  static_assert(sizeof(GatherParams<R>) < 32000, "kernel parameter limit");
  GatherParams<R> gp;
  memset(&gp, 0, sizeof(gp));
  gp.xs = p->rec3 ? (const double*)p->d_rec_user : p->d_xs;   // rec3: user-order 16-B records
  gp.perm = p->d_perm;
  gp.grid = p->d_grid;
  gp.out = out;
  gp.n = p->n;
  gp.L = p->L;
  gp.Ld = p->Ld;
  gp.Lf = (double)p->L;
  gp.batch = p->opts.batch;
  gp.bt = p->gather_bt;
  gp.smax = p->gather_smax;
  for (int t = 0; t < 3; ++t) {
    gp.log2W[t] = p->bin_log2[t];
    gp.nb[t] = p->nb_dim[t];
    gp.box[t] = t < p->opts.d ? (1 << p->bin_log2[t]) + 2 * p->opts.m - 1 : 1;
  }
  gp.box_elems = (int)gather_box_elems(p);
  gp.edge_sqrt = p->opts.window == BNFFT_SINH ? 1 : 0;
  gp.inv_m = (R)(1.0 / p->opts.m);
  gp.wp = p->wp;
  gp.boxcap = p->gather_box_cap;
  gp.xs_user = p->xs_user ? 1 : 0;
  gp.pre_w = (R*)p->d_pre_w;
  gp.sorted_out = (p->opts.flags & BNFFT_SORTED_OUTPUT) ? 1 : 0;
  gp.l2_hint = 3;   // y-sweep kernel: streaming outputs must not evict the grid boxes' halos from L2
  if (const char* s = getenv("BNFFT_L2_HINT")) gp.l2_hint = atoi(s);   // tuning knob (A/B)
  constexpr int NC = PolyN<R>::NC;
  constexpr int NH = PolyH<R>::NH;
  static_assert(2 * NH == NC, "even/odd split of the tap polynomials");
  if (p->tap_poly) {
    for (int i = 0; i < p->opts.m; ++i)      // taps i < m; the others by mirror symmetry
      for (int k = 0; k < NH; ++k) {
        gp.ceo[k][i][0] = (R)p->tap_coef[(size_t)i * NC + 2 * k];
        gp.ceo[k][i][1] = (R)p->tap_coef[(size_t)i * NC + 2 * k + 1];
      }
  }
  void* args[] = {&gp};
  if (prepsi) {   // grid-stride elementwise kernel, no shared memory
    unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((p->n + kGatherThreads - 1) / kGatherThreads, (int64_t)sm_count() * 16));
    cudaError_t e3 = cudaLaunchKernel(fn, dim3(nb), dim3(kGatherThreads), args, 0, p->stream);
    p->launches++;
    return e3;
  }
  gp.key_start = p->d_bin_start;
  gp.nkeys = p->nkeys;
  gp.nslice = p->gather_nslice;
  gp.bufstride = p->gather_bufstride;
  gp.nbuf = p->gather_nbuf;
  for (int t = 0; t < 3; ++t) gp.tbox[t] = p->gather_tbox[t];
  if (p->opts.d >= 2) {
    gp.box_elems = p->gather_box_elems;
    {
      int mb = 0;
      int64_t mx = std::max(p->nb_dim[0], std::max(p->nb_dim[1], p->nb_dim[2]));
      while (((int64_t)1 << mb) < mx) ++mb;
      gp.morton_bits = mb;
      gp.nkeys_morton = (p->nkeys / p->nbins) << (3 * mb);
      if (use_ysweep3(p)) {   // items of 8 x-lines; Morton order with per-dimension bit counts
        int bsum = 0;
        for (int64_t dim : {(p->L + 7) >> 3, p->nb_dim[1], p->nb_dim[2]}) {
          int b = 0;
          while (((int64_t)1 << b) < dim) ++b;
          bsum += b;
        }
        gp.nkeys_morton = (int64_t)1 << bsum;
      }
    }
    void* args2[] = {&gp, &p->d_tmap};
    unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(p->gather_grid1, p->nkeys));
    cudaError_t e2 = cudaLaunchKernel(fn, dim3(nb), dim3(p->gather_threads), args2, p->gather_smem, p->stream);
    p->launches++;
    return e2;
  }
  unsigned blocks;
  if (p->d1_binned) {
    blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(p->nkeys, p->gather_grid1));
    cudaError_t eb = cudaLaunchKernel(fn, dim3(blocks), dim3(kGather1bThreads), args, p->gather_smem, p->stream);
    p->launches++;
    return eb;
  }
  if (p->opts.d == 1 && p->opts.batch == 1) {
    const int64_t ch = (int64_t)kGatherThreads * NPT1<R>::v;
    blocks = (unsigned)std::min<int64_t>((p->n + ch - 1) / ch, p->gather_grid1);
  } else {
    blocks = (unsigned)((p->n + kGatherThreads - 1) / kGatherThreads);
  }
  cudaError_t e = cudaLaunchKernel(fn, dim3(blocks), dim3(kGatherThreads), args, p->gather_smem,
                                   p->stream);
  p->launches++;
  return e;
}

cudaError_t launch_gather(bnfft_plan_s* p, void* out) {
  if (p->n == 0) return cudaSuccess;
  const void* fn = select_kernel(p->opts.d, p->opts.m, p->c128, p->tap_poly, p->opts.batch > 1,
                                 (p->opts.flags & BNFFT_PRECOMPUTE_PSI) != 0, p->d1_binned);
  // d = 3, m = 4, complex64: the kernel chosen at plan creation (its launch shape is in the plan)
  if (use_coop3(p)) fn = coop3_kernel(p);
  if (use_coop2(p)) fn = gather2c_kernel_ptr(p->opts.m, p->tap_poly);
  if (!fn) return cudaErrorInvalidValue;
  return p->c128 ? launch_gather_t<double>(p, out, fn) : launch_gather_t<float>(p, out, fn);
}

// Algorithm 2 step 0(b): per-node tap weights for BNFFT_PRECOMPUTE_PSI (d = 1)
cudaError_t launch_prepsi(bnfft_plan_s* p) {
  if (p->n == 0) return cudaSuccess;
  const void* fn = p->c128 ? gather_kernel_1d(p->opts.m + 200, p->tap_poly) : gather_kernel_1f(p->opts.m + 200, p->tap_poly);
  if (!fn) return cudaErrorInvalidValue;
  return p->c128 ? launch_gather_t<double>(p, nullptr, fn, true) : launch_gather_t<float>(p, nullptr, fn, true);
}

int tap_coef_count(bool c128) { return c128 ? PolyN<double>::NC : PolyN<float>::NC; }

}  // namespace bnfft
