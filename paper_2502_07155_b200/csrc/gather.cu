// Row a6 gather: host-side dispatch and launch (kernels in gather_impl.cuh).
#include <cstring>

#include "gather_impl.cuh"

namespace bnfft {

static const void* select_kernel(int d, int m, bool c128, bool poly, bool batched = false) {
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
constexpr int kMaxSegPerRound = 32;

cudaError_t gather_prepare(bnfft_plan_s* p) {
  const void* fn = select_kernel(p->opts.d, p->opts.m, p->c128, p->tap_poly, p->opts.batch > 1);
  if (!fn) return cudaErrorInvalidValue;
  if (p->opts.d == 1 && p->opts.batch == 1) {
    // two contiguous windows (double buffer) of 12 KB each; persistent grid sized by occupancy
    p->gather_box_cap = (int)((12u << 10) / p->csize);
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
    p->gather_grid1 = (int64_t)std::max(1, per_sm) * nsm;
    return cudaSuccess;
  }
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
static cudaError_t launch_gather_t(bnfft_plan_s* p, void* out, const void* fn) {
  static_assert(sizeof(GatherParams<R>) < 32000, "kernel parameter limit");
  GatherParams<R> gp;
  memset(&gp, 0, sizeof(gp));
  gp.xs = p->d_xs;
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
  unsigned blocks;
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
  const void* fn = select_kernel(p->opts.d, p->opts.m, p->c128, p->tap_poly, p->opts.batch > 1);
  if (!fn) return cudaErrorInvalidValue;
  return p->c128 ? launch_gather_t<double>(p, out, fn) : launch_gather_t<float>(p, out, fn);
}

int tap_coef_count(bool c128) { return c128 ? PolyN<double>::NC : PolyN<float>::NC; }

}  // namespace bnfft
