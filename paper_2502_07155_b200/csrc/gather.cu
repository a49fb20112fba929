// Row a6 gather: host-side dispatch and launch (kernels in gather_impl.cuh).
#include "gather_impl.cuh"

namespace bnfft {

static const void* select_kernel(int d, int m, bool c128) {
  if (d == 1) return c128 ? gather_kernel_1d(m) : gather_kernel_1f(m);
  if (d == 2) return c128 ? gather_kernel_2d(m) : gather_kernel_2f(m);
  if (d == 3) return c128 ? gather_kernel_3d(m) : gather_kernel_3f(m);
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

cudaError_t gather_prepare(bnfft_plan_s* p) {
  const void* fn = select_kernel(p->opts.d, p->opts.m, p->c128);
  if (!fn) return cudaErrorInvalidValue;
  size_t per = gather_box_elems(p) * p->csize;
  int bt = (int)std::max<size_t>(1, std::min<size_t>((size_t)p->opts.batch, (48u << 10) / per));
  p->gather_bt = bt;
  p->gather_smem = per * bt;
  if (p->gather_smem > (48u << 10)) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)p->gather_smem);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_gather(bnfft_plan_s* p, void* out) {
  if (p->n == 0) return cudaSuccess;
  const void* fn = select_kernel(p->opts.d, p->opts.m, p->c128);
  if (!fn) return cudaErrorInvalidValue;
  GatherParams gp;
  gp.xs = p->d_xs;
  gp.perm = p->d_perm;
  gp.bin_start = p->d_bin_start;
  gp.grid = p->d_grid;
  gp.out = out;
  gp.n = p->n;
  gp.L = p->L;
  gp.Ld = p->Ld;
  gp.Lf = (double)p->L;
  gp.batch = p->opts.batch;
  gp.bt = p->gather_bt;
  for (int t = 0; t < 3; ++t) {
    gp.log2W[t] = p->bin_log2[t];
    gp.nb[t] = p->nb_dim[t];
    gp.box[t] = t < p->opts.d ? (1 << p->bin_log2[t]) + 2 * p->opts.m - 1 : 1;
  }
  gp.box_elems = (int)gather_box_elems(p);
  gp.wp = p->wp;
  void* args[] = {&gp};
  unsigned blocks = (unsigned)((p->n + kGatherThreads - 1) / kGatherThreads);
  cudaError_t e = cudaLaunchKernel(fn, dim3(blocks), dim3(kGatherThreads), args, p->gather_smem,
                                   p->stream);
  p->launches++;
  return e;
}

}  // namespace bnfft
