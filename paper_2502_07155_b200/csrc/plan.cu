// Host orchestration of the C ABI declared in include/bnfft.h: option validation (readings
// A1, A2, A7), device buffers, cuFFT plan, stage sequencing and per-stage CUDA-event timing.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "bnfft_internal.h"

using namespace bnfft;

namespace bnfft {

static thread_local std::string g_err;

void set_error(const std::string& s) { g_err = s; }

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  (void)cudaGetLastError();   // a failed launch must not be reported again by a later check
  if (e == cudaErrorMemoryAllocation) return BNFFT_E_OOM;
  return BNFFT_E_CUDA;
}

static cudaEvent_t get_event(bnfft_plan_s* p) {
  if (!p->pool.empty()) {
    cudaEvent_t e = p->pool.back();
    p->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;   // B200
    cached[dev] = n;
  }
  return cached[dev];
}

void timer_begin(bnfft_plan_s* p, int stage, cudaEvent_t* ev) {
  (void)stage;
  *ev = nullptr;
  if (!(p->opts.flags & BNFFT_TIMING)) return;
  *ev = get_event(p);
  cudaEventRecord(*ev, p->stream);
}

void timer_end(bnfft_plan_s* p, int stage, cudaEvent_t ev) {
  if (!(p->opts.flags & BNFFT_TIMING) || !ev) return;
  cudaEvent_t b = get_event(p);
  cudaEventRecord(b, p->stream);
  p->pending.push_back(Timer{stage, ev, b});
}

// Gauss-Legendre nodes/weights on [-1, 1] by Newton iteration on the three-term recurrence of
// P_n (long double), mapped to theta in [0, pi/2] (reading A4).  Independent of numpy.
static void gauss_legendre_theta(int n, double* theta, double* w) {
  const long double PI = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < n; ++i) {
    long double x = cosl(PI * (i + 0.75L) / (n + 0.5L));
    long double dp = 0;
    for (int it = 0; it < 100; ++it) {
      long double p0 = 1, p1 = x;
      for (int k = 2; k <= n; ++k) {
        long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1);
      long double dx = p1 / dp;
      x -= dx;
      if (fabsl(dx) < 1e-19L) break;
    }
    {
      long double p0 = 1, p1 = x;
      for (int k = 2; k <= n; ++k) {
        long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1);
    }
    long double wi = 2 / ((1 - x * x) * dp * dp);
    theta[i] = (double)((x + 1) * (PI / 4));
    w[i] = (double)(wi * (PI / 4));
  }
}

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

static int ceil_log2(int64_t v) {
  int b = 0;
  while (((int64_t)1 << b) < v) ++b;
  return b;
}

// plan-owned device allocations, counted in bnfft_info.device_bytes while they are live
cudaError_t dmalloc_bytes(bnfft_plan_s* p, void** ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaSuccess) {
    p->device_bytes += (int64_t)bytes;
    p->allocs.emplace_back(*ptr, bytes);
  }
  return e;
}

void dfree_plan(bnfft_plan_s* p, void* ptr) {
  if (!ptr) return;
  for (size_t i = 0; i < p->allocs.size(); ++i)
    if (p->allocs[i].first == ptr) {
      p->device_bytes -= (int64_t)p->allocs[i].second;
      p->allocs[i] = p->allocs.back();
      p->allocs.pop_back();
      break;
    }
  cudaFree(ptr);
}

template <typename T>
static cudaError_t dmalloc(bnfft_plan_s* p, T** ptr, size_t bytes) {
  return dmalloc_bytes(p, (void**)ptr, bytes);
}

static int collect_timing(bnfft_plan_s* p) {
  for (auto& t : p->pending) {
    cudaError_t e = cudaEventSynchronize(t.b);
    if (e != cudaSuccess) return cuda_fail(e, "timing event");
    float ms = 0;
    cudaEventElapsedTime(&ms, t.a, t.b);
    p->ms[t.stage] += ms;
    p->pool.push_back(t.a);
    p->pool.push_back(t.b);
  }
  p->pending.clear();
  return BNFFT_OK;
}

static void free_nodes(bnfft_plan_s* p) {
  dfree_plan(p, p->d_xs);
  dfree_plan(p, p->d_rec_user);
  p->d_rec_user = nullptr;
  dfree_plan(p, p->d_k0);
  dfree_plan(p, p->d_k1);
  dfree_plan(p, p->d_v0);
  dfree_plan(p, p->d_v1);
  p->d_xs = nullptr;
  p->d_k0 = p->d_k1 = p->d_v0 = p->d_v1 = nullptr;
  p->d_perm = p->d_skeys = nullptr;
  p->cap = 0;
}

}  // namespace bnfft

extern "C" {

const char* bnfft_status_string(int s) {
  switch (s) {
    case BNFFT_OK: return "ok";
    case BNFFT_E_BAD_DIM: return "bad dimension";
    case BNFFT_E_BAD_BANDWIDTH: return "bad bandwidth (M must be even and >= 2)";
    case BNFFT_E_BAD_SIGMA: return "bad oversampling factor (sigma >= 1)";
    case BNFFT_E_TRUNCATION_TOO_LARGE: return "truncation parameter out of range (1 <= m, 2m < L)";
    case BNFFT_E_BAD_WINDOW_PARAM: return "bad window or window parameter";
    case BNFFT_E_SPECTRAL_FACTOR_VANISHES: return "psi^ vanishes in band";
    case BNFFT_E_NODE_NOT_FINITE: return "node not finite";
    case BNFFT_E_NODE_OUT_OF_RANGE: return "node outside [-1/2, 1/2)^d";
    case BNFFT_E_NODE_OUTSIDE_FEASIBLE_BOX: return "node outside the feasible box";
    case BNFFT_E_NODES_NOT_SET: return "nodes not set";
    case BNFFT_E_CUDA: return "CUDA error";
    case BNFFT_E_CUFFT: return "cuFFT error";
    case BNFFT_E_OOM: return "out of device memory";
    case BNFFT_E_UNSUPPORTED: return "unsupported parameters";
    case BNFFT_E_INVALID_ARG: return "invalid argument";
    case BNFFT_E_NCCL: return "NCCL / multi-GPU transport error";
    default: return "unknown status";
  }
}

const char* bnfft_last_error(void) { return g_err.c_str(); }

const char* bnfft_build_info(void) {
  return "bnfft 0.1 (arXiv 2502.07155 Algorithm 2), target sm_100a";
}

int bnfft_destroy(bnfft_plan_s* p) {
  if (!p) return BNFFT_OK;
  cudaSetDevice(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  else cudaDeviceSynchronize();
  if (p->pre_stream) {
    cudaStreamSynchronize(p->pre_stream);
    cudaStreamDestroy(p->pre_stream);
  }
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_pre) cudaEventDestroy(p->ev_pre);
  if (p->fft_ok) cufftDestroy(p->fft);
  if (p->fft2_ok) cufftDestroy(p->fft2);
  dist_destroy(p);
  dfree_plan(p, p->d_fft_p);
  dfree_plan(p, p->d_gl);
  dfree_plan(p, p->d_psihat);
  dfree_plan(p, p->d_q);
  dfree_plan(p, p->d_flat);
  dfree_plan(p, p->d_fft_in);
  dfree_plan(p, p->d_grid);
  dfree_plan(p, p->d_bin_start);
  dfree_plan(p, p->d_hist);
  dfree_plan(p, p->d_scan_part);
  dfree_plan(p, p->d_bad);
  dfree_plan(p, p->d_x_stage);
  dfree_plan(p, p->d_fhat_stage);
  dfree_plan(p, p->d_f_stage);
  for (int k = 0; k < 2; ++k) {
    dfree_plan(p, p->d_xp[k]);
    dfree_plan(p, p->d_fhp[k]);
    dfree_plan(p, p->d_fp[k]);
    for (cudaEvent_t ev : {p->ev_h2d[k], p->ev_used[k], p->ev_f[k], p->ev_d2h[k]})
      if (ev) cudaEventDestroy(ev);
  }
  if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
  if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
  if (p->h_bads) cudaFreeHost(p->h_bads);
  dfree_plan(p, p->d_tmap);
  dfree_plan(p, p->d_pre_w);
  free_nodes(p);
  for (auto& a : p->allocs) cudaFree(a.first);   // anything a partially built plan still owns
  if (p->h_bad) cudaFreeHost(p->h_bad);
  for (auto& t : p->pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : p->pool) cudaEventDestroy(e);
  delete p;
  return BNFFT_OK;
}

// Step 0(a) is independent of the nodes: it runs on a plan-owned side stream forked from the plan's
// stream, so a following bnfft_set_nodes overlaps it; execute (the consumer of q) joins it.
int bnfft_precompute(bnfft_plan_s* p) {
  if (!p) return BNFFT_E_INVALID_ARG;
  cudaSetDevice(p->device);
  cudaError_t e = cudaEventRecord(p->ev_fork, p->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->pre_stream, p->ev_fork, 0);
  if (e != cudaSuccess) return cuda_fail(e, "precompute fork");
  cudaStream_t main_stream = p->stream;
  p->stream = p->pre_stream;   // launch_psihat and the stage timer use p->stream
  cudaEvent_t ev;
  timer_begin(p, ST_PSIHAT, &ev);
  e = launch_psihat(p);
  if (e == cudaSuccess) timer_end(p, ST_PSIHAT, ev);
  p->stream = main_stream;
  if (e != cudaSuccess) return cuda_fail(e, "psihat kernel");
  if ((e = cudaEventRecord(p->ev_pre, p->pre_stream)) != cudaSuccess) return cuda_fail(e, "precompute join");
  p->pre_pending = true;
  p->n_psihat++;
  return BNFFT_OK;
}

// make the plan's stream wait for the last precompute (before anything reads psi^ / q)
static cudaError_t join_precompute(bnfft_plan_s* p) {
  if (!p->pre_pending) return cudaSuccess;
  p->pre_pending = false;
  return cudaStreamWaitEvent(p->stream, p->ev_pre, 0);
}

int bnfft_plan_create(const bnfft_opts* o, bnfft_plan_s** out) {
  if (!out) return BNFFT_E_INVALID_ARG;
  *out = nullptr;
  if (!o) return BNFFT_E_INVALID_ARG;
  if (o->d < 1 || o->d > 3) { set_error("d must be 1..3"); return BNFFT_E_BAD_DIM; }
  if (o->M < 2 || (o->M & 1)) { set_error("M must be even and >= 2 (P:50)"); return BNFFT_E_BAD_BANDWIDTH; }
  if (!std::isfinite(o->sigma) || o->sigma < 1.0) { set_error("sigma >= 1 (P:86)"); return BNFFT_E_BAD_SIGMA; }
  // L = M_sigma = 2 ceil(ceil(sigma M)/2) (reading A7)
  double sm = std::ceil(o->sigma * (double)o->M);
  int64_t L = 2 * (int64_t)std::ceil(sm / 2.0);
  if (o->m < 1 || 2 * (int64_t)o->m >= L) { set_error("need 1 <= m and 2m < L"); return BNFFT_E_TRUNCATION_TOO_LARGE; }
  if (o->window != BNFFT_SINH && o->window != BNFFT_GAUSS && o->window != BNFFT_CKB) {
    set_error("unknown window");
    return BNFFT_E_BAD_WINDOW_PARAM;
  }
  if (o->prec != BNFFT_C64 && o->prec != BNFFT_C128) { set_error("prec"); return BNFFT_E_INVALID_ARG; }
  if (o->batch < 1) { set_error("batch >= 1"); return BNFFT_E_INVALID_ARG; }
  if (o->nranks > 1 && (o->rank < 0 || o->rank >= o->nranks)) { set_error("rank in [0, nranks)"); return BNFFT_E_INVALID_ARG; }
  const bool slab = o->nranks > 1 && o->dist == BNFFT_DIST_SLAB;
  if (!gather_supported(o->d, o->m)) { set_error("m outside the compiled range for this d"); return BNFFT_E_UNSUPPORTED; }
  const bool alg1 = (o->flags & BNFFT_ALG1) != 0;
  if ((o->flags & BNFFT_PRECOMPUTE_PSI) && (o->d != 1 || o->batch != 1)) {
    set_error("BNFFT_PRECOMPUTE_PSI is compiled for d = 1, batch 1");
    return BNFFT_E_UNSUPPORTED;
  }
  if (alg1 && (o->d != 1 || o->window == BNFFT_GAUSS || o->batch != 1)) {
    set_error("BNFFT_ALG1 is compiled for d = 1, batch 1, sinh/cKB windows");
    return BNFFT_E_UNSUPPORTED;
  }
  double shape = o->shape;
  if (!(shape > 0) && alg1) shape = 2.0 * M_PI * o->m * (1.0 - (double)o->M / (2.0 * (double)L));   // A17
  if (!(shape > 0)) {
    if (o->window == BNFFT_GAUSS) {
      if (L == o->M) { set_error("Gaussian default s needs L > M (reading A2)"); return BNFFT_E_BAD_WINDOW_PARAM; }
      shape = std::sqrt((double)o->m / (M_PI * (double)L * (double)(L - o->M)));  // A2
    } else {
      shape = M_PI * o->m * (1.0 - (double)o->M / (double)L);                        // A1
    }
  }
  if (!(shape > 0) || !std::isfinite(shape)) { set_error("window shape must be > 0"); return BNFFT_E_BAD_WINDOW_PARAM; }
  int64_t Ld = ipow(L, o->d), Md = ipow(o->M, o->d);
  if (Ld > ((int64_t)1 << 34)) { set_error("grid too large"); return BNFFT_E_UNSUPPORTED; }

  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0) {
    set_error(std::string("no CUDA device: ") + cudaGetErrorString(ce));
    return BNFFT_E_CUDA;
  }
  ce = cudaSetDevice(o->device);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaSetDevice");

  bnfft_plan_s* p = new bnfft_plan_s();
  p->opts = *o;
  p->device = o->device;
  p->stream = (cudaStream_t)o->stream;
  p->L = L;
  p->Ld = Ld;
  p->Md = Md;
  p->shape = shape;
  p->c128 = o->prec == BNFFT_C128;
  p->csize = p->c128 ? 16 : 8;

  WinParams& w = p->wp;
  w.window = o->window;
  w.alg1 = alg1 ? 1 : 0;
  w.m = o->m;
  w.inv_m = 1.0 / o->m;
  w.inv_m_f = (float)w.inv_m;
  w.beta = shape;
  w.beta_f = (float)shape;
  if (o->window == BNFFT_SINH) w.inv_norm = 1.0 / std::sinh(shape);
  else if (o->window == BNFFT_CKB) w.inv_norm = 1.0 / (std::cyl_bessel_i(0.0, shape) - 1.0);
  else w.inv_norm = 1.0;
  w.inv_norm_f = (float)w.inv_norm;
  w.gauss_b = (o->window == BNFFT_GAUSS) ? 1.0 / (2.0 * shape * shape * (double)L * (double)L) : 0.0;
  w.gauss_b_f = (float)w.gauss_b;
  if (!std::isfinite(w.inv_norm) || w.inv_norm <= 0) {
    delete p;
    set_error("window normalisation overflow (shape too large)");
    return BNFFT_E_BAD_WINDOW_PARAM;
  }

  // node binning geometry (row a1)
  int lg = 7;
  if (const char* ev = getenv("BNFFT_D1_BIN_LOG2")) lg = atoi(ev);   // tuning knob (d = 1)
  if (o->d == 2) lg = 4;
  if (o->d == 3) lg = o->batch > 1 ? 2 : 3;
  int lgL = 0;
  while (((int64_t)1 << (lgL + 1)) <= L) ++lgL;
  // d = 1, batch 1, large grids: bins wide enough that the key (bin index) fits one radix digit, when
  // a bin's window (bin + halo) fits three per CTA (<= 72 KB each); the gather then walks whole bins
  // (gather1b).  Otherwise 128-cell bins and the chunked window kernel.
  p->d1_binned = false;
  if (o->d == 1 && o->batch == 1 && !(o->flags & BNFFT_PRECOMPUTE_PSI) && lgL - lg > kMaxDigitBits &&
      !getenv("BNFFT_D1_CHUNKED")) {
    int lgc = 0;   // ceil(log2 L): at most 2^kMaxDigitBits bins even for L not a power of two
    while (((int64_t)1 << lgc) < L) ++lgc;
    const int lgb = lgc - kMaxDigitBits;
    const size_t win = (((size_t)1 << lgb) + 2 * (size_t)o->m + 2) * (size_t)p->csize;
    if (win <= ((size_t)(getenv("BNFFT_D1_WINMAX_KB") ? atoi(getenv("BNFFT_D1_WINMAX_KB")) : 72) << 10)) {   // 3 windows per CTA fit 227 KB
      lg = lgb;
      p->d1_binned = true;
    }
  }
  lg = std::min(lg, lgL);
  int64_t nbins = 1;
  // d = 3, m = 4, complex64, batch 1: the y-sweep gather (gather3y) sorts by x-line, bins of
  // 1 x 16 x 8 cells; the half-warp / z-sweep kernels (gather3c / gather3s, selectable) use bins of
  // 8 x 8 x 16 cells (innermost box extent 16 + 2m = 24: conflict-free shared-memory rows).
  const bool coop3 = o->d == 3 && o->m == 4 && o->prec == BNFFT_C64 && o->batch == 1 && lgL >= 4;
  p->g3_kind = getenv("BNFFT_GATHER3S") ? 2 : getenv("BNFFT_GATHER3C") ? 1 : getenv("BNFFT_GATHER3Q") ? 3 : 0;
  if ((p->g3_kind == 0 || p->g3_kind == 3) && L > 8192) p->g3_kind = 1;   // y-sweep item table: 10-bit item coordinates
  p->rec3 = coop3 && (p->g3_kind == 0 || p->g3_kind == 3);
  p->g2_coop = o->d == 2 && o->prec == BNFFT_C64 && o->batch == 1 && o->m <= 7 && !getenv("BNFFT_GATHER2N");
  for (int t = 0; t < 3; ++t) {
    int lt = lg;
    if (coop3) lt = p->rec3 ? (t == 0 ? 0 : t == 1 ? 4 : 3) : (t == 2 ? 4 : 3);
    p->bin_log2[t] = t < o->d ? lt : 0;
    p->nb_dim[t] = t < o->d ? (L + (1 << lt) - 1) >> lt : 1;
    nbins *= p->nb_dim[t];
  }
  p->nbins = nbins;
  p->col_bits = p->rec3 ? (p->g3_kind == 3 ? 5 : 4) : 0;
  p->key_bits = ceil_log2(nbins) + p->col_bits;
  p->sort_passes = (p->key_bits + kMaxDigitBits - 1) / kMaxDigitBits;
  p->digit_bits = p->sort_passes ? (p->key_bits + p->sort_passes - 1) / p->sort_passes : 0;
  // Sort key (user block, bin), row a1: for d <= 2 (grid resident in L2) nodes are binned inside
  // user blocks whose outputs (batch x csize each) span ~16 MiB, so the gather's writes to
  // f[perm[i]] stay within an L2-resident window; d = 3 uses one block (grid reuse dominates).
  {
    int64_t gbytes_one = Ld * (int64_t)o->batch * (int64_t)p->csize;
    if (o->d <= 2 && gbytes_one <= ((int64_t)48 << 20)) {
      int64_t per = (int64_t)o->batch * (int64_t)p->csize;
      int ub = kSortTileLog2;
      const int64_t target = (int64_t)16 << 20;   // measured best for cfg2 (both d = 1 kernels)
      while (ub < 31 && (((int64_t)1 << (ub + 1)) * per) <= target) ++ub;
      if (const char* s = getenv("BNFFT_UB_LOG2")) ub = atoi(s);
      ub = std::max(ub, kSortTileLog2);   // user blocks are whole sort tiles
      p->ub_log2 = std::min(ub, 31);
    } else {
      p->ub_log2 = 31;
    }
    // d = 1 one-pass plans: the single radix pass also writes the sorted node copy (radix1x)
    p->xs_user = p->ub_log2 < 31 && !p->d1_binned;
    if (getenv("BNFFT_XS_SORTED")) p->xs_user = false;
  }

  int rc = BNFFT_OK;
  cudaError_t e;
#define CK(call, what)                       \
  do {                                       \
    e = (call);                              \
    if (e != cudaSuccess) {                  \
      rc = cuda_fail(e, what);               \
      goto fail;                             \
    }                                        \
  } while (0)
  {
    CK(dmalloc(p, &p->d_gl, 2 * kQuadN * sizeof(double)), "alloc gl");
    CK(dmalloc(p, &p->d_psihat, o->M * sizeof(double)), "alloc psihat");
    CK(dmalloc(p, &p->d_q, o->M * sizeof(double)), "alloc q");
    CK(dmalloc(p, &p->d_flat, 2 * sizeof(double)), "alloc flat");
    size_t gbytes = (size_t)Ld * o->batch * p->csize;
    // BNFFT_DIST_SLAB: the grid is indexed globally but only the rank's slab and halos are written;
    // step 2 runs on the slab buffers of dist.cu (no whole-grid FFT input or plan)
    if (!slab) CK(dmalloc(p, &p->d_fft_in, gbytes), "alloc fft input");
    CK(dmalloc(p, &p->d_grid, gbytes), "alloc grid");
    CK(dmalloc(p, &p->d_bad, sizeof(unsigned long long)), "alloc status");
    CK(cudaMallocHost((void**)&p->h_bad, sizeof(unsigned long long)), "alloc pinned status");
    if (!slab) CK(cudaMemsetAsync(p->d_fft_in, 0, gbytes, p->stream), "zero fft input");
    p->pfft3 = !slab && o->d == 3 && o->batch == 1 && 2 * o->M <= L && !getenv("BNFFT_NO_PFFT");
    if (p->pfft3) {
      const size_t pb = (size_t)o->M * L * L * p->csize;
      CK(dmalloc(p, &p->d_fft_p, pb), "alloc pruned fft planes");
      CK(cudaMemsetAsync(p->d_fft_p, 0, pb, p->stream), "zero pruned fft planes");
    }
    CK(cudaMemsetAsync(p->d_grid, 0, gbytes, p->stream), "zero grid");
    double th[2 * kQuadN];
    gauss_legendre_theta(kQuadN, th, th + kQuadN);
    CK(cudaMemcpyAsync(p->d_gl, th, sizeof(th), cudaMemcpyHostToDevice, p->stream), "copy gl");
    {
      // tap polynomials of the gather (row a6): fit + accuracy check on the device
      const int T = 2 * o->m;
      const int NC = tap_coef_count(p->c128);
      double *d_coef = nullptr, *d_err = nullptr;
      CK(cudaMalloc((void**)&d_coef, (size_t)T * NC * sizeof(double)), "alloc tap coef");
      e = cudaMalloc((void**)&d_err, (size_t)T * sizeof(double));
      if (e == cudaSuccess) e = launch_tapfit(p, NC, d_coef, d_err);
      p->tap_coef.assign((size_t)T * NC, 0.0);
      std::vector<double> err(T, 0.0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(p->tap_coef.data(), d_coef, (size_t)T * NC * sizeof(double),
                            cudaMemcpyDeviceToHost, p->stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(err.data(), d_err, (size_t)T * sizeof(double), cudaMemcpyDeviceToHost,
                            p->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
      cudaFree(d_coef);
      if (d_err) cudaFree(d_err);
      if (e != cudaSuccess) { rc = cuda_fail(e, "tap fit"); goto fail; }
      double mx = 0;
      for (double v : err) mx = std::max(mx, v);
      p->tap_fit_err = mx;
      p->tap_nc = NC;
      p->tap_poly = std::isfinite(mx) && mx <= (p->c128 ? 1e-13 : 2e-6) &&
                    !(o->flags & BNFFT_EXACT_TAPS);
    }
    CK(gather_prepare(p), "gather kernel attributes");
    CK(sort_prepare(), "sort kernel attributes");

    int n[3] = {(int)L, (int)L, (int)L};
    size_t ws = 0;
    cufftResult fr = CUFFT_SUCCESS;
    if (!slab && !p->pfft3) {
      fr = cufftCreate(&p->fft);
      if (fr == CUFFT_SUCCESS) {
        p->fft_ok = true;
        fr = cufftMakePlanMany(p->fft, o->d, n, nullptr, 1, (int)Ld, nullptr, 1, (int)Ld,
                               p->c128 ? CUFFT_Z2Z : CUFFT_C2C, o->batch, &ws);
      }
      if (fr == CUFFT_SUCCESS) fr = cufftSetStream(p->fft, p->stream);
    } else if (p->pfft3) {
      // step 2 pruned (d = 3): 2-D FFTs over (k_2, k_3) on M/2 compact planes per call, then 1-D FFTs
      // along k_1 with stride L^2 over all L^2 lines
      const cufftType ty = p->c128 ? CUFFT_Z2Z : CUFFT_C2C;
      fr = cufftCreate(&p->fft2);
      if (fr == CUFFT_SUCCESS) {
        p->fft2_ok = true;
        int n2[2] = {(int)L, (int)L};
        fr = cufftMakePlanMany(p->fft2, 2, n2, nullptr, 1, (int)(L * L), nullptr, 1, (int)(L * L), ty,
                               (int)(o->M / 2), &ws);
        p->device_bytes += (int64_t)ws;
      }
      if (fr == CUFFT_SUCCESS) fr = cufftSetStream(p->fft2, p->stream);
      if (fr == CUFFT_SUCCESS) fr = cufftCreate(&p->fft);
      if (fr == CUFFT_SUCCESS) {
        p->fft_ok = true;
        int n1[1] = {(int)L};
        int nem[1] = {(int)L};
        fr = cufftMakePlanMany(p->fft, 1, n1, nem, (int)(L * L), 1, nem, (int)(L * L), 1, ty, (int)(L * L), &ws);
      }
      if (fr == CUFFT_SUCCESS) fr = cufftSetStream(p->fft, p->stream);
    }
    if (fr != CUFFT_SUCCESS) {
      char buf[96];
      snprintf(buf, sizeof(buf), "cuFFT plan failed (%d)", (int)fr);
      set_error(buf);
      rc = BNFFT_E_CUFFT;
      goto fail;
    }
    p->device_bytes += (int64_t)ws;

    CK(cudaStreamCreateWithFlags(&p->pre_stream, cudaStreamNonBlocking), "side stream");
    CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming), "fork event");
    CK(cudaEventCreateWithFlags(&p->ev_pre, cudaEventDisableTiming), "join event");
    rc = bnfft_precompute(p);
    if (rc != BNFFT_OK) goto fail;
    CK(join_precompute(p), "precompute join");
    double fl[2];
    CK(cudaMemcpyAsync(fl, p->d_flat, sizeof(fl), cudaMemcpyDeviceToHost, p->stream), "copy flat");
    CK(cudaStreamSynchronize(p->stream), "plan sync");
    p->flatness = fl[0];
    if (!(fl[1] >= 1e-12)) {
      set_error("|psi^_1(k)| < 1e-12 |psi^_1(0)| for some k in I_M (P:429)");
      rc = BNFFT_E_SPECTRAL_FACTOR_VANISHES;
      goto fail;
    }
    rc = dist_create(p);   // multi-GPU transport and slab buffers (nranks > 1)
    if (rc != BNFFT_OK) goto fail;
    CK(cudaStreamSynchronize(p->stream), "plan sync");
  }
#undef CK
  *out = p;
  return BNFFT_OK;
fail:
  bnfft_destroy(p);
  return rc;
}

int bnfft_set_nodes(bnfft_plan_s* p, int64_t n, const double* x, int64_t* first_bad) {
  if (first_bad) *first_bad = -1;
  if (!p) return BNFFT_E_INVALID_ARG;
  if (n < 0 || n >= ((int64_t)1 << 31) || (n > 0 && !x)) {
    set_error("n must be in [0, 2^31) and x non-NULL");
    return BNFFT_E_INVALID_ARG;
  }
  cudaSetDevice(p->device);
  if (p->dist) return dist_set_nodes(p, n, x, first_bad);
  return local_set_nodes(p, n, x, first_bad);
}

}  // extern "C"

// the one-rank body of bnfft_set_nodes (also the owner-side step of BNFFT_DIST_SLAB)
int bnfft::local_set_nodes(bnfft_plan_s* p, int64_t n, const double* x, int64_t* first_bad,
                           unsigned long long* h_bad_dst) {
  if (first_bad) *first_bad = -1;
  p->nodes_set = false;
  cudaError_t e;
  if (n > p->cap) {
    free_nodes(p);
    int64_t cap = std::max<int64_t>(n, 1);
    size_t b4 = (cap + 4) * sizeof(uint32_t);   // +4: 16-byte bulk copies of permutation ranges
    if ((p->rec3 && (e = dmalloc(p, &p->d_rec_user, cap * 16)) != cudaSuccess) ||
        (e = dmalloc(p, &p->d_xs, cap * std::max<size_t>(p->opts.d * sizeof(double), p->rec3 ? 16 : 0))) != cudaSuccess ||
        (e = dmalloc(p, &p->d_k0, b4)) != cudaSuccess || (e = dmalloc(p, &p->d_k1, b4)) != cudaSuccess ||
        (e = dmalloc(p, &p->d_v0, b4)) != cudaSuccess || (e = dmalloc(p, &p->d_v1, b4)) != cudaSuccess)
      return cuda_fail(e, "alloc nodes");
    p->cap = cap;
  }
  int64_t ntiles = (std::max<int64_t>(n, 1) + kSortTile - 1) / kSortTile;
  int64_t nh = ((int64_t)1 << std::max(p->digit_bits, 1)) * ntiles;
  if (nh > p->hist_cap) {
    dfree_plan(p, p->d_hist);
    p->d_hist = nullptr;
    if ((e = dmalloc(p, &p->d_hist, nh * sizeof(uint32_t))) != cudaSuccess) return cuda_fail(e, "alloc hist");
    p->hist_cap = nh;
  }
  int64_t np = (nh + 4095) / 4096 + 1;
  if (np > p->part_cap) {
    dfree_plan(p, p->d_scan_part);
    p->d_scan_part = nullptr;
    if ((e = dmalloc(p, &p->d_scan_part, np * sizeof(uint32_t))) != cudaSuccess) return cuda_fail(e, "alloc scan");
    p->part_cap = np;
  }

  {
    int64_t nblk = n > 0 ? ((n - 1) >> p->ub_log2) + 1 : 1;
    p->nkeys = nblk * p->nbins;
    if (p->nkeys + 1 > p->key_start_cap) {
      dfree_plan(p, p->d_bin_start);
      p->d_bin_start = nullptr;
      if ((e = dmalloc(p, &p->d_bin_start, (p->nkeys + 1) * sizeof(uint32_t))) != cudaSuccess)
        return cuda_fail(e, "alloc key offsets");
      p->key_start_cap = p->nkeys + 1;
    }
  }
  cudaEvent_t ev;
  timer_begin(p, ST_KEYS, &ev);
  if ((e = launch_keys(p, x, n)) != cudaSuccess) return cuda_fail(e, "keys kernel");
  timer_end(p, ST_KEYS, ev);
  if ((e = cudaMemcpyAsync(h_bad_dst ? h_bad_dst : p->h_bad, p->d_bad, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, p->stream)) != cudaSuccess)
    return cuda_fail(e, "status copy");
  timer_begin(p, ST_SORT, &ev);
  if ((e = launch_sort(p, x, n)) != cudaSuccess) return cuda_fail(e, "sort kernels");
  timer_end(p, ST_SORT, ev);
  if (p->opts.flags & BNFFT_PRECOMPUTE_PSI) {   // Algorithm 2 step 0(b)
    const size_t wb = (size_t)std::max<int64_t>(n, 1) * ((2 * p->opts.m + 3) / 4 * 4) * (p->csize / 2);   // rows padded to 16 B
    if (n > p->pre_cap) {
      dfree_plan(p, p->d_pre_w);
      p->d_pre_w = nullptr;
      if ((e = dmalloc(p, &p->d_pre_w, wb)) != cudaSuccess) return cuda_fail(e, "alloc psi table");
      p->pre_cap = std::max<int64_t>(n, 1);
    }
    const int64_t n_prev = p->n;
    p->n = n;   // the precompute kernel iterates over the new node set
    timer_begin(p, ST_BUILD, &ev);
    e = launch_prepsi(p);
    p->n = n_prev;
    if (e != cudaSuccess) return cuda_fail(e, "psi precompute");
    timer_end(p, ST_BUILD, ev);
  }
  p->offsets_valid = false;
  if (p->opts.d >= 2 || p->d1_binned) {   // key offsets for the binned gathers (else built on demand)
    timer_begin(p, ST_BUILD, &ev);
    if ((e = launch_build(p, x, n)) != cudaSuccess) return cuda_fail(e, "build kernel");
    timer_end(p, ST_BUILD, ev);
    p->offsets_valid = true;
  }
  if (h_bad_dst) {   // pipelined: the caller checks the validation word after synchronizing
    p->n = n;
    p->nodes_set = true;
    p->n_set++;
    return BNFFT_OK;
  }
  if ((e = cudaStreamSynchronize(p->stream)) != cudaSuccess) return cuda_fail(e, "set_nodes sync");
  unsigned long long bad = *p->h_bad;
  if (bad != ~0ull) {
    int64_t idx = (int64_t)(bad >> 4);
    int code = (int)(bad & 15);
    if (first_bad) *first_bad = idx;
    char buf[128];
    snprintf(buf, sizeof(buf), "node %lld rejected", (long long)idx);
    set_error(buf);
    p->n = 0;
    if (code == 1) return BNFFT_E_NODE_NOT_FINITE;
    if (code == 2) return BNFFT_E_NODE_OUT_OF_RANGE;
    return BNFFT_E_NODE_OUTSIDE_FEASIBLE_BOX;
  }
  p->n = n;
  p->nodes_set = true;
  p->n_set++;
  return BNFFT_OK;
}

// Steps 1 and 2 (deconvolution + zero-pad, inverse FFT) on p->stream: theta into d_grid
static int grid_stage(bnfft_plan_s* p, const void* fhat) {
  cudaError_t e;
  cudaEvent_t ev;
  timer_begin(p, ST_DECONV, &ev);
  if ((e = launch_deconv(p, fhat)) != cudaSuccess) return cuda_fail(e, "deconv kernel");
  timer_end(p, ST_DECONV, ev);
  timer_begin(p, ST_FFT, &ev);
  cufftResult fr = CUFFT_SUCCESS;
  if (p->pfft3) {   // planes k_1 in [0, M/2) -> [0, M/2), k_1 in [-M/2, 0) -> [L - M/2, L)
    const size_t pl = (size_t)p->L * p->L, half = (size_t)(p->opts.M / 2);
    for (int h = 0; h < 2 && fr == CUFFT_SUCCESS; ++h) {
      const size_t src = h * half * pl, dst = (h ? (size_t)p->L - half : 0) * pl;
      fr = p->c128 ? cufftExecZ2Z(p->fft2, (cufftDoubleComplex*)p->d_fft_p + src,
                                  (cufftDoubleComplex*)p->d_fft_in + dst, CUFFT_INVERSE)
                   : cufftExecC2C(p->fft2, (cufftComplex*)p->d_fft_p + src, (cufftComplex*)p->d_fft_in + dst,
                                  CUFFT_INVERSE);
    }
  }
  if (fr == CUFFT_SUCCESS)
    fr = p->c128 ? cufftExecZ2Z(p->fft, (cufftDoubleComplex*)p->d_fft_in, (cufftDoubleComplex*)p->d_grid,
                                CUFFT_INVERSE)
                 : cufftExecC2C(p->fft, (cufftComplex*)p->d_fft_in, (cufftComplex*)p->d_grid, CUFFT_INVERSE);
  if (fr != CUFFT_SUCCESS) {
    char buf[64];
    snprintf(buf, sizeof(buf), "cufftExec failed (%d)", (int)fr);
    set_error(buf);
    return BNFFT_E_CUFFT;
  }
  timer_end(p, ST_FFT, ev);
  return BNFFT_OK;
}

extern "C" {

int bnfft_execute(bnfft_plan_s* p, const void* fhat, void* f) {
  if (!p) return BNFFT_E_INVALID_ARG;
  if (!p->nodes_set) { set_error("call bnfft_set_nodes first"); return BNFFT_E_NODES_NOT_SET; }
  const int64_t n_out = (p->dist && p->opts.dist == BNFFT_DIST_SLAB) ? 1 : p->n;
  if (!fhat || (n_out > 0 && !f)) { set_error("NULL buffer"); return BNFFT_E_INVALID_ARG; }
  cudaSetDevice(p->device);
  cudaError_t e;
  if ((e = join_precompute(p)) != cudaSuccess) return cuda_fail(e, "precompute join");
  if (p->dist && p->opts.dist == BNFFT_DIST_SLAB) return dist_execute(p, fhat, f);
  int rc = grid_stage(p, fhat);
  if (rc != BNFFT_OK) return rc;
  cudaEvent_t ev;
  timer_begin(p, ST_GATHER, &ev);
  if ((e = launch_gather(p, f)) != cudaSuccess) return cuda_fail(e, "gather kernel");
  timer_end(p, ST_GATHER, ev);
  p->n_exec++;
  return BNFFT_OK;
}

/* One call for the whole of Algorithm 2 on device buffers (header: bnfft_transform). */
int bnfft_transform(bnfft_plan_s* p, int64_t n, const double* x, const void* fhat, void* f, int64_t* first_bad) {
  if (first_bad) *first_bad = -1;
  if (!p) return BNFFT_E_INVALID_ARG;
  if (n < 0 || n >= ((int64_t)1 << 31) || (n > 0 && !x) || !fhat || (n > 0 && !f)) {
    set_error("n must be in [0, 2^31), buffers non-NULL");
    return BNFFT_E_INVALID_ARG;
  }
  cudaSetDevice(p->device);
  int rc;
  if (p->dist) {   // multi-rank plans: the exchange steps order the stages
    if ((rc = bnfft_precompute(p)) != BNFFT_OK) return rc;
    if ((rc = bnfft_set_nodes(p, n, x, first_bad)) != BNFFT_OK) return rc;
    return bnfft_execute(p, fhat, f);
  }
  // fork: steps 0(a), 1, 2 on the side stream (they do not depend on the nodes) ...
  if ((rc = bnfft_precompute(p)) != BNFFT_OK) return rc;
  cudaStream_t main_stream = p->stream;
  cufftResult fr = cufftSetStream(p->fft, p->pre_stream);
  if (fr == CUFFT_SUCCESS && p->pfft3) fr = cufftSetStream(p->fft2, p->pre_stream);
  if (fr != CUFFT_SUCCESS) { set_error("cufftSetStream failed"); return BNFFT_E_CUFFT; }
  p->stream = p->pre_stream;
  rc = grid_stage(p, fhat);
  p->stream = main_stream;
  cudaError_t e = cudaEventRecord(p->ev_pre, p->pre_stream);   // the join now covers the grid stage
  fr = cufftSetStream(p->fft, main_stream);
  if (fr == CUFFT_SUCCESS && p->pfft3) fr = cufftSetStream(p->fft2, main_stream);
  if (rc != BNFFT_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "transform join");
  if (fr != CUFFT_SUCCESS) { set_error("cufftSetStream failed"); return BNFFT_E_CUFFT; }
  // ... while row a1 (validate, sort, offsets) runs on the plan's stream
  if ((rc = local_set_nodes(p, n, x, first_bad)) != BNFFT_OK) return rc;   // (a bad node: the join stays pending)
  if ((e = join_precompute(p)) != cudaSuccess) return cuda_fail(e, "transform join");
  cudaEvent_t ev;
  timer_begin(p, ST_GATHER, &ev);
  if ((e = launch_gather(p, f)) != cudaSuccess) return cuda_fail(e, "gather kernel");
  timer_end(p, ST_GATHER, ev);
  p->n_exec++;
  return BNFFT_OK;
}

int bnfft_interpolate(bnfft_plan_s* p, const void* samples, void* f) {
  if (!p) return BNFFT_E_INVALID_ARG;
  if (!p->nodes_set) { set_error("call bnfft_set_nodes first"); return BNFFT_E_NODES_NOT_SET; }
  if (!samples || (p->n > 0 && !f)) { set_error("NULL buffer"); return BNFFT_E_INVALID_ARG; }
  cudaSetDevice(p->device);
  cudaError_t e = cudaMemcpyAsync(p->d_grid, samples, (size_t)p->Ld * p->opts.batch * p->csize,
                                  cudaMemcpyDeviceToDevice, p->stream);
  if (e != cudaSuccess) return cuda_fail(e, "copy samples");
  cudaEvent_t ev;
  timer_begin(p, ST_GATHER, &ev);
  if ((e = launch_gather(p, f)) != cudaSuccess) return cuda_fail(e, "gather kernel");
  timer_end(p, ST_GATHER, ev);
  return BNFFT_OK;
}

int bnfft_kernel_hat(bnfft_plan_s* p, int64_t n, const double* v_host, double* out_host) {
  if (!p || n < 0 || (n > 0 && (!v_host || !out_host))) return BNFFT_E_INVALID_ARG;
  if (n == 0) return BNFFT_OK;
  cudaSetDevice(p->device);
  double* d = nullptr;
  cudaError_t e = cudaMalloc((void**)&d, 2 * n * sizeof(double));
  if (e != cudaSuccess) return cuda_fail(e, "alloc kernel_hat");
  e = cudaMemcpyAsync(d, v_host, n * sizeof(double), cudaMemcpyHostToDevice, p->stream);
  if (e == cudaSuccess) e = launch_kernel_hat(p, d, d + n, n);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_host, d + n, n * sizeof(double), cudaMemcpyDeviceToHost, p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  cudaFree(d);
  return e == cudaSuccess ? BNFFT_OK : cuda_fail(e, "kernel_hat");
}

int bnfft_transform_host(bnfft_plan_s* p, int64_t n, const double* x_host, const void* fhat_host,
                         void* f_host, int64_t* first_bad) {
  if (first_bad) *first_bad = -1;
  if (!p || !fhat_host || (n > 0 && (!x_host || !f_host))) return BNFFT_E_INVALID_ARG;
  if (n < 0 || n >= ((int64_t)1 << 31)) return BNFFT_E_INVALID_ARG;
  cudaSetDevice(p->device);
  cudaError_t e;
  size_t xb = (size_t)n * p->opts.d * sizeof(double);
  size_t fhb = (size_t)p->Md * p->opts.batch * p->csize;
  size_t fb = (size_t)n * p->opts.batch * p->csize;
  if (n > p->x_stage_cap) {
    dfree_plan(p, p->d_x_stage);
    dfree_plan(p, p->d_f_stage);
    p->d_x_stage = nullptr;
    p->d_f_stage = nullptr;
    if ((e = dmalloc(p, &p->d_x_stage, xb)) != cudaSuccess) return cuda_fail(e, "alloc x stage");
    if ((e = dmalloc(p, &p->d_f_stage, fb)) != cudaSuccess) return cuda_fail(e, "alloc f stage");
    p->x_stage_cap = n;
  }
  if (!p->d_fhat_stage && (e = dmalloc(p, &p->d_fhat_stage, fhb)) != cudaSuccess)
    return cuda_fail(e, "alloc fhat stage");
  if (n > 0 && (e = cudaMemcpyAsync(p->d_x_stage, x_host, xb, cudaMemcpyHostToDevice, p->stream)) != cudaSuccess)
    return cuda_fail(e, "H2D x");
  if ((e = cudaMemcpyAsync(p->d_fhat_stage, fhat_host, fhb, cudaMemcpyHostToDevice, p->stream)) != cudaSuccess)
    return cuda_fail(e, "H2D fhat");
  int rc = bnfft_set_nodes(p, n, p->d_x_stage, first_bad);
  if (rc != BNFFT_OK) return rc;
  rc = bnfft_execute(p, p->d_fhat_stage, p->d_f_stage);
  if (rc != BNFFT_OK) return rc;
  if (n > 0 && (e = cudaMemcpyAsync(f_host, p->d_f_stage, fb, cudaMemcpyDeviceToHost, p->stream)) != cudaSuccess)
    return cuda_fail(e, "D2H f");
  if ((e = cudaStreamSynchronize(p->stream)) != cudaSuccess) return cuda_fail(e, "transform sync");
  return BNFFT_OK;
}

int bnfft_transform_host_many(bnfft_plan_s* p, int32_t steps, int64_t n, const double* const* x_host,
                              const void* const* fhat_host, void* const* f_host, int64_t* first_bad) {
  if (first_bad) *first_bad = -1;
  if (!p || steps < 0 || (steps > 0 && (!x_host || !fhat_host || !f_host))) return BNFFT_E_INVALID_ARG;
  if (n < 0 || n >= ((int64_t)1 << 31)) return BNFFT_E_INVALID_ARG;
  for (int k = 0; k < steps; ++k)
    if (!fhat_host[k] || (n > 0 && (!x_host[k] || !f_host[k]))) return BNFFT_E_INVALID_ARG;
  if (p->dist) {   // multi-rank plans: the collectives order the steps; run them one by one
    for (int k = 0; k < steps; ++k) {
      int rc = bnfft_precompute(p);
      if (rc == BNFFT_OK) rc = bnfft_transform_host(p, n, x_host[k], fhat_host[k], f_host[k], first_bad);
      if (rc != BNFFT_OK) return rc;
    }
    return BNFFT_OK;
  }
  cudaSetDevice(p->device);
  cudaError_t e;
  const size_t xb = (size_t)n * p->opts.d * sizeof(double);
  const size_t fhb = (size_t)p->Md * p->opts.batch * p->csize;
  const size_t fb = (size_t)n * p->opts.batch * p->csize;
  if (!p->s_h2d) {
    if ((e = cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "copy streams");
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t* ev : {&p->ev_h2d[k], &p->ev_used[k], &p->ev_f[k], &p->ev_d2h[k]})
        if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "events");
  }
  if (n > p->pipe_cap) {
    for (int k = 0; k < 2; ++k) {
      dfree_plan(p, p->d_xp[k]);
      dfree_plan(p, p->d_fhp[k]);
      dfree_plan(p, p->d_fp[k]);
      p->d_xp[k] = nullptr;
      p->d_fhp[k] = p->d_fp[k] = nullptr;
      if ((e = dmalloc(p, &p->d_xp[k], std::max<size_t>(xb, 16))) != cudaSuccess ||
          (e = dmalloc(p, &p->d_fhp[k], fhb)) != cudaSuccess ||
          (e = dmalloc(p, &p->d_fp[k], std::max<size_t>(fb, 16))) != cudaSuccess)
        return cuda_fail(e, "alloc pipeline stages");
    }
    p->pipe_cap = n;
  }
  if (steps > p->h_bads_cap) {
    if (p->h_bads) cudaFreeHost(p->h_bads);
    p->h_bads = nullptr;
    if ((e = cudaMallocHost((void**)&p->h_bads, (size_t)steps * sizeof(unsigned long long))) != cudaSuccess)
      return cuda_fail(e, "alloc status ring");
    p->h_bads_cap = steps;
  }
  for (int k = 0; k < steps; ++k) {
    const int s = k & 1;
    // inputs of step k into slot s once step k-2 is done reading it
    if (k >= 2 && (e = cudaStreamWaitEvent(p->s_h2d, p->ev_used[s], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if (n > 0 && (e = cudaMemcpyAsync(p->d_xp[s], x_host[k], xb, cudaMemcpyHostToDevice, p->s_h2d)) != cudaSuccess)
      return cuda_fail(e, "H2D x");
    if ((e = cudaMemcpyAsync(p->d_fhp[s], fhat_host[k], fhb, cudaMemcpyHostToDevice, p->s_h2d)) != cudaSuccess)
      return cuda_fail(e, "H2D fhat");
    if ((e = cudaEventRecord(p->ev_h2d[s], p->s_h2d)) != cudaSuccess) return cuda_fail(e, "record");
    // compute on the plan's stream: step 0(a) (side stream), set_nodes, execute
    if ((e = cudaStreamWaitEvent(p->stream, p->ev_h2d[s], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if (k >= 2 && (e = cudaStreamWaitEvent(p->stream, p->ev_d2h[s], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    int rc = bnfft_precompute(p);
    if (rc == BNFFT_OK) rc = local_set_nodes(p, n, p->d_xp[s], nullptr, &p->h_bads[k]);
    if (rc == BNFFT_OK) rc = bnfft_execute(p, p->d_fhp[s], p->d_fp[s]);
    if (rc != BNFFT_OK) {
      cudaDeviceSynchronize();
      return rc;
    }
    if ((e = cudaEventRecord(p->ev_used[s], p->stream)) != cudaSuccess ||
        (e = cudaEventRecord(p->ev_f[s], p->stream)) != cudaSuccess)
      return cuda_fail(e, "record");
    // outputs of step k back while step k+1 runs
    if ((e = cudaStreamWaitEvent(p->s_d2h, p->ev_f[s], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if (n > 0 && (e = cudaMemcpyAsync(f_host[k], p->d_fp[s], fb, cudaMemcpyDeviceToHost, p->s_d2h)) != cudaSuccess)
      return cuda_fail(e, "D2H f");
    if ((e = cudaEventRecord(p->ev_d2h[s], p->s_d2h)) != cudaSuccess) return cuda_fail(e, "record");
  }
  if ((e = cudaStreamSynchronize(p->s_d2h)) != cudaSuccess || (e = cudaStreamSynchronize(p->stream)) != cudaSuccess)
    return cuda_fail(e, "pipeline sync");
  for (int k = 0; k < steps; ++k) {
    const unsigned long long bad = p->h_bads[k];
    if (bad == ~0ull) continue;
    const int64_t idx = (int64_t)(bad >> 4);
    const int code = (int)(bad & 15);
    if (first_bad) *first_bad = idx;
    char buf[128];
    snprintf(buf, sizeof(buf), "step %d: node %lld rejected", k, (long long)idx);
    set_error(buf);
    p->n = 0;
    p->nodes_set = false;
    if (code == 1) return BNFFT_E_NODE_NOT_FINITE;
    if (code == 2) return BNFFT_E_NODE_OUT_OF_RANGE;
    return BNFFT_E_NODE_OUTSIDE_FEASIBLE_BOX;
  }
  return BNFFT_OK;
}

int bnfft_get_info(const bnfft_plan_s* p, bnfft_info* o) {
  if (!p || !o) return BNFFT_E_INVALID_ARG;
  memset(o, 0, sizeof(*o));
  o->d = p->opts.d;
  o->M = p->opts.M;
  o->L = p->L;
  o->m = p->opts.m;
  o->window = p->opts.window;
  o->shape = p->shape;
  o->prec = p->opts.prec;
  o->batch = p->opts.batch;
  for (int t = 0; t < 3; ++t) {
    o->bin_log2[t] = p->bin_log2[t];
    o->bins_per_dim[t] = p->nb_dim[t];
  }
  o->nbins = p->nbins;
  o->user_block_log2 = p->ub_log2;
  o->nkeys = p->nkeys;
  o->key_col_bits = p->col_bits;
  o->tap_poly = p->tap_poly ? 1 : 0;
  o->tap_fit_err = p->tap_fit_err;
  o->key_bits = p->key_bits;
  o->sort_passes = p->sort_passes;
  o->flatness = p->flatness;
  o->n_nodes = p->nodes_set ? p->n : 0;
  o->grid_bytes = p->Ld * p->opts.batch * (int64_t)p->csize;
  o->device_bytes = p->device_bytes;
  dist_fill_info(p, o);
  if (p->opts.d == 1) {
    o->gather_kernel = p->opts.batch > 1 ? BNFFT_GK_SEGMENT
                       : (p->opts.flags & BNFFT_PRECOMPUTE_PSI) ? BNFFT_GK_PRE1
                       : p->d1_binned ? BNFFT_GK_BIN1 : BNFFT_GK_WINDOW1;
  } else {
    const bool coop3 = p->opts.d == 3 && p->opts.m == 4 && !p->c128 && p->opts.batch == 1;
    o->gather_kernel = p->g2_coop ? BNFFT_GK_COOP2 : !coop3 ? BNFFT_GK_BOX
                       : p->g3_kind == 0 ? BNFFT_GK_YSWEEP3 : p->g3_kind == 3 ? BNFFT_GK_YSWEEP3Q
                       : p->g3_kind == 1 ? BNFFT_GK_COOP3 : BNFFT_GK_SWEEP3;
  }
  return BNFFT_OK;
}

int bnfft_get_timing(bnfft_plan_s* p, bnfft_timing* o) {
  if (!p || !o) return BNFFT_E_INVALID_ARG;
  int rc = collect_timing(p);
  if (rc != BNFFT_OK) return rc;
  o->ms_psihat = p->ms[ST_PSIHAT];
  o->ms_keys = p->ms[ST_KEYS];
  o->ms_sort = p->ms[ST_SORT];
  o->ms_build = p->ms[ST_BUILD];
  o->ms_deconv = p->ms[ST_DECONV];
  o->ms_fft = p->ms[ST_FFT];
  o->ms_gather = p->ms[ST_GATHER];
  o->n_psihat = p->n_psihat;
  o->n_set_nodes = p->n_set;
  o->n_execute = p->n_exec;
  o->kernel_launches = p->launches;
  o->ms_exchange = p->ms[ST_EXCH];
  return BNFFT_OK;
}

int bnfft_reset_timing(bnfft_plan_s* p) {
  if (!p) return BNFFT_E_INVALID_ARG;
  int rc = collect_timing(p);
  for (int i = 0; i < ST_COUNT; ++i) p->ms[i] = 0;
  p->n_psihat = p->n_set = p->n_exec = p->launches = 0;
  return rc;
}

int bnfft_get_psihat(const bnfft_plan_s* p, double* host_out) {
  if (!p || !host_out) return BNFFT_E_INVALID_ARG;
  cudaSetDevice(p->device);
  cudaError_t e = cudaEventSynchronize(p->ev_pre);   // the last precompute has finished
  if (e == cudaSuccess) e = cudaMemcpyAsync(host_out, p->d_psihat, p->opts.M * sizeof(double),
                                  cudaMemcpyDeviceToHost, p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  return e == cudaSuccess ? BNFFT_OK : cuda_fail(e, "get_psihat");
}

int bnfft_get_grid(const bnfft_plan_s* p, void* dev_out) {
  if (!p || !dev_out) return BNFFT_E_INVALID_ARG;
  cudaSetDevice(p->device);
  cudaError_t e = cudaMemcpyAsync(dev_out, p->d_grid, (size_t)p->Ld * p->opts.batch * p->csize,
                                  cudaMemcpyDeviceToDevice, p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  return e == cudaSuccess ? BNFFT_OK : cuda_fail(e, "get_grid");
}

int bnfft_get_perm(const bnfft_plan_s* p, uint32_t* dev_out) {
  if (!p || !dev_out) return BNFFT_E_INVALID_ARG;
  if (!p->nodes_set) return BNFFT_E_NODES_NOT_SET;
  if (p->n == 0) return BNFFT_OK;
  cudaSetDevice(p->device);
  cudaError_t e = cudaMemcpyAsync(dev_out, p->d_perm, p->n * sizeof(uint32_t),
                                  cudaMemcpyDeviceToDevice, p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  return e == cudaSuccess ? BNFFT_OK : cuda_fail(e, "get_perm");
}

int bnfft_get_bin_offsets(bnfft_plan_s* p, uint32_t* dev_out) {
  if (!p || !dev_out) return BNFFT_E_INVALID_ARG;
  if (!p->nodes_set) return BNFFT_E_NODES_NOT_SET;
  cudaSetDevice(p->device);
  if (!p->offsets_valid) {   // user-order plans build the key offsets on demand
    cudaError_t eb = launch_build(p, nullptr, p->n);
    if (eb != cudaSuccess) return cuda_fail(eb, "build kernel");
    p->offsets_valid = true;
  }
  cudaError_t e = cudaMemcpyAsync(dev_out, p->d_bin_start, (p->nkeys + 1) * sizeof(uint32_t),
                                  cudaMemcpyDeviceToDevice, p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  return e == cudaSuccess ? BNFFT_OK : cuda_fail(e, "get_bin_offsets");
}

}  // extern "C"
