// Internal declarations of the bnfft library (product path).  Shares nothing with oracle/.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/bnfft.h"

namespace bnfft {

constexpr int kGatherThreads = 256;   // nodes per gather CTA chunk (one node per thread)
constexpr int kSortThreads = 512;
constexpr int kSortItems = 8;         // keys per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kSortTileLog2 = 12;
static_assert(kSortTile == (1 << kSortTileLog2), "sort tile is a power of two");
constexpr int kMaxDigitBits = 9;
constexpr int kQuadN = 64;            // Gauss-Legendre points for psi^ (reading A4)

// Window parameters in grid units tau = L x (|tau| <= m is the support).
struct WinParams {
  int window;        // bnfft_window
  int alg1;          // 1: classical NFFT (Algorithm 1): kernel phi instead of psi = sinc * phi
  int m;
  double inv_m;      // 1/m
  double beta;       // sinh / cKB shape
  double inv_norm;   // 1/sinh(beta) or 1/(I0(beta)-1)
  double gauss_b;    // Gaussian: phi(tau/L) = exp(-gauss_b tau^2), gauss_b = 1/(2 s^2 L^2)
  float beta_f, inv_norm_f, gauss_b_f, inv_m_f;
};

// phi(tau/L) (eq. varphisinh; cKB P:302-310; Gaussian reading A2), fp64.
__device__ __forceinline__ double phi_tau_d(double tau, const WinParams& w) {
  double t = tau * w.inv_m;
  if (fabs(t) > 1.0) return 0.0;
  double r = (1.0 - t) * (1.0 + t);
  if (w.window == BNFFT_SINH) return sinh(w.beta * sqrt(r)) * w.inv_norm;
  if (w.window == BNFFT_CKB) return (cyl_bessel_i0(w.beta * sqrt(r)) - 1.0) * w.inv_norm;
  return exp(-w.gauss_b * tau * tau);
}

// fp32 variant used by the complex64 path.
__device__ __forceinline__ float phi_tau_f(float tau, const WinParams& w) {
  float t = tau * w.inv_m_f;
  if (fabsf(t) > 1.0f) return 0.0f;
  float r = (1.0f - t) * (1.0f + t);
  if (w.window == BNFFT_SINH) {
    float a = w.beta_f * sqrtf(r);
    float e = expf(a);
    return 0.5f * (e - 1.0f / e) * w.inv_norm_f;
  }
  if (w.window == BNFFT_CKB) return (cyl_bessel_i0f(w.beta_f * sqrtf(r)) - 1.0f) * w.inv_norm_f;
  return expf(-w.gauss_b_f * tau * tau);
}

struct Timer {
  int stage;
  cudaEvent_t a, b;
};

enum Stage { ST_PSIHAT = 0, ST_KEYS, ST_SORT, ST_BUILD, ST_DECONV, ST_FFT, ST_GATHER, ST_EXCH, ST_COUNT };

struct DistState;   // multi-GPU state of a plan (dist.cu)

}  // namespace bnfft

struct bnfft_plan_s {
  bnfft_opts opts;
  int64_t L = 0, Ld = 0, Md = 0;
  double shape = 0;
  bnfft::WinParams wp{};
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t pre_stream = nullptr;   // step 0(a) runs here, overlapping node preprocessing
  cudaEvent_t ev_fork = nullptr, ev_pre = nullptr;
  bool pre_pending = false;            // main stream has not yet waited for the last precompute
  bool c128 = false;
  size_t csize = 8;  // bytes per complex

  // binning
  int bin_log2[3] = {0, 0, 0};
  int64_t nb_dim[3] = {1, 1, 1};
  int64_t nbins = 1;
  int key_bits = 0, sort_passes = 0, digit_bits = 0;
  int col_bits = 0;            // rec3: minor sort digit c_1 mod 16 below the bin (nodes of an x-line in
                               // column order); key offsets stay per bin
  int ub_log2 = 31;            // user-block size of the sort key (user block, bin); 31 = one block
  int64_t nkeys = 1;           // number of (user block, bin) keys of the current node set
  int64_t key_start_cap = 0;

  // gather tap polynomials (plan time, tapfit kernel)
  bool tap_poly = true;
  int tap_nc = 0;              // coefficients per tap
  double tap_fit_err = 0;      // max |poly - exact| over taps (plan-time check)
  std::vector<double> tap_coef;   // T x tap_nc, monomials in x = 2u - 1

  // plan-owned device buffers
  double* d_gl = nullptr;       // 2*kQuadN: theta_q, weights
  double* d_psihat = nullptr;   // M
  double* d_q = nullptr;        // M
  double* d_flat = nullptr;     // 2 doubles: flatness, min|psihat|/|psihat(0)|
  void* d_fft_in = nullptr;     // batch x L^d complex, zero outside I_M (set once)
  void* d_grid = nullptr;       // batch x L^d complex, theta (centred)
  cufftHandle fft = 0;
  bool fft_ok = false;
  // pruned step 2 (d = 3, batch 1, 2M <= L): the FFT input is zero outside I_M, so 2-D inverse FFTs
  // over (k_2, k_3) run only on the M nonzero k_1 planes (compact buffer d_fft_p, two affine batches:
  // k_1 >= 0 and k_1 < 0), into the nonzero planes of d_fft_in, then 1-D FFTs along k_1 (stride L^2)
  bool pfft3 = false;
  void* d_fft_p = nullptr;       // M x L x L complex: plane (k_1 mod M), rows k_2 mod L, k_3 mod L
  cufftHandle fft2 = 0;
  bool fft2_ok = false;
  double flatness = 0;

  // nodes
  int64_t n = 0, cap = 0;
  bool nodes_set = false;
  double* d_xs = nullptr;        // node copy n x d: user order (xs_user) or sorted (last radix pass);
                                 // rec3 plans: sorted 16-B node records (float4, see rec3)
  bool rec3 = false;             // y-sweep d = 3 plans: the keys kernel writes a 16-B record per node
                                 // (u_x, u_y, u_z as float; (c_y & 15) << 3 | (c_z & 7)) in user order
                                 // (d_rec_user); the last radix pass gathers the records, not x
  void* d_rec_user = nullptr;
  bool xs_user = false;          // d <= 2 user-blocked plans keep nodes in user order
  bool offsets_valid = false;    // key offsets built (lazily for xs_user plans)
  uint32_t* d_perm = nullptr;    // sorted pos -> user index
  uint32_t* d_skeys = nullptr;   // sorted keys (points into keys buffers)
  uint32_t* d_bin_start = nullptr;  // nkeys + 1: first sorted position of each (user block, bin)
  uint32_t *d_k0 = nullptr, *d_k1 = nullptr, *d_v0 = nullptr, *d_v1 = nullptr;
  uint32_t* d_hist = nullptr;    // digits x tiles
  uint32_t* d_scan_part = nullptr;
  int64_t hist_cap = 0, part_cap = 0;
  unsigned long long* d_bad = nullptr;   // (index << 4) | code
  unsigned long long* h_bad = nullptr;   // pinned

  // host transform staging
  double* d_x_stage = nullptr; int64_t x_stage_cap = 0;
  void* d_fhat_stage = nullptr;
  void* d_f_stage = nullptr; int64_t f_stage_cap = 0;
  // pipelined host transforms (bnfft_transform_host_many): two staging slots, copy streams, events
  double* d_xp[2] = {nullptr, nullptr};
  void* d_fhp[2] = {nullptr, nullptr};
  void* d_fp[2] = {nullptr, nullptr};
  int64_t pipe_cap = -1;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr}, ev_f[2] = {nullptr, nullptr},
              ev_d2h[2] = {nullptr, nullptr};
  unsigned long long* h_bads = nullptr; int32_t h_bads_cap = 0;

  int gather_bt = 1;          // batch slice per staged box
  int gather_smax = 1;        // segments (bins) staged per round
  int gather_box_cap = 0;     // d = 1: staged window capacity (complex elements)
  int64_t gather_grid1 = 0;   // persistent grid size (SMs x resident CTAs)
  int gather_nslice = 1, gather_box_elems = 0, gather_bufstride = 0;
  int gather_nbuf = 2;
  int gather_threads = 256;      // threads per CTA of the d >= 2 gather launch
  bool g2_coop = false;          // d = 2, complex64, batch 1, m <= 7: quarter-warp-cooperative kernel (gather2c)
  int g3_kind = 0;               // d = 3, m = 4, complex64, batch 1: 0 y-sweep (gather3y, default),
                                 // 1 half-warp (gather3c, BNFFT_GATHER3C), 2 z-sweep (gather3s, BNFFT_GATHER3S)
  int gather_tbox[3] = {1, 1, 1};
  bool d1_binned = false;         // d = 1: bins of 2^bin_log2 cells, one radix pass, per-bin gather
  void* d_pre_w = nullptr;        // BNFFT_PRECOMPUTE_PSI: [n][2m] weights of the sorted nodes
  int64_t pre_cap = 0;
  alignas(64) CUtensorMap tmap;   // d >= 2: TMA descriptor of the theta grid (host copy)
  CUtensorMap* d_tmap = nullptr;  // device (global memory) copy used by the kernel
  size_t gather_smem = 0;

  // timing
  std::vector<bnfft::Timer> pending;
  std::vector<cudaEvent_t> pool;
  double ms[bnfft::ST_COUNT] = {0};
  int64_t n_psihat = 0, n_set = 0, n_exec = 0, launches = 0;
  int64_t device_bytes = 0;
  std::vector<std::pair<void*, size_t>> allocs;   // live plan allocations (device_bytes accounting)

  // multi-GPU (nranks > 1): transport, slab geometry, node exchange (dist.cu)
  bnfft::DistState* dist = nullptr;
};

namespace bnfft {

// error helpers (plan.cu)
void set_error(const std::string& s);
int cuda_fail(cudaError_t e, const char* what);

// timing helpers
// SM count of the current device (cached per device): grid-stride launch caps are multiples of it
int sm_count();
void timer_begin(bnfft_plan_s* p, int stage, cudaEvent_t* ev);
void timer_end(bnfft_plan_s* p, int stage, cudaEvent_t ev);

// launchers
cudaError_t launch_psihat(bnfft_plan_s* p);
cudaError_t launch_tapfit(bnfft_plan_s* p, int NC, double* d_coef, double* d_err);
cudaError_t launch_kernel_hat(bnfft_plan_s* p, const double* v_dev, double* out_dev, int64_t n);
cudaError_t launch_keys(bnfft_plan_s* p, const double* x, int64_t n);
cudaError_t launch_sort(bnfft_plan_s* p, const double* x, int64_t n);
cudaError_t sort_prepare();
cudaError_t launch_build(bnfft_plan_s* p, const double* x, int64_t n);
cudaError_t launch_deconv(bnfft_plan_s* p, const void* fhat);
cudaError_t launch_gather(bnfft_plan_s* p, void* out);
int gather_supported(int d, int m);
size_t gather_box_elems(const bnfft_plan_s* p);
cudaError_t gather_prepare(bnfft_plan_s* p);
cudaError_t launch_prepsi(bnfft_plan_s* p);
int tap_coef_count(bool c128);
cudaError_t dmalloc_bytes(bnfft_plan_s* p, void** ptr, size_t bytes);   // plan-owned, counted
void dfree_plan(bnfft_plan_s* p, void* ptr);

// multi-GPU (dist.cu); nranks > 1 plans route set_nodes / execute through these
int dist_create(bnfft_plan_s* p);                 // plan_create: transport + slab geometry + FFT plans
void dist_destroy(bnfft_plan_s* p);
int dist_set_nodes(bnfft_plan_s* p, int64_t n, const double* x, int64_t* first_bad);
int dist_execute(bnfft_plan_s* p, const void* fhat, void* f);
void dist_fill_info(const bnfft_plan_s* p, bnfft_info* o);
// single-rank body of bnfft_set_nodes; with h_bad_dst the validation word is copied there
// asynchronously and the call returns without synchronizing (pipelined host transforms)
int local_set_nodes(bnfft_plan_s* p, int64_t n, const double* x, int64_t* first_bad,
                    unsigned long long* h_bad_dst = nullptr);
cudaError_t launch_deconv_slab(bnfft_plan_s* p, const void* fhat, void* out, int64_t k0_lo, int64_t k0_hi);

}  // namespace bnfft
