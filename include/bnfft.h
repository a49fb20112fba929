/*
 * bnfft -- B200-native hot path of Algorithm 2, "NFFT-like procedure for bandlimited
 * functions" (Kircheis & Potts, arXiv 2502.07155).  C ABI: plain pointers and sizes.
 *
 * Problem (Algorithm 2): given samples f^(k),
 * k in I_M = Z^d cap [-M/2, M/2)^d of the Fourier transform of a bandlimited f, and
 * nodes x_j in R^d, compute
 *     step 0(a)  psi^(k), k in I_M
 *     step 1     theta^(k) = f^(k)/psi^(k) on I_M, 0 on I_L \ I_M
 *     step 2     theta_l = L^{-d} sum_{k in I_L} theta^(k) e^{2 pi i k.l/L}, l in I_L
 *     step 3     f_j = sum_{l in J_{L,m}(x_j) cap I_L} theta_l psi(x_j - l/L)
 * with the regularized sinc psi(x) = sinc(L pi x) phi(x) (eq. sinc_reg) and a
 * window phi in Phi_{m,L}: sinh-type (eq. varphisinh), continuous
 * Kaiser-Bessel or the Gaussian of reading A2.  Matrix form:
 * f = Psi F D_psihat f^ (eq. function_eval).
 *
 * Readings where the paper is silent: L = M_sigma = 2 ceil(ceil(sigma M)/2)
 * (A7); default shape beta = pi m (1 - M/L) (A1), Gaussian s = sqrt(m/(pi L (L-M))) (A2);
 * tensor-product windows (A3); psi^ by 64-point Gauss-Legendre after t = (m/L) sin(theta) (A4);
 * nodes accepted on [-1/2, 1/2)^d with the literal I_L-truncated sum (A5).
 *
 * Execution model: every step runs on the GPU given at plan creation.  Step 2 calls cuFFT
 * (a separately timed stage, BASELINE north_star (c)); all other steps are this library's
 * own sm_100a kernels.  There is no CPU fallback: without a CUDA device every call that
 * would compute returns BNFFT_E_CUDA.
 *
 * Ownership: the caller owns every pointer it passes; the plan owns its device buffers
 * (psi^ table, FFT input/output grids, sorted nodes, permutation, bin offsets, scratch).
 * Thread safety: a plan is not re-entrant; distinct plans are independent.
 * Errors: every entry point returns 0 (BNFFT_OK) or a negative bnfft_status; no entry point
 * aborts the process.  bnfft_last_error() gives a human-readable detail for the calling thread.
 */
#ifndef BNFFT_H
#define BNFFT_H

#include <stdint.h>

#if defined(__GNUC__)
#define BNFFT_API __attribute__((visibility("default")))
#else
#define BNFFT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BNFFT_OK = 0,
  BNFFT_E_BAD_DIM = -1,                  /* d not in 1..3                                   */
  BNFFT_E_BAD_BANDWIDTH = -2,            /* M odd or < 2 ("M in 2N")                   */
  BNFFT_E_BAD_SIGMA = -3,                /* sigma < 1 or not finite                   */
  BNFFT_E_TRUNCATION_TOO_LARGE = -4,     /* m < 1 or 2m >= L ("2m << L")               */
  BNFFT_E_BAD_WINDOW_PARAM = -5,         /* unknown window, or shape <= 0 after defaults     */
  BNFFT_E_SPECTRAL_FACTOR_VANISHES = -6, /* |psi^_1(k)| < 1e-12 |psi^_1(0)|          */
  BNFFT_E_NODE_NOT_FINITE = -7,          /* a coordinate is NaN or +-Inf                     */
  BNFFT_E_NODE_OUT_OF_RANGE = -8,        /* a coordinate outside [-1/2, 1/2) (A5)            */
  BNFFT_E_NODE_OUTSIDE_FEASIBLE_BOX = -9,/* STRICT_DOMAIN: outside [-1/2+m/L, 1/2-m/L]*/
  BNFFT_E_NODES_NOT_SET = -10,           /* execute before a successful set_nodes            */
  BNFFT_E_CUDA = -11,                    /* CUDA runtime error (incl. no device)             */
  BNFFT_E_CUFFT = -12,                   /* cuFFT error                                      */
  BNFFT_E_OOM = -13,                     /* device allocation failed                         */
  BNFFT_E_UNSUPPORTED = -14,             /* parameters outside the compiled kernel set       */
  BNFFT_E_INVALID_ARG = -15,             /* NULL plan/pointer, n < 0, n >= 2^31, ...         */
  BNFFT_E_NCCL = -16                     /* NCCL (or local-group transport) error, or the NCCL
                                            library could not be loaded                      */
} bnfft_status;

typedef enum { BNFFT_SINH = 0, BNFFT_GAUSS = 1, BNFFT_CKB = 2 } bnfft_window;
typedef enum { BNFFT_C64 = 0, BNFFT_C128 = 1 } bnfft_prec;

enum {
  BNFFT_STRICT_DOMAIN = 1u,  /* reject nodes outside the closed feasible box   */
  BNFFT_TIMING = 8u,         /* record per-stage CUDA events (read with bnfft_get_timing)     */
  BNFFT_EXACT_TAPS = 16u,    /* gather evaluates sinc * phi directly (no tap polynomials)       */
  BNFFT_ALG1 = 32u           /* classical NFFT, Algorithm 1: phi^ deconvolution,
                                periodic short sums with the window phi (no sinc); nodes on the
                                torus [-1/2,1/2)^d.  d = 1; sinh / cKB windows; default shape
                                beta = 2 pi m (1 - 1/(2 sigma)) (reading A17)               */,
  BNFFT_PRECOMPUTE_PSI = 64u,/* Algorithm 2 step 0(b): set_nodes evaluates the kernel at every
                                (node, tap) once and stores it (2m values per node); execute reads
                                them instead of evaluating the tap polynomials.  d = 1, batch 1.
                                Costs 2m * (4|8) bytes per node of device memory.              */
  BNFFT_SORTED_OUTPUT = 128u,/* execute writes f in the plan's sorted node order (f_dev[i] is the value
                                of user node perm[i], bnfft_get_perm) instead of user order: the
                                gather's stores become sequential.  Single rank only.            */
  BNFFT_BALANCED_SLABS = 256u/* BNFFT_DIST_SLAB: slab cut points chosen from the all-reduced per-plane
                                node histogram (equal node counts) instead of equal plane counts */
};

/* Multi-GPU modes (bnfft_opts.dist; nranks > 1).  Step 3 is independent per node once theta exists
 * (P:510-513), so ranks exchange only grid planes and node records:
 *   BNFFT_DIST_REPLICATE  every rank computes the whole theta grid and evaluates its own nodes; no
 *                         communication (results bitwise equal to one GPU).
 *   BNFFT_DIST_SLAB       d = 3: rank r owns the theta planes l_2 in [a_r, b_r) (slab along the
 *                         second dimension).  Step 2 is a distributed slab FFT (per-rank 2-D FFTs over
 *                         (k_2, k_3) of its k_1 chunk, an all-to-all, 1-D FFTs along k_1), the m-halo
 *                         planes [a_r - m + 1, a_r) and [b_r, b_r + m) are exchanged with the
 *                         neighbours (zero beyond the global ends: Psi is not periodic),
 *                         set_nodes sends every node to the rank owning its cell and execute returns
 *                         the values to the originating rank, in its user order.
 * Transport: an NCCL communicator (nccl_comm = ncclComm_t, e.g. torch's ProcessGroupNCCL comm or
 * bnfft_nccl_comm_init) with one process per GPU, or a local group (local_group =
 * bnfft_group_create(nranks)) of nranks plans driven by nranks host threads of one process, on any
 * device(s) -- the same exchange code over cudaMemcpyAsync, for tests on one GPU. */
enum { BNFFT_DIST_REPLICATE = 0, BNFFT_DIST_SLAB = 1 };

/* Plan options.  d: 1..3.  M: even >= 2.  sigma >= 1, L = 2 ceil(ceil(sigma M)/2).
 * m: truncation parameter, 1 <= m, 2m < L; compiled range m <= 16 (d=1), 12 (d=2), 8 (d=3).
 * window: bnfft_window.  shape: beta (sinh, cKB) or s in x units (Gaussian); <= 0 selects the
 * default of readings A1/A2.  prec: arithmetic of steps 1-3 (C64: fp32 complex64 grid and
 * taps; C128: fp64).  Nodes are always float64.  batch >= 1 spectra share one node set.
 * flags: BNFFT_STRICT_DOMAIN | BNFFT_TIMING | BNFFT_EXACT_TAPS | BNFFT_ALG1 | BNFFT_PRECOMPUTE_PSI.  device: CUDA ordinal.  stream: cudaStream_t
 * (NULL = legacy default stream) on which every kernel and copy of this plan is issued. */
typedef struct {
  int32_t d;
  int64_t M;
  double sigma;
  int32_t m;
  int32_t window;
  double shape;
  int32_t prec;
  int32_t batch;
  uint32_t flags;
  int32_t device;
  void* stream;
  /* multi-GPU (all zero / NULL = one GPU) */
  int32_t rank, nranks;   /* this plan's rank in [0, nranks); nranks <= 1: single GPU            */
  void* nccl_comm;        /* ncclComm_t of nranks ranks (this plan's rank = its NCCL rank), or NULL */
  void* local_group;      /* bnfft_group handle (in-process transport), or NULL                   */
  int32_t dist;           /* BNFFT_DIST_REPLICATE or BNFFT_DIST_SLAB                              */
} bnfft_opts;

/* Plan description.  Node binning geometry (for the stable bin sort, row a1): the cell of
 * a node is c_t = floor(L x_t) + L/2 in [0, L) (clamped to L-1), its bin b_t = c_t >> bin_log2[t],
 * its bin index is row-major (dim 0 slowest) over bins_per_dim, and its sort key is
 * ((j >> user_block_log2) * nbins + bin) * 2^key_col_bits + minor for user index j, where minor =
 * c_1 mod 16 for key_col_bits = 4 (the d = 3 y-sweep gather: an x-line bin's nodes in y-column order),
 * minor = ((c_2 >> 2) & 1) * 16 + c_1 mod 16 for key_col_bits = 5 (gather3q: two column sweeps, one per
 * half of the bin's z extent), and no minor digit for key_col_bits = 0.
 * Nodes are sorted stably by that key (ties by user index); the key offsets (bnfft_get_bin_offsets)
 * are per (user block, bin): nkeys = ceil(n / 2^user_block_log2) * nbins for the current node set.
 * tap_poly: the gather evaluates psi by per-tap polynomials (fit error tap_fit_err, checked at
 * plan creation) rather than by direct sinc * phi evaluation. */
typedef struct {
  int32_t d;
  int64_t M;
  int64_t L;
  int32_t m;
  int32_t window;
  double shape;
  int32_t prec;
  int32_t batch;
  int32_t bin_log2[3];
  int64_t bins_per_dim[3];
  int64_t nbins;
  int32_t user_block_log2;
  int64_t nkeys;
  int32_t tap_poly;
  double tap_fit_err;
  int32_t key_bits;
  int32_t sort_passes;
  double flatness;          /* max_k |L psi^_1(k) - 1| on I_M                    */
  int64_t n_nodes;          /* nodes of the last successful set_nodes (0 if none)          */
  int64_t grid_bytes;       /* bytes of one theta grid (batch x L^d complex)               */
  int64_t device_bytes;     /* device memory currently owned by the plan                   */
  int32_t gather_kernel;    /* step-3 kernel execute launches: BNFFT_GK_*                  */
  int32_t rank, nranks, dist;
  int64_t slab_lo, slab_hi; /* DIST_SLAB: this rank's planes [slab_lo, slab_hi) of dimension 2 */
  int64_t n_owned;          /* DIST_SLAB: nodes this rank evaluates (its slab's nodes)      */
  int64_t halo_bytes;       /* DIST_SLAB: grid bytes received from the neighbours per execute */
  int32_t key_col_bits;     /* minor sort digit below the bin (see above)                  */
} bnfft_info;

/* bnfft_info.gather_kernel */
enum {
  BNFFT_GK_WINDOW1 = 0,   /* d = 1: chunked window kernel (gather1_kernel)                 */
  BNFFT_GK_BIN1 = 1,      /* d = 1, large grids: per-bin kernel (gather1b_kernel)           */
  BNFFT_GK_SEGMENT = 2,   /* d = 1 batched: generic segment kernel (gather_kernel)          */
  BNFFT_GK_BOX = 3,       /* d = 2, 3: binned TMA-box kernel (gatherN_kernel)               */
  BNFFT_GK_COOP3 = 4,     /* d = 3, m = 4, complex64: warp-cooperative kernel (gather3c)    */
  BNFFT_GK_PRE1 = 5,      /* d = 1 with BNFFT_PRECOMPUTE_PSI (gather1_kernel, stored taps)  */
  BNFFT_GK_SWEEP3 = 6,    /* d = 3, m = 4, complex64: z-sweep kernel (gather3s_kernel)       */
  BNFFT_GK_YSWEEP3 = 7,   /* d = 3, m = 4, complex64: y-sweep kernel (gather3y_kernel)       */
  BNFFT_GK_YSWEEP3Q = 8,  /* the same with half-height z sweeps, no z dispatch (gather3q_kernel) */
  BNFFT_GK_COOP2 = 9      /* d = 2, complex64, m <= 7: quarter-warp-cooperative kernel (gather2c) */
};

/* Per-stage device times (ms) accumulated since the last reset, and call counts.  Only
 * recorded with BNFFT_TIMING.  Events are recorded on the plan's stream around each stage's
 * kernels; reading them synchronizes with those events. */
typedef struct {
  double ms_psihat, ms_keys, ms_sort, ms_build, ms_deconv, ms_fft, ms_gather;
  int64_t n_psihat, n_set_nodes, n_execute;
  int64_t kernel_launches;  /* this library's own kernels launched (cuFFT not counted)    */
  double ms_exchange;       /* multi-GPU: node exchange, FFT all-to-all, halos, output return */
} bnfft_timing;

/* Create a plan: validates options, allocates device buffers, creates the cuFFT plan and runs
 * step 0(a) (bnfft_precompute).  Synchronous.  On error *out is NULL. */
BNFFT_API int bnfft_plan_create(const bnfft_opts* opts, struct bnfft_plan_s** out);

/* Algorithm 2 step 0(a): psi^_1(k), k in I_M, by quadrature on the device, and the
 * folded deconvolution factors q(k) = (-1)^k / (L psi^_1(k)) (A8, A9).  Asynchronous: the work
 * runs on a plan-owned side stream forked from the plan's stream (an event recorded on the plan's
 * stream at the call), so it overlaps a following bnfft_set_nodes; bnfft_execute makes the plan's
 * stream wait for it, and bnfft_get_psihat waits for it.  plan_create calls it and checks the
 * result. */
BNFFT_API int bnfft_precompute(struct bnfft_plan_s* plan);

/* Set the node set.  x_dev: device pointer, n x d float64, row-major, user order; may be freed
 * after return (the plan keeps a sorted copy).  n in [0, 2^31).  Validates every node (finite,
 * in [-1/2, 1/2)^d, and the feasible box with STRICT_DOMAIN), then sorts the nodes stably by bin
 * (row a1).  Synchronous (reads back the validation result).  On a bad node returns the code of
 * the lowest offending index and stores that index in *first_bad (if non-NULL; else -1). */
BNFFT_API int bnfft_set_nodes(struct bnfft_plan_s* plan, int64_t n, const double* x_dev, int64_t* first_bad);

/* Steps 1-3.  fhat_dev: device, batch x M^d complex (complex64 for C64, complex128 for C128;
 * interleaved re/im), centred row-major (index k_t + M/2, last dim fastest), batch slowest.
 * f_dev: device, batch x n complex of the same precision, user node order.  Stream-ordered and
 * asynchronous; errors of earlier asynchronous work surface as BNFFT_E_CUDA. */
BNFFT_API int bnfft_execute(struct bnfft_plan_s* plan, const void* fhat_dev, void* f_dev);

/* Algorithm 2 in one call on device buffers: step 0(a), row a1 (bnfft_set_nodes) and
 * steps 1-3 (bnfft_execute) for n nodes x_dev, spectrum fhat_dev, values into f_dev (layouts as in
 * those calls).  Steps 0(a), 1 and 2 do not depend on the nodes, and the bin sort does not depend on
 * f^: they run concurrently, the grid stage on the plan's side stream (forked from the plan's stream
 * at the call, so everything enqueued earlier on the plan's stream is visible to both), the sort on
 * the plan's stream; step 3 joins them.  Results are bitwise equal to precompute + set_nodes +
 * execute.  Synchronous up to the node validation (as bnfft_set_nodes); the gather is asynchronous
 * on the plan's stream.  Errors and first_bad as bnfft_set_nodes / bnfft_execute.  Multi-rank plans
 * run the three calls in sequence. */
BNFFT_API int bnfft_transform(struct bnfft_plan_s* plan, int64_t n, const double* x_dev, const void* fhat_dev,
                              void* f_dev, int64_t* first_bad);

/* Step 3 alone with caller-provided grid samples: f_j = sum_{l in I_L} s_l psi(x_j - l/L), i.e. the
 * regularized Shannon sampling formula with localized sampling (eq. Rmf(x)_multi) restricted
 * to l in I_L (first equality of P:463); with BNFFT_ALG1 the periodic sum with the window,
 * f~_j = sum_{l in I_{L,m}(x_j)} s_l phi~_m(x_j - l/L) (the matrix B of P:184-199).  samples_dev:
 * device, batch x L^d complex (plan precision), centred (l_t + L/2), row-major.  f_dev as in
 * bnfft_execute.  Stream-ordered; requires set_nodes. */
BNFFT_API int bnfft_interpolate(struct bnfft_plan_s* plan, const void* samples_dev, void* f_dev);

/* The kernel's Fourier transform at arbitrary real frequencies (the quadrature of step 0(a)):
 * psi^_1(v) = 2 int_0^{m/L} psi(t) cos(2 pi v t) dt, or phi^_1(v) with BNFFT_ALG1.  n values
 * from host v_host into host out_host (computed on the device; synchronous). */
BNFFT_API int bnfft_kernel_hat(struct bnfft_plan_s* plan, int64_t n, const double* v_host, double* out_host);

/* End-to-end helper with HOST buffers: copies x (n x d float64) and f^ host->device, runs
 * set_nodes and execute, copies f device->host, and synchronizes.  Pinned host memory gives
 * asynchronous DMA; pageable memory works but is staged by the CUDA driver. */
BNFFT_API int bnfft_transform_host(struct bnfft_plan_s* plan, int64_t n, const double* x_host,
                         const void* fhat_host, void* f_host, int64_t* first_bad);

/* Pipelined end-to-end transforms with HOST buffers: `steps` complete runs of Algorithm 2 (step 0(a),
 * set_nodes, execute) on node sets of n nodes each: step k reads x_host[k] (n x d float64, user order)
 * and fhat_host[k], and writes f_host[k] (layouts as bnfft_execute).  Step k+1's host->device copies,
 * step k's compute and step k-1's device->host copy run on three streams and overlap (two device
 * staging slots, owned by the plan); host buffers must be pinned for the copies to overlap.  Different
 * steps may share input buffers; output buffers of consecutive steps must differ.  Synchronous: returns
 * after the last copy.  A step with an invalid node returns that node's code (first_bad = its index in
 * that step's node set; bnfft_last_error names the step); outputs of that step are undefined.
 * Multi-rank plans run the steps one by one. */
BNFFT_API int bnfft_transform_host_many(struct bnfft_plan_s* plan, int32_t steps, int64_t n,
                                        const double* const* x_host, const void* const* fhat_host,
                                        void* const* f_host, int64_t* first_bad);

BNFFT_API int bnfft_get_info(const struct bnfft_plan_s* plan, bnfft_info* out);
BNFFT_API int bnfft_get_timing(struct bnfft_plan_s* plan, bnfft_timing* out);
BNFFT_API int bnfft_reset_timing(struct bnfft_plan_s* plan);

/* Stage outputs for parity checks (synchronous copies):
 *   bnfft_get_psihat: M float64 values psi^_1(k), k = -M/2..M/2-1, into host memory.
 *   bnfft_get_grid:   the theta grid of the last execute (batch x L^d complex, centred index
 *                     l_t + L/2, row-major) into a device buffer of grid_bytes.
 *   bnfft_get_perm:   n uint32: sorted position -> user index, into a device buffer.
 *   bnfft_get_bin_offsets: nkeys+1 uint32: first sorted position of each sort key (user block,
 *                     bin), into a device buffer (built on demand for plans that keep the nodes
 *                     in user order; see user_block_log2). */
BNFFT_API int bnfft_get_psihat(const struct bnfft_plan_s* plan, double* host_out);
BNFFT_API int bnfft_get_grid(const struct bnfft_plan_s* plan, void* dev_out);
BNFFT_API int bnfft_get_perm(const struct bnfft_plan_s* plan, uint32_t* dev_out);
BNFFT_API int bnfft_get_bin_offsets(struct bnfft_plan_s* plan, uint32_t* dev_out);

/* Release every resource of the plan (after synchronizing its stream).  NULL is a no-op. */
BNFFT_API int bnfft_destroy(struct bnfft_plan_s* plan);

/* ---- multi-GPU transport (see BNFFT_DIST_*) ----
 * bnfft_nccl_unique_id: 128 bytes (ncclUniqueId) into out128, to be broadcast to every rank.
 * bnfft_nccl_comm_init: ncclCommInitRank on `device`; *comm_out is an ncclComm_t for bnfft_opts.
 * bnfft_nccl_comm_destroy: ncclCommDestroy.  NCCL is loaded at run time (libnccl.so.2, the copy
 * already in the process if any); without it these return BNFFT_E_NCCL.
 * bnfft_nccl_selftest: collective check of the library's NCCL transport on `comm` (every rank of the
 * communicator calls it): each rank sends `bytes` bytes to every rank including itself through the
 * grouped ncclSend / ncclRecv exchange the slab path uses, and checks what it received and the host
 * all-gather; stream-ordered on `stream` (a cudaStream_t, may be NULL), synchronous.
 * bnfft_group_create / destroy: an in-process group of nranks ranks; each rank's plan is created
 * and driven by its own host thread (collective calls block until every rank has arrived). */
BNFFT_API int bnfft_nccl_unique_id(void* out128);
BNFFT_API int bnfft_nccl_comm_init(const void* id128, int32_t nranks, int32_t rank, int32_t device, void** comm_out);
BNFFT_API int bnfft_nccl_comm_destroy(void* comm);
BNFFT_API int bnfft_nccl_selftest(void* comm, int64_t bytes, void* stream);
BNFFT_API int bnfft_group_create(int32_t nranks, void** group_out);
BNFFT_API int bnfft_group_destroy(void* group);

/* Host-side partition logic of BNFFT_DIST_SLAB (pure functions, no device):
 * bnfft_slab_cuts: cut points cuts[0..nranks] (cuts[0] = 0, cuts[nranks] = L, multiples of `align`)
 *   of L planes; plane_counts == NULL gives equal plane counts, else (K10) the cuts that balance the
 *   cumulative node counts plane_counts[0..L) (each rank >= align planes when L allows).
 * bnfft_slab_owner: rank owning plane c (cuts as above).
 * bnfft_halo_ranges: for rank r, the planes it receives: [lo_from, a_r) from rank r-1 and
 *   [b_r, hi_from) from rank r+1, clipped to [0, L) (lower = m-1 planes, upper = m planes). */
BNFFT_API int bnfft_slab_cuts(const int64_t* plane_counts, int64_t L, int32_t nranks, int32_t align, int64_t* cuts);
BNFFT_API int32_t bnfft_slab_owner(const int64_t* cuts, int32_t nranks, int64_t c);
BNFFT_API int bnfft_halo_ranges(const int64_t* cuts, int32_t nranks, int32_t rank, int32_t m, int64_t L,
                                int64_t* below_lo, int64_t* above_hi);

/* Pipe-throughput microbenchmarks (the FP32 / FP64 / MUFU / shared-memory peaks the
 * gather kernels are measured against).  One full wave of independent dependency chains per
 * pipe; *_per_sm_clk = operations (bytes for LDS) per SM per SM cycle (clock64 inside the CTAs),
 * *_per_s = per second for the whole GPU (CUDA events), *_mhz = the SM clock that implies.
 * ffma: 3-register FFMA, counted in FMAs; ffma2: fma.rn.f32x2, counted in FMAs (2 per lane);
 * dfma: FP64 FMAs; ex2 / rsqrt / rcp: MUFU ops (approx.ftz); lds64 / lds128: bytes of
 * conflict-free 8- / 16-byte shared loads.  Synchronous; takes ~1 s on a B200. */
typedef struct {
  int32_t sms;
  double ffma_per_sm_clk, ffma_per_s, ffma_mhz;
  double ffma2_per_sm_clk, ffma2_per_s, ffma2_mhz;
  double dfma_per_sm_clk, dfma_per_s, dfma_mhz;
  double ex2_per_sm_clk, ex2_per_s, ex2_mhz;
  double rsqrt_per_sm_clk, rsqrt_per_s, rsqrt_mhz;
  double rcp_per_sm_clk, rcp_per_s, rcp_mhz;
  double lds64_per_sm_clk, lds64_per_s, lds64_mhz;
  double lds128_per_sm_clk, lds128_per_s, lds128_mhz;
} bnfft_peaks;
BNFFT_API int bnfft_measure_peaks(int32_t device, bnfft_peaks* out);

BNFFT_API const char* bnfft_status_string(int status);
BNFFT_API const char* bnfft_last_error(void);
/* Library version and the compiled target ("sm_100a"). */
BNFFT_API const char* bnfft_build_info(void);

typedef struct bnfft_plan_s* bnfft_plan;

#ifdef __cplusplus
}
#endif
#endif /* BNFFT_H */
