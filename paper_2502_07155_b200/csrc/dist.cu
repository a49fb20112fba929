// Multi-GPU execution of Algorithm 2 (bnfft_opts.nranks > 1; include/bnfft.h "Multi-GPU modes").
//
// Step 3 is independent per node once theta exists, and theta_l is only read within
// m planes of a node's cell, so ranks partition the grid into slabs of planes and exchange only
// the neighbourhood:
//   * slab geometry: rank r owns planes l_2 (array index, centred) in [cuts[r], cuts[r+1]) of the
//     second dimension, cut points multiples of the gather's bin height (bins stay rank-local),
//     equal plane counts or balanced by the all-reduced per-plane node histogram (K10);
//   * set_nodes: each rank partitions its user-order nodes by owning slab (stable), the counts are
//     all-gathered and the nodes sent to their owners (K9); the owner sorts them as a one-rank plan;
//   * execute: step 1 on the rank's k_1 chunk, 2-D inverse FFTs over (k_2, k_3), an all-to-all that
//     hands every rank all k_1 for its l_2 planes, 1-D inverse FFTs along k_1 into the slab (K11,
//     step 2), the halo planes [a-m+1, a) and [b, b+m) from the neighbours (K7; the
//     global ends stay zero: Psi is not periodic, and the gather's TMA zero-fills
//     out-of-range planes), the gather over the owned nodes, and the outputs' return to the
//     originating rank in its user order.
// Transports: NCCL (ncclSend/ncclRecv in a group, loaded at run time) or an in-process group of
// ranks driven by host threads (cudaMemcpyPeerAsync + events), the test transport on one GPU.
#include <dlfcn.h>
#include <nccl.h>   // types only: libnccl.so.2 is opened at run time

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>

#include "bnfft_internal.h"

namespace bnfft {

// ============================================================================ NCCL at run time
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  bool ok = false;
};

static NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the copy already in the process (torch's), so communicators are shared objects
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define BN_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    BN_SYM(GetUniqueId);
    BN_SYM(CommInitRank);
    BN_SYM(CommDestroy);
    BN_SYM(Send);
    BN_SYM(Recv);
    BN_SYM(GroupStart);
    BN_SYM(GroupEnd);
    BN_SYM(GetErrorString);
    BN_SYM(CommCount);
    BN_SYM(CommUserRank);
#undef BN_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
             api.GroupEnd && api.GetErrorString && api.CommCount && api.CommUserRank;
  });
  return api.ok ? &api : nullptr;
}

static int nccl_fail(ncclResult_t r, const char* what) {
  NcclApi* a = nccl_api();
  set_error(std::string(what) + ": " + (a ? a->GetErrorString(r) : "NCCL not loaded"));
  return BNFFT_E_NCCL;
}

// ============================================================================ transports
struct XOp {
  bool send;
  int peer;
  void* buf;
  size_t bytes;
};

struct Transport {
  int rank = 0, nranks = 1, device = 0;
  virtual ~Transport() {}
  // grouped point-to-point transfers, stream-ordered on s (all ranks call with matching ops)
  virtual int exchange(const std::vector<XOp>& ops, cudaStream_t s) = 0;
  // every rank's `bytes` of host data into all[nranks * bytes] (synchronous)
  virtual int allgather_host(const void* mine, size_t bytes, void* all, cudaStream_t s) = 0;
};

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  void* d_tmp = nullptr;
  size_t tmp_cap = 0;
  ~NcclTransport() override {
    if (d_tmp) cudaFree(d_tmp);
  }
  int exchange(const std::vector<XOp>& ops, cudaStream_t s) override {
    NcclApi* a = nccl_api();
    if (!a) return nccl_fail(ncclSystemError, "NCCL");
    ncclResult_t r = a->GroupStart();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    for (const XOp& op : ops) {
      if (!op.bytes) continue;
      r = op.send ? a->Send(op.buf, op.bytes, ncclUint8, op.peer, comm, s)
                  : a->Recv(op.buf, op.bytes, ncclUint8, op.peer, comm, s);
      if (r != ncclSuccess) {
        a->GroupEnd();
        return nccl_fail(r, op.send ? "ncclSend" : "ncclRecv");
      }
    }
    r = a->GroupEnd();
    return r == ncclSuccess ? BNFFT_OK : nccl_fail(r, "ncclGroupEnd");
  }
  int allgather_host(const void* mine, size_t bytes, void* all, cudaStream_t s) override {
    const size_t tot = bytes * (size_t)nranks;
    if (tot > tmp_cap) {
      if (d_tmp) cudaFree(d_tmp);
      d_tmp = nullptr;
      cudaError_t e = cudaMalloc(&d_tmp, tot);
      if (e != cudaSuccess) return cuda_fail(e, "allgather buffer");
      tmp_cap = tot;
    }
    unsigned char* d = (unsigned char*)d_tmp;
    cudaError_t e = cudaMemcpyAsync(d + rank * bytes, mine, bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "allgather H2D");
    std::vector<XOp> ops;
    for (int q = 0; q < nranks; ++q) {
      if (q == rank) continue;
      ops.push_back({true, q, d + rank * bytes, bytes});
      ops.push_back({false, q, d + q * bytes, bytes});
    }
    int rc = exchange(ops, s);
    if (rc != BNFFT_OK) return rc;
    e = cudaMemcpyAsync(all, d, tot, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? BNFFT_OK : cuda_fail(e, "allgather D2H");
  }
};

}  // namespace bnfft

// In-process group: nranks plans driven by nranks host threads (the test transport).
struct bnfft_group_s {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  uint64_t gen = 0;
  struct Post {
    int src, dst;
    const void* buf;
    size_t bytes;
    int dev;
  };
  std::vector<Post> posts;
  std::vector<cudaEvent_t> ready, done;
  std::vector<unsigned char> mailbox;
  // all n threads arrive; the last one runs `last` (under the lock) before releasing the others
  void barrier(const std::function<void()>& last = nullptr) {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++count == n) {
      if (last) last();
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace bnfft {

struct LocalTransport : Transport {
  bnfft_group_s* g = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  ~LocalTransport() override {
    if (ev_ready) cudaEventDestroy(ev_ready);
    if (ev_done) cudaEventDestroy(ev_done);
  }
  int exchange(const std::vector<XOp>& ops, cudaStream_t s) override {
    int rc = BNFFT_OK;
    cudaError_t e = cudaEventRecord(ev_ready, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "group exchange");
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->ready[rank] = ev_ready;
      g->done[rank] = ev_done;
      for (const XOp& op : ops)
        if (op.send) g->posts.push_back({rank, op.peer, op.buf, op.bytes, device});
    }
    g->barrier();
    // the k-th receive from peer q takes the k-th send q posted to this rank
    std::vector<int> seen(nranks, 0);
    for (const XOp& op : ops) {
      if (op.send) continue;
      int k = seen[op.peer]++, found = -1;
      for (size_t i = 0; i < g->posts.size(); ++i) {
        const auto& ps = g->posts[i];
        if (ps.src == op.peer && ps.dst == rank && k-- == 0) {
          found = (int)i;
          break;
        }
      }
      if (found < 0 || g->posts[found].bytes != op.bytes) {
        set_error("group exchange: unmatched or mis-sized transfer");
        rc = BNFFT_E_NCCL;
        continue;
      }
      if (!op.bytes) continue;
      const auto& ps = g->posts[found];
      e = cudaStreamWaitEvent(s, g->ready[op.peer], 0);
      if (e == cudaSuccess) e = cudaMemcpyPeerAsync(op.buf, device, ps.buf, ps.dev, op.bytes, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "group copy");
    }
    e = cudaEventRecord(ev_done, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "group exchange");
    g->barrier();
    // this rank's send buffers may be reused only after the receivers' copies
    for (const XOp& op : ops)
      if (op.send) cudaStreamWaitEvent(s, g->done[op.peer], 0);
    g->barrier([this] { g->posts.clear(); });
    return rc;
  }
  int allgather_host(const void* mine, size_t bytes, void* all, cudaStream_t) override {
    {
      std::lock_guard<std::mutex> lk(g->mu);
      if (g->mailbox.size() < bytes * (size_t)nranks) g->mailbox.resize(bytes * (size_t)nranks);
      memcpy(g->mailbox.data() + bytes * rank, mine, bytes);
    }
    g->barrier();
    memcpy(all, g->mailbox.data(), bytes * (size_t)nranks);
    g->barrier();
    return BNFFT_OK;
  }
};

// ============================================================================ host partition logic
static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static int slab_cuts(const int64_t* plane_counts, int64_t L, int P, int align, int64_t* cuts) {
  if (P < 1 || L < 1 || align < 1 || !cuts) return BNFFT_E_INVALID_ARG;
  const int64_t nblk = ceil_div(L, align);
  if (nblk < P) return BNFFT_E_UNSUPPORTED;
  cuts[0] = 0;
  if (!plane_counts) {
    for (int q = 1; q < P; ++q) cuts[q] = std::min<int64_t>(L, align * ((q * nblk) / P));
  } else {
    std::vector<int64_t> cum(nblk + 1, 0);
    for (int64_t b = 0; b < nblk; ++b) {
      int64_t s = 0;
      for (int64_t c = b * align; c < std::min<int64_t>(L, (b + 1) * align); ++c) s += plane_counts[c];
      cum[b + 1] = cum[b] + s;
    }
    const int64_t tot = cum[nblk];
    int64_t prev = 0;
    for (int q = 1; q < P; ++q) {
      // the block boundary whose cumulative count is closest to q/P of the total, keeping at least
      // one block per rank on both sides
      const double target = (double)tot * q / P;
      int64_t b = prev + 1;
      while (b < nblk - (P - q) && (double)cum[b] < target) ++b;
      if (b > prev + 1 && target - (double)cum[b - 1] < (double)cum[b] - target) --b;
      b = std::min<int64_t>(std::max<int64_t>(b, prev + 1), nblk - (P - q));
      cuts[q] = std::min<int64_t>(L, b * align);
      prev = b;
    }
  }
  cuts[P] = L;
  return BNFFT_OK;
}

static int slab_owner(const int64_t* cuts, int P, int64_t c) {
  int lo = 0, hi = P - 1;
  while (lo < hi) {   // largest q with cuts[q] <= c
    const int mid = (lo + hi + 1) / 2;
    if (cuts[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ============================================================================ device kernels
constexpr int kPartThreads = 1024;
constexpr int kMaxRanks = 64;

// validate + owner of every user node (slab of its cell's second coordinate) + per-block counts
__global__ void __launch_bounds__(kPartThreads) dist_owner_kernel(const double* __restrict__ x, int64_t n, int d,
                                                                  double Lf, int64_t L, const int64_t* __restrict__ cuts,
                                                                  int P, uint8_t* __restrict__ owner,
                                                                  uint32_t* __restrict__ blkcnt, int64_t nblk,
                                                                  unsigned long long* __restrict__ bad) {
  __shared__ int64_t s_cuts[kMaxRanks + 1];
  __shared__ uint32_t s_cnt[kMaxRanks];
  for (int q = threadIdx.x; q <= P; q += blockDim.x) s_cuts[q] = cuts[q];
  for (int q = threadIdx.x; q < P; q += blockDim.x) s_cnt[q] = 0;
  __syncthreads();
  const int64_t j = blockIdx.x * (int64_t)kPartThreads + threadIdx.x;
  if (j < n) {
    int code = 0;
    for (int t = 0; t < d; ++t) {
      const double v = x[j * d + t];
      if (!isfinite(v)) code = code ? code : 1;
      else if (v < -0.5 || v >= 0.5) code = code ? code : 2;
    }
    int o = 0;
    if (code) {
      atomicMin(bad, ((unsigned long long)j << 4) | (unsigned long long)code);
    } else {
      const double Lx = __dmul_rn(Lf, x[j * d + 1]);   // slab dimension: the second
      int64_t c = (int64_t)floor(Lx) + L / 2;
      c = c > L - 1 ? L - 1 : c;
      int lo = 0, hi = P - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (s_cuts[mid] <= c) lo = mid;
        else hi = mid - 1;
      }
      o = lo;
    }
    owner[j] = (uint8_t)o;
    atomicAdd(&s_cnt[o], 1u);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < P; q += blockDim.x) blkcnt[(int64_t)q * nblk + blockIdx.x] = s_cnt[q];
}

// per-plane histogram of the slab coordinate (BNFFT_BALANCED_SLABS, K10); invalid nodes skipped
__global__ void dist_plane_hist_kernel(const double* __restrict__ x, int64_t n, int d, double Lf, int64_t L,
                                       unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned int s_h[];
  for (int64_t c = threadIdx.x; c < L; c += blockDim.x) s_h[c] = 0;
  __syncthreads();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[j * d + 1];
    if (!(v >= -0.5 && v < 0.5)) continue;
    int64_t c = (int64_t)floor(__dmul_rn(Lf, v)) + L / 2;
    c = c > L - 1 ? L - 1 : c;
    atomicAdd(&s_h[c], 1u);
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < L; c += blockDim.x)
    if (s_h[c]) atomicAdd(&hist[c], (unsigned long long)s_h[c]);
}

// exclusive scan of blkcnt[q][0..nblk) per owner q (one CTA per owner); tot[q] = sum
__global__ void __launch_bounds__(1024) dist_scan_kernel(uint32_t* __restrict__ blkcnt, int64_t nblk,
                                                         int64_t* __restrict__ tot) {
  __shared__ uint32_t s_w[32];
  __shared__ uint64_t s_carry;
  uint32_t* c = blkcnt + (int64_t)blockIdx.x * nblk;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < nblk; b0 += 1024) {
    const int64_t b = b0 + threadIdx.x;
    const uint32_t v = b < nblk ? c[b] : 0u;
    uint32_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    uint32_t wb = 0, all = 0;
    for (int w = 0; w < 32; ++w) {
      wb += w < wid ? s_w[w] : 0u;
      all += s_w[w];
    }
    const uint64_t carry = s_carry;
    if (b < nblk) c[b] = (uint32_t)(carry + wb + incl - v);
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + all;
    __syncthreads();
  }
  if (threadIdx.x == 0) tot[blockIdx.x] = (int64_t)s_carry;
}

// stable scatter of the nodes into per-owner blocks: position = base[o] + block offset + rank of the
// node among the block's owner-o nodes in user order (MATCH.ANY within a warp, warp offsets in smem)
__global__ void __launch_bounds__(kPartThreads) dist_scatter_kernel(const double* __restrict__ x, int64_t n, int d,
                                                                    const uint8_t* __restrict__ owner, int P,
                                                                    const uint32_t* __restrict__ blkoff, int64_t nblk,
                                                                    const int64_t* __restrict__ base,
                                                                    double* __restrict__ xs,
                                                                    uint32_t* __restrict__ sendperm) {
  __shared__ uint32_t s_wc[32][kMaxRanks];
  __shared__ int64_t s_base[kMaxRanks];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 32 * kMaxRanks; i += blockDim.x) (&s_wc[0][0])[i] = 0;
  for (int q = threadIdx.x; q < P; q += blockDim.x) s_base[q] = base[q] + blkoff[(int64_t)q * nblk + blockIdx.x];
  __syncthreads();
  const int64_t j = blockIdx.x * (int64_t)kPartThreads + threadIdx.x;
  const bool act = j < n;
  const int o = act ? (int)owner[j] : kMaxRanks + 1;
  const unsigned peers = __match_any_sync(0xffffffffu, o);
  const int rk = __popc(peers & ((1u << lane) - 1u));
  if (act && rk == 0) s_wc[wid][o] = __popc(peers);
  __syncthreads();
  if (act) {
    uint32_t wo = 0;
    for (int w = 0; w < wid; ++w) wo += s_wc[w][o];
    const int64_t pos = s_base[o] + wo + rk;
    for (int t = 0; t < d; ++t) xs[pos * d + t] = x[j * d + t];
    sendperm[pos] = (uint32_t)j;
  }
}

// f[sendperm[pos]] = fret[pos] (outputs back in user order)
template <typename C>
__global__ void dist_unpermute_kernel(const C* __restrict__ fret, const uint32_t* __restrict__ sendperm, int64_t n,
                                      C* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[sendperm[i]] = fret[i];
}

// ============================================================================ plan state
struct DistState {
  Transport* tr = nullptr;
  int mode = BNFFT_DIST_REPLICATE;
  int P = 1, r = 0;
  int align = 8;
  std::vector<int64_t> cuts, kcut;
  int64_t* d_cuts = nullptr;
  // node exchange
  int64_t n_user = 0, n_owned = 0;
  int64_t owner_cap = 0, sendperm_cap = 0, xsend_cap = 0, owned_cap = 0, fown_cap = 0, fret_cap = 0;
  std::vector<int64_t> send_cnt, recv_cnt;
  uint8_t* d_owner = nullptr;
  uint32_t* d_sendperm = nullptr;
  double* d_xsend = nullptr;
  double* d_xrecv = nullptr;
  uint32_t* d_blkcnt = nullptr;
  int64_t blk_cap = 0, hist_cap = 0;
  int64_t* d_tot = nullptr;      // P totals + P bases
  unsigned long long* d_hist = nullptr;
  void* d_fown = nullptr;
  void* d_fret = nullptr;
  // distributed FFT
  int64_t nk = 0;                // this rank's k_1 chunk size
  void *d_ain = nullptr, *d_aout = nullptr, *d_sb = nullptr, *d_b = nullptr;
  void *d_hsend = nullptr, *d_hrecv = nullptr;
  int64_t b_ny = -1;             // slab width the 1-D FFT plan / B buffer are built for
  cufftHandle fft2 = 0, fft1 = 0;
  bool fft2_ok = false, fft1_ok = false;
  int64_t halo_bytes = 0;
};

static int64_t slab_w(const DistState* ds, int q) { return ds->cuts[q + 1] - ds->cuts[q]; }

// the 1-D FFT plan along k_1 and its input B for the current slab width
static int ensure_slab_fft(bnfft_plan_s* p) {
  DistState* ds = p->dist;
  const int64_t ny = slab_w(ds, ds->r);
  for (int q = 0; q < ds->P; ++q)
    if (slab_w(ds, q) < p->opts.m) {
      set_error("BNFFT_DIST_SLAB: a slab narrower than m planes (halo from one neighbour only)");
      return BNFFT_E_UNSUPPORTED;
    }
  if (ny == ds->b_ny) return BNFFT_OK;
  const int64_t L = p->L;
  if (ds->d_b) dfree_plan(p, ds->d_b);
  ds->d_b = nullptr;
  const size_t bb = (size_t)(L * ny * L) * p->csize;
  cudaError_t e = dmalloc_bytes(p, &ds->d_b, bb);
  if (e != cudaSuccess) return cuda_fail(e, "alloc slab FFT input");
  e = cudaMemsetAsync(ds->d_b, 0, bb, p->stream);   // planes k_1 outside I_M stay zero
  if (e != cudaSuccess) return cuda_fail(e, "zero slab FFT input");
  if (ds->fft1_ok) cufftDestroy(ds->fft1);
  ds->fft1_ok = false;
  int n1[1] = {(int)L};
  int inem[1] = {(int)L}, onem[1] = {(int)L};
  size_t ws = 0;
  cufftResult fr = cufftCreate(&ds->fft1);
  if (fr == CUFFT_SUCCESS) {
    ds->fft1_ok = true;
    fr = cufftMakePlanMany(ds->fft1, 1, n1, inem, (int)(ny * L), 1, onem, (int)(L * L), 1,
                           p->c128 ? CUFFT_Z2Z : CUFFT_C2C, (int)(ny * L), &ws);
  }
  if (fr == CUFFT_SUCCESS) fr = cufftSetStream(ds->fft1, p->stream);
  if (fr != CUFFT_SUCCESS) {
    set_error("cuFFT slab plan (1-D along k_1) failed");
    return BNFFT_E_CUFFT;
  }
  ds->b_ny = ny;
  return BNFFT_OK;
}

int dist_create(bnfft_plan_s* p) {
  const bnfft_opts& o = p->opts;
  if (o.nranks <= 1) return BNFFT_OK;
  if (o.rank < 0 || o.rank >= o.nranks || o.nranks > kMaxRanks) {
    set_error("rank / nranks");
    return BNFFT_E_INVALID_ARG;
  }
  if ((o.nccl_comm != nullptr) == (o.local_group != nullptr)) {
    set_error("nranks > 1 needs exactly one of nccl_comm and local_group");
    return BNFFT_E_INVALID_ARG;
  }
  if (o.dist != BNFFT_DIST_REPLICATE && o.dist != BNFFT_DIST_SLAB) {
    set_error("unknown dist mode");
    return BNFFT_E_INVALID_ARG;
  }
  if (o.dist == BNFFT_DIST_SLAB && (o.d != 3 || o.batch != 1 || (o.flags & (BNFFT_ALG1 | BNFFT_SORTED_OUTPUT)))) {
    set_error("BNFFT_DIST_SLAB is built for d = 3, batch 1, Algorithm 2, user-order output");
    return BNFFT_E_UNSUPPORTED;
  }
  DistState* ds = new DistState();
  p->dist = ds;
  ds->mode = o.dist;
  ds->P = o.nranks;
  ds->r = o.rank;
  if (o.nccl_comm) {
    NcclApi* a = nccl_api();
    if (!a) {
      set_error("libnccl.so.2 could not be loaded");
      return BNFFT_E_NCCL;
    }
    int cnt = 0, rk = 0;
    ncclResult_t r = a->CommCount((ncclComm_t)o.nccl_comm, &cnt);
    if (r == ncclSuccess) r = a->CommUserRank((ncclComm_t)o.nccl_comm, &rk);
    if (r != ncclSuccess) return nccl_fail(r, "NCCL communicator");
    if (cnt != o.nranks || rk != o.rank) {
      set_error("NCCL communicator size / rank differ from nranks / rank");
      return BNFFT_E_INVALID_ARG;
    }
    NcclTransport* t = new NcclTransport();
    t->comm = (ncclComm_t)o.nccl_comm;
    ds->tr = t;
  } else {
    bnfft_group_s* g = (bnfft_group_s*)o.local_group;
    if (g->n != o.nranks) {
      set_error("local group size differs from nranks");
      return BNFFT_E_INVALID_ARG;
    }
    LocalTransport* t = new LocalTransport();
    t->g = g;
    cudaEventCreateWithFlags(&t->ev_ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&t->ev_done, cudaEventDisableTiming);
    ds->tr = t;
  }
  ds->tr->rank = o.rank;
  ds->tr->nranks = o.nranks;
  ds->tr->device = p->device;
  if (ds->mode == BNFFT_DIST_REPLICATE) return BNFFT_OK;

  // ---- slab geometry and the distributed FFT's buffers
  const int64_t L = p->L, M = o.M;
  ds->align = 1 << p->bin_log2[1];
  ds->cuts.assign(ds->P + 1, 0);
  int rc = slab_cuts(nullptr, L, ds->P, ds->align, ds->cuts.data());
  if (rc != BNFFT_OK) {
    set_error("BNFFT_DIST_SLAB: fewer bin rows than ranks");
    return rc;
  }
  if (M < ds->P) {
    set_error("BNFFT_DIST_SLAB: M < nranks");
    return BNFFT_E_UNSUPPORTED;
  }
  ds->kcut.assign(ds->P + 1, 0);
  for (int q = 0; q <= ds->P; ++q) ds->kcut[q] = -M / 2 + (q * M) / ds->P;
  ds->nk = ds->kcut[ds->r + 1] - ds->kcut[ds->r];
  cudaError_t e;
  const size_t abytes = (size_t)(ds->nk * L * L) * p->csize;
  if ((e = dmalloc_bytes(p, &ds->d_ain, abytes)) != cudaSuccess ||
      (e = dmalloc_bytes(p, &ds->d_aout, abytes)) != cudaSuccess ||
      (e = dmalloc_bytes(p, &ds->d_sb, abytes)) != cudaSuccess ||
      (e = dmalloc_bytes(p, (void**)&ds->d_cuts, (ds->P + 1) * sizeof(int64_t))) != cudaSuccess ||
      (e = dmalloc_bytes(p, (void**)&ds->d_tot, 2 * ds->P * sizeof(int64_t))) != cudaSuccess)
    return cuda_fail(e, "alloc slab buffers");
  const size_t hb = (size_t)(2 * o.m * L * L) * p->csize;
  if ((e = dmalloc_bytes(p, &ds->d_hsend, hb)) != cudaSuccess || (e = dmalloc_bytes(p, &ds->d_hrecv, hb)) != cudaSuccess)
    return cuda_fail(e, "alloc halo buffers");
  if ((e = cudaMemsetAsync(ds->d_ain, 0, abytes, p->stream)) != cudaSuccess) return cuda_fail(e, "zero slab input");
  {
    int n2[2] = {(int)L, (int)L};
    size_t ws = 0;
    cufftResult fr = cufftCreate(&ds->fft2);
    if (fr == CUFFT_SUCCESS) {
      ds->fft2_ok = true;
      fr = cufftMakePlanMany(ds->fft2, 2, n2, nullptr, 1, (int)(L * L), nullptr, 1, (int)(L * L),
                             p->c128 ? CUFFT_Z2Z : CUFFT_C2C, (int)ds->nk, &ws);
    }
    if (fr == CUFFT_SUCCESS) fr = cufftSetStream(ds->fft2, p->stream);
    if (fr != CUFFT_SUCCESS) {
      set_error("cuFFT slab plan (2-D over k_2, k_3) failed");
      return BNFFT_E_CUFFT;
    }
  }
  return ensure_slab_fft(p);
}

void dist_destroy(bnfft_plan_s* p) {
  DistState* ds = p->dist;
  if (!ds) return;
  if (ds->fft2_ok) cufftDestroy(ds->fft2);
  if (ds->fft1_ok) cufftDestroy(ds->fft1);
  for (void* ptr : {(void*)ds->d_cuts, (void*)ds->d_owner, (void*)ds->d_sendperm, (void*)ds->d_xsend,
                    (void*)ds->d_xrecv, (void*)ds->d_blkcnt, (void*)ds->d_tot, (void*)ds->d_hist, ds->d_fown,
                    ds->d_fret, ds->d_ain, ds->d_aout, ds->d_sb, ds->d_b, ds->d_hsend, ds->d_hrecv})
    if (ptr) dfree_plan(p, ptr);
  delete ds->tr;
  delete ds;
  p->dist = nullptr;
}

static int grow(bnfft_plan_s* p, void** ptr, int64_t* cap, int64_t need, size_t elem, const char* what) {
  if (need <= *cap && *ptr) return BNFFT_OK;
  if (*ptr) dfree_plan(p, *ptr);
  *ptr = nullptr;
  const int64_t c = std::max<int64_t>(need, 1);
  cudaError_t e = dmalloc_bytes(p, ptr, (size_t)c * elem);
  if (e != cudaSuccess) return cuda_fail(e, what);
  *cap = c;
  return BNFFT_OK;
}

int dist_set_nodes(bnfft_plan_s* p, int64_t n, const double* x, int64_t* first_bad) {
  DistState* ds = p->dist;
  if (ds->mode == BNFFT_DIST_REPLICATE) return local_set_nodes(p, n, x, first_bad);
  const int P = ds->P, d = p->opts.d;
  const int64_t L = p->L;
  cudaStream_t s = p->stream;
  cudaError_t e;
  int rc;
  cudaEvent_t ev;
  timer_begin(p, ST_EXCH, &ev);
  // ---- cut points: equal planes, or balanced by the all-reduced plane histogram (K10)
  if (p->opts.flags & BNFFT_BALANCED_SLABS) {
    if ((rc = grow(p, (void**)&ds->d_hist, &ds->hist_cap, L, sizeof(unsigned long long), "alloc histogram")) != BNFFT_OK)
      return rc;
    if ((e = cudaMemsetAsync(ds->d_hist, 0, L * sizeof(unsigned long long), s)) != cudaSuccess)
      return cuda_fail(e, "zero histogram");
    if (n > 0) {
      dist_plane_hist_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), (int64_t)sm_count() * 8), 256, L * sizeof(unsigned), s>>>(
          x, n, d, (double)L, L, ds->d_hist);
      p->launches++;
    }
    std::vector<int64_t> h(L), all((size_t)L * P), tot(L, 0);
    if ((e = cudaMemcpyAsync(h.data(), ds->d_hist, L * sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
      return cuda_fail(e, "histogram");
    if ((rc = ds->tr->allgather_host(h.data(), L * sizeof(int64_t), all.data(), s)) != BNFFT_OK) return rc;
    for (int q = 0; q < P; ++q)
      for (int64_t c = 0; c < L; ++c) tot[c] += all[(size_t)q * L + c];
    std::vector<int64_t> cuts(P + 1);
    if ((rc = slab_cuts(tot.data(), L, P, ds->align, cuts.data())) != BNFFT_OK) return rc;
    ds->cuts = cuts;
    if ((rc = ensure_slab_fft(p)) != BNFFT_OK) return rc;
  }
  if ((e = cudaMemcpyAsync(ds->d_cuts, ds->cuts.data(), (P + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return cuda_fail(e, "copy cuts");
  // ---- validate + owners + stable partition by owner (K9)
  if ((rc = grow(p, (void**)&ds->d_owner, &ds->owner_cap, n, 1, "alloc owners")) != BNFFT_OK ||
      (rc = grow(p, (void**)&ds->d_sendperm, &ds->sendperm_cap, n, 4, "alloc node send order")) != BNFFT_OK ||
      (rc = grow(p, (void**)&ds->d_xsend, &ds->xsend_cap, n, (size_t)d * 8, "alloc node send buffer")) != BNFFT_OK ||
      (rc = grow(p, &ds->d_fret, &ds->fret_cap, n, p->csize, "alloc returned outputs")) != BNFFT_OK)
    return rc;
  const int64_t nblk = std::max<int64_t>(1, ceil_div(n, kPartThreads));
  if ((rc = grow(p, (void**)&ds->d_blkcnt, &ds->blk_cap, nblk * P, 4, "alloc block counts")) != BNFFT_OK) return rc;
  unsigned long long none = ~0ull;
  if ((e = cudaMemcpyAsync(p->d_bad, &none, sizeof(none), cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "status init");
  if ((e = cudaMemsetAsync(ds->d_blkcnt, 0, (size_t)nblk * P * 4, s)) != cudaSuccess) return cuda_fail(e, "zero counts");
  if (n > 0) {
    dist_owner_kernel<<<(unsigned)nblk, kPartThreads, 0, s>>>(x, n, d, (double)L, L, ds->d_cuts, P, ds->d_owner,
                                                             ds->d_blkcnt, nblk, p->d_bad);
    p->launches++;
  }
  dist_scan_kernel<<<P, 1024, 0, s>>>(ds->d_blkcnt, nblk, ds->d_tot);
  p->launches++;
  std::vector<int64_t> tot(2 * P, 0);
  unsigned long long bad = 0;
  if ((e = cudaMemcpyAsync(tot.data(), ds->d_tot, P * sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(&bad, p->d_bad, sizeof(bad), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(e, "partition counts");
  {
    int64_t acc = 0;
    for (int q = 0; q < P; ++q) {
      tot[P + q] = acc;
      acc += tot[q];
    }
  }
  // ---- counts (and every rank's validation status) to all ranks
  std::vector<int64_t> mine(P + 1), all((size_t)(P + 1) * P);
  for (int q = 0; q < P; ++q) mine[q] = tot[q];
  mine[P] = (int64_t)(bad == ~0ull ? -1 : (int64_t)bad);
  if ((rc = ds->tr->allgather_host(mine.data(), (P + 1) * sizeof(int64_t), all.data(), s)) != BNFFT_OK) return rc;
  int64_t worst = -1;
  for (int q = 0; q < P; ++q) {
    const int64_t bq = all[(size_t)q * (P + 1) + P];
    if (bq >= 0 && worst < 0) worst = bq;
  }
  if (worst >= 0) {   // every rank fails together (no rank enters the node exchange)
    p->n = 0;
    p->nodes_set = false;
    const int64_t own = mine[P];
    const int code = (int)((own >= 0 ? own : worst) & 15);
    if (own >= 0 && first_bad) *first_bad = own >> 4;
    set_error(own >= 0 ? "node rejected" : "a node of another rank was rejected");
    return code == 1 ? BNFFT_E_NODE_NOT_FINITE : BNFFT_E_NODE_OUT_OF_RANGE;
  }
  if ((e = cudaMemcpyAsync(ds->d_tot + P, tot.data() + P, P * sizeof(int64_t), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return cuda_fail(e, "partition bases");
  if (n > 0) {
    dist_scatter_kernel<<<(unsigned)nblk, kPartThreads, 0, s>>>(x, n, d, ds->d_owner, P, ds->d_blkcnt, nblk,
                                                               ds->d_tot + P, ds->d_xsend, ds->d_sendperm);
    p->launches++;
  }
  ds->send_cnt.assign(tot.begin(), tot.begin() + P);
  ds->recv_cnt.assign(P, 0);
  int64_t n_owned = 0;
  for (int q = 0; q < P; ++q) {
    ds->recv_cnt[q] = all[(size_t)q * (P + 1) + ds->r];
    n_owned += ds->recv_cnt[q];
  }
  if (n_owned >= ((int64_t)1 << 31)) {
    set_error("owned node count >= 2^31");
    return BNFFT_E_INVALID_ARG;
  }
  // ---- nodes to their owners
  if ((rc = grow(p, (void**)&ds->d_xrecv, &ds->owned_cap, n_owned, (size_t)d * 8, "alloc node receive buffer")) !=
      BNFFT_OK)
    return rc;
  if ((rc = grow(p, &ds->d_fown, &ds->fown_cap, n_owned, p->csize, "alloc owned outputs")) != BNFFT_OK) return rc;
  std::vector<XOp> ops;
  int64_t so = 0, ro = 0;
  for (int q = 0; q < P; ++q) {
    const size_t sb = (size_t)ds->send_cnt[q] * d * 8, rb = (size_t)ds->recv_cnt[q] * d * 8;
    if (q == ds->r) {
      if (sb && (e = cudaMemcpyAsync(ds->d_xrecv + ro * d, ds->d_xsend + so * d, sb, cudaMemcpyDeviceToDevice, s)) !=
                    cudaSuccess)
        return cuda_fail(e, "local node copy");
    } else {
      ops.push_back({true, q, ds->d_xsend + so * d, sb});
      ops.push_back({false, q, ds->d_xrecv + ro * d, rb});
    }
    so += ds->send_cnt[q];
    ro += ds->recv_cnt[q];
  }
  if ((rc = ds->tr->exchange(ops, s)) != BNFFT_OK) return rc;
  timer_end(p, ST_EXCH, ev);
  ds->n_user = n;
  ds->n_owned = n_owned;
  // ---- the owned nodes form this rank's one-rank problem (their order = receive order)
  int64_t fb = -1;
  rc = local_set_nodes(p, n_owned, ds->d_xrecv, &fb);
  if (rc != BNFFT_OK) return rc;
  return BNFFT_OK;
}

int dist_execute(bnfft_plan_s* p, const void* fhat, void* f) {
  DistState* ds = p->dist;
  const int P = ds->P, r = ds->r, m = p->opts.m;
  const int64_t L = p->L, cs = (int64_t)p->csize;
  cudaStream_t s = p->stream;
  cudaError_t e;
  int rc;
  cudaEvent_t ev;
  unsigned char* grid = (unsigned char*)p->d_grid;
  // ---- step 1 on this rank's k_1 chunk; 2-D inverse FFTs over (k_2, k_3)
  timer_begin(p, ST_DECONV, &ev);
  if ((e = launch_deconv_slab(p, fhat, ds->d_ain, ds->kcut[r], ds->kcut[r + 1])) != cudaSuccess)
    return cuda_fail(e, "slab deconv");
  timer_end(p, ST_DECONV, ev);
  timer_begin(p, ST_FFT, &ev);
  cufftResult fr = p->c128 ? cufftExecZ2Z(ds->fft2, (cufftDoubleComplex*)ds->d_ain, (cufftDoubleComplex*)ds->d_aout,
                                          CUFFT_INVERSE)
                           : cufftExecC2C(ds->fft2, (cufftComplex*)ds->d_ain, (cufftComplex*)ds->d_aout, CUFFT_INVERSE);
  if (fr != CUFFT_SUCCESS) {
    set_error("cufftExec (slab 2-D)");
    return BNFFT_E_CUFFT;
  }
  timer_end(p, ST_FFT, ev);
  // ---- all-to-all: rank q receives planes l_2 in its slab of every rank's k_1 chunk
  timer_begin(p, ST_EXCH, &ev);
  const int64_t nk = ds->nk;
  unsigned char* sb = (unsigned char*)ds->d_sb;
  unsigned char* B = (unsigned char*)ds->d_b;
  const int64_t nyr = slab_w(ds, r);
  std::vector<int64_t> sboff(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    const int64_t nyq = slab_w(ds, q);
    sboff[q + 1] = sboff[q] + nk * nyq * L;
    if (nyq == 0 || nk == 0) continue;
    e = cudaMemcpy2DAsync(sb + sboff[q] * cs, (size_t)(nyq * L * cs), (unsigned char*)ds->d_aout + ds->cuts[q] * L * cs,
                          (size_t)(L * L * cs), (size_t)(nyq * L * cs), (size_t)nk, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "pack slab planes");
  }
  // chunk q's k_1 values split at 0: [kcut[q], min(0, kcut[q+1])) -> planes k_1 + L, the rest -> k_1
  auto parts = [&](int q, int64_t* k_a, int64_t* n_a, int64_t* k_b, int64_t* n_b) {
    const int64_t a = ds->kcut[q], b = ds->kcut[q + 1];
    *n_a = std::max<int64_t>(0, std::min<int64_t>(b, 0) - a);
    *k_a = a + L;
    *n_b = (b - a) - *n_a;
    *k_b = a + *n_a;
  };
  std::vector<XOp> ops;
  for (int q = 0; q < P; ++q) {
    // send: my chunk's planes for rank q's slab, in the two parts of MY chunk
    int64_t ka, na, kb, nb;
    parts(r, &ka, &na, &kb, &nb);
    const int64_t nyq = slab_w(ds, q);
    const size_t pa = (size_t)(na * nyq * L * cs), pb = (size_t)(nb * nyq * L * cs);
    unsigned char* src = sb + sboff[q] * cs;
    // receive: rank q's chunk planes of my slab into B (two parts of ITS chunk)
    int64_t qka, qna, qkb, qnb;
    parts(q, &qka, &qna, &qkb, &qnb);
    unsigned char* dA = B + qka * nyr * L * cs;
    unsigned char* dB = B + qkb * nyr * L * cs;
    const size_t ra = (size_t)(qna * nyr * L * cs), rb = (size_t)(qnb * nyr * L * cs);
    if (q == r) {
      if (pa && (e = cudaMemcpyAsync(dA, src, pa, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "local slab copy");
      if (pb && (e = cudaMemcpyAsync(dB, src + pa, pb, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "local slab copy");
      continue;
    }
    ops.push_back({true, q, src, pa});
    ops.push_back({true, q, src + pa, pb});
    ops.push_back({false, q, dA, ra});
    ops.push_back({false, q, dB, rb});
  }
  if ((rc = ds->tr->exchange(ops, s)) != BNFFT_OK) return rc;
  timer_end(p, ST_EXCH, ev);
  // ---- 1-D inverse FFTs along k_1 into the slab of the (globally indexed) grid
  timer_begin(p, ST_FFT, &ev);
  if (nyr > 0) {
    unsigned char* gout = grid + ds->cuts[r] * L * cs;
    fr = p->c128 ? cufftExecZ2Z(ds->fft1, (cufftDoubleComplex*)ds->d_b, (cufftDoubleComplex*)gout, CUFFT_INVERSE)
                 : cufftExecC2C(ds->fft1, (cufftComplex*)ds->d_b, (cufftComplex*)gout, CUFFT_INVERSE);
    if (fr != CUFFT_SUCCESS) {
      set_error("cufftExec (slab 1-D)");
      return BNFFT_E_CUFFT;
    }
  }
  timer_end(p, ST_FFT, ev);
  // ---- halo planes (K7): [a - m + 1, a) from rank r-1, [b, b + m) from rank r+1
  timer_begin(p, ST_EXCH, &ev);
  {
    const int64_t a = ds->cuts[r], b = ds->cuts[r + 1];
    const size_t row = (size_t)(L * cs), pitch = (size_t)(L * L * cs);
    unsigned char* hs = (unsigned char*)ds->d_hsend;
    unsigned char* hr = (unsigned char*)ds->d_hrecv;
    const size_t lo_bytes = (size_t)(m - 1) * row * L, hi_bytes = (size_t)m * row * L;
    std::vector<XOp> hops;
    // to r-1: my planes [a, a + m) (its upper halo); to r+1: [b - m + 1, b) (its lower halo)
    if (r > 0) {
      if ((e = cudaMemcpy2DAsync(hs, m * row, grid + a * row, pitch, m * row, L, cudaMemcpyDeviceToDevice, s)) !=
          cudaSuccess)
        return cuda_fail(e, "pack halo");
      hops.push_back({true, r - 1, hs, hi_bytes});
      hops.push_back({false, r - 1, hr, lo_bytes});
    }
    if (r < P - 1) {
      if (m > 1 && (e = cudaMemcpy2DAsync(hs + hi_bytes, (m - 1) * row, grid + (b - (m - 1)) * row, pitch, (m - 1) * row,
                                          L, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "pack halo");
      hops.push_back({true, r + 1, hs + hi_bytes, lo_bytes});
      hops.push_back({false, r + 1, hr + lo_bytes, hi_bytes});
    }
    if ((rc = ds->tr->exchange(hops, s)) != BNFFT_OK) return rc;
    if (r > 0 && m > 1 &&
        (e = cudaMemcpy2DAsync(grid + (a - (m - 1)) * row, pitch, hr, (m - 1) * row, (m - 1) * row, L,
                               cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "unpack halo");
    if (r < P - 1 && (e = cudaMemcpy2DAsync(grid + b * row, pitch, hr + lo_bytes, m * row, m * row, L,
                                            cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "unpack halo");
    ds->halo_bytes = (int64_t)((r > 0 ? lo_bytes : 0) + (r < P - 1 ? hi_bytes : 0));
  }
  timer_end(p, ST_EXCH, ev);
  // ---- step 3 on the owned nodes
  timer_begin(p, ST_GATHER, &ev);
  if ((e = launch_gather(p, ds->d_fown)) != cudaSuccess) return cuda_fail(e, "gather kernel");
  timer_end(p, ST_GATHER, ev);
  // ---- values back to the originating ranks, then into user order
  timer_begin(p, ST_EXCH, &ev);
  {
    std::vector<XOp> rops;
    int64_t ro = 0, so = 0;
    unsigned char* fo = (unsigned char*)ds->d_fown;
    unsigned char* fr2 = (unsigned char*)ds->d_fret;
    for (int q = 0; q < P; ++q) {
      const size_t back = (size_t)(ds->recv_cnt[q] * cs), mineb = (size_t)(ds->send_cnt[q] * cs);
      if (q == r) {
        if (back && (e = cudaMemcpyAsync(fr2 + so * cs, fo + ro * cs, back, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
          return cuda_fail(e, "local output copy");
      } else {
        rops.push_back({true, q, fo + ro * cs, back});
        rops.push_back({false, q, fr2 + so * cs, mineb});
      }
      ro += ds->recv_cnt[q];
      so += ds->send_cnt[q];
    }
    if ((rc = ds->tr->exchange(rops, s)) != BNFFT_OK) return rc;
    if (ds->n_user > 0) {
      const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(ds->n_user, 256), (int64_t)sm_count() * 16);
      if (p->c128)
        dist_unpermute_kernel<double2><<<blocks, 256, 0, s>>>((const double2*)ds->d_fret, ds->d_sendperm, ds->n_user,
                                                              (double2*)f);
      else
        dist_unpermute_kernel<float2><<<blocks, 256, 0, s>>>((const float2*)ds->d_fret, ds->d_sendperm, ds->n_user,
                                                             (float2*)f);
      p->launches++;
      if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "unpermute kernel");
    }
  }
  timer_end(p, ST_EXCH, ev);
  p->n_exec++;
  return BNFFT_OK;
}

void dist_fill_info(const bnfft_plan_s* p, bnfft_info* o) {
  o->rank = p->opts.nranks > 1 ? p->opts.rank : 0;
  o->nranks = std::max(1, p->opts.nranks);
  o->dist = p->opts.nranks > 1 ? p->opts.dist : BNFFT_DIST_REPLICATE;
  const DistState* ds = p->dist;
  if (ds && ds->mode == BNFFT_DIST_SLAB) {
    o->slab_lo = ds->cuts[ds->r];
    o->slab_hi = ds->cuts[ds->r + 1];
    o->n_owned = ds->n_owned;
    o->halo_bytes = ds->halo_bytes;
  } else {
    o->slab_lo = 0;
    o->slab_hi = p->L;
    o->n_owned = p->nodes_set ? p->n : 0;
    o->halo_bytes = 0;
  }
}

}  // namespace bnfft

using namespace bnfft;

extern "C" {

int bnfft_nccl_unique_id(void* out128) {
  if (!out128) return BNFFT_E_INVALID_ARG;
  NcclApi* a = nccl_api();
  if (!a) {
    set_error("libnccl.so.2 could not be loaded");
    return BNFFT_E_NCCL;
  }
  ncclUniqueId id;
  ncclResult_t r = a->GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
  return BNFFT_OK;
}

int bnfft_nccl_comm_init(const void* id128, int32_t nranks, int32_t rank, int32_t device, void** comm_out) {
  if (!id128 || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return BNFFT_E_INVALID_ARG;
  *comm_out = nullptr;
  NcclApi* a = nccl_api();
  if (!a) {
    set_error("libnccl.so.2 could not be loaded");
    return BNFFT_E_NCCL;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  ncclResult_t r = a->CommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm_out = c;
  return BNFFT_OK;
}

int bnfft_nccl_comm_destroy(void* comm) {
  if (!comm) return BNFFT_OK;
  NcclApi* a = nccl_api();
  if (!a) return BNFFT_E_NCCL;
  ncclResult_t r = a->CommDestroy((ncclComm_t)comm);
  return r == ncclSuccess ? BNFFT_OK : nccl_fail(r, "ncclCommDestroy");
}

// Collective self-test of the NCCL transport (header: bnfft_nccl_selftest): the library's own exchange and
// all-gather code over `comm`, every rank sending `bytes` bytes to every rank (itself included).
int bnfft_nccl_selftest(void* comm, int64_t bytes, void* stream) {
  if (!comm || bytes < 1 || bytes > ((int64_t)1 << 30)) return BNFFT_E_INVALID_ARG;
  NcclApi* a = nccl_api();
  if (!a) {
    set_error("libnccl.so.2 could not be loaded");
    return BNFFT_E_NCCL;
  }
  NcclTransport t;
  t.comm = (ncclComm_t)comm;
  ncclResult_t r = a->CommCount(t.comm, &t.nranks);
  if (r == ncclSuccess) r = a->CommUserRank(t.comm, &t.rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommCount");
  cudaGetDevice(&t.device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nb = (size_t)bytes, P = (size_t)t.nranks;
  unsigned char *d_src = nullptr, *d_dst = nullptr;
  cudaError_t e = cudaMalloc((void**)&d_src, nb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&d_dst, nb * P);
  std::vector<unsigned char> h(nb), back(nb * P);
  for (size_t i = 0; i < nb; ++i) h[i] = (unsigned char)(t.rank * 37 + i * 11 + (i >> 8));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_src, h.data(), nb, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_dst, 0xee, nb * P, s);
  int rc = e == cudaSuccess ? BNFFT_OK : cuda_fail(e, "selftest buffers");
  if (rc == BNFFT_OK) {
    std::vector<XOp> ops;
    for (int q = 0; q < t.nranks; ++q) {
      ops.push_back({true, q, d_src, nb});
      ops.push_back({false, q, d_dst + (size_t)q * nb, nb});
    }
    rc = t.exchange(ops, s);
  }
  if (rc == BNFFT_OK) {
    e = cudaMemcpyAsync(back.data(), d_dst, nb * P, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "selftest copy");
  }
  if (rc == BNFFT_OK) {
    for (size_t q = 0; q < P && rc == BNFFT_OK; ++q)
      for (size_t i = 0; i < nb; ++i)
        if (back[q * nb + i] != (unsigned char)(q * 37 + i * 11 + (i >> 8))) {
          set_error("NCCL self-test: wrong byte received from rank " + std::to_string(q));
          rc = BNFFT_E_NCCL;
          break;
        }
  }
  if (rc == BNFFT_OK) {   // the host all-gather used for counts and cut points
    int64_t mine[2] = {t.rank, bytes + t.rank}, all[2 * kMaxRanks];
    rc = t.allgather_host(mine, sizeof(mine), all, s);
    for (int q = 0; q < t.nranks && rc == BNFFT_OK; ++q)
      if (all[2 * q] != q || all[2 * q + 1] != bytes + q) {
        set_error("NCCL self-test: wrong all-gather entry");
        rc = BNFFT_E_NCCL;
      }
  }
  cudaFree(d_src);
  cudaFree(d_dst);
  return rc;
}

int bnfft_group_create(int32_t nranks, void** group_out) {
  if (!group_out || nranks < 1 || nranks > kMaxRanks) return BNFFT_E_INVALID_ARG;
  bnfft_group_s* g = new bnfft_group_s();
  g->n = nranks;
  g->ready.assign(nranks, nullptr);
  g->done.assign(nranks, nullptr);
  *group_out = g;
  return BNFFT_OK;
}

int bnfft_group_destroy(void* group) {
  delete (bnfft_group_s*)group;
  return BNFFT_OK;
}

int bnfft_slab_cuts(const int64_t* plane_counts, int64_t L, int32_t nranks, int32_t align, int64_t* cuts) {
  if (nranks > kMaxRanks) return BNFFT_E_INVALID_ARG;
  return slab_cuts(plane_counts, L, nranks, align, cuts);
}

int32_t bnfft_slab_owner(const int64_t* cuts, int32_t nranks, int64_t c) {
  if (!cuts || nranks < 1) return -1;
  return slab_owner(cuts, nranks, c);
}

int bnfft_halo_ranges(const int64_t* cuts, int32_t nranks, int32_t rank, int32_t m, int64_t L, int64_t* below_lo,
                      int64_t* above_hi) {
  if (!cuts || !below_lo || !above_hi || rank < 0 || rank >= nranks || m < 1) return BNFFT_E_INVALID_ARG;
  *below_lo = std::max<int64_t>(0, cuts[rank] - (m - 1));
  *above_hi = std::min<int64_t>(L, cuts[rank + 1] + m);
  return BNFFT_OK;
}

}  // extern "C"
