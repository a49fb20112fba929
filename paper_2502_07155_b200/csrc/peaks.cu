// Throughput microbenchmarks of the SM pipes the gather kernels are bound by (SURVEY §8(d)
// "Microbenchmark FP32/FP64 FMA, XU and LDS peaks once per box"): FFMA (3-register form),
// FFMA2 (fma.rn.f32x2), DFMA, MUFU ex2 / rsqrt / rcp and conflict-free LDS.64 / LDS.128.
//
// Each kernel runs one full wave (every SM filled to its occupancy limit) of independent
// dependency chains; the rate is counted operations / (SMs x elapsed SM cycles), the cycles taken
// from clock64 inside every CTA (max over CTAs), and per second from CUDA events around the
// launch.  These are the roofline denominators bench.py reports against (bnfft_measure_peaks).
#include <cuda_runtime.h>

#include <cstring>

#include "bnfft_internal.h"

namespace bnfft {

constexpr int kPkThreads = 512;
constexpr int kPkIters = 4096;

__device__ unsigned long long g_pk_cycles;
__device__ float g_pk_sink;

__device__ __forceinline__ void pk_start(unsigned long long& t0) {
  __syncthreads();
  t0 = clock64();
}
__device__ __forceinline__ void pk_stop(unsigned long long t0) {
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_pk_cycles, clock64() - t0);
}

// 8 independent chains of a = a * b + c with b, c in registers (3-register FFMA)
__global__ void __launch_bounds__(kPkThreads) pk_ffma(float b, float c, int iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  unsigned long long t0;
  pk_start(t0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
  }
  pk_stop(t0);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345f) g_pk_sink = s;
}

__global__ void __launch_bounds__(kPkThreads) pk_ffma2(float b, float c, int iters) {
  float2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 bb = make_float2(b, b * 0.5f), cc = make_float2(c, c * 0.25f);
  unsigned long long t0;
  pk_start(t0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], bb, cc);
  }
  pk_stop(t0);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 1.2345f) g_pk_sink = s;
}

__global__ void __launch_bounds__(kPkThreads) pk_dfma(double b, double c, int iters) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  unsigned long long t0;
  pk_start(t0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  pk_stop(t0);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) g_pk_sink = (float)s;
}

template <int OP>
__device__ __forceinline__ float mufu(float v) {
  float r;
  if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  else if (OP == 1) asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  else asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

template <int OP>
__global__ void __launch_bounds__(kPkThreads) pk_mufu(float c, int iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 0.5f + threadIdx.x * 1e-6f + i * 1e-3f;
  unsigned long long t0;
  pk_start(t0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = mufu<OP>(a[i]) * c;   // FMUL keeps the value in range
  }
  pk_stop(t0);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345f) g_pk_sink = s;
}

// conflict-free shared loads: lane l of a warp reads word (base + l) of W bytes; 4 independent
// loads per step at addresses rotating through a 16 KB buffer
template <int W>
__global__ void __launch_bounds__(kPkThreads) pk_lds(int iters) {
  __shared__ __align__(16) float buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = (float)i;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(buf);
  constexpr int WPL = W / 4;   // words per lane
  const uint32_t span = 32 * W;
  float acc = 0;
  unsigned long long t0;
  pk_start(t0);
  uint32_t off = (uint32_t)((wid * span) % 16384u);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t a = base + ((off + r * span) & 16383u) + lane * W;
      if (WPL == 2) {
        float x, y;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
        acc += x + y;
      } else {
        float x, y, z, w;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
        acc += (x + y) + (z + w);
      }
    }
    off += 4 * span;
  }
  pk_stop(t0);
  if (acc == 1.2345f) g_pk_sink = acc;
}

}  // namespace bnfft

using namespace bnfft;

namespace {

struct PkRun {
  double per_sm_clk;   // operations (or bytes) per SM per cycle
  double per_s;        // operations (or bytes) per second, whole GPU
  double mhz;          // cycles / event time
};

template <typename Launch>
static int pk_time(Launch launch, double ops_per_thread, PkRun* out) {
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const void* fn = launch(0, 0, true);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPkThreads, 0) != cudaSuccess || per_sm < 1)
    return BNFFT_E_CUDA;
  const int blocks = nsm * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch(blocks, kPkIters / 8, false);   // warm-up
  double best = 1e30;
  unsigned long long best_cyc = 0;
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z = 0;
    cudaMemcpyToSymbol(g_pk_cycles, &z, sizeof(z));
    cudaEventRecord(a);
    launch(blocks, kPkIters, false);
    cudaEventRecord(b);
    if (cudaEventSynchronize(b) != cudaSuccess) return cuda_fail(cudaGetLastError(), "peaks");
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc = 0;
    cudaMemcpyFromSymbol(&cyc, g_pk_cycles, sizeof(cyc));
    if (ms < best) {
      best = ms;
      best_cyc = cyc;
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const double total = ops_per_thread * (double)kPkIters * (double)blocks * kPkThreads;
  out->per_sm_clk = total / ((double)nsm * (double)best_cyc);
  out->per_s = total / (best * 1e-3);
  out->mhz = (double)best_cyc / (best * 1e-3) * 1e-6;
  return BNFFT_OK;
}

}  // namespace

extern "C" int bnfft_measure_peaks(int device, bnfft_peaks* o) {
  if (!o) return BNFFT_E_INVALID_ARG;
  memset(o, 0, sizeof(*o));
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device");
    return BNFFT_E_CUDA;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaDeviceGetAttribute(&o->sms, cudaDevAttrMultiProcessorCount, device);
  const float fb = 0.999f, fc = 1e-7f;
  PkRun r;
  int rc;
#define PK(field, kern, ops, ...)                                                                  \
  rc = pk_time(                                                                                    \
      [&](int blocks, int iters, bool get) -> const void* {                                        \
        if (get) return (const void*)kern;                                                         \
        kern<<<blocks, kPkThreads>>>(__VA_ARGS__ iters);                                           \
        return nullptr;                                                                            \
      },                                                                                           \
      ops, &r);                                                                                    \
  if (rc != BNFFT_OK) return rc;                                                                   \
  o->field##_per_sm_clk = r.per_sm_clk;                                                            \
  o->field##_per_s = r.per_s;                                                                      \
  o->field##_mhz = r.mhz;
  PK(ffma, pk_ffma, 16.0 * 8.0, fb, fc, )
  PK(ffma2, pk_ffma2, 16.0 * 8.0 * 2.0, fb, fc, )
  PK(dfma, pk_dfma, 4.0 * 8.0, (double)fb, (double)fc, )
  PK(ex2, pk_mufu<0>, 4.0 * 8.0, 0.5f, )
  PK(rsqrt, pk_mufu<1>, 4.0 * 8.0, 1.5f, )
  PK(rcp, pk_mufu<2>, 4.0 * 8.0, 1.5f, )
  PK(lds64, pk_lds<8>, 4.0 * 8.0, )
  PK(lds128, pk_lds<16>, 4.0 * 16.0, )
#undef PK
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "peaks");
  return BNFFT_OK;
}
