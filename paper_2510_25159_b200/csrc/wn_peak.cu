// wn_peak.cu -- measured FP64 / FP32 pipe peaks of the device (diagnostics).
//
// The roofline of the query kernel is stated against the FP64 (or FP32) pipe
// ("148 SMs x 64 FP64 lanes/clk x f ... must be MEASURED by a
// DFMA/FFMA throughput microbenchmark on the box, with the SM clock logged").
// k_fma_peak runs CH independent dependent-FMA chains per thread (enough
// independent work per scheduler to cover the pipe latency), with a grid of
// 148 x 4 CTAs of 256 threads; the result is lane-FMA instructions per second
// (x2 = FLOP/s).  The SM clock during the run is measured in the kernel from
// clock64() cycles against the %globaltimer nanoseconds of CTA 0.
#include "wn_common.cuh"

namespace wn {
namespace {

constexpr int PK_CH = 8;        // independent chains per thread
constexpr int PK_UNROLL = 16;   // FMAs per chain per loop iteration

template <typename R>
__global__ void __launch_bounds__(256) k_fma_peak(int iters, R a, R b, R *sink, unsigned long long *clk) {
  R x[PK_CH];
#pragma unroll
  for (int c = 0; c < PK_CH; ++c) x[c] = (R)(threadIdx.x + c) * (R)1e-3;
  unsigned long long c0 = 0, g0 = 0;
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    c0 = clock64();
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < PK_UNROLL; ++u)
#pragma unroll
      for (int c = 0; c < PK_CH; ++c) x[c] = fma(x[c], a, b);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long g1;
    const unsigned long long c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    clk[0] = c1 - c0;
    clk[1] = g1 - g0;
  }
  R s = 0;
#pragma unroll
  for (int c = 0; c < PK_CH; ++c) s += x[c];
  if (s == (R)12345.678) sink[0] = s;   // keeps the chains live; never true in practice
}

template <typename R>
wn_status_t measure(double seconds, double *rate, double *mhz) {
  int dev = 0, nsm = 0;
  WN_CUDA(cudaGetDevice(&dev));
  WN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  R *sink = nullptr;
  unsigned long long *clk = nullptr;
  WN_CUDA(cudaMalloc(&sink, sizeof(R)));
  WN_CUDA(cudaMalloc(&clk, 2 * sizeof(unsigned long long)));
  cudaStream_t st;
  WN_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  WN_CUDA(cudaEventCreate(&e0));
  WN_CUDA(cudaEventCreate(&e1));
  const int blocks = nsm * 4, threads = 256;
  const R a = (R)0.999999, b = (R)1e-7;
  // calibrate the iteration count to ~`seconds` per launch
  int iters = 256;
  float ms = 0.f;
  for (int k = 0; k < 12; ++k) {
    WN_CUDA(cudaEventRecord(e0, st));
    k_fma_peak<R><<<blocks, threads, 0, st>>>(iters, a, b, sink, clk);
    WN_CUDA(cudaEventRecord(e1, st));
    WN_CUDA(cudaEventSynchronize(e1));
    WN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms > 1e3 * seconds * 0.5) break;
    iters *= 2;
  }
  double best = 0.0, best_mhz = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    WN_CUDA(cudaEventRecord(e0, st));
    k_fma_peak<R><<<blocks, threads, 0, st>>>(iters, a, b, sink, clk);
    WN_CUDA(cudaEventRecord(e1, st));
    WN_CUDA(cudaEventSynchronize(e1));
    WN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    unsigned long long h[2];
    WN_CUDA(cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost));
    const double lanes = (double)blocks * threads * (double)iters * PK_UNROLL * PK_CH;
    const double r = lanes / (ms * 1e-3);
    if (r > best) {
      best = r;
      best_mhz = h[1] ? (double)h[0] / (double)h[1] * 1e3 : 0.0;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaFree(sink);
  cudaFree(clk);
  *rate = best;
  if (mhz) *mhz = best_mhz;
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

}  // namespace
}  // namespace wn

extern "C" wn_status_t wn_measure_fp_peak(int fp32, double seconds, double *lane_fma_per_s, double *sm_mhz) {
  if (!lane_fma_per_s || seconds <= 0.0) {
    wn::set_error("wn_measure_fp_peak: bad arguments");
    return WN_ERR_ARG;
  }
  return fp32 ? wn::measure<float>(seconds, lane_fma_per_s, sm_mhz)
              : wn::measure<double>(seconds, lane_fma_per_s, sm_mhz);
}
