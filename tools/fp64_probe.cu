// FP64 peak probe: the DFMA throughput of one B200, measured (the roofline
// denominator for the gradient pass's FP64 work; MEASURED_PEAKS.json has no
// FP64 figure).  Every thread runs kChains independent DFMA chains, so the
// pipe, not the dependency latency, bounds the loop.  Built by
// __graft_entry__.build() into paper_2312_09888_b200/lib/libnkbprobe.so and
// called by bench.py through ctypes:
//     int nkb_probe_fp64(double* tflops_best, double* tflops_median, int reps)
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = __fma_rn(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;   // keeps the chains live
}

}  // namespace

extern "C" int nkb_probe_fp64(double* tflops_best, double* tflops_median, int reps) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 1;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 1;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);   // warm-up
  std::vector<double> tf;
  for (int r = 0; r < std::max(reps, 1); ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * kChains * (double)kIters * blocks * threads;
    tf.push_back(flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return 1;
  std::sort(tf.begin(), tf.end());
  *tflops_best = tf.back();
  *tflops_median = tf[tf.size() / 2];
  return 0;
}
