// Library plumbing: last-error text, version, FP64 peak probe.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace bfmm {

static thread_local char g_err[4096] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

namespace {

// Eight independent DFMA chains per thread; the compiler cannot fold them.
__global__ void __launch_bounds__(256) dfma_probe_kernel(double *out, int iters,
                                                         double a, double b) {
  double x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = threadIdx.x * 1e-3 + u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = fma(x[u], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += x[u];
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}

}  // namespace
}  // namespace bfmm

using namespace bfmm;

extern "C" const char *bfmm_last_error(void) { return g_err; }

extern "C" int bfmm_version(void) { return 1; }

extern "C" int bfmm_device_fp64_probe(double *gflops, bfmm_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  double *out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) {
    set_error("bfmm_device_fp64_probe: cudaMalloc failed");
    return 1;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int iters = 1 << 14;
  dim3 grid(sms * 8), block(256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_probe_kernel<<<grid, block, 0, st>>>(out, iters, 0.999999, 1e-9);  // warm
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, st);
    dfma_probe_kernel<<<grid, block, 0, st>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (check_launch("dfma_probe_kernel")) return 1;
  const double flops = 2.0 * 8.0 * iters * double(grid.x) * block.x;
  *gflops = flops / (best * 1e-3) / 1e9;
  return 0;
}
