// Microbenchmark: FP64 pipe throughput of DFMA streams by operand pattern.
//  A: acc_k = fma(acc_k, a, b)              (two shared operands)
//  B: complex MAC, 4 targets x 6 taps in registers (stencil inner loop)
//  C: acc_k = fma(x_k, y_k, acc_k)          (three distinct register pairs)
// nvcc -arch=sm_100a -O3 -o dfma_operands dfma_operands.cu && ./dfma_operands
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(128) k(double *out, int iters, double a, double b) {
  double acc[16], x[16], y[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    acc[i] = threadIdx.x * 1e-3 + i;
    x[i] = a + i * 1e-9 + threadIdx.x * 1e-12;
    y[i] = b + i * 1e-9;
  }
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    } else if (MODE == 1) {
      // 6 taps (x[0..5] re, y[0..5] im) x 4 targets: sources x[8+..], y[8+..]
#pragma unroll
      for (int c = 0; c < 6; ++c)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const double vx = x[8 + ((c + 2 * kk) & 7)], vy = y[8 + ((c + 2 * kk) & 7)];
          acc[2 * kk] = fma(x[c], vx, fma(-y[c], vy, acc[2 * kk]));
          acc[2 * kk + 1] = fma(x[c], vy, fma(y[c], vx, acc[2 * kk + 1]));
        }
    } else {
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(x[(i + r) & 15], y[(i + 3 * r) & 15], acc[i]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 123.456) *out = s;
}

int main() {
  double *out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 1 << 14;
  for (int wps = 4; wps <= 16; wps *= 2) {
    for (int mode = 0; mode < 3; ++mode) {
      dim3 grid(sms * wps / 4), block(128);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<grid, block>>>(out, iters, 0.999999, 1e-9);
        if (mode == 1) k<1><<<grid, block>>>(out, iters, 0.999999, 1e-9);
        if (mode == 2) k<2><<<grid, block>>>(out, iters, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double dfma = 96.0 * iters * grid.x * 128.0;
      printf("warps/SM %2d mode %d: %.3f ms  %.2f TFLOP/s  (%.1f%% of %d SMs x 64 x 2 x %.3f GHz)\n", wps,
             mode, best, 2 * dfma / best / 1e9, 100 * 2 * dfma / (best * 1e-3) / (sms * 128.0 * clk * 1e3),
             sms, clk * 1e-6);
    }
  }
  return 0;
}
