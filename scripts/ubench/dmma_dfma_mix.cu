// Microbenchmark: do FP64 tensor-core MMAs (mma.sync m8n8k4.f64, SASS DMMA)
// and DFMA share one pipe on B200?  Warps of a CTA run either a DMMA chain
// loop or a DFMA chain loop; the rates alone and mixed tell.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_dfma_mix dmma_dfma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// mode bit 0: DMMA warps active, bit 1: DFMA warps active; warps with
// (warp & 1) == 0 are DMMA warps, the others DFMA warps
__global__ void __launch_bounds__(256) k(double *out, int iters, int mode, double a, double b) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if ((warp & 1) == 0) {
    if (!(mode & 1)) return;
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[2 * i], c[2 * i + 1], a, b);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
  } else {
    if (!(mode & 2)) return;
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
  }
  if (s == 123.456) *out = s;
}

int main() {
  double *out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 1 << 13;
  for (int mode = 1; mode <= 3; ++mode) {
    dim3 grid(sms * 4), block(256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      k<<<grid, block>>>(out, iters, mode, 0.999999, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    // per CTA: 4 DMMA warps x 32 DMMA x 512 flop, 4 DFMA warps x 128 DFMA x 64 flop, per iteration
    const double dmma_fl = (mode & 1) ? 4.0 * 32 * 512 * iters * grid.x : 0;
    const double dfma_fl = (mode & 2) ? 4.0 * 128 * 64 * iters * grid.x : 0;
    printf("mode %d (%s): %.3f ms  DMMA %.2f TF  DFMA %.2f TF  total %.2f TF\n", mode,
           mode == 1 ? "DMMA only" : mode == 2 ? "DFMA only" : "both", best, dmma_fl / best / 1e9,
           dfma_fl / best / 1e9, (dmma_fl + dfma_fl) / best / 1e9);
  }
  return 0;
}
