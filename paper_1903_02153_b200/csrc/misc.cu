// Library plumbing: last-error text, version, FP64 peak probe.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "common.cuh"
#include "tcgen05.cuh"

namespace bfmm {

static thread_local char g_err[4096] = "";
static std::atomic<long long> g_launches{0};

void add_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

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

// Eight independent m8n8k4 f64 MMA chains per warp (FP64 tensor cores).
__global__ void __launch_bounds__(256) dmma_probe_kernel(double *out, int iters) {
  double c[8][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
#pragma unroll
  for (int u = 0; u < 8; ++u) c[u][0] = c[u][1] = u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, "
          "{%3}, {%0, %1};\n"
          : "+d"(c[u][0]), "+d"(c[u][1])
          : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
  if (s == 12345.678) out[0] = s;
}

// C independent m8n8k4 chains per warp (microarchitecture sweep).
template <int C>
__global__ void dmma_chain_kernel(double *out, int iters) {
  double c[C][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
#pragma unroll
  for (int u = 0; u < C; ++u) c[u][0] = c[u][1] = u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < C; ++u)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, "
          "{%3}, {%0, %1};\n"
          : "+d"(c[u][0]), "+d"(c[u][1])
          : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < C; ++u) s += c[u][0] + c[u][1];
  if (s == 12345.678) out[0] = s;
}

template <class F>
float best_ms(F launch, cudaStream_t st) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, st);
    launch();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

}  // namespace
}  // namespace bfmm

using namespace bfmm;

// Diagnostics: DMMA throughput with `warps_per_sm` resident warps (one CTA
// of that many warps per SM) each running `chains` independent chains.
extern "C" int bfmm_device_dmma_sweep(int warps_per_sm, int chains,
                                      double *gflops, bfmm_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  double *out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int iters = (1 << 13) / chains;
  dim3 grid(sms), block(32 * warps_per_sm);
  float ms = 0.f;
  switch (chains) {
    case 1: ms = best_ms([&] { dmma_chain_kernel<1><<<grid, block, 0, st>>>(out, iters); }, st); break;
    case 2: ms = best_ms([&] { dmma_chain_kernel<2><<<grid, block, 0, st>>>(out, iters); }, st); break;
    case 4: ms = best_ms([&] { dmma_chain_kernel<4><<<grid, block, 0, st>>>(out, iters); }, st); break;
    case 8: ms = best_ms([&] { dmma_chain_kernel<8><<<grid, block, 0, st>>>(out, iters); }, st); break;
    default: ms = best_ms([&] { dmma_chain_kernel<16><<<grid, block, 0, st>>>(out, iters); }, st); chains = 16; break;
  }
  cudaFree(out);
  if (check_launch("dmma_chain_kernel")) return 1;
  *gflops = 512.0 * chains * iters * double(grid.x) * warps_per_sm / (ms * 1e-3) / 1e9;
  return 0;
}

extern "C" int bfmm_device_dmma_probe(double *gflops, bfmm_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  double *out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) {
    set_error("bfmm_device_dmma_probe: cudaMalloc failed");
    return 1;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int iters = 1 << 12;
  dim3 grid(sms * 4), block(256);
  float ms = best_ms([&] { dmma_probe_kernel<<<grid, block, 0, st>>>(out, iters); }, st);
  cudaFree(out);
  if (check_launch("dmma_probe_kernel")) return 1;
  // 8 chains x 256 FMA (512 flops) per warp per iteration
  const double flops = 512.0 * 8 * iters * double(grid.x) * (block.x / 32);
  *gflops = flops / (ms * 1e-3) / 1e9;
  return 0;
}

extern "C" const char *bfmm_last_error(void) { return g_err; }

extern "C" int bfmm_version(void) { return 1; }

extern "C" long long bfmm_launch_count(void) {
  return g_launches.load(std::memory_order_relaxed);
}

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

// ---- tcgen05 int8 self-test: D (128 x 64, int32) = A (128 x K) B (64 x K)^T ----
namespace bfmm {
namespace {
__global__ void __launch_bounds__(128)
tc_i8_selftest_kernel(const int8_t *__restrict__ A, const int8_t *__restrict__ B, int K,
                      int32_t *__restrict__ D) {
  using namespace bfmm;
  __shared__ __align__(128) int8_t sA[128 * 32];
  __shared__ __align__(128) int8_t sB[64 * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) tc::alloc(&tmem_base, 64);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = tc::idesc_i8(128, 64);
  int phase = 0;
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int e = tid; e < 128 * 2; e += 128) {
      const int row = e >> 1, h = e & 1;
      *reinterpret_cast<int4 *>(sA + tc::kmajor_off(row, 16 * h)) =
          *reinterpret_cast<const int4 *>(A + (size_t)row * K + k0 + 16 * h);
    }
    for (int e = tid; e < 64 * 2; e += 128) {
      const int row = e >> 1, h = e & 1;
      *reinterpret_cast<int4 *>(sB + tc::kmajor_off(row, 16 * h)) =
          *reinterpret_cast<const int4 *>(B + (size_t)row * K + k0 + 16 * h);
    }
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      tc::mma_i8(tmem, tc::desc_kmajor(tc::smem_u32(sA), 128, 256),
                 tc::desc_kmajor(tc::smem_u32(sB), 128, 256), idesc, k0 > 0 ? 1u : 0u);
      tc::commit(&mbar);
    }
    // wait for the MMA before the tile is overwritten
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            tc::smem_u32(&mbar)),
        "r"(phase)
        : "memory");
    phase ^= 1;
    tc::fence_after();
  }
  uint32_t v[16];
  for (int c = 0; c < 64; c += 16) {
    tc::ld16(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
    tc::wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) D[(32 * warp + lane) * 64 + c + j] = (int32_t)v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 64);
}
}  // namespace
}  // namespace bfmm

extern "C" int bfmm_tc_i8_selftest(const int8_t *A, const int8_t *B, int K, int32_t *D,
                                   bfmm_stream_t stream) {
  if (K <= 0 || K % 32) {
    set_error("bfmm_tc_i8_selftest: K=%d must be a positive multiple of 32", K);
    return 2;
  }
  bfmm::tc_i8_selftest_kernel<<<1, 128, 0, as_stream(stream)>>>(A, B, K, D);
  return check_launch("tc_i8_selftest_kernel");
}

// ---- tcgen05 kind::i8 throughput probe: back-to-back 128 x N x 32 MMAs ----
namespace bfmm {
namespace {
template <int N>
__global__ void __launch_bounds__(128, 1) tc_i8_probe_kernel(int iters, int32_t *sink) {
  __shared__ __align__(1024) int8_t sA[128 * 32];
  __shared__ __align__(1024) int8_t sB[N * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 32; e += 128) sA[e] = (int8_t)(e & 7);
  for (int e = tid; e < N * 32; e += 128) sB[e] = (int8_t)(e & 3);
  if (warp == 0) tc::alloc(&tmem_base, 512);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t da = tc::desc_kmajor(tc::smem_u32(sA), 128, 256);
    const uint64_t db = tc::desc_kmajor(tc::smem_u32(sB), 128, 256);
    const uint32_t idesc = tc::idesc_i8(128, N);
    for (int i = 0; i < iters; ++i) tc::mma_i8(tmem + (uint32_t)((i & 1) * N), da, db, idesc, 1u);
    tc::commit(&mbar);
  }
  if (warp == 0) {  // tcgen05.ld is warp-collective
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
            tc::smem_u32(&mbar))
        : "memory");
    tc::fence_after();
    uint32_t v[16];
    tc::ld16(tmem, v);
    tc::wait_ld();
    if (v[0] == 0x7fffffffu) sink[blockIdx.x] = (int32_t)v[1];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 512);
}
}  // namespace
}  // namespace bfmm

extern "C" int bfmm_device_i8_probe_n(int N, double *tops, bfmm_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  int32_t *sink = nullptr;
  if (cudaMalloc(&sink, 4096 * sizeof(int32_t)) != cudaSuccess) return 1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int iters = 1 << 14;
  float ms = 0;
  switch (N) {
    case 64: ms = best_ms([&] { bfmm::tc_i8_probe_kernel<64><<<sms, 128, 0, st>>>(iters, sink); }, st); break;
    case 128: ms = best_ms([&] { bfmm::tc_i8_probe_kernel<128><<<sms, 128, 0, st>>>(iters, sink); }, st); break;
    case 192: ms = best_ms([&] { bfmm::tc_i8_probe_kernel<192><<<sms, 128, 0, st>>>(iters, sink); }, st); break;
    default: ms = best_ms([&] { bfmm::tc_i8_probe_kernel<256><<<sms, 128, 0, st>>>(iters, sink); }, st); N = 256; break;
  }
  cudaFree(sink);
  if (check_launch("tc_i8_probe_kernel")) return 1;
  *tops = 2.0 * 128 * N * 32 * double(iters) * sms / (ms * 1e-3) / 1e12;
  return 0;
}

extern "C" int bfmm_device_i8_probe(double *tops, bfmm_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  int32_t *sink = nullptr;
  if (cudaMalloc(&sink, 4096 * sizeof(int32_t)) != cudaSuccess) {
    set_error("bfmm_device_i8_probe: cudaMalloc failed");
    return 1;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int iters = 1 << 14;
  float ms = best_ms([&] { bfmm::tc_i8_probe_kernel<256><<<sms, 128, 0, st>>>(iters, sink); }, st);
  cudaFree(sink);
  if (check_launch("tc_i8_probe_kernel")) return 1;
  const double ops = 2.0 * 128 * 256 * 32 * double(iters) * sms;
  *tops = ops / (ms * 1e-3) / 1e12;
  return 0;
}
