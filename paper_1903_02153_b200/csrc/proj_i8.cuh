// Basis projections on the int8 tensor cores (included by m2l_cheb.cu after
// m2l_i8.cuh): C[r, n] = alpha * sum_k A[r, k] B[k, n] for the row-major
// GEMMs z = M V and locals = s lt U^T (engine.py:233, 252-255) with
// K, N <= 128 -- FP64-accurate by the same error-free digit splitting as the
// M2L (m2l_i8.cuh), but with a scale per A ROW (a plain GEMM allows it):
//   A[r, :] / 2^(e_r - 6) = sum_a 2^(-8a) D_a   (six signed 8-bit digits)
//   B[:, n] / 2^(e_n - 6) = sum_b 2^(-8b) C_b   (host-built, as the cores)
// so C[r, n] = 2^(e_r + e_n - 12) sum_{a+b<6} 2^(-8(a+b)) (D_a C_b^T)[r, n],
// the 21 digit products accumulated exactly in int32 TMEM (|D C| <= 2^14,
// K <= 128, <= 6 products per accumulator: < 2^24).  Truncation ~2^-46 of
// the row / column scales, against the FP64 DMMA projection's 2^-53 K:
// either is far inside the M2L's own digit truncation.
//
// Persistent CTA per SM, 288 threads: warp 0 allocates TMEM and issues the
// MMAs; warps 1-4 slice 128-row tiles of A straight from HBM into the
// K-major digit planes (a warp per 32 rows, lane l holding k = 4l .. 4l+3,
// the row maximum by a warp reduction); warps 5-8 drain the S int32
// accumulators of each 64-column N tile to FP64, so the slicing of tile t+1
// overlaps the drain of tile t.  B's digit image (<= 96 KB) is bulk-copied
// once per CTA.  Memory-bound: A is read once, C written once.
#pragma once

constexpr int kPjS = 6;           // 8-bit digits
constexpr int kPjThreads = 288;

template <int KC, int NTN>
struct PjI8Shape {
  static constexpr int A_PLANE = 128 * 32, B_PLANE = 64 * 32;
  static constexpr int A_BYTES = KC * kPjS * A_PLANE;
  static constexpr int B_BYTES = NTN * KC * kPjS * B_PLANE;
  static constexpr size_t smem = (size_t)A_BYTES + B_BYTES + 256 * sizeof(double) + 64;
};

template <int KC, int NTN>
__global__ void __launch_bounds__(kPjThreads, 1)
proj_i8_kernel(const double *__restrict__ A, int64_t rows, int lda, int K,
               const int8_t *__restrict__ bdig, const double *__restrict__ bpow, int N,
               double *__restrict__ C, double alpha, unsigned long long *__restrict__ zmax) {
  using Sh = PjI8Shape<KC, NTN>;
  constexpr int S = kPjS;
  extern __shared__ __align__(1024) uint8_t sp[];
  uint8_t *const sA = sp;
  uint8_t *const sB = sp + Sh::A_BYTES;
  // row scales of the tile being sliced / drained (two: by tile parity)
  double *const s_rs = reinterpret_cast<double *>(sB + Sh::B_BYTES);
  uint64_t *bars = reinterpret_cast<uint64_t *>(s_rs + 256);
  uint64_t *bar_b = bars, *bar_full = bars + 1, *bar_done = bars + 2, *bar_free = bars + 3,
           *bar_aempty = bars + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 5);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ntiles = (rows + 127) / 128;

  if (warp == 0) bfmm::tc::alloc(tmem_slot, 512);
  if (threadIdx.x == 32) {
    mbar_init(bar_b, 1);
    mbar_init(bar_full, 4);
    mbar_init(bar_done, 1);
    mbar_init(bar_free, 4);
    mbar_init(bar_aempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  bfmm::tc::fence_before();
  __syncthreads();
  bfmm::tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 32) {  // B's digit image, once per CTA
    mbar_expect_tx(bar_b, Sh::B_BYTES);
    for (int off = 0; off < Sh::B_BYTES; off += 16384)
      bulk_g2s(sB + off, bdig + off, min(16384, Sh::B_BYTES - off), bar_b);
  }

  if (warp == 0) {
    // ---------------- MMA issue ----------------
    const uint64_t dA0 = bfmm::tc::desc_kmajor(bfmm::tc::smem_u32(sA), 128, 256);
    const uint64_t dB0 = bfmm::tc::desc_kmajor(bfmm::tc::smem_u32(sB), 128, 256);
    if (lane == 0) mbar_wait(bar_b, 0);
    __syncwarp();
    uint32_t ph_full = 0, ph_free = 0;
    int batch = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      if (lane == 0) mbar_wait(bar_full, ph_full);
      __syncwarp();
      ph_full ^= 1u;
      for (int nt = 0; nt < NTN; ++nt, ++batch) {
        if (batch > 0) {  // the previous batch's accumulators have been drained
          if (lane == 0) mbar_wait(bar_free, ph_free);
          __syncwarp();
          ph_free ^= 1u;
        }
        bfmm::tc::fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kc = 0; kc < KC; ++kc) {
            const uint64_t dA = dA0 + (uint64_t)((kc * S * Sh::A_PLANE) >> 4);
            const uint64_t dB = dB0 + (uint64_t)(((nt * KC + kc) * S * Sh::B_PLANE) >> 4);
#pragma unroll
            for (int a = 0; a < S; ++a) {
#pragma unroll
              for (int b0 = 0; b0 < S - a; b0 += 4) {
                const int nb = min(4, S - a - b0);
                bfmm::tc::mma_i8(tmem + (uint32_t)((a + b0) * 64),
                                 dA + (uint64_t)((a * Sh::A_PLANE) >> 4),
                                 dB + (uint64_t)((b0 * Sh::B_PLANE) >> 4),
                                 bfmm::tc::idesc_i8(128, 64 * nb),
                                 (kc > 0 || a > 0) ? 1u : 0u);
              }
            }
          }
          bfmm::tc::commit(bar_done);
          if (nt == NTN - 1) bfmm::tc::commit(bar_aempty);  // A may be refilled
        }
        __syncwarp();
      }
    }
  } else if (warp <= 4) {
    // ---------------- slice A tiles, drain accumulators ----------------
    // rows 32 quarter .. + 31 of a tile and the same TMEM lanes: a warp may
    // only touch TMEM lanes 32 (warp % 4) .. + 31
    const int quarter = warp & 3;
    uint32_t ph_ae = 0;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      double *rs = s_rs + 128 * (it & 1);
      for (int rb = 0; rb < 4; ++rb) {
        double v[8][4];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int64_t r = t * 128 + quarter * 32 + rb * 8 + rr;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = 4 * lane + u;
            v[rr][u] = (r < rows && k < K) ? A[r * lda + k] : 0.0;
          }
        }
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int row = quarter * 32 + rb * 8 + rr;
          unsigned long long mx = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned long long bits =
                (unsigned long long)__double_as_longlong(v[rr][u]) & 0x7fffffffffffffffull;
            mx = bits > mx ? bits : mx;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = m2 > mx ? m2 : mx;
          }
          const double amax = __longlong_as_double((long long)mx);
          int e = 0;
          const bool fin = amax <= 1.7976931348623157e308;  // false for inf / NaN
          if (fin && amax > 0) frexp(amax, &e);
          if (rb == 0 && rr == 0 && it > 0) {
            // the previous tile's MMAs released A (and, through bar_free, the
            // drain of the tile before it released this half of s_rs); this
            // tile's first rows are already in flight
            mbar_wait(bar_aempty, ph_ae);
            ph_ae ^= 1u;
          }
          if (lane == 0)
            rs[row] = fin ? ldexp(1.0, e - 12) : __longlong_as_double(0x7ff8000000000000ll);
          const double inv = ldexp(1.0, 6 - e);  // first digit of x / 2^(e - 6) in [-64, 64]
          uint32_t w[S];
#pragma unroll
          for (int j = 0; j < S; ++j) w[j] = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double x = fin ? v[rr][u] * inv : 0.0;
            int64_t X = (int64_t)rint(ldexp(x, 8 * (S - 1)));
#pragma unroll
            for (int j = S - 1; j >= 0; --j) {
              const int8_t dg = j > 0 ? (int8_t)(X & 0xff) : (int8_t)X;
              X = (X - dg) >> 8;
              w[j] |= ((uint32_t)(uint8_t)dg) << (8 * u);
            }
          }
          // k = 4 lane .. 4 lane + 3: chunk kc = lane / 8, byte 4 (lane % 8)
          const int kc = lane >> 3;
          const uint32_t off = bfmm::tc::kmajor_off(row, 4 * (lane & 7));
#pragma unroll
          for (int j = 0; j < S; ++j)
            if (kc < KC)
              *reinterpret_cast<uint32_t *>(sA + (kc * S + j) * Sh::A_PLANE + off) = w[j];
        }
      }
      bfmm::tc::fence_proxy_async();  // generic-proxy writes -> tensor core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_full);
    }
  } else {
    // ---------------- drain the accumulators (warps 5-8) ----------------
    const int quarter = warp & 3;
    uint32_t ph_done = 0;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int row = quarter * 32 + lane;
      const int64_t r = t * 128 + row;
      for (int nt = 0; nt < NTN; ++nt) {
        mbar_wait(bar_done, ph_done);
        ph_done ^= 1u;
        bfmm::tc::fence_after();
        const double rs = s_rs[128 * (it & 1) + row] * alpha;
        double amax = 0.0;
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 8) {
          uint32_t acc[S][8];
#pragma unroll
          for (int d = 0; d < S; ++d)
            bfmm::tc::ld8(tmem + ((uint32_t)(32 * quarter) << 16) + d * 64 + c0, acc[d]);
          bfmm::tc::wait_ld();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int n = nt * 64 + c0 + jj;
            double x = (double)(int32_t)acc[S - 1][jj];
#pragma unroll
            for (int d = S - 2; d >= 0; --d) x = fma(x, 0.00390625, (double)(int32_t)acc[d][jj]);
            if (r < rows && n < N) {
              const double val = x * rs * bpow[n];
              C[r * N + n] = val;
              amax = fmax(amax, fabs(val));
            }
          }
        }
        if (zmax) {  // max |C| (one weight column): the int8 M2L's digit scale
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
          if (lane == 0 && amax > 0)
            atomicMax(zmax, (unsigned long long)__double_as_longlong(amax));
        }
        bfmm::tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_free);
      }
    }
  }
  bfmm::tc::fence_before();
  __syncthreads();
  if (warp == 0) bfmm::tc::dealloc(tmem, 512);
}

template <int KC, int NTN>
int launch_proj_i8(const double *A, int64_t rows, int lda, int K, const int8_t *bdig,
                   const double *bpow, int N, double *C, double alpha,
                   unsigned long long *zmax, cudaStream_t st) {
  using Sh = PjI8Shape<KC, NTN>;
  static unsigned long long attr = 0;
  if (first_on_device(&attr))
    cudaFuncSetAttribute(proj_i8_kernel<KC, NTN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Sh::smem);
  const int64_t ntiles = (rows + 127) / 128;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, kNumSMs);
  proj_i8_kernel<KC, NTN><<<grid, kPjThreads, Sh::smem, st>>>(A, rows, lda, K, bdig, bpow, N, C,
                                                             alpha, zmax);
  return check_launch("proj_i8_kernel");
}
