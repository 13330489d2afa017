// Chebyshev far field (engine.py:228-256) as FP64 GEMMs.
//
//  * bfmm_rows_gemm: C = alpha * A @ B + beta * C, the basis projections
//    z = M V and locals = scale * lt U^T (engine.py:233, 252-255).
//  * bfmm_m2l_cheb: the 316-offset translation as ONE implicit GEMM per
//    child octant.  Every target cell c of octant o needs exactly the 189
//    offsets t whose +/-3 components match c's coordinate parity
//    (octree.py:128-145); so per octant the operation is
//        lt[c, i] = sum_{t in valid(o)} sum_k z[c + t, k] * C_t[i, k]
//    i.e. a GEMM with K = 189 * rp whose A operand is gathered on the fly
//    (rows of z at the shifted cells; zero-filled when the source leaves the
//    grid, exactly the pairs cell_pairs_for_offset omits, octree.py:202-221).
//    The MMA is the FP64 tensor-core instruction (DMMA, mma.sync m8n8k4 f64;
//    tcgen05 has no f64 kind), operands staged by a 3-stage cp.async ring.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace bfmm {
namespace {

constexpr int TM = 64, TN = 64, KC = 8, kThreads = 256;

// Output row of A row r: r itself, or -- for the compact rows of listed
// cells -- groups[r / group_rows] * group_rows + r % group_rows.
__device__ __forceinline__ int64_t c_row(int64_t r, const int64_t *groups,
                                         int64_t group_rows) {
  if (!groups) return r;
  const int64_t g = r / group_rows;
  return groups[g] * group_rows + (r - g * group_rows);
}

// ----------------------------------------------------------------------------
// Generic tiled DGEMM for row-major (rows x K) @ (K x N); the A operand may
// be stored as a_splits blocks per row that are summed on load.
__global__ void __launch_bounds__(kThreads)
rows_gemm_kernel(const double *__restrict__ A, int64_t rows, int K,
                 int a_splits, const double *__restrict__ B, int N,
                 double *__restrict__ C, double alpha, double beta,
                 const int64_t *__restrict__ groups, int64_t group_rows) {
  __shared__ double As[2][KC][TM];
  __shared__ double Bs[2][KC][TN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = int64_t(blockIdx.x) * TM;
  const int n0 = blockIdx.y * TN;
  double acc[4][4] = {};
  const int la_r = threadIdx.x >> 2, la_k = (threadIdx.x & 3) * 2;
  const int lb_k = threadIdx.x >> 5, lb_n = (threadIdx.x & 31) * 2;
  double ra[2], rb[2];
  auto load = [&](int k0) {
    const int64_t r = r0 + la_r;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = k0 + la_k + u;
      // row stride a_splits * K: split block 0 holds the reduced sum
      ra[u] = (r < rows && k < K) ? A[(r * a_splits) * K + k] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = k0 + lb_k, n = n0 + lb_n + u;
      rb[u] = (k < K && n < N) ? B[(int64_t)k * N + n] : 0.0;
    }
  };
  auto store = [&](int buf) {
    As[buf][la_k][la_r] = ra[0];
    As[buf][la_k + 1][la_r] = ra[1];
    Bs[buf][lb_k][lb_n] = rb[0];
    Bs[buf][lb_k][lb_n + 1] = rb[1];
  };
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += KC) {
    const bool more = k0 + KC < K;
    if (more) load(k0 + KC);
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty + 16 * i;
    if (r >= rows) continue;
    const int64_t cr = c_row(r, groups, group_rows);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      double v = alpha * acc[i][j];
      if (beta != 0.0) v += beta * C[cr * N + n];
      C[cr * N + n] = v;
    }
  }
}

// A[r][0][k] = sum_s A[r][s][k] in place, fixed order (M2L split blocks).
__global__ void reduce_splits_kernel(double *__restrict__ A, int64_t rows, int K,
                                     int a_splits) {
  const int64_t total = rows * K;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / K;
    const int k = (int)(e - r * K);
    double *a = A + r * a_splits * K + k;
    double v = a[0];
    for (int sp = 1; sp < a_splits; ++sp) v += a[(int64_t)sp * K];
    a[0] = v;
  }
}

// One thread per output for small (coarse-level) projections: a single 64-row
// tile would serialise the whole K loop on one SM.
__global__ void __launch_bounds__(128)
small_gemm_kernel(const double *__restrict__ A, int64_t rows, int K,
                  int a_splits, const double *__restrict__ B, int N,
                  double *__restrict__ C, double alpha, double beta,
                  const int64_t *__restrict__ groups, int64_t group_rows) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= rows * N) return;
  const int64_t r = e / N;
  const int n = (int)(e - r * N);
  const double *a = A + r * a_splits * K;  // split block 0 holds the sum
  // four independent partial sums (fixed order) keep the FMA chain short
  double acc4[4] = {0.0, 0.0, 0.0, 0.0};
  int k = 0;
  for (; k + 4 <= K; k += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) acc4[u] = fma(a[k + u], B[(int64_t)(k + u) * N + n], acc4[u]);
  }
  for (; k < K; ++k) acc4[0] = fma(a[k], B[(int64_t)k * N + n], acc4[0]);
  const double acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
  const int64_t ce = c_row(r, groups, group_rows) * N + n;
  double out = alpha * acc;
  if (beta != 0.0) out += beta * C[ce];
  C[ce] = out;
}

// ----------------------------------------------------------------------------
// 316 far offsets in the reference's lexicographic order (octree.py:110-119)
// and, per child octant, the 189 of them its parity admits (in that order).
__constant__ signed char c_offsets[316][3];
__constant__ short c_valid[8][189];
bool g_offsets_ready = false;

void ensure_offsets() {
  if (g_offsets_ready) return;
  signed char h[316][3];
  short v[8][189];
  int n = 0;
  for (int a = -3; a <= 3; ++a)
    for (int b = -3; b <= 3; ++b)
      for (int c = -3; c <= 3; ++c) {
        int mx = std::max(abs(a), std::max(abs(b), abs(c)));
        if (mx >= 2) {
          h[n][0] = (signed char)a;
          h[n][1] = (signed char)b;
          h[n][2] = (signed char)c;
          ++n;
        }
      }
  for (int o = 0; o < 8; ++o) {
    int k = 0;
    const int bit[3] = {(o >> 2) & 1, (o >> 1) & 1, o & 1};
    for (int t = 0; t < 316; ++t) {
      bool ok = true;
      for (int a = 0; a < 3; ++a) {
        // the parity half of far_axis_ok: +3 needs even, -3 needs odd
        if (h[t][a] == 3 && bit[a]) ok = false;
        if (h[t][a] == -3 && !bit[a]) ok = false;
      }
      if (ok) v[o][k++] = (short)t;
    }
  }
  cudaMemcpyToSymbol(c_offsets, h, sizeof(h));
  cudaMemcpyToSymbol(c_valid, v, sizeof(v));
  g_offsets_ready = true;
}

// ---- DMMA helpers -------------------------------------------------------------
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a,
                                           double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, "
      "{%0, %1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem,
                                           bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s),
               "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

#include "m2l_ws.cuh"

// ----------------------------------------------------------------------------
// Explicit far list for one offset, in the reference's meshgrid(ij) order
// (x slowest, z fastest), built from the same far_pair() predicate the M2L
// kernel applies.  Diagnostics / parity only.
__global__ void far_flags_kernel(int level, int t, int32_t *flag) {
  const int n = 1 << level;
  const int64_t total = int64_t(n) * n * n;
  const int t0 = c_offsets[t][0], t1 = c_offsets[t][1], t2 = c_offsets[t][2];
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int ix = (int)(e / (int64_t(n) * n)), iy = (int)((e / n) % n),
              iz = (int)(e % n);
    flag[e] = far_pair(n, ix, iy, iz, t0, t1, t2) ? 1 : 0;
  }
}

__global__ void far_emit_kernel(int level, int t, const int32_t *flag,
                                const int32_t *pos, int64_t *tg, int64_t *sr,
                                int64_t *count) {
  const int n = 1 << level;
  const int64_t total = int64_t(n) * n * n;
  const int t0 = c_offsets[t][0], t1 = c_offsets[t][1], t2 = c_offsets[t][2];
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int ix = (int)(e / (int64_t(n) * n)), iy = (int)((e / n) % n),
              iz = (int)(e % n);
    if (flag[e]) {
      tg[pos[e]] = (int64_t)morton3(ix, iy, iz);
      sr[pos[e]] = (int64_t)morton3(ix + t0, iy + t1, iz + t2);
    }
    if (e == total - 1) *count = (int64_t)pos[e] + flag[e];
  }
}

}  // namespace
}  // namespace bfmm

using namespace bfmm;

extern "C" size_t bfmm_far_pairs_scratch_bytes(int level) {
  const int64_t total = int64_t(1) << (3 * level);
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int32_t *)nullptr,
                                (int32_t *)nullptr, (int)total);
  return 2 * ((total * sizeof(int32_t) + 255) & ~size_t(255)) + cub_bytes;
}

extern "C" int bfmm_far_pairs(int level, int t_index, int64_t *tg, int64_t *sr,
                              int64_t *count, void *scratch,
                              size_t scratch_bytes, bfmm_stream_t stream) {
  if (level < 2 || level > 9 || t_index < 0 || t_index >= 316) {
    set_error("bfmm_far_pairs: bad level %d / offset %d", level, t_index);
    return 2;
  }
  if (scratch_bytes < bfmm_far_pairs_scratch_bytes(level)) {
    set_error("bfmm_far_pairs: scratch too small");
    return 2;
  }
  ensure_offsets();
  cudaStream_t st = as_stream(stream);
  const int64_t total = int64_t(1) << (3 * level);
  const size_t a = (total * sizeof(int32_t) + 255) & ~size_t(255);
  int32_t *flag = static_cast<int32_t *>(scratch);
  int32_t *pos = reinterpret_cast<int32_t *>(static_cast<char *>(scratch) + a);
  void *tmp = static_cast<char *>(scratch) + 2 * a;
  size_t tb = scratch_bytes - 2 * a;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(total, 256), 4096);
  far_flags_kernel<<<grid, 256, 0, st>>>(level, t_index, flag);
  if (check_launch("far_flags_kernel")) return 1;
  if (cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, (int)total, st) !=
      cudaSuccess) {
    set_error("bfmm_far_pairs: scan failed");
    return 1;
  }
  far_emit_kernel<<<grid, 256, 0, st>>>(level, t_index, flag, pos, tg, sr,
                                        count);
  return check_launch("far_emit_kernel");
}

static int rows_gemm(const double *A, int64_t rows, int K, const double *B, int N,
                     double *C, double alpha, double beta, int a_splits,
                     const int64_t *groups, int64_t group_rows,
                     bfmm_stream_t stream) {
  if (rows <= 0 || N <= 0) return 0;
  if (a_splits < 1) {
    set_error("bfmm_rows_gemm: a_splits=%d < 1", a_splits);
    return 2;
  }
  cudaStream_t st = as_stream(stream);
  if (a_splits > 1) {
    reduce_splits_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * K, 256), 4096), 256,
                           0, st>>>(const_cast<double *>(A), rows, K, a_splits);
    if (check_launch("reduce_splits_kernel")) return 1;
  }
  if (rows * N <= (int64_t(1) << 17)) {
    // small problem (coarse tree levels): one thread per output, full K
    small_gemm_kernel<<<(unsigned)ceil_div(rows * N, 128), 128, 0, st>>>(
        A, rows, K, a_splits, B, N, C, alpha, beta, groups, group_rows);
    return check_launch("small_gemm_kernel");
  }
  dim3 grid((unsigned)ceil_div(rows, TM), (unsigned)ceil_div(N, TN));
  rows_gemm_kernel<<<grid, kThreads, 0, st>>>(A, rows, K, a_splits, B, N, C,
                                              alpha, beta, groups, group_rows);
  return check_launch("rows_gemm_kernel");
}

extern "C" int bfmm_rows_gemm(const double *A, int64_t rows, int K,
                              const double *B, int N, double *C, double alpha,
                              double beta, int a_splits, bfmm_stream_t stream) {
  return rows_gemm(A, rows, K, B, N, C, alpha, beta, a_splits, nullptr, 1, stream);
}

extern "C" int bfmm_rows_gemm_scatter(const double *A, int64_t rows, int K,
                                      const double *B, int N, double *C,
                                      double alpha, double beta, int a_splits,
                                      const int64_t *groups, int64_t group_rows,
                                      bfmm_stream_t stream) {
  if (!groups || group_rows < 1) {
    set_error("bfmm_rows_gemm_scatter: groups=%p group_rows=%lld", (const void *)groups,
              (long long)group_rows);
    return 2;
  }
  return rows_gemm(A, rows, K, B, N, C, alpha, beta, a_splits, groups, group_rows, stream);
}

extern "C" int bfmm_m2l_cheb_splits(int level, int m, int rp, int64_t nq) {
  const int64_t rows = nq * m;
  const int64_t ctas = ceil_div(rows, 64 * m2l_mw(rows)) * ceil_div(rp, 8 * m2l_nt8(rp)) * 8;
  const double slots = 2.0 * kNumSMs;
  // coarse levels: too few tiles to fill the GPU, so split the 189 offsets
  // finely (down to one per CTA; measured faster than one fat wave) and let
  // the U projection sum the blocks
  if (ctas * 4 < slots) return (int)std::min<int64_t>(189, ceil_div(4 * (int64_t)slots, ctas));
  // otherwise pick the split count whose last wave (2 CTAs per SM) is
  // fullest, with a small penalty per split for the extra lt traffic
  int best = 1;
  double best_score = -1e30;
  for (int s = 1; s <= 16; ++s) {
    const double waves = ctas * s / slots;
    const double score = waves / std::ceil(waves) - 0.004 * s;
    if (score > best_score + 1e-12) {
      best_score = score;
      best = s;
    }
  }
  return best;
}

extern "C" int bfmm_m2l_cheb(const double *z, double *lt, int level, int m,
                             int rp, int nsplit, int64_t q_lo, int64_t nq,
                             const double *cores, bfmm_stream_t stream) {
  if (rp % 8 != 0 || rp <= 0 || level < 2 || level > 10) {
    set_error("bfmm_m2l_cheb: rp=%d must be a positive multiple of 8, level=%d",
              rp, level);
    return 2;
  }
  if (nsplit < 1 || nsplit > 189) {
    set_error("bfmm_m2l_cheb: nsplit=%d outside [1, 189]", nsplit);
    return 2;
  }
  const int64_t nparent = int64_t(1) << (3 * level - 3);
  if (q_lo < 0 || nq < 0 || q_lo + nq > nparent) {
    set_error("bfmm_m2l_cheb: parent range [%lld, %lld) outside [0, %lld)",
              (long long)q_lo, (long long)(q_lo + nq), (long long)nparent);
    return 2;
  }
  ensure_offsets();
  M2LCall a{z, lt, level, m, rp, nsplit, q_lo, nq, nullptr, cores, as_stream(stream)};
  return dispatch_ws(m2l_mw(nq * m), m2l_nt8(rp), a);
}

extern "C" int bfmm_m2l_cheb_list(const double *z, double *lt, int level, int m,
                                  int rp, int nsplit, const int64_t *qlist,
                                  int64_t nq, const double *cores,
                                  bfmm_stream_t stream) {
  if (rp % 8 != 0 || rp <= 0 || level < 2 || level > 10) {
    set_error("bfmm_m2l_cheb_list: rp=%d must be a positive multiple of 8, level=%d",
              rp, level);
    return 2;
  }
  if (nsplit < 1 || nsplit > 189) {
    set_error("bfmm_m2l_cheb_list: nsplit=%d outside [1, 189]", nsplit);
    return 2;
  }
  if (nq < 0 || nq > (int64_t(1) << (3 * level - 3)) || (nq > 0 && !qlist)) {
    set_error("bfmm_m2l_cheb_list: %lld listed parents invalid at level %d",
              (long long)nq, level);
    return 2;
  }
  ensure_offsets();
  M2LCall a{z, lt, level, m, rp, nsplit, 0, nq, qlist, cores, as_stream(stream)};
  return dispatch_ws(m2l_mw(nq * m), m2l_nt8(rp), a);
}
