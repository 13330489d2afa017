// Chebyshev far field (engine.py:228-256) as FP64 GEMMs.
//
//  * bfmm_rows_gemm: C = alpha * A @ B + beta * C, the basis projections
//    z = M V and locals = scale * lt U^T (engine.py:233, 252-255).
//  * bfmm_m2l_cheb: the 316-offset translation as ONE implicit GEMM per
//    child octant.  Every target cell c of octant o needs exactly the 189
//    offsets t whose +/-3 components match c's coordinate parity
//    (octree.py:128-145); so per octant the operation is
//        lt[c, :] = sum_{t in valid(o)} z[c + t, :] @ coresT[t]
//    i.e. a GEMM with K = 189 * rp whose A operand is gathered on the fly
//    (rows of z at the shifted cells; zero when the source leaves the grid,
//    exactly the pairs cell_pairs_for_offset omits, octree.py:202-221).
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

namespace bfmm {
namespace {

constexpr int TM = 64, TN = 64, KC = 8, kThreads = 256;

// ----------------------------------------------------------------------------
// Generic tiled DGEMM for row-major (rows x K) @ (K x N).
__global__ void __launch_bounds__(kThreads)
rows_gemm_kernel(const double *__restrict__ A, int64_t rows, int K,
                 const double *__restrict__ B, int N, double *__restrict__ C,
                 double alpha, double beta) {
  __shared__ double As[2][KC][TM];
  __shared__ double Bs[2][KC][TN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = int64_t(blockIdx.x) * TM;
  const int n0 = blockIdx.y * TN;
  double acc[4][4] = {};
  // loader mapping: A tile TM x KC -> thread loads 2 elements
  const int la_r = threadIdx.x >> 2, la_k = (threadIdx.x & 3) * 2;
  const int lb_k = threadIdx.x >> 5, lb_n = (threadIdx.x & 31) * 2;
  double ra[2], rb[2];
  auto load = [&](int k0) {
    const int64_t r = r0 + la_r;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = k0 + la_k + u;
      ra[u] = (r < rows && k < K) ? A[r * K + k] : 0.0;
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
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      double v = alpha * acc[i][j];
      if (beta != 0.0) v += beta * C[r * N + n];
      C[r * N + n] = v;
    }
  }
}

// ----------------------------------------------------------------------------
// 316 far offsets in the reference's lexicographic order (octree.py:110-119).
__constant__ signed char c_offsets[316][3];
bool g_offsets_ready = false;

void ensure_offsets() {
  if (g_offsets_ready) return;
  signed char h[316][3];
  int n = 0;
  for (int a = -3; a <= 3; ++a)
    for (int b = -3; b <= 3; ++b)
      for (int c = -3; c <= 3; ++c) {
        int mx = abs(a) > abs(b) ? abs(a) : abs(b);
        mx = mx > abs(c) ? mx : abs(c);
        if (mx >= 2) {
          h[n][0] = (signed char)a;
          h[n][1] = (signed char)b;
          h[n][2] = (signed char)c;
          ++n;
        }
      }
  cudaMemcpyToSymbol(c_offsets, h, sizeof(h));
  g_offsets_ready = true;
}

__device__ inline bool offset_valid_for_octant(int o, int t0, int t1, int t2) {
  // +3 needs an even coordinate (octant bit 0), -3 an odd one (bit 1)
  const int bx = (o >> 2) & 1, by = (o >> 1) & 1, bz = o & 1;
  if (t0 == 3 && bx) return false;
  if (t0 == -3 && !bx) return false;
  if (t1 == 3 && by) return false;
  if (t1 == -3 && !by) return false;
  if (t2 == 3 && bz) return false;
  if (t2 == -3 && !bz) return false;
  return true;
}

// Implicit-GEMM M2L.  Grid: (row tiles, column tiles, 8 octants).
// Rows are (target cell of octant o, weight column) pairs.
__global__ void __launch_bounds__(kThreads)
m2l_cheb_kernel(const double *__restrict__ z, double *__restrict__ lt,
                int level, int m, int rp, const double *__restrict__ coresT) {
  __shared__ double As[2][KC][TM];
  __shared__ double Bs[2][KC][TN];
  const int o = blockIdx.z;
  const int n = 1 << level;
  const int64_t ncell = int64_t(1) << (3 * level);
  const int64_t rows = (ncell >> 3) * m;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = int64_t(blockIdx.x) * TM;
  const int n0 = blockIdx.y * TN;

  // loader: A tile TM rows x KC -> each thread one double2 (row, k pair)
  const int la_r = threadIdx.x >> 2, la_k = (threadIdx.x & 3) * 2;
  const int lb_k = threadIdx.x >> 5, lb_n = (threadIdx.x & 31) * 2;
  const int64_t my_row = r0 + la_r;
  int cx = 0, cy = 0, cz = 0, col = 0;
  const bool row_ok = my_row < rows;
  if (row_ok) {
    const int64_t q = my_row / m;
    col = (int)(my_row - q * m);
    unmorton3((uint64_t)(8 * q + o), cx, cy, cz);
  }
  const int kchunks = rp / KC;

  double acc[4][4] = {};
  double2 ra;
  double rb[2];
  // iterate over (offset, k-chunk) steps
  int t = -1, kc = kchunks;  // current step
  int64_t src_base = -1;
  auto advance = [&]() -> bool {
    ++kc;
    if (kc >= kchunks) {
      kc = 0;
      for (++t; t < 316; ++t)
        if (offset_valid_for_octant(o, c_offsets[t][0], c_offsets[t][1],
                                    c_offsets[t][2]))
          break;
      if (t >= 316) return false;
      const int t0 = c_offsets[t][0], t1 = c_offsets[t][1], t2 = c_offsets[t][2];
      if (row_ok && far_pair(n, cx, cy, cz, t0, t1, t2))
        src_base =
            ((int64_t)morton3(cx + t0, cy + t1, cz + t2) * m + col) * rp;
      else
        src_base = -1;
    }
    return true;
  };
  auto load = [&]() {
    const int k = kc * KC;
    if (src_base >= 0)
      ra = *reinterpret_cast<const double2 *>(z + src_base + k + la_k);
    else
      ra = make_double2(0.0, 0.0);
    const double *bt = coresT + ((int64_t)t * rp + k + lb_k) * rp;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int nn = n0 + lb_n + u;
      rb[u] = nn < rp ? bt[nn] : 0.0;
    }
  };
  auto store = [&](int buf) {
    As[buf][la_k][la_r] = ra.x;
    As[buf][la_k + 1][la_r] = ra.y;
    Bs[buf][lb_k][lb_n] = rb[0];
    Bs[buf][lb_k][lb_n + 1] = rb[1];
  };
  if (!advance()) return;
  load();
  store(0);
  __syncthreads();
  int buf = 0;
  while (true) {
    const bool more = advance();
    if (more) load();
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
    if (!more) break;
    store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty + 16 * i;
    if (r >= rows) continue;
    const int64_t q = r / m;
    const int c = (int)(r - q * m);
    double *dst = lt + ((8 * q + o) * m + c) * rp;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int nn = n0 + tx + 16 * j;
      if (nn < rp) dst[nn] = acc[i][j];
    }
  }
}

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

extern "C" int bfmm_rows_gemm(const double *A, int64_t rows, int K,
                              const double *B, int N, double *C, double alpha,
                              double beta, bfmm_stream_t stream) {
  if (rows <= 0 || N <= 0) return 0;
  dim3 grid((unsigned)ceil_div(rows, TM), (unsigned)ceil_div(N, TN));
  rows_gemm_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(A, rows, K, B, N,
                                                             C, alpha, beta);
  return check_launch("rows_gemm_kernel");
}

extern "C" int bfmm_m2l_cheb(const double *z, double *lt, int level, int m,
                             int rp, const double *coresT,
                             bfmm_stream_t stream) {
  if (rp % KC != 0 || level < 2 || level > 10) {
    set_error("bfmm_m2l_cheb: rp=%d must be a multiple of %d, level=%d", rp, KC,
              level);
    return 2;
  }
  ensure_offsets();
  const int64_t rows = (int64_t(1) << (3 * level - 3)) * m;
  dim3 grid((unsigned)ceil_div(rows, TM), (unsigned)ceil_div(rp, TN), 8);
  m2l_cheb_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(z, lt, level, m, rp,
                                                            coresT);
  return check_launch("m2l_cheb_kernel");
}
