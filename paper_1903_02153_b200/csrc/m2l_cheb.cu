// Chebyshev far field (engine.py:228-256) as FP64 GEMMs.
//
//  * bfmm_rows_gemm: C = alpha * A @ B + beta * C, the basis projections
//    z = M V and locals = scale * lt U^T (engine.py:233, 252-255), on the
//    FP64 tensor cores with a cp.async ring (proj_gemm_kernel).
//  * bfmm_m2l_cheb: the 316-offset translation as ONE implicit GEMM per
//    child octant.  Every target cell c of octant o needs exactly the 189
//    offsets t whose +/-3 components match c's coordinate parity
//    (octree.py:128-145); so per octant the operation is
//        lt[c, i] = sum_{t in valid(o)} sum_k z[c + t, k] * C_t[i, k]
//    i.e. a GEMM with K = 189 * rp whose A operand is gathered on the fly
//    (rows of z at the shifted cells; zero-filled when the source leaves the
//    grid, exactly the pairs cell_pairs_for_offset omits, octree.py:202-221).
//    The MMA is the FP64 tensor-core instruction (DMMA, mma.sync m8n8k4 f64;
//    tcgen05 has no f64 kind); a producer warp stages the operands with
//    cp.async into an 8-stage mbarrier ring (m2l_ws.cuh).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include <mutex>

#include "common.cuh"
#include "tcgen05.cuh"

namespace bfmm {
namespace {

// Output row of A row r: r itself, or -- for the compact rows of listed
// cells -- groups[r / group_rows] * group_rows + r % group_rows.
__device__ __forceinline__ int64_t c_row(int64_t r, const int64_t *groups,
                                         int64_t group_rows) {
  if (!groups) return r;
  const int64_t g = r / group_rows;
  return groups[g] * group_rows + (r - g * group_rows);
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
#pragma unroll 4
    for (int sp = 1; sp < a_splits; ++sp) v += a[(int64_t)sp * K];
    a[0] = v;
  }
}

// ----------------------------------------------------------------------------
// 316 far offsets in the reference's lexicographic order (octree.py:110-119)
// and, per child octant, the 189 of them its parity admits (in that order).
__constant__ signed char c_offsets[316][3];
__constant__ short c_valid[8][189];
// offsets as dilated (Morton-interleaved) 10-bit two's-complement integers,
// x / y / z in bit positions 3b+2 / 3b+1 / 3b: cell + t is one masked add
// per axis for levels <= 10 (m2l_i8.cuh)
__constant__ uint32_t c_dil[316][3];
// per octant, its 189 offsets ordered by plane group g = (t_x + 3) * 4 +
// ((o_y + t_y) & 1) * 2 + ((o_z + t_z) & 1); group g is
// c_grp[o][c_grp_off[o][g] .. c_grp_off[o][g + 1]) (m2l_i8p_kernel)
__constant__ short c_grp[8][189];
__constant__ unsigned char c_grp_off[8][29];
std::mutex g_offsets_mu;
unsigned long long g_offsets_ready = 0;  // one bit per device (its own __constant__ bank)

void ensure_offsets() {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lock(g_offsets_mu);
  if (g_offsets_ready & bit) return;
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
  uint32_t dl[316][3];
  for (int t = 0; t < 316; ++t)
    for (int a = 0; a < 3; ++a)
      dl[t][a] = (uint32_t)(spread3((uint64_t)(h[t][a] & 1023)) << (2 - a));
  cudaMemcpyToSymbol(c_dil, dl, sizeof(dl));
  short gr[8][189];
  unsigned char go[8][29];
  for (int o = 0; o < 8; ++o) {
    const int oy = (o >> 1) & 1, oz = o & 1;
    int k = 0;
    for (int g = 0; g < 28; ++g) {
      go[o][g] = (unsigned char)k;
      for (int e = 0; e < 189; ++e) {
        const int t = v[o][e];
        const int gg = (h[t][0] + 3) * 4 + ((oy + h[t][1]) & 1) * 2 + ((oz + h[t][2]) & 1);
        if (gg == g) gr[o][k++] = (short)t;
      }
    }
    go[o][28] = (unsigned char)k;
  }
  cudaMemcpyToSymbol(c_grp, gr, sizeof(gr));
  cudaMemcpyToSymbol(c_grp_off, go, sizeof(go));
  g_offsets_ready |= bit;
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
#include "m2l_i8.cuh"
#include "proj_i8.cuh"

// ----------------------------------------------------------------------------
// Basis projections on the FP64 tensor cores: C = alpha * A @ B (+ beta C),
// A row-major (rows, K) with row stride lda, B row-major (K, N).  CTA tile
// 64 rows x 64*WN columns, warp (wr, wc) owns rows 16 wr.. and columns
// 64 wc..; K is staged 16 at a time through a kPjStages-deep cp.async ring
// (8-byte copies: rows of 125 doubles are not 16-byte aligned), each thread
// owning fixed tile slots so a refill is a handful of pointer bumps.
// Strides: A 20 doubles, B 64*WN + 8, so each 8 x 4 DMMA fragment load is two
// conflict-free wavefronts.
constexpr int kPjTM = 64, kPjKC = 16, kPjLDA = 20, kPjStages = 4;

template <int WN>
constexpr int pj_ldb() { return 64 * WN + 8; }
template <int WN>
constexpr size_t pj_smem() {
  return sizeof(double) * kPjStages * (kPjTM * kPjLDA + kPjKC * pj_ldb<WN>());
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}

template <int WN>
__global__ void __launch_bounds__(128 * WN)
proj_gemm_kernel(const double *__restrict__ A, int64_t rows, int64_t lda, int K,
                 const double *__restrict__ B, int N, double *__restrict__ C, double alpha,
                 double beta, const int64_t *__restrict__ groups, int64_t group_rows,
                 int gather_a) {
  constexpr int TN = 64 * WN, NT = 8, LDB = pj_ldb<WN>(), NTH = 128 * WN;
  constexpr int A_ELEMS = kPjTM * kPjLDA, STAGE = A_ELEMS + kPjKC * LDB;
  constexpr int AEPT = kPjTM * kPjKC / NTH;  // A slots per thread
  constexpr int BEPT = kPjKC * TN / NTH;      // B slots per thread (8)
  constexpr int AR_STEP = NTH / kPjKC;        // rows between a thread's A slots
  constexpr int BK_STEP = NTH / TN;           // k rows between its B slots
  extern __shared__ __align__(16) double pj[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t row0 = int64_t(blockIdx.x) * kPjTM;
  const int n0 = blockIdx.y * TN;
  const int nk = (K + kPjKC - 1) / kPjKC;
  // slot u of a thread: A (row ar + u AR_STEP, k ak), B (k bk + u BK_STEP,
  // column bn): consecutive lanes walk consecutive k of a row (A) and
  // consecutive columns (B), so each copy instruction touches 2-4 lines
  const int ar = tid / kPjKC, ak = tid % kPjKC;
  const int bk = tid / TN, bn = tid % TN;
  const bool bn_ok = n0 + bn < N;
  auto issue = [&](int chunk) {
    double *As = pj + (chunk % kPjStages) * STAGE, *Bs = As + A_ELEMS;
    const int k0 = chunk * kPjKC;
    const bool akv = k0 + ak < K;
#pragma unroll
    for (int u = 0; u < AEPT; ++u) {
      const int64_t r = row0 + ar + u * AR_STEP;
      const bool v = akv && r < rows;
      // gather_a: A rows live at their cells too (row map as for C)
      const int64_t ra = (gather_a && v) ? c_row(r, groups, group_rows) : r;
      cp_async8(As + (ar + u * AR_STEP) * kPjLDA + ak, v ? A + ra * lda + k0 + ak : A, v);
    }
#pragma unroll
    for (int u = 0; u < BEPT; ++u) {
      const int k = k0 + bk + u * BK_STEP;
      const bool v = bn_ok && k < K;
      cp_async8(Bs + (bk + u * BK_STEP) * LDB + bn, v ? B + (int64_t)k * N + n0 + bn : B, v);
    }
  };
  double acc[2][NT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int st = 0; st < kPjStages - 1; ++st) {
    if (st < nk) issue(st);
    cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<kPjStages - 2>();
    __syncthreads();
    // refill the stage consumed last iteration (everyone is past it now)
    if (kc + kPjStages - 1 < nk) issue(kc + kPjStages - 1);
    cp_async_commit();
    const double *As = pj + (kc % kPjStages) * STAGE, *Bs = As + A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < kPjKC; ks += 4) {
      double a[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = As[(wr * 16 + i * 8 + g) * kPjLDA + ks + t4];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const double b = Bs[(ks + t4) * LDB + wc * 64 + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 2; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b);
      }
    }
  }
  cp_async_wait<0>();
  if (WN == 2 && !groups && beta == 0.0 && gridDim.y == 1) {
    // all N columns in this CTA and a plain row range: stage the 64 x N tile
    // in the (now idle) ring and write it as one contiguous block of C, rows
    // whole, instead of 8-byte stores spread over 8 rows per instruction
    constexpr int CLD = 64 * WN + 2;
    __syncthreads();
    double *Cs = pj;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int rl = wr * 16 + i * 8 + g;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int n = wc * 64 + j * 8 + 2 * t4;
        Cs[rl * CLD + n] = alpha * acc[i][j][0];
        Cs[rl * CLD + n + 1] = alpha * acc[i][j][1];
      }
    }
    __syncthreads();
    const int nr = rows - row0 < kPjTM ? (int)(rows - row0) : kPjTM;
    double *cblk = C + row0 * N;
    for (int e = tid; e < nr * N; e += NTH) {
      const int rl = e / N, n = e - rl * N;
      cblk[e] = Cs[rl * CLD + n];
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t r = row0 + wr * 16 + i * 8 + g;
    if (r >= rows) continue;
    double *crow = C + c_row(r, groups, group_rows) * N;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wc * 64 + j * 8 + 2 * t4 + h;
        if (n >= N) continue;
        double v = alpha * acc[i][j][h];
        if (beta != 0.0) v += beta * crow[n];
        crow[n] = v;
      }
    }
  }
}

// Persistent variant for the big levels (no split blocks, no row groups):
// the whole B (<= 128 x 136 doubles, 70-74 KB) is staged once per CTA and
// stays resident, and the A ring runs across row tiles without draining --
// the per-stage B copies and the per-tile pipeline restarts of
// proj_gemm_kernel go away.  Two CTAs per SM (3-stage ring).  Optional
// epilogue: zmax = max |C| (bit pattern, atomicMax; one weight column),
// the digit scale of the int8 M2L, which then skips its absmax pass.
constexpr int kPjResStages = 3;
// WN = 2 (N > 64, e.g. locals = lt U^T with N = p^3 = 125): the tile's
// 64 x N outputs are staged in shared memory and written as whole rows
// (the tile is one contiguous 64 N-double block of C), instead of 8-byte
// stores scattered over 8 rows per instruction
constexpr int kPjCLD = 130;
constexpr int kPjResMaxK2 = 80;  // WN = 2: resident B + ring + C stage <= 184 KB
template <int WN>
constexpr size_t pj_res_smem(int K) {
  return sizeof(double) * ((size_t)((K + kPjKC - 1) / kPjKC) * kPjKC * pj_ldb<WN>() +
                           kPjResStages * kPjTM * kPjLDA + (WN == 2 ? kPjTM * kPjCLD : 0));
}

template <int WN>
__global__ void __launch_bounds__(128 * WN, 2)
proj_gemm_res_kernel(const double *__restrict__ A, int64_t rows, int64_t lda, int K,
                     const double *__restrict__ B, int N, double *__restrict__ C, double alpha,
                     unsigned long long *__restrict__ zmax) {
  constexpr int TN = 64 * WN, NT = 8, LDB = pj_ldb<WN>(), NTH = 128 * WN;
  constexpr int A_ELEMS = kPjTM * kPjLDA;
  constexpr int AEPT = kPjTM * kPjKC / NTH;  // A slots per thread
  constexpr int AR_STEP = NTH / kPjKC;
  extern __shared__ __align__(16) double pj[];
  const int nk = (K + kPjKC - 1) / kPjKC;
  double *Bs = pj;                         // [nk * 16][LDB], resident
  double *As0 = pj + (size_t)nk * kPjKC * LDB;  // [kPjResStages][A_ELEMS]
  double *Cs = As0 + kPjResStages * A_ELEMS;    // [64][kPjCLD] (WN == 2)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t ntiles = (rows + kPjTM - 1) / kPjTM;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // B once: rows k < K, columns n < N, zeros elsewhere
  for (int e = tid; e < nk * kPjKC * TN; e += NTH) {
    const int k = e / TN, n = e - k * TN;
    const bool v = k < K && n < N;
    cp_async8(Bs + k * LDB + n, v ? B + (int64_t)k * N + n : B, v);
  }
  cp_async_commit();
  const int ar = tid / kPjKC, ak = tid % kPjKC;
  // chunk q of this CTA: tile index q / nk of its sequence, k chunk q % nk
  auto issue = [&](int64_t q) {
    double *As = As0 + (q % kPjResStages) * A_ELEMS;
    const int64_t row0 = (blockIdx.x + (q / nk) * gridDim.x) * kPjTM;
    const int k0 = (int)(q % nk) * kPjKC;
    const bool akv = k0 + ak < K;
#pragma unroll
    for (int u = 0; u < AEPT; ++u) {
      const int64_t r = row0 + ar + u * AR_STEP;
      const bool v = akv && r < rows;
      cp_async8(As + (ar + u * AR_STEP) * kPjLDA + ak, v ? A + r * lda + k0 + ak : A, v);
    }
  };
  const int64_t nq = my_tiles * nk;
#pragma unroll
  for (int st = 0; st < kPjResStages - 1; ++st) {
    if (st < nq) issue(st);
    cp_async_commit();
  }
  double amax = 0.0;
  for (int64_t i = 0; i < my_tiles; ++i) {
    double acc[2][NT][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[a][j][0] = acc[a][j][1] = 0.0;
    for (int kc = 0; kc < nk; ++kc) {
      const int64_t q = i * nk + kc;
      cp_async_wait<kPjResStages - 2>();
      __syncthreads();
      if (q + kPjResStages - 1 < nq) issue(q + kPjResStages - 1);
      cp_async_commit();
      const double *As = As0 + (q % kPjResStages) * A_ELEMS;
      const double *Bk = Bs + kc * kPjKC * LDB;
#pragma unroll
      for (int ks = 0; ks < kPjKC; ks += 4) {
        double a[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) a[u] = As[(wr * 16 + u * 8 + g) * kPjLDA + ks + t4];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const double b = Bk[(ks + t4) * LDB + wc * 64 + j * 8 + g];
#pragma unroll
          for (int u = 0; u < 2; ++u) dmma_8x8x4(acc[u][j][0], acc[u][j][1], a[u], b);
        }
      }
    }
    const int64_t row0 = (blockIdx.x + i * gridDim.x) * kPjTM;
    if constexpr (WN == 2) {
      // stage, then whole contiguous rows (the A ring is untouched: Cs is its own)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int rl = wr * 16 + u * 8 + g;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int n = wc * 64 + j * 8 + 2 * t4;
          Cs[rl * kPjCLD + n] = alpha * acc[u][j][0];
          Cs[rl * kPjCLD + n + 1] = alpha * acc[u][j][1];
        }
      }
      __syncthreads();
      const int nr = rows - row0 < kPjTM ? (int)(rows - row0) : kPjTM;
      double *cblk = C + row0 * N;
      for (int e = tid; e < nr * N; e += NTH) {
        const int rl = e / N, n = e - rl * N;
        const double v = Cs[rl * kPjCLD + n];
        cblk[e] = v;
        amax = fmax(amax, fabs(v));
      }
      __syncthreads();  // Cs is rewritten by the next tile
    } else {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t r = row0 + wr * 16 + u * 8 + g;
        if (r >= rows) continue;
        double *crow = C + r * N;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int n = wc * 64 + j * 8 + 2 * t4;
          const double v0 = alpha * acc[u][j][0], v1 = alpha * acc[u][j][1];
          if (n + 1 < N && (N % 2 == 0)) {  // 16-byte aligned pair (even row stride)
            *reinterpret_cast<double2 *>(crow + n) = make_double2(v0, v1);
          } else {
            if (n < N) crow[n] = v0;
            if (n + 1 < N) crow[n + 1] = v1;
          }
          if (n < N) amax = fmax(amax, fabs(v0));
          if (n + 1 < N) amax = fmax(amax, fabs(v1));
        }
      }
    }
  }
  cp_async_wait<0>();
  if (zmax) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0 && amax > 0) atomicMax(zmax, (unsigned long long)__double_as_longlong(amax));
  }
}

// A[r][0][k] = sum_s A[r][s][k] in place for many splits: CTA per row, the
// splits dealt round-robin to G = 256 / K thread groups that sum theirs in
// order, then the G partials are added in group order (fixed tree, so the
// result is the same on every run).
__global__ void __launch_bounds__(256)
reduce_splits_wide_kernel(double *__restrict__ A, int64_t rows, int K, int a_splits) {
  __shared__ double part[256];
  const int G = 256 / K;
  const int t = threadIdx.x, k = t % K, grp = t / K;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    double *a = A + r * a_splits * (int64_t)K;
    double v = 0.0;
    if (grp < G) {
#pragma unroll 4
      for (int sp = grp; sp < a_splits; sp += G) v += a[(int64_t)sp * K + k];
      part[grp * K + k] = v;
    }
    __syncthreads();
    if (t < K) {
      double s = part[t];
      for (int gi = 1; gi < G; ++gi) s += part[gi * K + t];
      a[t] = s;
    }
    __syncthreads();
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

static int rows_gemm_res(const double *A, int64_t rows, int64_t lda, int K, const double *B,
                         int N, double *C, double alpha, unsigned long long *zmax,
                         cudaStream_t st) {
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(proj_gemm_res_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)pj_res_smem<1>(128));
    cudaFuncSetAttribute(proj_gemm_res_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)pj_res_smem<2>(kPjResMaxK2));
  }
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(rows, kPjTM), 2 * kNumSMs);
  if (N > 64)
    proj_gemm_res_kernel<2><<<grid, 256, pj_res_smem<2>(K), st>>>(A, rows, lda, K, B, N, C, alpha,
                                                                  zmax);
  else
    proj_gemm_res_kernel<1><<<grid, 128, pj_res_smem<1>(K), st>>>(A, rows, lda, K, B, N, C, alpha,
                                                                  zmax);
  return check_launch("proj_gemm_res_kernel");
}

static int rows_gemm(const double *A, int64_t rows, int K, const double *B, int N,
                     double *C, double alpha, double beta, int a_splits,
                     const int64_t *groups, int64_t group_rows,
                     bfmm_stream_t stream, int gather_a = 0) {
  if (rows <= 0 || N <= 0) return 0;
  if (a_splits < 1 || K < 1) {
    set_error("bfmm_rows_gemm: a_splits=%d K=%d", a_splits, K);
    return 2;
  }
  cudaStream_t st = as_stream(stream);
  // split blocks are first summed in place into block 0, in a fixed order
  if (a_splits > 16 && K <= 256) {
    reduce_splits_wide_kernel<<<(unsigned)std::min<int64_t>(rows, 65535), 256, 0, st>>>(
        const_cast<double *>(A), rows, K, a_splits);
    if (check_launch("reduce_splits_wide_kernel")) return 1;
  } else if (a_splits > 1) {
    reduce_splits_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * K, 256), 8192), 256, 0,
                           st>>>(const_cast<double *>(A), rows, K, a_splits);
    if (check_launch("reduce_splits_kernel")) return 1;
  }
  const int64_t lda = (int64_t)a_splits * K;
  // big plain levels: the persistent kernel with B resident
  // (N <= 64 only: for N = p^3 = 125 the staged WN = 2 variant measured
  // slower than the tiled kernel -- one CTA per SM, C5 Uᵀ 16.0 -> 19.7 ms)
  if (!groups && K <= 128 && N <= 64 && beta == 0.0 && ceil_div(rows, kPjTM) >= 8 * kNumSMs &&
      !getenv("BFMM_PJ_TILED"))
    return rows_gemm_res(A, rows, lda, K, B, N, C, alpha, nullptr, st);
  // one CTA spans all N <= 128 columns, so A is read once -- unless that
  // leaves most SMs idle (small levels): then 64-column tiles, twice the CTAs
  const int wn = (N > 64 && ceil_div(rows, kPjTM) >= kNumSMs) ? 2 : 1;
  dim3 grid((unsigned)ceil_div(rows, kPjTM), (unsigned)ceil_div(N, 64 * wn));
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(proj_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)pj_smem<1>());
    cudaFuncSetAttribute(proj_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)pj_smem<2>());
  }
  if (wn == 2)
    proj_gemm_kernel<2><<<grid, 256, pj_smem<2>(), st>>>(A, rows, lda, K, B, N, C, alpha,
                                                        beta, groups, group_rows, gather_a);
  else
    proj_gemm_kernel<1><<<grid, 128, pj_smem<1>(), st>>>(A, rows, lda, K, B, N, C, alpha,
                                                        beta, groups, group_rows, gather_a);
  return check_launch("proj_gemm_kernel");
}

extern "C" int bfmm_rows_gemm(const double *A, int64_t rows, int K,
                              const double *B, int N, double *C, double alpha,
                              double beta, int a_splits, bfmm_stream_t stream) {
  return rows_gemm(A, rows, K, B, N, C, alpha, beta, a_splits, nullptr, 1, stream);
}

extern "C" int bfmm_rows_gemm_max(const double *A, int64_t rows, int K, const double *B, int N,
                                  double *C, double alpha, unsigned long long *zmax,
                                  bfmm_stream_t stream) {
  if (K < 1 || K > 128 || N < 1 || N > 128 || rows < 0 || !zmax) {
    set_error("bfmm_rows_gemm_max: K=%d N=%d (1..128), zmax=%p", K, N, (void *)zmax);
    return 2;
  }
  if (rows == 0) return 0;
  if (N > 64 && K > kPjResMaxK2) {
    set_error("bfmm_rows_gemm_max: K=%d > %d with N=%d > 64", K, kPjResMaxK2, N);
    return 2;
  }
  return rows_gemm_res(A, rows, K, K, B, N, C, alpha, zmax, as_stream(stream));
}

extern "C" int bfmm_rows_gemm_i8(const double *A, int64_t rows, int K, const int8_t *bdig,
                                 const double *bpow, int N, double *C, double alpha,
                                 unsigned long long *zmax, bfmm_stream_t stream) {
  if (K < 1 || K > 128 || N < 1 || N > 128 || rows < 0) {
    set_error("bfmm_rows_gemm_i8: K=%d N=%d (1..128)", K, N);
    return 2;
  }
  if (rows == 0) return 0;
  cudaStream_t st = as_stream(stream);
  const int kc = (int)ceil_div(K, 32), ntn = (int)ceil_div(N, 64);
#define BFMM_PJ(KC, NT)                                                                   \
  if (kc == KC && ntn == NT)                                                              \
    return launch_proj_i8<KC, NT>(A, rows, K, K, bdig, bpow, N, C, alpha, zmax, st);
  BFMM_PJ(1, 1) BFMM_PJ(2, 1) BFMM_PJ(3, 1) BFMM_PJ(4, 1)
  BFMM_PJ(1, 2) BFMM_PJ(2, 2) BFMM_PJ(3, 2) BFMM_PJ(4, 2)
#undef BFMM_PJ
  set_error("bfmm_rows_gemm_i8: unreachable K=%d N=%d", K, N);
  return 2;
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

extern "C" int bfmm_rows_gemm_cells(const double *A, int64_t rows, int K, const double *B,
                                    int N, double *C, double alpha, const int64_t *groups,
                                    int64_t group_rows, bfmm_stream_t stream) {
  if (!groups || group_rows < 1) {
    set_error("bfmm_rows_gemm_cells: groups=%p group_rows=%lld", (const void *)groups,
              (long long)group_rows);
    return 2;
  }
  return rows_gemm(A, rows, K, B, N, C, alpha, 0.0, 1, groups, group_rows, stream, 1);
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
  M2LCall a{z, lt, level, m, rp, nsplit, q_lo, nq, OctList{nullptr, {}}, cores,
            as_stream(stream)};
  return dispatch_ws(m2l_mw(nq * m), m2l_nt8(rp), a);
}

extern "C" int bfmm_m2l_cheb_cells(const double *z, double *lt, int level, int m,
                                   int rp, int nsplit, const int64_t *cells,
                                   const int64_t *oct_off, const double *cores,
                                   bfmm_stream_t stream) {
  if (rp % 8 != 0 || rp <= 0 || level < 2 || level > 10) {
    set_error("bfmm_m2l_cheb_cells: rp=%d must be a positive multiple of 8, level=%d",
              rp, level);
    return 2;
  }
  if (nsplit < 1 || nsplit > 189) {
    set_error("bfmm_m2l_cheb_cells: nsplit=%d outside [1, 189]", nsplit);
    return 2;
  }
  OctList act{cells, {}};
  int64_t longest = 0;
  for (int o = 0; o <= 8; ++o) {
    act.off[o] = oct_off[o];
    if (o > 0 && (oct_off[o] < oct_off[o - 1])) {
      set_error("bfmm_m2l_cheb_cells: octant offsets not ascending");
      return 2;
    }
    if (o > 0) longest = std::max(longest, oct_off[o] - oct_off[o - 1]);
  }
  if (oct_off[8] > (int64_t(1) << (3 * level)) || (oct_off[8] > 0 && !cells)) {
    set_error("bfmm_m2l_cheb_cells: %lld listed cells invalid at level %d",
              (long long)oct_off[8], level);
    return 2;
  }
  if (oct_off[8] == 0) return 0;
  ensure_offsets();
  M2LCall a{z, lt, level, m, rp, nsplit, 0, 0, act, cores, as_stream(stream)};
  return dispatch_ws(m2l_mw(longest * m), m2l_nt8(rp), a);
}

// ---- int8 tensor-core M2L (m2l_i8.cuh) ----
// S argument: digits per operand, | BFMM_I8_BASE256 for 8-bit digits
static void i8_digits(int Sarg, int *S, int *B) {
  *B = (Sarg & BFMM_I8_BASE256) ? 8 : 7;
  *S = Sarg & 0xff;
}

extern "C" size_t bfmm_m2l_i8_zs_bytes(int64_t rows, int rp, int Sarg) {
  return (size_t)rows * ceil_div(rp, 32) * (Sarg & 0xff) * 32;
}

static int i8_zmax(const double *z, int64_t rows, int m, int rp, unsigned long long *zmax,
                   const int64_t *groups, bfmm_stream_t stream) {
  if (rp <= 0 || rows < 0 || m < 1 || m > 65535 || rows % m) {
    set_error("bfmm_m2l_i8_zmax: rp=%d, m=%d, rows=%lld", rp, m, (long long)rows);
    return 2;
  }
  cudaStream_t st = as_stream(stream);
  if (cudaMemsetAsync(zmax, 0, sizeof(unsigned long long) * m, st) != cudaSuccess) {
    set_error("bfmm_m2l_i8_zmax: memset failed");
    return 1;
  }
  if (rows == 0) return 0;
  const int64_t n = rows / m * rp;
  absmax_bits_kernel<<<dim3((unsigned)std::min<int64_t>(ceil_div(n, 256), 4 * kNumSMs), m), 256,
                       0, st>>>(z, rows, rp, m, zmax, groups);
  return check_launch("absmax_bits_kernel");
}

extern "C" int bfmm_m2l_i8_zmax(const double *z, int64_t rows, int m, int rp,
                                unsigned long long *zmax, bfmm_stream_t stream) {
  return i8_zmax(z, rows, m, rp, zmax, nullptr, stream);
}

static int i8_slice_z(const double *z, int64_t rows, int m, int rp, int Sarg, int8_t *zs,
                      unsigned long long *zmax, const int64_t *groups, bfmm_stream_t stream) {
  int S, B;
  i8_digits(Sarg, &S, &B);
  if (rp <= 0 || rp > 256 || S < 5 || S > 8 || (B == 8 && S != 6) || rows < 0 || m < 1 ||
      m > 65535 || rows % m) {
    set_error("bfmm_m2l_i8_slice_z: rp=%d (1..256), S=%d (5..8; 6 for 8-bit digits), rows=%lld",
              rp, S, (long long)rows);
    return 2;
  }
  cudaStream_t st = as_stream(stream);
  if (!(Sarg & BFMM_I8_ZMAX_GIVEN)) {
    if (int rc = i8_zmax(z, rows, m, rp, zmax, groups, stream)) return rc;
  }
  if (rows == 0) return 0;
  const int kc_n = (int)ceil_div(rp, 32);
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(rows * kc_n * 2, 256), 16 * kNumSMs);
  if (B == 8) {
    z_slice_kernel<6, 8><<<grid, 256, 0, st>>>(z, rows, rp, kc_n, m, zmax, zs, groups);
  } else {
    switch (S) {
      case 5: z_slice_kernel<5, 7><<<grid, 256, 0, st>>>(z, rows, rp, kc_n, m, zmax, zs, groups); break;
      case 6: z_slice_kernel<6, 7><<<grid, 256, 0, st>>>(z, rows, rp, kc_n, m, zmax, zs, groups); break;
      case 7: z_slice_kernel<7, 7><<<grid, 256, 0, st>>>(z, rows, rp, kc_n, m, zmax, zs, groups); break;
      default: z_slice_kernel<8, 7><<<grid, 256, 0, st>>>(z, rows, rp, kc_n, m, zmax, zs, groups); break;
    }
  }
  return check_launch("z_slice_kernel");
}

extern "C" int bfmm_m2l_i8_slice_z(const double *z, int64_t rows, int m, int rp, int Sarg,
                                   int8_t *zs, unsigned long long *zmax, bfmm_stream_t stream) {
  return i8_slice_z(z, rows, m, rp, Sarg, zs, zmax, nullptr, stream);
}

extern "C" int bfmm_m2l_i8_slice_z_cells(const double *z, int64_t rows, int m, int rp, int Sarg,
                                         int8_t *zs, unsigned long long *zmax,
                                         const int64_t *cells, bfmm_stream_t stream) {
  if (!cells) {
    set_error("bfmm_m2l_i8_slice_z_cells: cell list required");
    return 2;
  }
  return i8_slice_z(z, rows, m, rp, Sarg, zs, zmax, cells, stream);
}

extern "C" int bfmm_m2l_i8_splits(int level, int m, int rp, int64_t nq) {
  if (level <= 3) {  // mixed-octant rows, 316 offsets (m2l_i8_kernel)
    const int64_t ctas = ceil_div(8 * nq * m, kI8TM) * ceil_div(rp, kI8TN);
    return (int)std::max<int64_t>(1, std::min<int64_t>(79, ceil_div(kNumSMs, ctas)));
  }
  const int64_t ctas = ceil_div(nq * m, kI8TM) * ceil_div(rp, kI8TN) * 8;
  const double slots = kNumSMs;  // one CTA per SM (TMEM 512 columns, ~215 KB smem)
  if (ctas * 4 < slots) return (int)std::min<int64_t>(189, ceil_div(4 * (int64_t)slots, ctas));
  int best = 1;
  double best_score = -1e30;
  for (int s = 1; s <= 16; ++s) {
    const double waves = ctas * s / slots;
    const double score = waves / std::ceil(waves) - 0.006 * s;
    if (score > best_score + 1e-12) {
      best_score = score;
      best = s;
    }
  }
  return best;
}

static int i8_check(const char *fn, int level, int m, int rp, int S, int B, int nsplit,
                    bool listed) {
  if (B == 8) {
    // 8-bit digits: |digit product| <= 2^14, at most 6 products per
    // accumulator, K = offsets x 32 x ceil(rp/32) terms each: the exact
    // int32 accumulation needs 6 K 2^14 < 2^31 (189 offsets per octant; the
    // mixed-octant rows of dense levels <= 3 walk all 316)
    const int64_t offs = (level <= 3 && !listed) ? 316 : 189;
    if (S != 6 || 6 * offs * 32 * ceil_div(rp, 32) * 16384 >= (int64_t(1) << 31)) {
      set_error("%s: 8-bit digits need S = 6 and 6 K 2^14 < 2^31 (rp=%d, level=%d)", fn, rp,
                level);
      return 2;
    }
  }
  if (m < 1 || (int64_t(1) << (3 * level)) * m >= (int64_t(1) << 31)) {
    set_error("%s: 8^%d cells x %d columns exceed the 32-bit row index", fn, level, m);
    return 2;
  }
  if (rp % 8 != 0 || rp <= 0 || rp > 256 || level < 2 || level > 10 || S < 5 || S > 8) {
    set_error("%s: rp=%d (multiple of 8, <= 256), level=%d, S=%d (5..8)", fn, rp, level, S);
    return 2;
  }
  if (nsplit < 1 || nsplit > 316) {
    set_error("%s: nsplit=%d outside [1, 316]", fn, nsplit);
    return 2;
  }
  return 0;
}

extern "C" int bfmm_m2l_i8(const int8_t *zs, const unsigned long long *zmax, const int8_t *cs,
                           const double *cpow, double *lt, int level, int m, int rp, int Sarg,
                           int nsplit, int64_t q_lo, int64_t nq, bfmm_stream_t stream) {
  int S, B;
  i8_digits(Sarg, &S, &B);
  if (int rc = i8_check("bfmm_m2l_i8", level, m, rp, S, B, nsplit, false)) return rc;
  const int64_t nparent = int64_t(1) << (3 * level - 3);
  if (q_lo < 0 || nq < 0 || q_lo + nq > nparent) {
    set_error("bfmm_m2l_i8: parent range [%lld, %lld) outside [0, %lld)", (long long)q_lo,
              (long long)(q_lo + nq), (long long)nparent);
    return 2;
  }
  ensure_offsets();
  I8Call a{zs, zmax, cs, cpow, lt, level, m, rp, (int)ceil_div(rp, 32), (int)ceil_div(rp, kI8TN),
           nsplit, q_lo, nq, OctList{nullptr, {}}, as_stream(stream)};
  return dispatch_i8(S, B, a);
}

extern "C" int bfmm_m2l_i8_cells(const int8_t *zs, const unsigned long long *zmax,
                                 const int8_t *cs, const double *cpow, double *lt, int level,
                                 int m, int rp, int Sarg, int nsplit, const int64_t *cells,
                                 const int64_t *oct_off, bfmm_stream_t stream) {
  int S, B;
  i8_digits(Sarg, &S, &B);
  if (int rc = i8_check("bfmm_m2l_i8_cells", level, m, rp, S, B, nsplit, true)) return rc;
  OctList act{cells, {}};
  for (int o = 0; o <= 8; ++o) {
    act.off[o] = oct_off[o];
    if (o > 0 && oct_off[o] < oct_off[o - 1]) {
      set_error("bfmm_m2l_i8_cells: octant offsets not ascending");
      return 2;
    }
  }
  if (oct_off[8] > (int64_t(1) << (3 * level)) || (oct_off[8] > 0 && !cells)) {
    set_error("bfmm_m2l_i8_cells: %lld listed cells invalid at level %d", (long long)oct_off[8],
              level);
    return 2;
  }
  if (oct_off[8] == 0) return 0;
  ensure_offsets();
  I8Call a{zs, zmax, cs, cpow, lt, level, m, rp, (int)ceil_div(rp, 32), (int)ceil_div(rp, kI8TN),
           nsplit, 0, 0, act, as_stream(stream)};
  return dispatch_i8(S, B, a);
}

#ifdef BFMM_I8_TRACE
extern "C" int bfmm_i8_trace_read(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, bfmm::g_i8_trace, sizeof(long long) * 8192);
}
#endif
