// Uniform-grid far field (engine.py:258-292): the 316 translation operators
// are nested-Toeplitz on the equispaced node grid, so each is a circulant
// convolution on a q^3 grid (q = 2p - 1) and diagonal in the real-FFT basis.
//
// Per level and per chunk of weight columns:
//   1. fft_fwd_kernel : X[col][f][cell] = rfftn(pad_q(M[cell, col]))[f]
//   2. stencil_kernel : Y[col][f][c] = sum_{t valid} S_t[f] X[col][f][c + t]
//   3. fft_inv_kernel : L[c, col] = scale * irfftn(Y[col][:][c])[:p,:p,:p]
// f = (kx*q + ky)*(q/2+1) + kz indexes numpy's rfftn output layout
// (ops:156-159), so the symbols S_t are the reference's table verbatim.
//
// Spectra are stored frequency-major with cells in lexicographic (x, y, z)
// order: for one frequency the Hadamard accumulation is a 3-D stencil with
// 189 complex taps over the cell grid, which stencil_kernel
// tiles through shared memory (an 8 x 8 x 8 target tile plus its 3-cell
// halo) and blocks in registers along z (each thread owns 4 same-parity
// targets, so one z-column of 13 sources serves 7 taps x 4 targets).
// The transforms are direct DFTs along each axis with exactly tabulated
// twiddles: zero padding makes them cheaper than a generic FFT.
#include <algorithm>

#include <mutex>

#include "common.cuh"


namespace bfmm {
namespace {

constexpr int kMaxQ = 23;  // p <= 12

struct FftGeom {
  int p, q, h;  // h = q/2 + 1 bins along z
  double c[kMaxQ], s[kMaxQ];  // cos / sin(2 pi r / q)
};

__device__ __forceinline__ int64_t lex_of(int x, int y, int z, int n) {
  return ((int64_t)x * n + y) * n + z;
}

// The transforms work on G lexicographically consecutive cells (a z-run)
// per CTA pass, so the frequency-major spectra are written / read as
// G * 16-byte runs instead of isolated 16-byte values, and every
// spectrum value is touched once.  Twiddles come from a q x q shared table
// tw[a][b] = e^{2 pi i (a b mod q) / q} (no integer modulo in the loops).
// G = 2 cells per run when the tiles fit in shared memory, else 1 (large
// p); fft_group() picks it.

__device__ __forceinline__ void stage_twiddles(const FftGeom &g, double2 *tw) {
  for (int e = threadIdx.x; e < g.q * g.q; e += blockDim.x) {
    const int r = ((e / g.q) * (e % g.q)) % g.q;
    tw[e] = make_double2(g.c[r], g.s[r]);
  }
}

inline size_t fft_fwd_smem(const FftGeom &g, int G) {
  const size_t F = size_t(g.q) * g.q * g.h;
  return sizeof(double2) * (g.q * g.q + G * (g.p * g.p * g.h + g.p * g.q * g.h) + F * G) +
         sizeof(double) * G * g.p * g.p * g.p;
}

// ---- 1. forward transform: X[col][f][lex] = rfftn(pad_q(M[cell, col]))[f] ---
// P is a template parameter so the short DFT sums unroll and each thread's
// independent outputs (2 per pass iteration) interleave their FMA chains.
template <int P>
__global__ void __launch_bounds__(128)
fft_fwd_kernel(const double *__restrict__ moments, int level, int m, int c0,
               int cc, FftGeom g, int G, double2 *__restrict__ X) {
  extern __shared__ double2 sm2[];
  constexpr int p = P, q = 2 * P - 1, h = q / 2 + 1, F = q * q * h;
  const int P3 = p * p * p, PPH = p * p * h, PQH = p * q * h;
  const int n = 1 << level;
  const int64_t ncell = int64_t(1) << (3 * level);
  const int64_t ngroups = ncell / G;
  double2 *tw = sm2;                   // [q][q]
  double2 *A = tw + q * q;             // [G][p][p][h]  z transformed
  double2 *B = A + G * PPH;        // [G][p][q][h]  y transformed
  double2 *stage = B + G * PQH;    // [F][G]        x transformed
  double *in = reinterpret_cast<double *>(stage + F * G);  // [G][p^3]
  stage_twiddles(g, tw);
  for (int64_t w = blockIdx.x; w < ngroups * cc; w += gridDim.x) {
    const int crel = (int)(w / ngroups);
    const int64_t lex0 = (w - crel * ngroups) * G;
    __syncthreads();
    #pragma unroll 2
    for (int e = threadIdx.x; e < G * P3; e += blockDim.x) {
      const int gi = e / P3, r = e - gi * P3;
      const int64_t lex = lex0 + gi;
      const int x = (int)(lex / ((int64_t)n * n)), y = (int)((lex / n) % n), z = (int)(lex % n);
      in[e] = moments[((int64_t)morton3(x, y, z) * m + c0 + crel) * P3 + r];
    }
    __syncthreads();
    // z: real -> h complex bins, e^{-2 pi i k kz / q}
    #pragma unroll 2
    for (int e = threadIdx.x; e < G * PPH; e += blockDim.x) {
      const int gi = e / PPH, r = e - gi * PPH, ij = r / h, kz = r - ij * h;
      const double *v = in + gi * P3 + ij * p;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int k = 0; k < p; ++k) {
        const double2 t = tw[k * q + kz];
        re = fma(v[k], t.x, re);
        im = fma(-v[k], t.y, im);
      }
      A[e] = make_double2(re, im);
    }
    __syncthreads();
    // y: p inputs -> q bins
    #pragma unroll 2
    for (int e = threadIdx.x; e < G * PQH; e += blockDim.x) {
      const int gi = e / PQH, r = e - gi * PQH;
      const int i = r / (q * h), rem = r - i * q * h, ky = rem / h, kz = rem - ky * h;
      const double2 *a = A + gi * PPH + i * p * h + kz;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int j = 0; j < p; ++j) {
        const double2 t = tw[j * q + ky], v = a[j * h];
        re = fma(v.x, t.x, fma(v.y, t.y, re));  // (v.x + i v.y)(c - i s)
        im = fma(v.y, t.x, fma(-v.x, t.y, im));
      }
      B[e] = make_double2(re, im);
    }
    __syncthreads();
    // x: p inputs -> q bins, into the [f][cell] staging tile
    #pragma unroll 2
    for (int e = threadIdx.x; e < F * G; e += blockDim.x) {
      const int f = e / G, gi = e - f * G;
      const int kx = f / (q * h), rem = f - kx * q * h;
      const double2 *b = B + gi * PQH + rem;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int i = 0; i < p; ++i) {
        const double2 t = tw[i * q + kx], v = b[i * q * h];
        re = fma(v.x, t.x, fma(v.y, t.y, re));
        im = fma(v.y, t.x, fma(-v.x, t.y, im));
      }
      stage[e] = make_double2(re, im);
    }
    __syncthreads();
    double2 *dst = X + (int64_t)crel * F * ncell + lex0;
    #pragma unroll 2
    for (int e = threadIdx.x; e < F * G; e += blockDim.x) {
      const int f = e / G, gi = e - f * G;
      dst[(int64_t)f * ncell + gi] = stage[e];
    }
  }
}

// ---- 2. Hadamard accumulation as a per-frequency 3-D stencil ------------------
// 8 x 8 x 8 targets, 128 threads x 4: a 47 KB halo keeps 4 CTAs per SM
// (measured: 16-deep z tiles reuse each source more but fit only 3 CTAs and
// run 3 % slower, the kernel being shared-memory-latency bound)
constexpr int kTX = 8, kTY = 8, kTZ = 8, kR = kTZ / 2;
constexpr int kHX = kTX + 6, kHY = kTY + 6, kHZ = kTZ + 6;
// Bank layout: an LDS.128 is served 8 lanes (one quarter-warp phase) at a
// time, and those 8 lanes must hit 8 distinct 16-byte slots (mod 8).  A
// phase's lanes vary z parity (stride 1) and 4 same-parity x positions
// (stride 2 * HYP * HZP), so the halo is padded to HYP = 15, HZP = 15:
// 2 * 15 * 15 = 450 = 2 (mod 8) -> slots {0,2,4,6} + {0,1}, conflict-free
// (the unpadded 14 x 14 layout is 2-way conflicted).
constexpr int kHYP = kHY + 1, kHZP = kHZ + 1;

// grid: (tiles, frequencies, columns); block (8, 8, 2): thread (ix, iy, pz)
// owns targets (x0+ix, y0+iy, z0+pz+2k), k < kR -- one parity class, so one
// valid-offset set (octree.py:128-145).  The symbol of every offset t sits in
// a 7^3 table (zero for the 27 near offsets).
__global__ void __launch_bounds__(128)
stencil_kernel(const double2 *__restrict__ X, double2 *__restrict__ Y, int level,
               int F, const double2 *__restrict__ S, const short *__restrict__ tap_index,
               int64_t cell_lo, int64_t cell_hi) {
  extern __shared__ double2 sm2[];
  auto halo = reinterpret_cast<double2 (*)[kHYP][kHZP]>(sm2);                   // [kHX][kHYP][kHZP]
  auto taps = reinterpret_cast<double2 (*)[7][7]>(sm2 + kHX * kHYP * kHZP);    // [7][7][7]
  const int n = 1 << level;
  const int64_t ncell = int64_t(1) << (3 * level);
  const int tilesx = (n + kTX - 1) / kTX, tilesy = (n + kTY - 1) / kTY;
  const int tile = blockIdx.x;
  const int tz = tile / (tilesx * tilesy), trem = tile - tz * tilesx * tilesy;
  const int x0 = (trem / tilesy) * kTX, y0 = (trem % tilesy) * kTY, z0 = tz * kTZ;
  const int f = blockIdx.y, col = blockIdx.z;
  // warp w handles the (x, y) parity class (w >> 1, w & 1): its 32 lanes are
  // 2 z-parities (lane bit 0) x 4 same-parity x (bits 1-2) x 4 same-parity y
  // (bits 3-4), so the +-3 offset skips below are warp-uniform (no
  // divergence) and each 8-lane phase of an LDS.128 is conflict-free
  const int tid = (threadIdx.z * kTY + threadIdx.y) * kTX + threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int ix = ((w >> 1) & 1) + 2 * ((lane >> 1) & 3), iy = (w & 1) + 2 * ((lane >> 3) & 3);
  const int pz = lane & 1;
  const int x = x0 + ix, y = y0 + iy;
  // shard filter: skip the tile when none of its targets is ours
  bool mine = false;
#pragma unroll
  for (int k = 0; k < kR; ++k) {
    const int z = z0 + pz + 2 * k;
    if (x < n && y < n && z < n) {
      const int64_t id = (int64_t)morton3(x, y, z);
      mine |= id >= cell_lo && id < cell_hi;
    }
  }
  if (!__syncthreads_or(mine)) return;
  const double2 *Xf = X + ((int64_t)col * F + f) * ncell;
  for (int e = tid; e < kHX * kHY * kHZ; e += 128) {
    const int hx = e / (kHY * kHZ), hr = e - hx * kHY * kHZ, hy = hr / kHZ, hz = hr - hy * kHZ;
    const int sx = x0 + hx - 3, sy = y0 + hy - 3, sz = z0 + hz - 3;
    double2 v = make_double2(0.0, 0.0);
    if (sx >= 0 && sx < n && sy >= 0 && sy < n && sz >= 0 && sz < n) v = Xf[lex_of(sx, sy, sz, n)];
    halo[hx][hy][hz] = v;
  }
  for (int e = tid; e < 343; e += 128) {
    const int t = tap_index[e];
    (&taps[0][0][0])[e] = t >= 0 ? S[(int64_t)t * F + f] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2 acc[kR];
#pragma unroll
  for (int k = 0; k < kR; ++k) acc[k] = make_double2(0.0, 0.0);
  // parity rule: +3 needs an even target coordinate, -3 an odd one
  const int px = x & 1, py = y & 1, pzz = (z0 + pz) & 1;
  for (int a = -3; a <= 3; ++a) {
    if ((a == 3 && px) || (a == -3 && !px)) continue;
    for (int b = -3; b <= 3; ++b) {
      if ((b == 3 && py) || (b == -3 && !py)) continue;
      // the z column of sources for all 8 targets and all 7 z offsets
      double2 seg[kR * 2 + 5];
      const double2 *col_src = &halo[ix + 3 + a][iy + 3 + b][pz];
#pragma unroll
      for (int u = 0; u < kR * 2 + 5; ++u) seg[u] = col_src[u];
#pragma unroll
      for (int c = -3; c <= 3; ++c) {
        if ((c == 3 && pzz) || (c == -3 && !pzz)) continue;
        const double2 s = taps[a + 3][b + 3][c + 3];  // zero for near offsets
#pragma unroll
        for (int k = 0; k < kR; ++k) {
          const double2 v = seg[c + 3 + 2 * k];
          acc[k].x = fma(s.x, v.x, fma(-s.y, v.y, acc[k].x));
          acc[k].y = fma(s.x, v.y, fma(s.y, v.x, acc[k].y));
        }
      }
    }
  }
  double2 *Yf = Y + ((int64_t)col * F + f) * ncell;
#pragma unroll
  for (int k = 0; k < kR; ++k) {
    const int z = z0 + pz + 2 * k;
    if (x < n && y < n && z < n) Yf[lex_of(x, y, z, n)] = acc[k];
  }
}

// ---- 3. inverse transform + crop + scale ------------------------------------
inline size_t fft_inv_smem(const FftGeom &g, int G) {
  const size_t F = size_t(g.q) * g.q * g.h;
  return sizeof(double2) * (g.q * g.q + F * G + G * (g.p * g.q * g.h + g.p * g.p * g.h));
}

inline int fft_group(const FftGeom &g) {
  // measured on C3 (p = 6): G = 2 (4 CTAs/SM) 661 ms, G = 4 763 ms, G = 1 712 ms
  for (int G = 2; G > 1; G /= 2)
    if (std::max(fft_fwd_smem(g, G), fft_inv_smem(g, G)) <= 200 * 1024) return G;
  return 1;
}

template <int P>
__global__ void __launch_bounds__(128)
fft_inv_kernel(const double2 *__restrict__ Y, int level, int64_t cell_lo, int64_t cell_hi,
               int m, int c0, int cc, FftGeom g, int G, double scale,
               double *__restrict__ locals) {
  extern __shared__ double2 sm2[];
  constexpr int p = P, q = 2 * P - 1, h = q / 2 + 1, F = q * q * h;
  const int P3 = p * p * p, PPH = p * p * h, PQH = p * q * h;
  const int n = 1 << level;
  const int64_t ncell = int64_t(1) << (3 * level);
  const int64_t ngroups = ncell / G;
  double2 *tw = sm2;                 // [q][q]
  double2 *stage = tw + q * q;       // [F][G]
  double2 *C = stage + F * G;    // [G][p][q][h]  x inverted, i < p
  double2 *D = C + G * PQH;      // [G][p][p][h]  y inverted, j < p
  const double norm = scale / ((double)q * q * q);
  stage_twiddles(g, tw);
  for (int64_t w = blockIdx.x; w < ngroups * cc; w += gridDim.x) {
    const int crel = (int)(w / ngroups);
    const int64_t lex0 = (w - crel * ngroups) * G;
    const int x = (int)(lex0 / ((int64_t)n * n)), y = (int)((lex0 / n) % n), z0 = (int)(lex0 % n);
    // the run's cells in this call's Morton range (a shard's own targets)
    bool any = false;
    for (int gi = 0; gi < G; ++gi) {
      const int64_t id = (int64_t)morton3(x, y, z0 + gi);
      any |= id >= cell_lo && id < cell_hi;
    }
    if (!any) continue;  // uniform across the CTA
    __syncthreads();
    const double2 *src = Y + (int64_t)crel * F * ncell + lex0;
    #pragma unroll 2
    for (int e = threadIdx.x; e < F * G; e += blockDim.x) {
      const int f = e / G, gi = e - f * G;
      stage[e] = src[(int64_t)f * ncell + gi];
    }
    __syncthreads();
    // x: q bins -> p outputs, e^{+2 pi i i kx / q}
    #pragma unroll 2
    for (int e = threadIdx.x; e < G * PQH; e += blockDim.x) {
      const int gi = e / PQH, r = e - gi * PQH, i = r / (q * h), rem = r - i * q * h;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int kx = 0; kx < q; ++kx) {
        const double2 t = tw[i * q + kx], v = stage[(kx * q * h + rem) * G + gi];
        re = fma(v.x, t.x, fma(-v.y, t.y, re));
        im = fma(v.y, t.x, fma(v.x, t.y, im));
      }
      C[e] = make_double2(re, im);
    }
    __syncthreads();
    // y: q bins -> p outputs
    #pragma unroll 2
    for (int e = threadIdx.x; e < G * PPH; e += blockDim.x) {
      const int gi = e / PPH, r = e - gi * PPH, i = r / (p * h), rem = r - i * p * h;
      const int j = rem / h, kz = rem - j * h;
      const double2 *c = C + gi * PQH + i * q * h + kz;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int ky = 0; ky < q; ++ky) {
        const double2 t = tw[j * q + ky], v = c[ky * h];
        re = fma(v.x, t.x, fma(-v.y, t.y, re));
        im = fma(v.y, t.x, fma(v.x, t.y, im));
      }
      D[e] = make_double2(re, im);
    }
    __syncthreads();
    // z: Hermitian half spectrum -> p real outputs (irfft: DC imaginary
    // part dropped, bins 1..q/2 counted twice; q is odd so no Nyquist bin)
    #pragma unroll 2
    for (int e = threadIdx.x; e < G * P3; e += blockDim.x) {
      const int gi = e / P3, r = e - gi * P3, ij = r / p, k = r - ij * p;
      const int64_t cell = (int64_t)morton3(x, y, z0 + gi);
      if (cell < cell_lo || cell >= cell_hi) continue;
      const double2 *d = D + gi * PPH + ij * h;
      double v = d[0].x;
#pragma unroll
      for (int kz = 1; kz < h; ++kz) {
        const double2 t = tw[k * q + kz];
        v = fma(2.0 * d[kz].x, t.x, fma(-2.0 * d[kz].y, t.y, v));
      }
      locals[(cell * m + c0 + crel) * (int64_t)P3 + r] = norm * v;
    }
  }
}

FftGeom make_geom(int p) {
  FftGeom g{};
  g.p = p;
  g.q = 2 * p - 1;
  g.h = g.q / 2 + 1;
  for (int r = 0; r < g.q; ++r) {
    // exact-angle table: every twiddle e^{+-2 pi i j k / q} is one of these
    g.c[r] = cospi(2.0 * r / g.q);
    g.s[r] = sinpi(2.0 * r / g.q);
  }
  return g;
}

// 7^3 table: offset (a, b, c) -> index among the 316 far offsets
// (lexicographic, octree.py:110-119), -1 for the 27 near offsets.
short *tap_table() {
  // one copy per device (the table is read by that device's kernels)
  static std::mutex mu;
  static short *per_dev[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  std::lock_guard<std::mutex> lock(mu);
  short *&dev = per_dev[d & 63];
  if (dev) return dev;
  short h[343];
  int t = 0;
  for (int a = -3; a <= 3; ++a)
    for (int b = -3; b <= 3; ++b)
      for (int c = -3; c <= 3; ++c) {
        const int e = ((a + 3) * 7 + (b + 3)) * 7 + (c + 3);
        h[e] = (std::max(abs(a), std::max(abs(b), abs(c))) >= 2) ? (short)t++ : (short)-1;
      }
  cudaMalloc(&dev, sizeof(h));
  cudaMemcpy(dev, h, sizeof(h), cudaMemcpyHostToDevice);
  return dev;
}

}  // namespace
}  // namespace bfmm

using namespace bfmm;

// Scratch for a chunk of `cc` columns: X and Y spectra, 2 x 8^l x cc x F x 16 B.
extern "C" int bfmm_m2l_fft_scratch_bytes(int level, int cc, int p, size_t *bytes) {
  const int q = 2 * p - 1;
  const int64_t F = int64_t(q) * q * (q / 2 + 1);
  *bytes = 2 * sizeof(double2) * (size_t(1) << (3 * level)) * size_t(cc) * F;
  return 0;
}

extern "C" int bfmm_m2l_fft(const double *moments, double *locals, int level,
                            int m, int p, const double *symbols, double scale,
                            int64_t q_lo, int64_t nq, void *scratch,
                            size_t scratch_bytes, bfmm_stream_t stream) {
  if (p < 2 || p > 12 || level < 2 || level > 10) {
    set_error("bfmm_m2l_fft: unsupported p=%d level=%d", p, level);
    return 2;
  }
  cudaStream_t st = as_stream(stream);
  const FftGeom g = make_geom(p);
  const int64_t F = int64_t(g.q) * g.q * g.h;
  const int64_t ncell = int64_t(1) << (3 * level);
  const size_t per_col = 2 * sizeof(double2) * ncell * F;
  const int cc = (int)std::min<size_t>((size_t)m, scratch_bytes / per_col);
  if (cc < 1) {
    set_error("bfmm_m2l_fft: scratch %zu B holds no column (need %zu)", scratch_bytes,
              per_col);
    return 2;
  }
  const short *taps = tap_table();
  double2 *X = static_cast<double2 *>(scratch);
  double2 *Y = X + ncell * cc * F;
  const int G = fft_group(g);
  const size_t smem_f = fft_fwd_smem(g, G), smem_i = fft_inv_smem(g, G);
  const int n = 1 << level;
  const unsigned tiles = (unsigned)(ceil_div(n, kTX) * ceil_div(n, kTY) * ceil_div(n, kTZ));
  const size_t smem_s = sizeof(double2) * (kHX * kHYP * kHZP + 343);
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(stencil_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_s);
  }
  int rc = 0;
  switch (p) {
#define BFMM_FFT_ATTR(PP)                                                                      \
  case PP:                                                                                     \
    cudaFuncSetAttribute(fft_fwd_kernel<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                         (int)smem_f);                                                         \
    cudaFuncSetAttribute(fft_inv_kernel<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                         (int)smem_i);                                                         \
    break;
    BFMM_FFT_ATTR(2) BFMM_FFT_ATTR(3) BFMM_FFT_ATTR(4) BFMM_FFT_ATTR(5) BFMM_FFT_ATTR(6)
    BFMM_FFT_ATTR(7) BFMM_FFT_ATTR(8) BFMM_FFT_ATTR(9) BFMM_FFT_ATTR(10) BFMM_FFT_ATTR(11)
    BFMM_FFT_ATTR(12)
#undef BFMM_FFT_ATTR
  }
  (void)rc;
  for (int c0 = 0; c0 < m; c0 += cc) {
    const int ccur = std::min(cc, m - c0);
    const int64_t groups = ncell / G * ccur;
    const unsigned gcell = (unsigned)std::min<int64_t>(groups, kNumSMs * 16);
    switch (p) {
#define BFMM_FFT_FWD(PP)                                                                       \
  case PP:                                                                                     \
    fft_fwd_kernel<PP><<<gcell, 128, smem_f, st>>>(moments, level, m, c0, ccur, g, G, X);      \
    break;
      BFMM_FFT_FWD(2) BFMM_FFT_FWD(3) BFMM_FFT_FWD(4) BFMM_FFT_FWD(5) BFMM_FFT_FWD(6)
      BFMM_FFT_FWD(7) BFMM_FFT_FWD(8) BFMM_FFT_FWD(9) BFMM_FFT_FWD(10) BFMM_FFT_FWD(11)
      BFMM_FFT_FWD(12)
#undef BFMM_FFT_FWD
    }
    if (check_launch("fft_fwd_kernel")) return 1;
    stencil_kernel<<<dim3(tiles, (unsigned)F, (unsigned)ccur), dim3(kTX, kTY, 2), smem_s, st>>>(
        X, Y, level, (int)F, reinterpret_cast<const double2 *>(symbols), taps, 8 * q_lo,
        8 * (q_lo + nq));
    if (check_launch("stencil_kernel")) return 1;
    const unsigned gi = (unsigned)std::min<int64_t>(groups, kNumSMs * 16);
    switch (p) {
#define BFMM_FFT_INV(PP)                                                                       \
  case PP:                                                                                     \
    fft_inv_kernel<PP><<<gi, 128, smem_i, st>>>(Y, level, 8 * q_lo, 8 * (q_lo + nq), m, c0,     \
                                                ccur, g, G, scale, locals);                    \
    break;
      BFMM_FFT_INV(2) BFMM_FFT_INV(3) BFMM_FFT_INV(4) BFMM_FFT_INV(5) BFMM_FFT_INV(6)
      BFMM_FFT_INV(7) BFMM_FFT_INV(8) BFMM_FFT_INV(9) BFMM_FFT_INV(10) BFMM_FFT_INV(11)
      BFMM_FFT_INV(12)
#undef BFMM_FFT_INV
    }
    if (check_launch("fft_inv_kernel")) return 1;
  }
  return 0;
}
