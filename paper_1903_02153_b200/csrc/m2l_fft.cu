// Uniform-grid far field (engine.py:258-292): the 316 translation operators
// are nested-Toeplitz on the equispaced node grid, so each is a circulant
// convolution on a q^3 grid (q = 2p - 1) and diagonal in the real-FFT basis.
//
// Per level and per chunk of weight columns:
//   1. fft_fwd_kernel : X[c][f] = rfftn(pad_q(M[c]))           (pass z, y, x)
//   2. hadamard_kernel: Y[c][f] = sum_{t valid} S_t[f] * X[c + t][f]
//   3. fft_inv_kernel : L[c]    = scale * irfftn(Y[c], s=(q,q,q))[:p,:p,:p]
// f = (kx*q + ky)*(q/2+1) + kz indexes numpy's rfftn output layout
// (ops:156-159), so the symbols S_t are the reference's table verbatim.
// The transforms are direct DFTs along each axis with exactly tabulated
// twiddles (q <= 23): zero padding makes them cheaper than a generic FFT
// and their cost is a few percent of the Hadamard sum.
#include <algorithm>

#include "common.cuh"

namespace bfmm {
namespace {

constexpr int kMaxQ = 23;  // p <= 12

struct FftGeom {
  int p, q, h;  // h = q/2 + 1 bins along z
  double c[kMaxQ], s[kMaxQ];  // cos / sin(2 pi r / q)
};

// ---- 1. forward transform: one CTA per (cell, column) ------------------------
__global__ void __launch_bounds__(128)
fft_fwd_kernel(const double *__restrict__ moments, int64_t ncell, int m, int c0,
               int cc, FftGeom g, double2 *__restrict__ X) {
  extern __shared__ double2 sm2[];
  const int p = g.p, q = g.q, h = g.h, F = q * q * h;
  double2 *A = sm2;            // [p][p][h]
  double2 *B = A + p * p * h;  // [p][q][h]
  double *in = reinterpret_cast<double *>(B + p * q * h);  // [p][p][p]
  for (int64_t w = blockIdx.x; w < ncell * cc; w += gridDim.x) {
    const int64_t cell = w / cc;
    const int col = c0 + (int)(w - cell * cc);
    const double *src = moments + (cell * m + col) * (int64_t)(p * p * p);
    __syncthreads();
    for (int e = threadIdx.x; e < p * p * p; e += blockDim.x) in[e] = src[e];
    __syncthreads();
    // z: real -> h complex bins, e^{-2 pi i k kz / q}
    for (int e = threadIdx.x; e < p * p * h; e += blockDim.x) {
      const int ij = e / h, kz = e - ij * h;
      double re = 0.0, im = 0.0;
      for (int k = 0; k < p; ++k) {
        const int r = (k * kz) % q;
        const double v = in[ij * p + k];
        re = fma(v, g.c[r], re);
        im = fma(-v, g.s[r], im);
      }
      A[e] = make_double2(re, im);
    }
    __syncthreads();
    // y: p inputs -> q bins
    for (int e = threadIdx.x; e < p * q * h; e += blockDim.x) {
      const int i = e / (q * h), rem = e - i * q * h, ky = rem / h, kz = rem - ky * h;
      double re = 0.0, im = 0.0;
      for (int j = 0; j < p; ++j) {
        const int r = (j * ky) % q;
        const double2 a = A[(i * p + j) * h + kz];
        // (a.x + i a.y)(c - i s)
        re = fma(a.x, g.c[r], fma(a.y, g.s[r], re));
        im = fma(a.y, g.c[r], fma(-a.x, g.s[r], im));
      }
      B[e] = make_double2(re, im);
    }
    __syncthreads();
    // x: p inputs -> q bins, straight to global
    double2 *dst = X + w * (int64_t)F;
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      const int kx = f / (q * h), rem = f - kx * q * h;
      double re = 0.0, im = 0.0;
      for (int i = 0; i < p; ++i) {
        const int r = (i * kx) % q;
        const double2 b = B[i * q * h + rem];
        re = fma(b.x, g.c[r], fma(b.y, g.s[r], re));
        im = fma(b.y, g.c[r], fma(-b.x, g.s[r], im));
      }
      dst[f] = make_double2(re, im);
    }
  }
}

// ---- 2. Hadamard accumulation over the far offsets ----------------------------
__constant__ signed char c_off[316][3];
bool g_off_ready = false;

void ensure_off() {
  if (g_off_ready) return;
  signed char h[316][3];
  int n = 0;
  for (int a = -3; a <= 3; ++a)
    for (int b = -3; b <= 3; ++b)
      for (int c = -3; c <= 3; ++c)
        if (std::max(abs(a), std::max(abs(b), abs(c))) >= 2) {
          h[n][0] = (signed char)a;
          h[n][1] = (signed char)b;
          h[n][2] = (signed char)c;
          ++n;
        }
  cudaMemcpyToSymbol(c_off, h, sizeof(h));
  g_off_ready = true;
}

// thread per (target cell, column, frequency); frequencies fastest so a warp
// reads 32 consecutive bins of one source spectrum and of one symbol.
__global__ void __launch_bounds__(256)
hadamard_kernel(const double2 *__restrict__ X, double2 *__restrict__ Y,
                int level, int cc, int F, const double2 *__restrict__ S,
                int64_t cell_lo, int64_t ncell) {
  // targets: cells [cell_lo, cell_lo + ncell); X holds every cell
  const int n = 1 << level;
  const int64_t total = ncell * cc * F;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cw = e / F;
    const int f = (int)(e - cw * F);
    const int64_t rel = cw / cc;
    const int col = (int)(cw - rel * cc);
    const int64_t cell = cell_lo + rel;
    int cx, cy, cz;
    unmorton3((uint64_t)cell, cx, cy, cz);
    double re = 0.0, im = 0.0;
    for (int t = 0; t < 316; ++t) {
      const int t0 = c_off[t][0], t1 = c_off[t][1], t2 = c_off[t][2];
      if (!far_pair(n, cx, cy, cz, t0, t1, t2)) continue;
      const int64_t src = (int64_t)morton3(cx + t0, cy + t1, cz + t2);
      const double2 x = X[(src * cc + col) * F + f];
      const double2 s = S[(int64_t)t * F + f];
      re = fma(s.x, x.x, fma(-s.y, x.y, re));
      im = fma(s.x, x.y, fma(s.y, x.x, im));
    }
    Y[e] = make_double2(re, im);
  }
}

// ---- 3. inverse transform + crop + scale: one CTA per (cell, column) ---------
__global__ void __launch_bounds__(128)
fft_inv_kernel(const double2 *__restrict__ Y, int64_t cell_lo, int64_t ncell,
               int m, int c0, int cc, FftGeom g, double scale,
               double *__restrict__ locals) {
  extern __shared__ double2 sm2[];
  const int p = g.p, q = g.q, h = g.h, F = q * q * h;
  double2 *C = sm2;            // [p][q][h]   x inverted, i < p
  double2 *D = C + p * q * h;  // [p][p][h]   y inverted, j < p
  const double norm = scale / ((double)q * q * q);
  for (int64_t w = blockIdx.x; w < ncell * cc; w += gridDim.x) {
    const int64_t rel = w / cc;
    const int col = c0 + (int)(w - rel * cc);
    const int64_t cell = cell_lo + rel;
    const double2 *src = Y + w * (int64_t)F;
    __syncthreads();
    // x: q bins -> p outputs, e^{+2 pi i i kx / q}
    for (int e = threadIdx.x; e < p * q * h; e += blockDim.x) {
      const int i = e / (q * h), rem = e - i * q * h;
      double re = 0.0, im = 0.0;
      for (int kx = 0; kx < q; ++kx) {
        const int r = (i * kx) % q;
        const double2 y = src[kx * q * h + rem];
        re = fma(y.x, g.c[r], fma(-y.y, g.s[r], re));
        im = fma(y.y, g.c[r], fma(y.x, g.s[r], im));
      }
      C[e] = make_double2(re, im);
    }
    __syncthreads();
    // y: q bins -> p outputs
    for (int e = threadIdx.x; e < p * p * h; e += blockDim.x) {
      const int i = e / (p * h), rem = e - i * p * h, j = rem / h, kz = rem - j * h;
      double re = 0.0, im = 0.0;
      for (int ky = 0; ky < q; ++ky) {
        const int r = (j * ky) % q;
        const double2 c = C[(i * q + ky) * h + kz];
        re = fma(c.x, g.c[r], fma(-c.y, g.s[r], re));
        im = fma(c.y, g.c[r], fma(c.x, g.s[r], im));
      }
      D[e] = make_double2(re, im);
    }
    __syncthreads();
    // z: Hermitian half spectrum -> p real outputs (irfft: DC imaginary
    // part dropped, bins 1..q/2 counted twice; q is odd so no Nyquist bin)
    double *dst = locals + (cell * m + col) * (int64_t)(p * p * p);
    for (int e = threadIdx.x; e < p * p * p; e += blockDim.x) {
      const int ij = e / p, k = e - ij * p;
      const double2 *d = D + ij * h;
      double v = d[0].x;
      for (int kz = 1; kz < h; ++kz) {
        const int r = (k * kz) % q;
        v = fma(2.0 * d[kz].x, g.c[r], fma(-2.0 * d[kz].y, g.s[r], v));
      }
      dst[e] = norm * v;
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
  ensure_off();
  cudaStream_t st = as_stream(stream);
  const FftGeom g = make_geom(p);
  const int64_t F = int64_t(g.q) * g.q * g.h;
  const int64_t ncell = int64_t(1) << (3 * level);
  const size_t per_col = 2 * sizeof(double2) * ncell * F;
  int cc = (int)std::min<size_t>((size_t)m, scratch_bytes / per_col);
  if (cc < 1) {
    set_error("bfmm_m2l_fft: scratch %zu B holds no column (need %zu)", scratch_bytes,
              per_col);
    return 2;
  }
  double2 *X = static_cast<double2 *>(scratch);
  double2 *Y = X + ncell * cc * F;
  const size_t smem_f = sizeof(double2) * (g.p * g.p * g.h + g.p * g.q * g.h) +
                        sizeof(double) * g.p * g.p * g.p;
  const size_t smem_i = sizeof(double2) * (g.p * g.q * g.h + g.p * g.p * g.h);
  for (int c0 = 0; c0 < m; c0 += cc) {
    const int ccur = std::min(cc, m - c0);
    const int64_t work = ncell * ccur;
    const unsigned gcell = (unsigned)std::min<int64_t>(work, kNumSMs * 16);
    fft_fwd_kernel<<<gcell, 128, smem_f, st>>>(moments, ncell, m, c0, ccur, g, X);
    if (check_launch("fft_fwd_kernel")) return 1;
    const int64_t tgt = 8 * nq * ccur;
    const unsigned gh = (unsigned)std::min<int64_t>(ceil_div(tgt * F, 256), kNumSMs * 64);
    hadamard_kernel<<<gh, 256, 0, st>>>(X, Y, level, ccur, (int)F,
                                        reinterpret_cast<const double2 *>(symbols),
                                        8 * q_lo, 8 * nq);
    if (check_launch("hadamard_kernel")) return 1;
    const unsigned gi = (unsigned)std::min<int64_t>(std::max<int64_t>(tgt, 1), kNumSMs * 16);
    fft_inv_kernel<<<gi, 128, smem_i, st>>>(Y, 8 * q_lo, 8 * nq, m, c0, ccur, g, scale,
                                            locals);
    if (check_launch("fft_inv_kernel")) return 1;
  }
  return 0;
}
