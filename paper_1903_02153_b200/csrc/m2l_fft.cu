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

// 16-byte global -> shared copy on the async path (zero-filled when !valid):
// a CTA's whole halo is in flight at once instead of one load round trip per
// element (the stencils' halo load was latency-bound: ncu long_scoreboard)
__device__ __forceinline__ void cp_async16z(void *smem, const void *gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// The transforms work on G lexicographically consecutive cells (a z-run)
// per CTA pass, so the frequency-major spectra are written / read as
// G * 16-byte runs, and every spectrum value is touched once.  Each 1-D DFT
// line (p inputs -> q bins, or back) is computed by ONE thread in
// registers: its inputs are loaded once, every output is an independent
// FMA chain, and the twiddles e^{2 pi i r / q} are read from the kernel
// parameter bank at compile-time indices (r = j k mod q, all loops
// unrolled on P) -- so a line costs p loads + q stores for 4pq DFMAs,
// instead of one shared-memory twiddle and one input load per MAC.
template <int P, int G>
struct FftShape {
  static constexpr int p = P, q = 2 * P - 1, h = q / 2 + 1, F = q * q * h;
  static constexpr int P3 = p * p * p, PPH = p * p * h, PQH = p * q * h;
  // forward: {in [G][p^3] real, B [G][p][q][h]} share storage (in dies
  // before B is written), then A [G][p][p][h]; the x pass writes its bins
  // straight to the spectrum (no [F][G] staging tile: lanes run over the G
  // cells of a bin first, so a bin's G values still leave as one G * 16-byte
  // run -- and the 46 KB the tile took at p = 6 buys two more CTAs per SM)
  static constexpr size_t U1 = (sizeof(double) * G * P3 > sizeof(double2) * G * PQH)
                                   ? sizeof(double) * G * P3 : sizeof(double2) * G * PQH;
  static constexpr size_t U2 = sizeof(double2) * G * PPH;
  static constexpr size_t smem = U1 + U2;
  // inverse: D [G][p][p][h] and C [G][p][q][h]; the x pass reads its q
  // bins straight from the spectrum into registers
  static constexpr size_t V1 = PPH * sizeof(double2) * G;
  static constexpr size_t smem_inv = V1 + sizeof(double2) * G * PQH;
  static constexpr size_t most = smem > smem_inv ? smem : smem_inv;
};

// cells per CTA pass: 4 when both kernels fit 3 CTAs per SM, else fewer
template <int P>
constexpr int fft_cells() {
  return FftShape<P, 4>::most <= 72 * 1024 ? 4 : FftShape<P, 2>::most <= 100 * 1024 ? 2 : 1;
};

// Threads per CTA: the three DFT passes run G p^2, G p h and G q h
// independent lines, one per thread, between block barriers; with 128
// threads P = 6 (144, 144, 264 lines) needs 2 + 2 + 3 rounds whose last ones
// are mostly idle.  Rounding G p^2 up to a whole warp (160 threads for
// P = 6: 1 + 1 + 2 rounds) nearly halves the passes' time.
template <int P, int G>
constexpr int fft_threads() {
  const int t = (G * P * P + 31) / 32 * 32;
  return t < 128 ? 128 : t > 256 ? 256 : t;
}

template <int P, int G>
__global__ void __launch_bounds__(fft_threads<P, G>())
fft_fwd_kernel(const double *__restrict__ moments, int level, int m, int c0,
               int cc, FftGeom g, double2 *__restrict__ X) {
  using Sh = FftShape<P, G>;
  constexpr int p = Sh::p, q = Sh::q, h = Sh::h, F = Sh::F;
  constexpr int P3 = Sh::P3, PPH = Sh::PPH, PQH = Sh::PQH;
  extern __shared__ __align__(16) unsigned char smraw[];
  double *in = reinterpret_cast<double *>(smraw);            // [G][p^3]
  double2 *B = reinterpret_cast<double2 *>(smraw);           // [G][p][q][h]
  double2 *A = reinterpret_cast<double2 *>(smraw + Sh::U1);  // [G][p][p][h]
  const int n = 1 << level;
  const int64_t ncell = int64_t(1) << (3 * level);
  const int64_t ngroups = ncell / G;
  for (int64_t w = blockIdx.x; w < ngroups * cc; w += gridDim.x) {
    const int crel = (int)(w / ngroups);
    const int64_t lex0 = (w - crel * ngroups) * G;
    const int x = (int)(lex0 / ((int64_t)n * n)), y = (int)((lex0 / n) % n), z0 = (int)(lex0 % n);
    __syncthreads();
    if (P3 % 2 == 0) {  // 16-byte rows: the whole block's moments in flight at once
      for (int e = threadIdx.x; e < G * P3 / 2; e += blockDim.x) {
        const int gi = (2 * e) / P3, r = 2 * e - gi * P3;
        cp_async16z(in + 2 * e,
                    moments + ((int64_t)morton3(x, y, z0 + gi) * m + c0 + crel) * P3 + r, true);
      }
      cp_async_all();
    } else {
      for (int e = threadIdx.x; e < G * P3; e += blockDim.x) {
        const int gi = e / P3, r = e - gi * P3;
        in[e] = moments[((int64_t)morton3(x, y, z0 + gi) * m + c0 + crel) * P3 + r];
      }
    }
    __syncthreads();
    // z: p reals -> h bins, e^{-2 pi i k kz / q}; one line (gi, i, j) per thread
    for (int l = threadIdx.x; l < G * p * p; l += blockDim.x) {
      double v[p];
#pragma unroll
      for (int k = 0; k < p; ++k) v[k] = in[l * p + k];
      double2 *dst = A + l * h;
#pragma unroll
      for (int kz = 0; kz < h; ++kz) {
        double re = v[0], im = 0.0;
#pragma unroll
        for (int k = 1; k < p; ++k) {
          const int r = (k * kz) % q;
          re = fma(v[k], g.c[r], re);
          im = fma(-v[k], g.s[r], im);
        }
        dst[kz] = make_double2(re, im);
      }
    }
    __syncthreads();
    // y: p inputs -> q bins; line (gi, i, kz)
    for (int l = threadIdx.x; l < G * p * h; l += blockDim.x) {
      const int gi = l / (p * h), r0 = l - gi * p * h, i = r0 / h, kz = r0 - i * h;
      const double2 *a = A + gi * PPH + i * p * h + kz;
      double2 v[p];
#pragma unroll
      for (int j = 0; j < p; ++j) v[j] = a[j * h];
      double2 *dst = B + gi * PQH + i * q * h + kz;
#pragma unroll
      for (int ky = 0; ky < q; ++ky) {
        double re = v[0].x, im = v[0].y;
#pragma unroll
        for (int j = 1; j < p; ++j) {
          const int r = (j * ky) % q;  // (v.x + i v.y)(c - i s)
          re = fma(v[j].x, g.c[r], fma(v[j].y, g.s[r], re));
          im = fma(v[j].y, g.c[r], fma(-v[j].x, g.s[r], im));
        }
        dst[ky * h] = make_double2(re, im);
      }
    }
    __syncthreads();
    // x: p inputs -> q bins, straight into the [f][cell] spectrum; line
    // (ky, kz, gi) with the cell index fastest across lanes: the G cells of
    // a bin are one G * 16-byte run in global memory
    double2 *dst = X + (int64_t)crel * F * ncell + lex0;
    for (int l = threadIdx.x; l < G * q * h; l += blockDim.x) {
      const int rem = l / G, gi = l - rem * G;
      const double2 *b = B + gi * PQH + rem;
      double2 v[p];
#pragma unroll
      for (int i = 0; i < p; ++i) v[i] = b[i * q * h];
#pragma unroll
      for (int kx = 0; kx < q; ++kx) {
        double re = v[0].x, im = v[0].y;
#pragma unroll
        for (int i = 1; i < p; ++i) {
          const int r = (i * kx) % q;
          re = fma(v[i].x, g.c[r], fma(v[i].y, g.s[r], re));
          im = fma(v[i].y, g.c[r], fma(-v[i].x, g.s[r], im));
        }
        dst[(int64_t)(kx * q * h + rem) * ncell + gi] = make_double2(re, im);
      }
    }
  }
}

// ---- 2. Hadamard accumulation as a per-frequency 3-D stencil ------------------
// 8 x 8 x 8 targets, 128 threads x 4: a 47 KB halo keeps 4 CTAs per SM
// (measured: 16-deep z tiles reuse each source more but fit only 3 CTAs and
// run 3 % slower, the kernel being shared-memory-latency bound)
constexpr int kTX = 8, kTY = 8, kTZ = 8, kR = kTZ / 2;
constexpr int kHX = kTX + 6, kHY = kTY + 6, kHZ = kTZ + 6;
// Bank layout (round-1 reasoning): an LDS.128 is served 8 lanes (one
// quarter-warp phase) at a time, and those 8 lanes must hit 8 distinct
// 16-byte slots (mod 8).  A phase's lanes vary z parity (stride 1) and 4
// same-parity x positions (stride 2 * HYP * HZP), so the halo is padded to
// HYP = 15, HZP = 15: 2 * 15 * 15 = 450 = 2 (mod 8) -> slots {0,2,4,6} +
// {0,1} (the unpadded 14 x 14 layout is 2-way conflicted).  ncu on full C3
// showed the rule is warp-wide, not per phase: a wavefront serves any lanes
// with distinct slots, this kernel's 16 distinct source addresses per warp
// all fall on even slots, and 40 % of its shared-memory wavefronts are
// conflict replays (profiles/r02_ncu_c3_stencil_variants.txt) -- what
// stencil3_kernel's skewed layout fixes.  Kept as the bitwise reference.
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
    const bool v = sx >= 0 && sx < n && sy >= 0 && sy < n && sz >= 0 && sz < n;
    cp_async16z(&halo[hx][hy][hz], v ? Xf + lex_of(sx, sy, sz, n) : Xf, v);
  }
  for (int e = tid; e < 343; e += 128) {
    const int t = tap_index[e];
    cp_async16z(&taps[0][0][0] + e, t >= 0 ? S + (int64_t)t * F + f : S, t >= 0);
  }
  cp_async_all();
  __syncthreads();
  double2 acc[kR];
#pragma unroll
  for (int k = 0; k < kR; ++k) acc[k] = make_double2(0.0, 0.0);
  // Parity rule (octree.py:128-145): +3 needs an even target coordinate,
  // -3 an odd one, so a target of parity p along an axis takes the offsets
  // t = t' - p, t' in [-2, 3].  x and y parities are warp-uniform; along z
  // the tile starts even, so target z0 + pz + 2k with source offset
  // c = c' - pz reads source z0 + 2k + c' -- the same source column for both
  // z parities (only the tap differs per lane): no divergence, no skipped
  // lanes, 12 source loads serve 6 x 4 complex MACs.  For the near (a, b)
  // columns (|a|, |b| <= 1) only |c| >= 2 taps are nonzero: c' in
  // {-2, -1, 2, 3} covers both parities (one of the four is zero per lane).
  const int px = x & 1, py = y & 1;
  for (int ap = -2; ap <= 3; ++ap) {
    const int a = ap - px;
#pragma unroll 2
    for (int bp = -2; bp <= 3; ++bp) {
      const int b = bp - py;
      double2 seg[2 * kR + 4];
      const double2 *col_src = &halo[ix + 3 + a][iy + 3 + b][1];  // source z0 - 2
#pragma unroll
      for (int u = 0; u < 2 * kR + 4; ++u) seg[u] = col_src[u];
      const double2 *tp = &taps[a + 3][b + 3][3 - pz];  // tap of c' = tp[c']
      const bool near_col = a >= -1 && a <= 1 && b >= -1 && b <= 1;  // warp-uniform
#pragma unroll
      for (int cp = -2; cp <= 3; ++cp) {
        if (near_col && (cp == 0 || cp == 1)) continue;
        const double2 s = tp[cp];
#pragma unroll
        for (int k = 0; k < kR; ++k) {
          const double2 v = seg[cp + 2 + 2 * k];
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

// ---- 2b. the same stencil with two x targets per thread ----------------------
// Tile 16 x 8 x 8: thread (ix4, iy, pz) of (x, y) parity class w owns the
// targets x_a = x0 + px + 4 ix4 and x_a + 2 (same parity), y = y0 + iy, and
// z = z0 + pz + 2k.  A source x-column x_a + alpha, alpha' = alpha + px in
// [-2, 5], serves target x_a with tap a = alpha (alpha' <= 3) and target
// x_a + 2 with tap alpha - 2 (alpha' >= 0): 8 column loads per (b, 2
// targets) instead of 12, the shared-memory operand traffic that bounds
// stencil_kernel (ncu: FP64 pipe ~55 %, LSU busy).  Same taps, same
// per-target accumulation order (a, b, c ascending) as stencil_kernel:
// bitwise-equal spectra.
constexpr int kT2X = 16, kH2X = kT2X + 6;
// lanes: bit 0 = pz (halo z stride 1), bits 1-2 = same-parity y (stride
// 2 * HZP = 30 = 6 mod 8), bits 3-4 = x pair index: an 8-lane LDS.128 phase
// (pz, y) covers 16-byte slots {0,1,6,7,4,5,2,3} (mod 8) -- conflict-free.
__global__ void __launch_bounds__(128, 2)
stencil2_kernel(const double2 *__restrict__ X, double2 *__restrict__ Y, int level, int F,
                const double2 *__restrict__ S, const short *__restrict__ tap_index,
                int64_t cell_lo, int64_t cell_hi) {
  extern __shared__ double2 sm2[];
  auto halo = reinterpret_cast<double2 (*)[kHYP][kHZP]>(sm2);                    // [kH2X][kHYP][kHZP]
  auto taps = reinterpret_cast<double2 (*)[7][7]>(sm2 + kH2X * kHYP * kHZP);    // [7][7][7]
  const int n = 1 << level;
  const int64_t ncell = int64_t(1) << (3 * level);
  const int tilesx = (n + kT2X - 1) / kT2X, tilesy = (n + kTY - 1) / kTY;
  const int tile = blockIdx.x;
  const int tz = tile / (tilesx * tilesy), trem = tile - tz * tilesx * tilesy;
  const int x0 = (trem / tilesy) * kT2X, y0 = (trem % tilesy) * kTY, z0 = tz * kTZ;
  const int f = blockIdx.y, col = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int px = w >> 1, py = w & 1;
  const int pz = lane & 1, iy = py + 2 * ((lane >> 1) & 3), ix4 = (lane >> 3) & 3;
  const int xa = x0 + px + 4 * ix4, y = y0 + iy;
  bool mine = false;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int k = 0; k < kR; ++k) {
      const int x = xa + 2 * u, z = z0 + pz + 2 * k;
      if (x < n && y < n && z < n) {
        const int64_t id = (int64_t)morton3(x, y, z);
        mine |= id >= cell_lo && id < cell_hi;
      }
    }
  if (!__syncthreads_or(mine)) return;
  const double2 *Xf = X + ((int64_t)col * F + f) * ncell;
  for (int e = tid; e < kH2X * kHY * kHZ; e += 128) {
    const int hx = e / (kHY * kHZ), hr = e - hx * kHY * kHZ, hy = hr / kHZ, hz = hr - hy * kHZ;
    const int sx = x0 + hx - 3, sy = y0 + hy - 3, sz = z0 + hz - 3;
    const bool v = sx >= 0 && sx < n && sy >= 0 && sy < n && sz >= 0 && sz < n;
    cp_async16z(&halo[hx][hy][hz], v ? Xf + lex_of(sx, sy, sz, n) : Xf, v);
  }
  for (int e = tid; e < 343; e += 128) {
    const int t = tap_index[e];
    cp_async16z(&taps[0][0][0] + e, t >= 0 ? S + (int64_t)t * F + f : S, t >= 0);
  }
  cp_async_all();
  __syncthreads();
  double2 acc[2][kR];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int k = 0; k < kR; ++k) acc[u][k] = make_double2(0.0, 0.0);
  const int hx0 = px + 4 * ix4 + 3;  // halo x of target x_a
  // target x_a takes a = alpha' - px for alpha' in [-2, 3], target x_a + 2
  // a = alpha' - 2 - px for alpha' in [0, 5]; with b inside alpha' each
  // target sees its (a, b, c) taps in stencil_kernel's order
#pragma unroll
  for (int ap = -2; ap <= 5; ++ap) {
#pragma unroll 2
    for (int bp = -2; bp <= 3; ++bp) {
      const int b = bp - py;
      double2 seg[2 * kR + 4];
      const double2 *col_src = &halo[hx0 + ap - px][iy + 3 + b][1];  // source z0 - 2
#pragma unroll
      for (int uu = 0; uu < 2 * kR + 4; ++uu) seg[uu] = col_src[uu];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if ((u == 0 && ap > 3) || (u == 1 && ap < 0)) continue;  // compile-time
        const int a = ap - px - 2 * u;
        const double2 *tp = &taps[a + 3][b + 3][3 - pz];
        const bool near_col = a >= -1 && a <= 1 && b >= -1 && b <= 1;  // warp-uniform
#pragma unroll
        for (int cp = -2; cp <= 3; ++cp) {
          if (near_col && (cp == 0 || cp == 1)) continue;
          const double2 s = tp[cp];
#pragma unroll
          for (int k = 0; k < kR; ++k) {
            const double2 v = seg[cp + 2 + 2 * k];
            acc[u][k].x = fma(s.x, v.x, fma(-s.y, v.y, acc[u][k].x));
            acc[u][k].y = fma(s.x, v.y, fma(s.y, v.x, acc[u][k].y));
          }
        }
      }
    }
  }
  double2 *Yf = Y + ((int64_t)col * F + f) * ncell;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int k = 0; k < kR; ++k) {
      const int x = xa + 2 * u, z = z0 + pz + 2 * k;
      if (x < n && y < n && z < n) Yf[lex_of(x, y, z, n)] = acc[u][k];
    }
}

// ---- 2c. the stencil with both z parities per thread (the default) -----------
// ncu on full C3 (profiles/r02_ncu_c3_stencil_variants.txt): stencil_kernel
// keeps the shared-memory data pipe 85 % busy -- 40 % of its wavefronts are
// bank-conflict replays (a wavefront serves lanes with distinct 16-byte
// slots mod 8 across the WHOLE warp, and its 16 distinct source addresses
// all fall on even slots) -- and spends a quarter of its instructions on the
// per-element halo index arithmetic.  Here
//  * a thread owns 4 CONSECUTIVE z targets (both parities) of its (x, y):
//    the 8 sources of an (a, b) column feed 24 complex MACs and the 7 taps
//    c = -3..3 of the column serve both parities (15 LDS.128 per 96 DFMAs
//    instead of 18);
//  * the y parity takes over the role z parity plays in stencil_kernel: a
//    lane pair (py = 0, 1) reads the SAME source column y0 + 2 jy + 3 + b'
//    with taps b = b' - py (octree.py:128-145), so the +-3 skips stay
//    divergence-free;
//  * halo rows are skewed by one slot for every other x pair
//    (z index + ((hx >> 1) & 1), rows of 15), so the 16 distinct source
//    addresses of a warp -- 4 y (stride 30 = 6 mod 8) x 4 x -- cover every
//    slot exactly twice: 2 wavefronts per LDS.128, the minimum;
//  * a thread copies whole halo rows (14 contiguous values, immediate
//    offsets) instead of one element per loop trip.
// Tile 8 x 8 x 8, 128 threads: warp = (z half, x parity), lane = (py, jy, jx).
// Same taps in the same per-target order (a, b, c ascending) as
// stencil_kernel: bitwise-equal spectra (only zero taps are skipped
// differently).
constexpr int kH3ZP = kHZ + 1;  // 15: odd z stride + room for the skew; y needs no padding
constexpr int kZT = 4;          // z targets per thread
__global__ void __launch_bounds__(128, 4)
stencil3_kernel(const double2 *__restrict__ X, double2 *__restrict__ Y, int level, int F,
                const double2 *__restrict__ S, const short *__restrict__ tap_index,
                int64_t cell_lo, int64_t cell_hi) {
  extern __shared__ double2 sm2[];
  auto halo = reinterpret_cast<double2 (*)[kHY][kH3ZP]>(sm2);                  // [kHX][kHY][kH3ZP]
  auto taps = reinterpret_cast<double2 (*)[7][7]>(sm2 + kHX * kHY * kH3ZP);   // [7][7][7]
  const int n = 1 << level;
  const int64_t ncell = int64_t(1) << (3 * level);
  const int tilesx = (n + kTX - 1) / kTX, tilesy = (n + kTY - 1) / kTY;
  const int tile = blockIdx.x;
  const int tz = tile / (tilesx * tilesy), trem = tile - tz * tilesx * tilesy;
  const int x0 = (trem / tilesy) * kTX, y0 = (trem % tilesy) * kTY, z0 = tz * kTZ;
  const int f = blockIdx.y, col = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int px = w & 1, zb = kZT * (w >> 1), py = lane & 1;
  const int ix = px + 2 * ((lane >> 3) & 3), iy = py + 2 * ((lane >> 1) & 3);
  const int x = x0 + ix, y = y0 + iy;
  // shard filter: skip the tile when none of its targets is ours
  if (cell_lo > 0 || cell_hi < ncell) {
    bool mine = false;
#pragma unroll
    for (int k = 0; k < kZT; ++k) {
      const int z = z0 + zb + k;
      if (x < n && y < n && z < n) {
        const int64_t id = (int64_t)morton3(x, y, z);
        mine |= id >= cell_lo && id < cell_hi;
      }
    }
    if (!__syncthreads_or(mine)) return;
  }
  const double2 *Xf = X + ((int64_t)col * F + f) * ncell;
  for (int r = tid; r < kHX * kHY; r += 128) {
    const int hx = r / kHY, hy = r - hx * kHY;
    const int sx = x0 + hx - 3, sy = y0 + hy - 3;
    const bool vr = sx >= 0 && sx < n && sy >= 0 && sy < n;
    const double2 *row = Xf + (vr ? lex_of(sx, sy, 0, n) : 0);
    double2 *dst = &halo[hx][hy][(hx >> 1) & 1];
#pragma unroll
    for (int hz = 0; hz < kHZ; ++hz) {
      const int sz = z0 + hz - 3;
      const bool v = vr && sz >= 0 && sz < n;
      cp_async16z(dst + hz, row + (v ? sz : 0), v);
    }
  }
  for (int e = tid; e < 343; e += 128) {
    const int t = tap_index[e];
    cp_async16z(&taps[0][0][0] + e, t >= 0 ? S + (int64_t)t * F + f : S, t >= 0);
  }
  cp_async_all();
  __syncthreads();
  double2 acc[kZT];
#pragma unroll
  for (int k = 0; k < kZT; ++k) acc[k] = make_double2(0.0, 0.0);
  // target z0 + zb + zi (zi = 2k + pz) takes c = c' - pz, c' in [-2, 3],
  // from source z0 + zb + 2k + c' = seg[c' + 2 + 2k] with tap tp[c + 3]
#pragma unroll 1
  for (int ap = -2; ap <= 3; ++ap) {
    const int a = ap - px;
    const int hx = ix + 3 + a;
#pragma unroll 2
    for (int bp = -2; bp <= 3; ++bp) {
      const int b = bp - py;
      double2 seg[kZT + 4];
      // source z0 + zb - 2 = halo z index zb + 1, plus the row's skew
      const double2 *col_src = &halo[hx][iy + 3 + b][zb + 1 + ((hx >> 1) & 1)];
#pragma unroll
      for (int u = 0; u < kZT + 4; ++u) seg[u] = col_src[u];
      const double2 *tp = &taps[a + 3][b + 3][0];
      // zero taps |c| <= 1 of the near columns: skipped where the column is
      // near for both y parities of the warp (b' in {0, 1})
      const bool near_col = a >= -1 && a <= 1 && (bp == 0 || bp == 1);  // warp-uniform
#pragma unroll
      for (int c = -3; c <= 3; ++c) {
        if (near_col && c >= -1 && c <= 1) continue;
        const double2 s = tp[c + 3];
#pragma unroll
        for (int zi = 0; zi < kZT; ++zi) {
          const int pz = zi & 1, cp = c + pz;
          if (cp < -2 || cp > 3) continue;  // compile-time: the parity rule
          const double2 v = seg[cp + 2 + (zi - pz)];
          acc[zi].x = fma(s.x, v.x, fma(-s.y, v.y, acc[zi].x));
          acc[zi].y = fma(s.x, v.y, fma(s.y, v.x, acc[zi].y));
        }
      }
    }
  }
  double2 *Yf = Y + ((int64_t)col * F + f) * ncell;
  if (x < n && y < n) {
    double2 *dst = Yf + lex_of(x, y, z0 + zb, n);
#pragma unroll
    for (int k = 0; k < kZT; ++k)
      if (z0 + zb + k < n) dst[k] = acc[k];
  }
}

// ---- 3. inverse transform + crop + scale ------------------------------------
template <int P, int G>
__global__ void __launch_bounds__(fft_threads<P, G>())
fft_inv_kernel(const double2 *__restrict__ Y, int level, int64_t cell_lo, int64_t cell_hi,
               int m, int c0, int cc, FftGeom g, double scale,
               double *__restrict__ locals) {
  using Sh = FftShape<P, G>;
  constexpr int p = Sh::p, q = Sh::q, h = Sh::h, F = Sh::F;
  constexpr int P3 = Sh::P3, PPH = Sh::PPH, PQH = Sh::PQH;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2 *D = reinterpret_cast<double2 *>(smraw);               // [G][p][p][h]  y inverted, j < p
  double2 *C = reinterpret_cast<double2 *>(smraw + Sh::V1);      // [G][p][q][h]  x inverted, i < p
  const int n = 1 << level;
  const int64_t ncell = int64_t(1) << (3 * level);
  const int64_t ngroups = ncell / G;
  const double norm = scale / ((double)q * q * q);
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
    __syncthreads();  // the previous run's readers of C and D are done
    const double2 *src = Y + (int64_t)crel * F * ncell + lex0;
    // x: q bins -> p outputs, e^{+2 pi i i kx / q}; line (ky, kz, gi), the
    // cell index fastest across lanes (G * 16-byte runs), its q bins loaded
    // from the spectrum into registers (all in flight at once)
    for (int l = threadIdx.x; l < G * q * h; l += blockDim.x) {
      const int rem = l / G, gi = l - rem * G;
      double2 v[q];
#pragma unroll
      for (int kx = 0; kx < q; ++kx) v[kx] = src[(int64_t)(kx * q * h + rem) * ncell + gi];
      double2 *dst = C + gi * PQH + rem;
#pragma unroll
      for (int i = 0; i < p; ++i) {
        double re = v[0].x, im = v[0].y;
#pragma unroll
        for (int kx = 1; kx < q; ++kx) {
          const int r = (i * kx) % q;
          re = fma(v[kx].x, g.c[r], fma(-v[kx].y, g.s[r], re));
          im = fma(v[kx].y, g.c[r], fma(v[kx].x, g.s[r], im));
        }
        dst[i * q * h] = make_double2(re, im);
      }
    }
    __syncthreads();
    // y: q bins -> p outputs; line (gi, i, kz)
    for (int l = threadIdx.x; l < G * p * h; l += blockDim.x) {
      const int gi = l / (p * h), r0 = l - gi * p * h, i = r0 / h, kz = r0 - i * h;
      const double2 *c = C + gi * PQH + i * q * h + kz;
      double2 v[q];
#pragma unroll
      for (int ky = 0; ky < q; ++ky) v[ky] = c[ky * h];
      double2 *dst = D + gi * PPH + i * p * h + kz;
#pragma unroll
      for (int j = 0; j < p; ++j) {
        double re = v[0].x, im = v[0].y;
#pragma unroll
        for (int ky = 1; ky < q; ++ky) {
          const int r = (j * ky) % q;
          re = fma(v[ky].x, g.c[r], fma(-v[ky].y, g.s[r], re));
          im = fma(v[ky].y, g.c[r], fma(v[ky].x, g.s[r], im));
        }
        dst[j * h] = make_double2(re, im);
      }
    }
    __syncthreads();
    // z: Hermitian half spectrum -> p real outputs (irfft: DC imaginary part
    // dropped, bins 1..q/2 counted twice; q is odd so no Nyquist bin);
    // line (gi, i, j)
    for (int l = threadIdx.x; l < G * p * p; l += blockDim.x) {
      const int gi = l / (p * p), ij = l - gi * p * p;
      const int64_t cell = (int64_t)morton3(x, y, z0 + gi);
      if (cell < cell_lo || cell >= cell_hi) continue;
      const double2 *d = D + gi * PPH + ij * h;
      double2 v[h];
#pragma unroll
      for (int kz = 0; kz < h; ++kz) v[kz] = d[kz];
      double *out = locals + (cell * m + c0 + crel) * (int64_t)P3 + ij * p;
#pragma unroll
      for (int k = 0; k < p; ++k) {
        double t = v[0].x;
#pragma unroll
        for (int kz = 1; kz < h; ++kz) {
          const int r = (k * kz) % q;
          t = fma(2.0 * v[kz].x, g.c[r], fma(-2.0 * v[kz].y, g.s[r], t));
        }
        out[k] = norm * t;
      }
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

template <int P>
int launch_fft(bool fwd, const double *moments, const double2 *Y, int level, int64_t cell_lo,
               int64_t cell_hi, int m, int c0, int ccur, const FftGeom &g, double scale,
               double2 *X, double *locals, cudaStream_t st) {
  constexpr int G = fft_cells<P>();
  using Sh = FftShape<P, G>;
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(fft_fwd_kernel<P, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Sh::smem);
    cudaFuncSetAttribute(fft_inv_kernel<P, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Sh::smem_inv);
  }
  const int64_t ncell = int64_t(1) << (3 * level);
  const unsigned grid = (unsigned)std::min<int64_t>(ncell / G * ccur, kNumSMs * 24);
  if (fwd) {
    fft_fwd_kernel<P, G><<<grid, fft_threads<P, G>(), Sh::smem, st>>>(moments, level, m, c0, ccur, g, X);
    return check_launch("fft_fwd_kernel");
  }
  fft_inv_kernel<P, G><<<grid, fft_threads<P, G>(), Sh::smem_inv, st>>>(Y, level, cell_lo, cell_hi, m, c0, ccur,
                                                        g, scale, locals);
  return check_launch("fft_inv_kernel");
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
  const int n = 1 << level;
  const unsigned tiles = (unsigned)(ceil_div(n, kTX) * ceil_div(n, kTY) * ceil_div(n, kTZ));
  const size_t smem_s = sizeof(double2) * (kHX * kHYP * kHZP + 343);
  const size_t smem_s2 = sizeof(double2) * (kH2X * kHYP * kHZP + 343);
  const unsigned tiles2 = (unsigned)(ceil_div(n, kT2X) * ceil_div(n, kTY) * ceil_div(n, kTZ));
  // BFMM_STENCIL=2: the two-x-targets-per-thread kernel (fewer halo
  // reads, but 85 KB tiles leave 2 CTAs/SM; measured slower on C3)
  const char *sv = getenv("BFMM_STENCIL");
  const int stencil = sv && sv[0] >= '1' && sv[0] <= '3' ? sv[0] - '0' : 3;
  const bool stencil1 = stencil == 1;
  const size_t smem_s3 = sizeof(double2) * (kHX * kHY * kH3ZP + 343);
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(stencil_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_s);
    cudaFuncSetAttribute(stencil2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_s2);
    cudaFuncSetAttribute(stencil3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_s3);
  }
  for (int c0 = 0; c0 < m; c0 += cc) {
    const int ccur = std::min(cc, m - c0);
    int rc = 0;
    switch (p) {
#define BFMM_FFT_FWD(PP)                                                                       \
  case PP:                                                                                     \
    rc = launch_fft<PP>(true, moments, nullptr, level, 0, 0, m, c0, ccur, g, 1.0, X, nullptr,  \
                        st);                                                                   \
    break;
      BFMM_FFT_FWD(2) BFMM_FFT_FWD(3) BFMM_FFT_FWD(4) BFMM_FFT_FWD(5) BFMM_FFT_FWD(6)
      BFMM_FFT_FWD(7) BFMM_FFT_FWD(8) BFMM_FFT_FWD(9) BFMM_FFT_FWD(10) BFMM_FFT_FWD(11)
      BFMM_FFT_FWD(12)
#undef BFMM_FFT_FWD
    }
    if (rc) return rc;
    if (stencil == 3) {
      stencil3_kernel<<<dim3(tiles, (unsigned)F, (unsigned)ccur), 128, smem_s3, st>>>(
          X, Y, level, (int)F, reinterpret_cast<const double2 *>(symbols), taps, 8 * q_lo,
          8 * (q_lo + nq));
      if (check_launch("stencil3_kernel")) return 1;
    } else if (stencil1) {
      stencil_kernel<<<dim3(tiles, (unsigned)F, (unsigned)ccur), dim3(kTX, kTY, 2), smem_s, st>>>(
          X, Y, level, (int)F, reinterpret_cast<const double2 *>(symbols), taps, 8 * q_lo,
          8 * (q_lo + nq));
      if (check_launch("stencil_kernel")) return 1;
    } else {
      stencil2_kernel<<<dim3(tiles2, (unsigned)F, (unsigned)ccur), 128, smem_s2, st>>>(
          X, Y, level, (int)F, reinterpret_cast<const double2 *>(symbols), taps, 8 * q_lo,
          8 * (q_lo + nq));
      if (check_launch("stencil2_kernel")) return 1;
    }
    switch (p) {
#define BFMM_FFT_INV(PP)                                                                       \
  case PP:                                                                                     \
    rc = launch_fft<PP>(false, nullptr, Y, level, 8 * q_lo, 8 * (q_lo + nq), m, c0, ccur, g,   \
                        scale, nullptr, locals, st);                                           \
    break;
      BFMM_FFT_INV(2) BFMM_FFT_INV(3) BFMM_FFT_INV(4) BFMM_FFT_INV(5) BFMM_FFT_INV(6)
      BFMM_FFT_INV(7) BFMM_FFT_INV(8) BFMM_FFT_INV(9) BFMM_FFT_INV(10) BFMM_FFT_INV(11)
      BFMM_FFT_INV(12)
#undef BFMM_FFT_INV
    }
    if (rc) return rc;
  }
  return 0;
}
