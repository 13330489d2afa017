// Warp-per-leaf P2M / L2P specialised on the interpolation order P (included
// by interp.cu; the production path for p <= 8).
//
// A warp owns one leaf at a time.  P2M: lanes compute the 3 x P weights of up
// to 32 points into the warp's shared slice; lane l then owns the node pairs
// (i, j) = divmod(l + 32u, P) and accumulates all P nodes k of each, i.e.
// M[i][j][k] += ((wx_i wy_j) wz_k) w over the leaf's points in sorted order
// (the product order of interp_matrix_3d and the reduceat order of
// engine.py:176-182).  L2P: lanes own points; the leaf's locals of one column
// sit in shared memory and every lane contracts them with its weights.
#pragma once

// 1-D weights from the basis staged in shared memory (sS = S[n][j] for
// Chebyshev, sN = nodes for uniform): keeping the P^2 coefficients out of
// registers is what lets these kernels run at full occupancy.
template <int P>
__device__ __forceinline__ void weights_s(const double *sS, const double *sN, int scheme,
                                          double x, double *w) {
  if (scheme == 0) {
    x = fmin(1.0, fmax(-1.0, x));
    double T[P];
    T[0] = 1.0;
    if (P > 1) T[1] = x;
#pragma unroll
    for (int n = 2; n < P; ++n) T[n] = fma(2.0 * x, T[n - 1], -T[n - 2]);
#pragma unroll
    for (int j = 0; j < P; ++j) {
      double s = 0.0;
#pragma unroll
      for (int n = 0; n < P; ++n) s = fma(T[n], sS[n * P + j], s);
      w[j] = s;
    }
  } else {
    // Lagrange products in the reference's factor order, with the inverse
    // node differences staged in sS (one rounding per factor off the
    // reference's division, far inside the 1e-10 parity bar)
#pragma unroll
    for (int j = 0; j < P; ++j) {
      double v = 1.0;
#pragma unroll
      for (int k = 0; k < P; ++k)
        if (k != j) v *= (x - sN[k]) * sS[j * P + k];
      w[j] = v;
    }
  }
}

// weights_s at two coordinates (a leaf's and its parent's frame) sharing
// every basis load from shared memory; same arithmetic per output as
// weights_s (bitwise equal to two calls)
template <int P>
__device__ __forceinline__ void weights2_s(const double *sS, const double *sN, int scheme,
                                           double x, double y, double *w, double *v) {
  if (scheme == 0) {
    x = fmin(1.0, fmax(-1.0, x));
    y = fmin(1.0, fmax(-1.0, y));
    double T[P], U[P];
    T[0] = 1.0;
    U[0] = 1.0;
    if (P > 1) {
      T[1] = x;
      U[1] = y;
    }
#pragma unroll
    for (int n = 2; n < P; ++n) {
      T[n] = fma(2.0 * x, T[n - 1], -T[n - 2]);
      U[n] = fma(2.0 * y, U[n - 1], -U[n - 2]);
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      double s = 0.0, t = 0.0;
#pragma unroll
      for (int n = 0; n < P; ++n) {
        const double b = sS[n * P + j];
        s = fma(T[n], b, s);
        t = fma(U[n], b, t);
      }
      w[j] = s;
      v[j] = t;
    }
  } else {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      double a = 1.0, b = 1.0;
#pragma unroll
      for (int k = 0; k < P; ++k)
        if (k != j) {
          const double nk = sN[k], f = sS[j * P + k];
          a *= (x - nk) * f;
          b *= (y - nk) * f;
        }
      w[j] = a;
      v[j] = b;
    }
  }
}

template <int P>
__device__ __forceinline__ void stage_basis(const Interp &ip, double *sS, double *sN) {
  // static indices into the parameter block (a dynamic index would make the
  // compiler materialise the whole Interp struct)
  if (threadIdx.x < P) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (threadIdx.x == k) sN[k] = ip.nodes[k];
#pragma unroll
      for (int j = 0; j < P; ++j)
        if (threadIdx.x == j)
          sS[j * P + k] = ip.scheme == 0 ? ip.S[j * P + k]
                                         : (j != k ? 1.0 / (ip.nodes[j] - ip.nodes[k]) : 0.0);
    }
  }
  __syncthreads();
}

// Leaf-frame coordinate like ref_coord, scaled by the precomputed 1 / hw.
__device__ __forceinline__ double ref_coord_m(double x, double lo, double h, double inv_hw,
                                             int cell, int32_t *flag) {
  const double center = lo + ((double)cell + 0.5) * h;
  const double r = (x - center) * inv_hw;
  if (fabs(r) > 1.0 + 1e-9) atomicOr(flag, 1);
  return fmin(1.0, fmax(-1.0, r));
}

// The leaf cell of a coordinate, computed exactly like the tree build
// (tree.cu leaf_keys_kernel): IEEE subtraction and division, floor, clip.
__device__ __forceinline__ int leaf_coord(double x, double lo, double h, int nmax) {
  const double f = floor(__ddiv_rn(__dsub_rn(x, lo), h));
  const int64_t v = (int64_t)f;
  return (int)(v < 0 ? 0 : (v > nmax ? nmax : v));
}

template <int P>
__global__ void __launch_bounds__(32 * kLeafWarps)
p2m_leaf_kernel(const double *__restrict__ pts4, const double *__restrict__ ws,
                int m, const int64_t *__restrict__ leaves,
                const int64_t *__restrict__ starts,
                const int64_t *__restrict__ counts,
                const int64_t *__restrict__ n_leaves, Interp ip, LeafGeom g,
                double *__restrict__ moments, int32_t *flag) {
  constexpr int NP = (P * P + 31) / 32;  // (i, j) pairs per lane
  __shared__ double s_w[kLeafWarps][32][3 * P];
  __shared__ double s_v[kLeafWarps][32];
  __shared__ double sS[P * P], sN[P];
  stage_basis<P>(ip, sS, sN);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nl = *n_leaves;
  for (int64_t leaf = int64_t(blockIdx.x) * kLeafWarps + wid; leaf < nl;
       leaf += int64_t(gridDim.x) * kLeafWarps) {
    const int64_t cell = leaves[leaf];
    if (cell < g.cell_lo || cell >= g.cell_hi) continue;  // other rank's shard
    const int64_t s0 = starts[leaf], cnt = counts[leaf];
    int cx, cy, cz;
    unmorton3((uint64_t)cell, cx, cy, cz);
    for (int c = 0; c < m; ++c) {
      double acc[NP][P];
#pragma unroll
      for (int u = 0; u < NP; ++u)
#pragma unroll
        for (int k = 0; k < P; ++k) acc[u][k] = 0.0;
      for (int64_t c0 = 0; c0 < cnt; c0 += 32) {
        const int nb = (int)(cnt - c0 < 32 ? cnt - c0 : 32);
        __syncwarp();
        if (lane < nb) {
          const int64_t i = s0 + c0 + lane;
          const double4 q = reinterpret_cast<const double4 *>(pts4)[i];
          weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.x, g.lo[0], g.h, 1.0 / g.hw, cx, flag),
                       &s_w[wid][lane][0]);
          weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.y, g.lo[1], g.h, 1.0 / g.hw, cy, flag),
                       &s_w[wid][lane][P]);
          weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.z, g.lo[2], g.h, 1.0 / g.hw, cz, flag),
                       &s_w[wid][lane][2 * P]);
          s_v[wid][lane] = ws[i * m + c];
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < NP; ++u) {
          const int pr = lane + 32 * u;
          if (pr < P * P) {
            const int ii = pr / P, jj = pr - ii * P;
            for (int t = 0; t < nb; ++t) {
              const double *wt = s_w[wid][t];
              const double wxy = wt[ii] * wt[P + jj], v = s_v[wid][t];
#pragma unroll
              for (int k = 0; k < P; ++k) acc[u][k] += (wxy * wt[2 * P + k]) * v;
            }
          }
        }
      }
      double *dst = moments + (cell * m + c) * (int64_t)(P * P * P);
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int pr = lane + 32 * u;
        if (pr < P * P) {
#pragma unroll
          for (int k = 0; k < P; ++k) dst[pr * P + k] = acc[u][k];
        }
      }
    }
  }
}

// P2M for sparse leaves (a few points each): one thread per (leaf, x-node
// i) accumulating the P x P moments M[i][j][k] over the leaf's points in
// sorted order, with the same products as p2m_leaf_kernel -- no idle lanes,
// and the threads of a leaf read its points as L1 broadcasts.
template <int P>
__global__ void __launch_bounds__(128)
p2m_thread_kernel(const double *__restrict__ pts4, const double *__restrict__ ws,
                  int m, const int64_t *__restrict__ leaves,
                  const int64_t *__restrict__ starts,
                  const int64_t *__restrict__ counts,
                  const int64_t *__restrict__ n_leaves, Interp ip, LeafGeom g,
                  double *__restrict__ moments, int32_t *flag) {
  __shared__ double sS[P * P], sN[P];
  stage_basis<P>(ip, sS, sN);
  const int64_t nl = *n_leaves;
  const double inv_hw = 1.0 / g.hw;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nl * P;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t leaf = t / P;
    const int ii = (int)(t - leaf * P);
    const int64_t cell = leaves[leaf];
    if (cell < g.cell_lo || cell >= g.cell_hi) continue;  // other rank's shard
    const int64_t s0 = starts[leaf], cnt = counts[leaf];
    int cx, cy, cz;
    unmorton3((uint64_t)cell, cx, cy, cz);
    for (int c = 0; c < m; ++c) {
      double acc[P][P];
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int k = 0; k < P; ++k) acc[j][k] = 0.0;
      for (int64_t pt = 0; pt < cnt; ++pt) {
        const int64_t i = s0 + pt;
        const double4 q = reinterpret_cast<const double4 *>(pts4)[i];
        double wx[P], wy[P], wz[P];
        weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.x, g.lo[0], g.h, inv_hw, cx, flag), wx);
        weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.y, g.lo[1], g.h, inv_hw, cy, flag), wy);
        weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.z, g.lo[2], g.h, inv_hw, cz, flag), wz);
        double wxi = wx[0];
#pragma unroll
        for (int u = 1; u < P; ++u) wxi = ii == u ? wx[u] : wxi;
        const double v = ws[i * m + c];
#pragma unroll
        for (int j = 0; j < P; ++j) {
          const double wxy = wxi * wy[j];
#pragma unroll
          for (int k = 0; k < P; ++k) acc[j][k] += (wxy * wz[k]) * v;
        }
      }
      double *dst = moments + (cell * m + c) * (int64_t)(P * P * P) + ii * P * P;
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int k = 0; k < P; ++k) dst[j * P + k] = acc[j][k];
    }
  }
}

// L2P (engine.py:313-347), one warp per leaf: the leaf's locals (one column
// at a time) are brought into the warp's shared slice with coalesced loads;
// each lane evaluates its point's weights, parks the P^2 products wx wy in
// its own shared column, and contracts the locals pair by pair (broadcast
// reads of L, z weights in registers), which keeps the kernel at ~40
// registers and full occupancy.
template <int P>
constexpr int l2p_warps() { return P <= 6 ? kLeafWarps : 1; }  // static smem < 48 KB

template <int P>
__global__ void __launch_bounds__(32 * l2p_warps<P>())
l2p_warp_kernel(const double *__restrict__ pts4, int m,
                const int64_t *__restrict__ leaves, const int64_t *__restrict__ starts,
                const int64_t *__restrict__ counts, const int64_t *__restrict__ n_leaves,
                Interp ip, LeafGeom g, const double *__restrict__ locals,
                double *__restrict__ phi, int32_t *flag) {
  constexpr int P2 = P * P, P3 = P2 * P, W = l2p_warps<P>();
  __shared__ double sL[W][P3];
  __shared__ double sWxy[W][P2][32];
  __shared__ double sS[P * P], sN[P];
  stage_basis<P>(ip, sS, sN);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double inv_hw = 1.0 / g.hw;
  const int64_t nl = *n_leaves;
  for (int64_t leaf = int64_t(blockIdx.x) * W + wid; leaf < nl;
       leaf += int64_t(gridDim.x) * W) {
    const int64_t cell = leaves[leaf];
    if (cell < g.cell_lo || cell >= g.cell_hi) continue;  // other rank's shard
    const int64_t s0 = starts[leaf], cnt = counts[leaf];
    int cx, cy, cz;
    unmorton3((uint64_t)cell, cx, cy, cz);
    for (int64_t c0 = 0; c0 < cnt; c0 += 32) {
      const bool have = c0 + lane < cnt;
      const int64_t i = s0 + c0 + (have ? lane : 0);
      double wz[P];
      const double4 q = reinterpret_cast<const double4 *>(pts4)[i];
      // column 0's locals are loaded into registers before the weights are
      // evaluated, so the global-memory latency overlaps that arithmetic
      constexpr int NL = (P3 + 31) / 32;
      double lpre[NL];
      {
        const double *src0 = locals + (cell * m) * (int64_t)P3;
#pragma unroll
        for (int u = 0; u < NL; ++u) {
          const int e = lane + 32 * u;
          lpre[u] = e < P3 ? src0[e] : 0.0;
        }
      }
      {
        double wx[P], wy[P];
        weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.x, g.lo[0], g.h, inv_hw, cx, flag), wx);
        weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.y, g.lo[1], g.h, inv_hw, cy, flag), wy);
        __syncwarp();
#pragma unroll
        for (int a = 0; a < P; ++a)
#pragma unroll
          for (int b = 0; b < P; ++b) sWxy[wid][a * P + b][lane] = wx[a] * wy[b];
      }
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.z, g.lo[2], g.h, inv_hw, cz, flag), wz);
      for (int c = 0; c < m; ++c) {
        __syncwarp();
        if (c == 0) {
#pragma unroll
          for (int u = 0; u < NL; ++u) {
            const int e = lane + 32 * u;
            if (e < P3) sL[wid][e] = lpre[u];
          }
        } else {
          const double *src = locals + (cell * m + c) * (int64_t)P3;
          for (int e = lane; e < P3; e += 32) sL[wid][e] = src[e];
        }
        __syncwarp();
        const double *L = sL[wid];
        // one partial sum per x node a (P independent chains), added in a
        // fixed order -- the same arithmetic as l2p_point_kernel
        double sa[P];
#pragma unroll
        for (int a = 0; a < P; ++a) {
          sa[a] = 0.0;
#pragma unroll
          for (int b = 0; b < P; ++b) {
            const int ab = a * P + b;
            double sb = 0.0;
#pragma unroll
            for (int k = 0; k < P; ++k) sb = fma(wz[k], L[ab * P + k], sb);
            sa[a] = fma(sWxy[wid][ab][lane], sb, sa[a]);
          }
        }
        double s = sa[0];
#pragma unroll
        for (int a = 1; a < P; ++a) s += sa[a];
        if (have) phi[i * m + c] = s;
      }
    }
  }
}

// P2M for sparse clouds (a few points per leaf, e.g. C5's 3.8), over CELL
// chunks: a CTA owns kP2MCells consecutive leaf cells of [cell_lo, cell_hi)
// and writes ALL of their moments -- zeros for empty cells, so the level-L
// array needs no memset.  The chunk's points (contiguous in sorted order)
// get their 3 x P weights once, one thread per point, into shared memory;
// then one thread per output (cell, column, node) sums its cell's points in
// sorted order (the reduceat order of engine.py:176-182, the products of
// p2m_leaf_kernel), so consecutive threads write consecutive moments.
constexpr int kP2MCells = 32, kP2MThreads = 256;
// points per batch: the 3 x P weights in <= 40 KB of static shared memory
template <int P>
constexpr int p2m_pts() {
  return (40 * 1024 / (24 * P)) / 32 * 32 > 512 ? 512 : (40 * 1024 / (24 * P)) / 32 * 32;
}

template <int P>
__global__ void __launch_bounds__(kP2MThreads, 3)
p2m_cells_kernel(const double *__restrict__ pts4, const double *__restrict__ ws, int m,
                 const int32_t *__restrict__ cell_start, const int32_t *__restrict__ cell_count,
                 Interp ip, LeafGeom g, double *__restrict__ moments, int32_t *flag) {
  constexpr int P3 = P * P * P, kP2MPts = p2m_pts<P>();
  __shared__ double s_w[kP2MPts][3 * P];
  __shared__ int s_off[kP2MCells + 1];
  __shared__ int64_t s_first;
  __shared__ double sS[P * P], sN[P];
  stage_basis<P>(ip, sS, sN);
  const double inv_hw = 1.0 / g.hw;
  const int64_t ncells = g.cell_hi - g.cell_lo;
  const int64_t nchunks = (ncells + kP2MCells - 1) / kP2MCells;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t c0 = g.cell_lo + ch * kP2MCells;
    const int nc = (int)(g.cell_hi - c0 < kP2MCells ? g.cell_hi - c0 : kP2MCells);
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      const int cnt = lane < nc ? cell_count[c0 + lane] : 0;
      int inc = cnt;  // inclusive scan of the counts
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += v;
      }
      s_off[lane + 1] = inc;
      if (lane == 0) s_off[0] = 0;
      // first point of the chunk: the start of its first occupied cell
      const unsigned occ = __ballot_sync(0xffffffffu, cnt > 0);
      if (lane == 0) s_first = occ ? (int64_t)cell_start[c0 + __ffs(occ) - 1] : 0;
    }
    __syncthreads();
    const int npts = s_off[nc];
    const int64_t first = s_first;
    const int nout = nc * m * P3;
    // points in batches of kP2MPts (a crowded chunk takes several)
    for (int b0 = 0; b0 < max(npts, 1); b0 += kP2MPts) {
      const int nb = min(kP2MPts, npts - b0);
      if (b0 > 0) __syncthreads();
      for (int t = threadIdx.x; t < nb; t += kP2MThreads) {
        const int64_t i = first + b0 + t;
        const double4 q = reinterpret_cast<const double4 *>(pts4)[i];
        // the point's cell: the last chunk cell whose offset is <= b0 + t
        int lo = 0;
#pragma unroll
        for (int step = kP2MCells / 2; step > 0; step >>= 1)
          if (lo + step <= nc && s_off[lo + step] <= b0 + t) lo += step;
        int cx, cy, cz;
        unmorton3((uint64_t)(c0 + lo), cx, cy, cz);
        weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.x, g.lo[0], g.h, inv_hw, cx, flag),
                     &s_w[t][0]);
        weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.y, g.lo[1], g.h, inv_hw, cy, flag),
                     &s_w[t][P]);
        weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.z, g.lo[2], g.h, inv_hw, cz, flag),
                     &s_w[t][2 * P]);
      }
      __syncthreads();
      for (int o = threadIdx.x; o < nout; o += kP2MThreads) {
        const int cl = o / (m * P3), rem = o - cl * m * P3, c = rem / P3, a = rem - c * P3;
        const int ii = a / (P * P), jj = (a / P) % P, kk = a % P;
        const int p0 = max(s_off[cl], b0), p1 = min(s_off[cl + 1], b0 + nb);
        double acc = 0.0;
        for (int pt = p0; pt < p1; ++pt) {
          const double *wt = s_w[pt - b0];
          acc += ((wt[ii] * wt[P + jj]) * wt[2 * P + kk]) * ws[(first + pt) * m + c];
        }
        double *dst = moments + (c0 * m) * (int64_t)P3 + o;
        *dst = b0 == 0 ? acc : *dst + acc;
      }
    }
  }
}

// L2P for sparse leaves (a few points each, e.g. C5's 3.8): one thread per
// sorted point instead of one warp per leaf, so no lanes idle.  The point's
// leaf is recomputed from its coordinates (bit-identical to the tree build),
// its weights evaluated once, and the leaf's locals contracted z, y, x
// straight from global memory (neighbouring threads share a leaf: L1
// broadcasts).  Same arithmetic as l2p_warp_kernel.
template <int P>
__global__ void __launch_bounds__(128)
l2p_point_kernel(const double *__restrict__ pts4, int m,
                 const int64_t *__restrict__ starts, const int64_t *__restrict__ counts,
                 const int64_t *__restrict__ n_leaves, int levels, Interp ip, LeafGeom g,
                 const double *__restrict__ locals, double *__restrict__ phi,
                 int32_t *flag) {
  constexpr int P2 = P * P, P3 = P2 * P;
  __shared__ double sS[P * P], sN[P];
  stage_basis<P>(ip, sS, sN);
  const int64_t nl = *n_leaves;
  if (nl == 0) return;
  const int64_t n = starts[nl - 1] + counts[nl - 1];
  const int nmax = (1 << levels) - 1;
  const double inv_hw = 1.0 / g.hw;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double4 q = reinterpret_cast<const double4 *>(pts4)[i];
    const int cx = leaf_coord(q.x, g.lo[0], g.h, nmax), cy = leaf_coord(q.y, g.lo[1], g.h, nmax),
              cz = leaf_coord(q.z, g.lo[2], g.h, nmax);
    const int64_t cell = (int64_t)morton3(cx, cy, cz);
    if (cell < g.cell_lo || cell >= g.cell_hi) continue;  // other rank's shard
    double wx[P], wy[P], wz[P];
    weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.x, g.lo[0], g.h, inv_hw, cx, flag), wx);
    weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.y, g.lo[1], g.h, inv_hw, cy, flag), wy);
    weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.z, g.lo[2], g.h, inv_hw, cz, flag), wz);
    for (int c = 0; c < m; ++c) {
      const double *L = locals + (cell * m + c) * (int64_t)P3;
      double sa[P];
#pragma unroll
      for (int a = 0; a < P; ++a) {
        sa[a] = 0.0;
#pragma unroll
        for (int b = 0; b < P; ++b) {
          const double *Lab = L + (a * P + b) * P;
          double sb = 0.0;
#pragma unroll
          for (int k = 0; k < P; ++k) sb = fma(wz[k], Lab[k], sb);
          sa[a] = fma(wx[a] * wy[b], sb, sa[a]);  // same products as the warp kernel
        }
      }
      double s = sa[0];
#pragma unroll
      for (int a = 1; a < P; ++a) s += sa[a];
      phi[i * m + c] = s;
    }
  }
}

struct LeafCall {
  const double *pts4, *ws;
  int m;
  const int64_t *leaves, *starts, *counts, *n_leaves;
  int64_t max_leaves;
  int levels;
  bool per_point;  // L2P: thread per point (sparse leaves)
  Interp ip;
  LeafGeom g;
  const double *locals;
  double *out;  // moments (P2M) or phi (L2P)
  int32_t *flag;
  cudaStream_t st;
};

template <int P>
int launch_leaf(bool p2m, const LeafCall &a) {
  const unsigned grid = (unsigned)grid_cap(ceil_div(a.max_leaves, kLeafWarps), 16);
  if (p2m && a.per_point) {
    p2m_thread_kernel<P><<<(unsigned)grid_cap(ceil_div(a.max_leaves * P, 128), 16), 128, 0,
                           a.st>>>(a.pts4, a.ws, a.m, a.leaves, a.starts, a.counts,
                                   a.n_leaves, a.ip, a.g, a.out, a.flag);
    return check_launch("p2m_thread_kernel");
  }
  if (p2m) {
    p2m_leaf_kernel<P><<<grid, 32 * kLeafWarps, 0, a.st>>>(
        a.pts4, a.ws, a.m, a.leaves, a.starts, a.counts, a.n_leaves, a.ip, a.g, a.out,
        a.flag);
    return check_launch("p2m_leaf_kernel");
  }
  if (a.per_point) {
    l2p_point_kernel<P><<<(unsigned)(kNumSMs * 16), 128, 0, a.st>>>(
        a.pts4, a.m, a.starts, a.counts, a.n_leaves, a.levels, a.ip, a.g, a.locals, a.out,
        a.flag);
    return check_launch("l2p_point_kernel");
  }
  l2p_warp_kernel<P><<<(unsigned)grid_cap(ceil_div(a.max_leaves, l2p_warps<P>()), 16),
                       32 * l2p_warps<P>(), 0, a.st>>>(
      a.pts4, a.m, a.leaves, a.starts, a.counts, a.n_leaves, a.ip, a.g, a.locals, a.out,
      a.flag);
  return check_launch("l2p_warp_kernel");
}

// L2P for sparse clouds over leaf-CELL chunks: a CTA stages the locals of
// cc consecutive cells in shared memory with coalesced loads, then one
// thread per point of the chunk (contiguous in sorted order) contracts them
// with the same arithmetic as l2p_point_kernel (bitwise equal).
template <int P>
__global__ void __launch_bounds__(kP2MThreads, 2)
l2p_cells_kernel(const double *__restrict__ pts4, int m, int cc,
                 const int32_t *__restrict__ cell_start, const int32_t *__restrict__ cell_count,
                 Interp ip, LeafGeom g, const double *__restrict__ locals,
                 double *__restrict__ phi, int32_t *flag) {
  constexpr int P3 = P * P * P;
  extern __shared__ double sLoc[];  // [cc][m][P^3]
  __shared__ int s_off[kP2MCells + 1];
  __shared__ int64_t s_first;
  __shared__ double sS[P * P], sN[P];
  stage_basis<P>(ip, sS, sN);
  const double inv_hw = 1.0 / g.hw;
  const int64_t ncells = g.cell_hi - g.cell_lo;
  const int64_t nchunks = (ncells + cc - 1) / cc;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t c0 = g.cell_lo + ch * cc;
    const int nc = (int)(g.cell_hi - c0 < cc ? g.cell_hi - c0 : cc);
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      const int cnt = lane < nc ? cell_count[c0 + lane] : 0;
      int inc = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += v;
      }
      s_off[lane + 1] = inc;
      if (lane == 0) s_off[0] = 0;
      const unsigned occ = __ballot_sync(0xffffffffu, cnt > 0);
      if (lane == 0) s_first = occ ? (int64_t)cell_start[c0 + __ffs(occ) - 1] : 0;
    }
    const double *src = locals + c0 * (int64_t)m * P3;
    for (int e = threadIdx.x; e < nc * m * P3; e += kP2MThreads) sLoc[e] = src[e];
    __syncthreads();
    const int npts = s_off[nc];
    const int64_t first = s_first;
    for (int t = threadIdx.x; t < npts; t += kP2MThreads) {
      int lo = 0;
#pragma unroll
      for (int step = kP2MCells / 2; step > 0; step >>= 1)
        if (lo + step <= nc && s_off[lo + step] <= t) lo += step;
      int cx, cy, cz;
      unmorton3((uint64_t)(c0 + lo), cx, cy, cz);
      const int64_t i = first + t;
      const double4 q = reinterpret_cast<const double4 *>(pts4)[i];
      double wx[P], wy[P], wz[P];
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.x, g.lo[0], g.h, inv_hw, cx, flag), wx);
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.y, g.lo[1], g.h, inv_hw, cy, flag), wy);
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(q.z, g.lo[2], g.h, inv_hw, cz, flag), wz);
      for (int c = 0; c < m; ++c) {
        const double *L = sLoc + (lo * m + c) * P3;
        double sa[P];
#pragma unroll
        for (int a = 0; a < P; ++a) {
          sa[a] = 0.0;
#pragma unroll
          for (int b = 0; b < P; ++b) {
            const double *Lab = L + (a * P + b) * P;
            double sb = 0.0;
#pragma unroll
            for (int k = 0; k < P; ++k) sb = fma(wz[k], Lab[k], sb);
            sa[a] = fma(wx[a] * wy[b], sb, sa[a]);
          }
        }
        double s = sa[0];
#pragma unroll
        for (int a = 1; a < P; ++a) s += sa[a];
        phi[i * m + c] = s;
      }
    }
  }
}

template <int P>
int launch_l2p_cells(const LeafCall &a, const int32_t *cell_start, const int32_t *cell_count) {
  constexpr int P3 = P * P * P;
  int cc = kP2MCells;
  while (cc > 1 && (size_t)cc * a.m * P3 * sizeof(double) > 96 * 1024) cc >>= 1;
  const size_t smem = (size_t)cc * a.m * P3 * sizeof(double);
  if (smem > 96 * 1024) {
    set_error("bfmm_l2p_cells: m * p^3 = %d too large", a.m * P3);
    return 2;
  }
  static unsigned long long attr = 0;
  if (first_on_device(&attr))
    cudaFuncSetAttribute(l2p_cells_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         96 * 1024);
  const int64_t chunks = ceil_div(a.g.cell_hi - a.g.cell_lo, cc);
  if (chunks <= 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>(chunks, (int64_t)kNumSMs * 8);
  l2p_cells_kernel<P><<<grid, kP2MThreads, smem, a.st>>>(a.pts4, a.m, cc, cell_start,
                                                         cell_count, a.ip, a.g, a.locals, a.out,
                                                         a.flag);
  return check_launch("l2p_cells_kernel");
}

inline int dispatch_l2p_cells(int p, const LeafCall &a, const int32_t *cs, const int32_t *cc) {
  switch (p) {
    case 2: return launch_l2p_cells<2>(a, cs, cc);
    case 3: return launch_l2p_cells<3>(a, cs, cc);
    case 4: return launch_l2p_cells<4>(a, cs, cc);
    case 5: return launch_l2p_cells<5>(a, cs, cc);
    case 6: return launch_l2p_cells<6>(a, cs, cc);
    case 7: return launch_l2p_cells<7>(a, cs, cc);
    default: return launch_l2p_cells<8>(a, cs, cc);
  }
}

template <int P>
int launch_p2m_cells(const LeafCall &a, const int32_t *cell_start, const int32_t *cell_count) {
  const int64_t chunks = ceil_div(a.g.cell_hi - a.g.cell_lo, kP2MCells);
  if (chunks <= 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>(chunks, (int64_t)kNumSMs * 8);
  p2m_cells_kernel<P><<<grid, kP2MThreads, 0, a.st>>>(a.pts4, a.ws, a.m, cell_start, cell_count,
                                                       a.ip, a.g, a.out, a.flag);
  return check_launch("p2m_cells_kernel");
}

inline int dispatch_p2m_cells(int p, const LeafCall &a, const int32_t *cs, const int32_t *cc) {
  switch (p) {
    case 2: return launch_p2m_cells<2>(a, cs, cc);
    case 3: return launch_p2m_cells<3>(a, cs, cc);
    case 4: return launch_p2m_cells<4>(a, cs, cc);
    case 5: return launch_p2m_cells<5>(a, cs, cc);
    case 6: return launch_p2m_cells<6>(a, cs, cc);
    case 7: return launch_p2m_cells<7>(a, cs, cc);
    default: return launch_p2m_cells<8>(a, cs, cc);
  }
}

inline int dispatch_leaf(int p, bool p2m, const LeafCall &a) {
  switch (p) {
    case 2: return launch_leaf<2>(p2m, a);
    case 3: return launch_leaf<3>(p2m, a);
    case 4: return launch_leaf<4>(p2m, a);
    case 5: return launch_leaf<5>(p2m, a);
    case 6: return launch_leaf<6>(p2m, a);
    case 7: return launch_leaf<7>(p2m, a);
    default: return launch_leaf<8>(p2m, a);
  }
}

// ---------------------------------------------------------------------------
// Leaf "pair" kernels for sparse clouds (one weight column): a warp owns one
// parent cell q of level L-1 and its eight leaf children 8q .. 8q+7 (whose
// points are contiguous in sorted order).
//
// p2m_pair_kernel writes the leaf moments of the eight children (as
// p2m_cells_kernel: the same products in sorted order, zeros for empty
// cells) AND the parent's moments straight from the points,
//   M_{L-1}[q] = sum_{i in q} S_{L-1}(x_i) w_i,
// which is M2M(M_L) exactly in exact arithmetic (the child's Chebyshev
// interpolant of the parent basis polynomial is the polynomial itself, the
// identity behind engine.py:187-204), so the level-L -> L-1 M2M pass and its
// 16.8 GB (C5) re-read of the leaf moments disappear.
//
// l2p_pair_kernel evaluates phi_i = S_L(x_i) . loc_L[c] + S_{L-1}(x_i) .
// loc_{L-1}[q] where loc_L holds ONLY the level-L M2L locals: the parent's
// contribution L2L(loc_{L-1}) interpolated at x_i equals the parent's own
// expansion at x_i (same identity, engine.py:296-311 then :315-327), so
// the L-1 -> L L2L pass (a read-modify-write of the leaf locals) disappears.
template <int P>
constexpr int pair_warps() { return P <= 6 ? 4 : 2; }
// tuning overrides (scripts/pair_sweep.sh): -DBFMM_PAIR_MINB / -DBFMM_PAIR_BATCH
#ifdef BFMM_PAIR_MINB
template <int P>
constexpr int pair_minb() { return BFMM_PAIR_MINB; }
#else
template <int P>
constexpr int pair_minb() { return P == 5 ? 4 : 2; }  // <= 128 registers for C5 (p = 5)
#endif
#ifdef BFMM_PAIR_BATCH
template <int P>
constexpr int pair_batch() { return BFMM_PAIR_BATCH; }
#else
template <int P>
constexpr int pair_batch() {  // points staged per pass
  // p = 5: 48 points = 47.6 KB per CTA -> 4 CTAs per SM (C5 P2M 11.8 -> 9.9 ms
  // against 64); p = 6 keeps 64 (C4's crowded leaves take several passes, each
  // a read-modify-write of the moments: 48 measured 6.8 -> 8.1 ms there)
  return P == 5 ? 48 : P <= 6 ? 64 : 32;
}
#endif
template <int P>
constexpr size_t p2m_pair_smem() {
  return sizeof(double) * pair_warps<P>() * pair_batch<P>() * (6 * P + 1);
}
template <int P>
constexpr size_t l2p_pair_smem() {
  return sizeof(double) * pair_warps<P>() * 2 * ((9 * P * P * P + 1) & ~1);
}

// the eight children's counts of parent q: lanes < 8 hold child lane's
// count; returns the inclusive prefix (lanes < 8) and the first point
__device__ __forceinline__ int pair_scan(const int32_t *cell_start, const int32_t *cell_count,
                                         int64_t q, int lane, int &total, int64_t &first) {
  const int cnt = lane < 8 ? cell_count[8 * q + lane] : 0;
  int inc = cnt;
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += v;
  }
  total = __shfl_sync(0xffffffffu, inc, 7);
  const unsigned occ = __ballot_sync(0xffffffffu, lane < 8 && cnt > 0);
  const int fl = occ ? __ffs(occ) - 1 : 0;
  const int st = lane < 8 && lane == fl && occ ? cell_start[8 * q + lane] : 0;
  first = (int64_t)__shfl_sync(0xffffffffu, st, fl);
  return inc;
}

template <int P>
__global__ void __launch_bounds__(32 * pair_warps<P>(), pair_minb<P>())
p2m_pair_kernel(const double *__restrict__ pts4, const double *__restrict__ ws,
                const int32_t *__restrict__ cell_start, const int32_t *__restrict__ cell_count,
                Interp ip, LeafGeom g, double *__restrict__ mom_leaf,
                double *__restrict__ mom_par, int32_t *flag) {
  constexpr int P3 = P * P * P, B = pair_batch<P>(), W = pair_warps<P>(), R = 6 * P + 1;
  extern __shared__ __align__(16) double s_pair[];
  __shared__ double sS[P * P], sN[P];
  __shared__ int s_off[W][9];
  stage_basis<P>(ip, sS, sN);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *sw = s_pair + (size_t)wid * B * R;  // [B][R]: w_L (3P), w_{L-1} (3P), weight
  const double inv_hw = 1.0 / g.hw, inv_hp = 1.0 / g.h, hp = 2.0 * g.h;
  const int64_t q_lo = g.cell_lo / 8, q_hi = (g.cell_hi + 7) / 8;
  for (int64_t q = q_lo + int64_t(blockIdx.x) * W + wid; q < q_hi; q += int64_t(gridDim.x) * W) {
    int total;
    int64_t first;
    __syncwarp();  // the previous parent's readers of s_off / sw are done
    const int inc = pair_scan(cell_start, cell_count, q, lane, total, first);
    if (lane < 8) s_off[wid][lane + 1] = inc;
    if (lane == 0) s_off[wid][0] = 0;
    __syncwarp();
    int px, py, pz;
    unmorton3((uint64_t)q, px, py, pz);
    for (int b0 = 0; b0 < max(total, 1); b0 += B) {
      const int nb = min(B, total - b0);
      __syncwarp();
      for (int t = lane; t < nb; t += 32) {
        const int e = b0 + t;
        int ch = 0;
#pragma unroll
        for (int k = 1; k < 8; ++k) ch += s_off[wid][k] <= e ? 1 : 0;
        const int64_t i = first + e;
        const double4 x = reinterpret_cast<const double4 *>(pts4)[i];
        const int cx = 2 * px + ((ch >> 2) & 1), cy = 2 * py + ((ch >> 1) & 1),
                  cz = 2 * pz + (ch & 1);
        double *row = sw + t * R;
        weights2_s<P>(sS, sN, ip.scheme, ref_coord_m(x.x, g.lo[0], g.h, inv_hw, cx, flag),
                      ref_coord_m(x.x, g.lo[0], hp, inv_hp, px, flag), row, row + 3 * P);
        weights2_s<P>(sS, sN, ip.scheme, ref_coord_m(x.y, g.lo[1], g.h, inv_hw, cy, flag),
                      ref_coord_m(x.y, g.lo[1], hp, inv_hp, py, flag), row + P, row + 4 * P);
        weights2_s<P>(sS, sN, ip.scheme, ref_coord_m(x.z, g.lo[2], g.h, inv_hw, cz, flag),
                      ref_coord_m(x.z, g.lo[2], hp, inv_hp, pz, flag), row + 2 * P, row + 5 * P);
        row[6 * P] = ws[i];
      }
      __syncwarp();
      // the eight children's moments: slot (child, i, j) owns the P
      // moments M[i][j][0..P) -- one (wx_i wy_j w) product per point, then a
      // P-wide FMA row against the broadcast wz (no per-output index math)
      double *leaf = mom_leaf + 8 * q * (int64_t)P3;
      for (int sl = lane; sl < 8 * P * P; sl += 32) {
        const int ch = sl / (P * P), ij = sl - ch * P * P, ii = ij / P, jj = ij - ii * P;
        const int p0 = max(s_off[wid][ch], b0), p1 = min(s_off[wid][ch + 1], b0 + nb);
        double acc[P];
#pragma unroll
        for (int k = 0; k < P; ++k) acc[k] = 0.0;
        for (int pt = p0; pt < p1; ++pt) {
          const double *wt = sw + (pt - b0) * R;
          const double wxyw = (wt[ii] * wt[P + jj]) * wt[6 * P];
#pragma unroll
          for (int k = 0; k < P; ++k) acc[k] = fma(wxyw, wt[2 * P + k], acc[k]);
        }
        double *dst = leaf + ch * P3 + ij * P;
#pragma unroll
        for (int k = 0; k < P; ++k) {
          if (b0 == 0) {
            dst[k] = acc[k];
          } else {
            dst[k] += acc[k];
          }
        }
      }
      // the parent's moments from the same points, slot (i, j)
      double *par = mom_par + q * (int64_t)P3;
      for (int ij = lane; ij < P * P; ij += 32) {
        const int ii = ij / P, jj = ij - ii * P;
        double acc[P];
#pragma unroll
        for (int k = 0; k < P; ++k) acc[k] = 0.0;
        for (int pt = 0; pt < nb; ++pt) {
          const double *wt = sw + pt * R + 3 * P;
          const double wxyw = (wt[ii] * wt[P + jj]) * wt[3 * P];
#pragma unroll
          for (int k = 0; k < P; ++k) acc[k] = fma(wxyw, wt[2 * P + k], acc[k]);
        }
        double *dst = par + ij * P;
#pragma unroll
        for (int k = 0; k < P; ++k) {
          if (b0 == 0) {
            dst[k] = acc[k];
          } else {
            dst[k] += acc[k];
          }
        }
      }
    }
  }
}

template <int P>
__device__ __forceinline__ double l2p_contract(const double *wx, const double *wy,
                                               const double *wz, const double *L) {
  double sa[P];
#pragma unroll
  for (int a = 0; a < P; ++a) {
    sa[a] = 0.0;
#pragma unroll
    for (int b = 0; b < P; ++b) {
      const double *Lab = L + (a * P + b) * P;
      double sb = 0.0;
#pragma unroll
      for (int k = 0; k < P; ++k) sb = fma(wz[k], Lab[k], sb);
      sa[a] = fma(wx[a] * wy[b], sb, sa[a]);
    }
  }
  double s = sa[0];
#pragma unroll
  for (int a = 1; a < P; ++a) s += sa[a];
  return s;
}

// async 8-byte global -> shared copy (the parent's locals are 8-byte aligned)
__device__ __forceinline__ void cp_async8_pair(double *smem, const double *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16_pair(double *smem, const double *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

template <int P>
__global__ void __launch_bounds__(32 * pair_warps<P>(), pair_minb<P>())
l2p_pair_kernel(const double *__restrict__ pts4, const int32_t *__restrict__ cell_start,
                const int32_t *__restrict__ cell_count, Interp ip, LeafGeom g,
                const double *__restrict__ loc_leaf, const double *__restrict__ loc_par,
                double *__restrict__ phi, int32_t *flag) {
  // buffer stride rounded up to an even number of doubles: 16-byte aligned
  // cp.async destinations for every P
  constexpr int P3 = P * P * P, W = pair_warps<P>(), SL = (9 * P3 + 1) & ~1;
  extern __shared__ __align__(16) double s_pair[];
  __shared__ double sS[P * P], sN[P];
  __shared__ int s_off[W][9];
  stage_basis<P>(ip, sS, sN);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // two buffers per warp (the next parent's locals stream in while this
  // one's points are evaluated): 8 children's locals, then the parent's
  double *sl2 = s_pair + (size_t)wid * 2 * SL;
  const double inv_hw = 1.0 / g.hw, inv_hp = 1.0 / g.h, hp = 2.0 * g.h;
  const int64_t q_lo = g.cell_lo / 8, q_hi = (g.cell_hi + 7) / 8;
  const int64_t stride = int64_t(gridDim.x) * W;
  // the children's block (8 P^3 doubles) starts 16-byte aligned when 8 P^3
  // is even -- always -- so it moves in 16-byte chunks; the parent's row in
  // 8-byte ones
  auto prefetch = [&](int64_t q, double *dst) {
    const double *src = loc_leaf + 8 * q * (int64_t)P3;
    for (int e = lane; e < 4 * P3; e += 32) cp_async16_pair(dst + 2 * e, src + 2 * e);
    const double *srp = loc_par + q * (int64_t)P3;
    for (int e = lane; e < P3; e += 32) cp_async8_pair(dst + 8 * P3 + e, srp + e);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int64_t q = q_lo + int64_t(blockIdx.x) * W + wid;
  int buf = 0;
  if (q < q_hi) prefetch(q, sl2);
  for (; q < q_hi; q += stride) {
    const bool more = q + stride < q_hi;
    if (more) prefetch(q + stride, sl2 + (buf ^ 1) * SL);
    int total;
    int64_t first;
    const int inc = pair_scan(cell_start, cell_count, q, lane, total, first);
    if (lane < 8) s_off[wid][lane + 1] = inc;
    if (lane == 0) s_off[wid][0] = 0;
    if (more) {
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncwarp();
    const double *sl = sl2 + buf * SL;
    int px, py, pz;
    unmorton3((uint64_t)q, px, py, pz);
    for (int t = lane; t < total; t += 32) {
      int ch = 0;
#pragma unroll
      for (int k = 1; k < 8; ++k) ch += s_off[wid][k] <= t ? 1 : 0;
      const int64_t i = first + t;
      const double4 x = reinterpret_cast<const double4 *>(pts4)[i];
      const int cx = 2 * px + ((ch >> 2) & 1), cy = 2 * py + ((ch >> 1) & 1),
                cz = 2 * pz + (ch & 1);
      double wx[P], wy[P], wz[P];
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(x.x, g.lo[0], g.h, inv_hw, cx, flag), wx);
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(x.y, g.lo[1], g.h, inv_hw, cy, flag), wy);
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(x.z, g.lo[2], g.h, inv_hw, cz, flag), wz);
      const double s_leaf = l2p_contract<P>(wx, wy, wz, sl + ch * P3);
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(x.x, g.lo[0], hp, inv_hp, px, flag), wx);
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(x.y, g.lo[1], hp, inv_hp, py, flag), wy);
      weights_s<P>(sS, sN, ip.scheme, ref_coord_m(x.z, g.lo[2], hp, inv_hp, pz, flag), wz);
      phi[i] = s_leaf + l2p_contract<P>(wx, wy, wz, sl + 8 * P3);
    }
    __syncwarp();  // buffer buf is refilled two parents on
    buf ^= 1;
  }
}

template <int P>
int launch_p2m_pair(const LeafCall &a, const int32_t *cs, const int32_t *cc, double *mom_par) {
  constexpr size_t smem = p2m_pair_smem<P>();
  static unsigned long long attr = 0;
  if (first_on_device(&attr) && smem > 48 * 1024)
    cudaFuncSetAttribute(p2m_pair_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int64_t parents = (a.g.cell_hi + 7) / 8 - a.g.cell_lo / 8;
  if (parents <= 0) return 0;
  const unsigned grid =
      (unsigned)std::min<int64_t>(ceil_div(parents, pair_warps<P>()), (int64_t)kNumSMs * 16);
  p2m_pair_kernel<P><<<grid, 32 * pair_warps<P>(), smem, a.st>>>(a.pts4, a.ws, cs, cc, a.ip, a.g,
                                                                  a.out, mom_par, a.flag);
  return check_launch("p2m_pair_kernel");
}

template <int P>
int launch_l2p_pair(const LeafCall &a, const int32_t *cs, const int32_t *cc,
                    const double *loc_par) {
  constexpr size_t smem = l2p_pair_smem<P>();
  static unsigned long long attr = 0;
  if (first_on_device(&attr) && smem > 48 * 1024)
    cudaFuncSetAttribute(l2p_pair_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int64_t parents = (a.g.cell_hi + 7) / 8 - a.g.cell_lo / 8;
  if (parents <= 0) return 0;
  const unsigned grid =
      (unsigned)std::min<int64_t>(ceil_div(parents, pair_warps<P>()), (int64_t)kNumSMs * 16);
  l2p_pair_kernel<P><<<grid, 32 * pair_warps<P>(), smem, a.st>>>(a.pts4, cs, cc, a.ip, a.g,
                                                                  a.locals, loc_par, a.out, a.flag);
  return check_launch("l2p_pair_kernel");
}

inline int dispatch_p2m_pair(int p, const LeafCall &a, const int32_t *cs, const int32_t *cc,
                             double *mom_par) {
  switch (p) {
    case 2: return launch_p2m_pair<2>(a, cs, cc, mom_par);
    case 3: return launch_p2m_pair<3>(a, cs, cc, mom_par);
    case 4: return launch_p2m_pair<4>(a, cs, cc, mom_par);
    case 5: return launch_p2m_pair<5>(a, cs, cc, mom_par);
    case 6: return launch_p2m_pair<6>(a, cs, cc, mom_par);
    case 7: return launch_p2m_pair<7>(a, cs, cc, mom_par);
    default: return launch_p2m_pair<8>(a, cs, cc, mom_par);
  }
}

inline int dispatch_l2p_pair(int p, const LeafCall &a, const int32_t *cs, const int32_t *cc,
                             const double *loc_par) {
  switch (p) {
    case 2: return launch_l2p_pair<2>(a, cs, cc, loc_par);
    case 3: return launch_l2p_pair<3>(a, cs, cc, loc_par);
    case 4: return launch_l2p_pair<4>(a, cs, cc, loc_par);
    case 5: return launch_l2p_pair<5>(a, cs, cc, loc_par);
    case 6: return launch_l2p_pair<6>(a, cs, cc, loc_par);
    case 7: return launch_l2p_pair<7>(a, cs, cc, loc_par);
    default: return launch_l2p_pair<8>(a, cs, cc, loc_par);
  }
}
