// Leaf-facing interpolation passes and tree transfers:
//   P2M  leaf_moments     (engine.py:159-185)
//   L2P  read_potentials  (engine.py:313-337)
//   M2M  ascend           (engine.py:187-204)
//   L2L  descend          (engine.py:296-311)
// Coefficient layout per cell is (m, p^3) with the node index
// a = (i*p + j)*p + k, z fastest (interpolation.py:93-102).
#include <algorithm>

#include "common.cuh"

namespace bfmm {
namespace {

constexpr int kMaxP = 12;

struct Interp {
  int p, scheme;
  double nodes[kMaxP];
  double S[kMaxP * kMaxP];  // Chebyshev: S[n][j] = c_n T_n(x_j)
};

struct LeafGeom {
  double lo[3], h, hw;
  int64_t cell_lo, cell_hi;  // leaf cells this call handles (Morton range)
};

inline LeafGeom make_leaf_geom(const double *geom) {
  // host geom = {lo_x, lo_y, lo_z, h_leaf, cell_lo, cell_hi}
  return LeafGeom{{geom[0], geom[1], geom[2]}, geom[3], 0.5 * geom[3],
                  (int64_t)geom[4], (int64_t)geom[5]};
}

// 1-D weights of node j at x (interpolation.py:66-90).  Chebyshev:
// sum_n T_n(x) S[n][j]; the reference evaluates T_n(x) = cos(n arccos x),
// here the three-term recurrence T_{n+1} = 2x T_n - T_{n-1} gives the same
// polynomials (agreement to a few ulp on [-1, 1]) without transcendentals.
// Uniform: Lagrange products with the reference's factor order.
__device__ inline void weights_1d(const Interp &ip, double x, double *w) {
  const int p = ip.p;
  if (ip.scheme == 0) {
    x = fmin(1.0, fmax(-1.0, x));
    double T[kMaxP];
    T[0] = 1.0;
    if (p > 1) T[1] = x;
    for (int n = 2; n < p; ++n) T[n] = fma(2.0 * x, T[n - 1], -T[n - 2]);
    for (int j = 0; j < p; ++j) {
      double s = 0.0;
      for (int n = 0; n < p; ++n) s = fma(T[n], ip.S[n * p + j], s);
      w[j] = s;
    }
  } else {
    for (int j = 0; j < p; ++j) {
      double v = 1.0;
      for (int k = 0; k < p; ++k)
        if (k != j) v *= (x - ip.nodes[k]) / (ip.nodes[j] - ip.nodes[k]);
      w[j] = v;
    }
  }
}

// Leaf-frame coordinate (engine.py:176, 330 and 339-345): (x - center)/hw,
// bound-checked at 1 + 1e-9, then clipped to [-1, 1].
__device__ inline double ref_coord(double x, double lo, double h, double hw,
                                   int cell, int32_t *flag) {
  double center = lo + ((double)cell + 0.5) * h;
  double r = (x - center) / hw;
  if (fabs(r) > 1.0 + 1e-9) atomicOr(flag, 1);
  return fmin(1.0, fmax(-1.0, r));
}

// ---------------------------------------------------------------------------
// P2M: one CTA per nonempty leaf; points staged through shared memory in
// chunks; each thread owns (column, node) outputs and sums the leaf's points
// in sorted order (the add.reduceat order of engine.py:181-182).
constexpr int kLeafThreads = 128;

__global__ void __launch_bounds__(kLeafThreads)
p2m_kernel(const double *__restrict__ pts4, const double *__restrict__ ws,
           int m, int ncmax, const int64_t *__restrict__ leaves,
           const int64_t *__restrict__ starts,
           const int64_t *__restrict__ counts,
           const int64_t *__restrict__ n_leaves, int levels, Interp ip,
           LeafGeom g, double *__restrict__ moments, int32_t *flag) {
  extern __shared__ double sm[];
  const int p = ip.p, p3 = p * p * p;
  double *wx = sm;                          // [kLeafThreads][p]
  double *wy = wx + kLeafThreads * p;
  double *wz = wy + kLeafThreads * p;
  double *wv = wz + kLeafThreads * p;       // [kLeafThreads][ncmax]: the pass's columns
  const int64_t nl = *n_leaves;
  for (int64_t leaf = blockIdx.x; leaf < nl; leaf += gridDim.x) {
    const int64_t cell = leaves[leaf];
    if (cell < g.cell_lo || cell >= g.cell_hi) continue;  // other rank's shard
    const int64_t s0 = starts[leaf], cnt = counts[leaf];
    int cx, cy, cz;
    unmorton3((uint64_t)cell, cx, cy, cz);
    const int nout = m * p3;
    // outputs in passes of up to 27 accumulators per thread (any m * p^3;
    // the leaf's points are re-staged for every pass)
    for (int o0 = 0; o0 < nout; o0 += 27 * kLeafThreads) {
      const int nrem = nout - o0 < 27 * kLeafThreads ? nout - o0 : 27 * kLeafThreads;
      double acc[27];
      const int per = (nrem + kLeafThreads - 1) / kLeafThreads;
      const int cl = o0 / p3, nc = (o0 + nrem - 1) / p3 - cl + 1;  // columns of this pass
      for (int u = 0; u < per; ++u) acc[u] = 0.0;
      for (int64_t c0 = 0; c0 < cnt; c0 += kLeafThreads) {
        const int nb = (int)(cnt - c0 < kLeafThreads ? cnt - c0 : kLeafThreads);
        __syncthreads();
        if (threadIdx.x < nb) {
          const int64_t i = s0 + c0 + threadIdx.x;
          const double4 q = reinterpret_cast<const double4 *>(pts4)[i];
          double w1[kMaxP];
          weights_1d(ip, ref_coord(q.x, g.lo[0], g.h, g.hw, cx, flag), w1);
          for (int j = 0; j < p; ++j) wx[threadIdx.x * p + j] = w1[j];
          weights_1d(ip, ref_coord(q.y, g.lo[1], g.h, g.hw, cy, flag), w1);
          for (int j = 0; j < p; ++j) wy[threadIdx.x * p + j] = w1[j];
          weights_1d(ip, ref_coord(q.z, g.lo[2], g.h, g.hw, cz, flag), w1);
          for (int j = 0; j < p; ++j) wz[threadIdx.x * p + j] = w1[j];
          for (int c = 0; c < nc; ++c) wv[threadIdx.x * ncmax + c] = ws[i * m + cl + c];
        }
        __syncthreads();
        for (int u = 0; u < per; ++u) {
          const int o = o0 + threadIdx.x + u * kLeafThreads;
          if (o >= nout) break;
          const int c = o / p3, a = o - c * p3;
          const int i = a / (p * p), j = (a / p) % p, k = a % p;
          double s = acc[u];
          for (int t = 0; t < nb; ++t)
            s += ((wx[t * p + i] * wy[t * p + j]) * wz[t * p + k]) * wv[t * ncmax + c - cl];
          acc[u] = s;
        }
      }
      double *dst = moments + cell * (int64_t)nout;
      for (int u = 0; u < per; ++u) {
        const int o = o0 + threadIdx.x + u * kLeafThreads;
        if (o >= nout) break;
        dst[o] = acc[u];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// L2P: one CTA per nonempty leaf, leaf locals in shared memory, one thread
// per target point.
__global__ void __launch_bounds__(kLeafThreads)
l2p_kernel(const double *__restrict__ pts4, int m, int mc,
           const int64_t *__restrict__ leaves,
           const int64_t *__restrict__ starts,
           const int64_t *__restrict__ counts,
           const int64_t *__restrict__ n_leaves, Interp ip, LeafGeom g,
           const double *__restrict__ locals, double *__restrict__ phi,
           int32_t *flag) {
  // mc columns of the leaf's locals staged per pass (any m * p^3)
  extern __shared__ double sm[];
  const int p = ip.p, p3 = p * p * p;
  const int nout = m * p3;
  const int64_t nl = *n_leaves;
  for (int64_t leaf = blockIdx.x; leaf < nl; leaf += gridDim.x) {
    const int64_t cell = leaves[leaf];
    if (cell < g.cell_lo || cell >= g.cell_hi) continue;  // other rank's shard
    const int64_t s0 = starts[leaf], cnt = counts[leaf];
    int cx, cy, cz;
    unmorton3((uint64_t)cell, cx, cy, cz);
    for (int c0 = 0; c0 < m; c0 += mc) {
      const int nc = m - c0 < mc ? m - c0 : mc;
      __syncthreads();
      for (int o = threadIdx.x; o < nc * p3; o += kLeafThreads)
        sm[o] = locals[cell * (int64_t)nout + (int64_t)c0 * p3 + o];
      __syncthreads();
      for (int64_t t = threadIdx.x; t < cnt; t += kLeafThreads) {
        const int64_t i = s0 + t;
        const double4 q = reinterpret_cast<const double4 *>(pts4)[i];
        double wx[kMaxP], wy[kMaxP], wz[kMaxP];
        weights_1d(ip, ref_coord(q.x, g.lo[0], g.h, g.hw, cx, flag), wx);
        weights_1d(ip, ref_coord(q.y, g.lo[1], g.h, g.hw, cy, flag), wy);
        weights_1d(ip, ref_coord(q.z, g.lo[2], g.h, g.hw, cz, flag), wz);
        for (int c = 0; c < nc; ++c) {
          const double *L = sm + c * p3;
          double s = 0.0;
          int a = 0;
          for (int ii = 0; ii < p; ++ii)
            for (int jj = 0; jj < p; ++jj) {
              const double wxy = wx[ii] * wy[jj];
              for (int kk = 0; kk < p; ++kk, ++a) s = fma(wxy * wz[kk], L[a], s);
            }
          phi[i * m + c0 + c] = s;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Kronecker transfers.  T[o] = kron(H[sx], kron(H[sy], H[sz])) where
// H[s][a][b] is the weight of parent node a at child node b
// (interpolation.py:136-155).  Three successive p x p contractions.
struct Halves {
  double H[2][kMaxP * kMaxP];
};

constexpr int kXferThreads = 128;

// in/out are p^3 tensors in shared memory; tmp same size.
// up=true : out[a] = sum_b T[o][a][b] in[b]     (M2M)
// up=false: out[b] = sum_a T[o][a][b] in[a]     (L2L, transpose)
__device__ inline void kron_apply(const Halves &hv, int p, int o, bool up,
                                  const double *in, double *tmp1,
                                  double *tmp2, double *out, bool accumulate) {
  const int p3 = p * p * p;
  const double *Hx = hv.H[(o >> 2) & 1];
  const double *Hy = hv.H[(o >> 1) & 1];
  const double *Hz = hv.H[o & 1];
  // contract z
  for (int e = threadIdx.x; e < p3; e += blockDim.x) {
    const int i = e / (p * p), j = (e / p) % p, k = e % p;
    const double *row = in + (i * p + j) * p;
    double s = 0.0;
    for (int q = 0; q < p; ++q)
      s = fma(up ? Hz[k * p + q] : Hz[q * p + k], row[q], s);
    tmp1[e] = s;
  }
  __syncthreads();
  // contract y
  for (int e = threadIdx.x; e < p3; e += blockDim.x) {
    const int i = e / (p * p), j = (e / p) % p, k = e % p;
    double s = 0.0;
    for (int q = 0; q < p; ++q)
      s = fma(up ? Hy[j * p + q] : Hy[q * p + j], tmp1[(i * p + q) * p + k], s);
    tmp2[e] = s;
  }
  __syncthreads();
  // contract x
  for (int e = threadIdx.x; e < p3; e += blockDim.x) {
    const int i = e / (p * p), j = (e / p) % p, k = e % p;
    double s = 0.0;
    for (int q = 0; q < p; ++q)
      s = fma(up ? Hx[i * p + q] : Hx[q * p + i], tmp2[(q * p + j) * p + k], s);
    out[e] = accumulate ? out[e] + s : s;
  }
  __syncthreads();
}

// One CTA per (parent, column): parent = sum_o T[o] child[8q+o].
__global__ void __launch_bounds__(kXferThreads)
m2m_kernel(const double *__restrict__ child, double *__restrict__ parent,
           int64_t n_parent, int p, int m, Halves hv) {
  extern __shared__ double sm[];
  const int p3 = p * p * p;
  double *in = sm, *t1 = in + p3, *t2 = t1 + p3, *acc = t2 + p3;
  for (int64_t w = blockIdx.x; w < n_parent * m; w += gridDim.x) {
    const int64_t q = w / m;
    const int c = (int)(w - q * m);
    for (int o = 0; o < 8; ++o) {
      const double *src = child + ((8 * q + o) * m + c) * (int64_t)p3;
      for (int e = threadIdx.x; e < p3; e += blockDim.x) in[e] = src[e];
      __syncthreads();
      kron_apply(hv, p, o, true, in, t1, t2, acc, o > 0);
    }
    double *dst = parent + (q * m + c) * (int64_t)p3;
    for (int e = threadIdx.x; e < p3; e += blockDim.x) dst[e] = acc[e];
    __syncthreads();
  }
}

// One CTA per (parent, column): child[8q+o] += T[o]^T parent[q].
__global__ void __launch_bounds__(kXferThreads)
l2l_kernel(const double *__restrict__ parent, double *__restrict__ child,
           int64_t n_parent, int p, int m, Halves hv) {
  extern __shared__ double sm[];
  const int p3 = p * p * p;
  double *in = sm, *t1 = in + p3, *t2 = t1 + p3, *out = t2 + p3;
  for (int64_t w = blockIdx.x; w < n_parent * m; w += gridDim.x) {
    const int64_t q = w / m;
    const int c = (int)(w - q * m);
    const double *src = parent + (q * m + c) * (int64_t)p3;
    for (int e = threadIdx.x; e < p3; e += blockDim.x) in[e] = src[e];
    __syncthreads();
    for (int o = 0; o < 8; ++o) {
      double *dst = child + ((8 * q + o) * m + c) * (int64_t)p3;
      for (int e = threadIdx.x; e < p3; e += blockDim.x) out[e] = dst[e];
      __syncthreads();
      kron_apply(hv, p, o, false, in, t1, t2, out, true);
      for (int e = threadIdx.x; e < p3; e += blockDim.x) dst[e] = out[e];
      __syncthreads();
    }
  }
}

constexpr int kLeafWarps = 4;

Interp make_interp(int p, int scheme, const double *host) {
  Interp ip{};
  ip.p = p;
  ip.scheme = scheme;
  for (int j = 0; j < p; ++j) ip.nodes[j] = host[j];
  for (int e = 0; e < p * p; ++e) ip.S[e] = host[p + e];
  return ip;
}

int grid_cap(int64_t work, int per_sm) {
  int64_t cap = int64_t(kNumSMs) * per_sm;
  return (int)(work < 1 ? 1 : (work < cap ? work : cap));
}

#include "leaf_kernels.cuh"
#include "transfer_kernels.cuh"

}  // namespace
}  // namespace bfmm

using namespace bfmm;

static int p2m_impl(const double *pts4, const double *wsorted, int m,
                    const int64_t *leaves, const int64_t *starts,
                    const int64_t *counts, const int64_t *n_leaves,
                    int64_t max_leaves, int levels, int p, int scheme,
                    const double *interp, const double *geom,
                    double *moments, int32_t *ref_flag, bool per_thread,
                    bfmm_stream_t stream) {
  if (p < 1 || p > kMaxP || m < 1) {
    set_error("bfmm_p2m: unsupported p=%d m=%d", p, m);
    return 2;
  }
  if (max_leaves <= 0) return 0;
  Interp ip = make_interp(p, scheme, interp);
  const LeafGeom g = make_leaf_geom(geom);
  if (p >= 2 && p <= 8) {
    LeafCall a{pts4, wsorted, m, leaves, starts, counts, n_leaves, max_leaves, levels, per_thread, ip, g,
               nullptr, moments, ref_flag, as_stream(stream)};
    return dispatch_leaf(p, true, a);
  }
  const int p3 = p * p * p;
  const int ncmax = std::min(m, 27 * kLeafThreads / p3 + 2);  // columns one output pass spans
  size_t smem = sizeof(double) * kLeafThreads * (3 * p + ncmax);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(p2m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  p2m_kernel<<<grid_cap(max_leaves, 16), kLeafThreads, smem,
               as_stream(stream)>>>(pts4, wsorted, m, ncmax, leaves, starts, counts,
                                    n_leaves, levels, ip, g, moments, ref_flag);
  return check_launch("p2m_kernel");
}

static int l2p_impl(const double *pts4, int m, const int64_t *leaves,
                    const int64_t *starts, const int64_t *counts,
                    const int64_t *n_leaves, int64_t max_leaves, int levels,
                    int p, int scheme, const double *interp,
                    const double *geom, const double *locals,
                    double *phi_sorted, int32_t *ref_flag, bool per_point,
                    bfmm_stream_t stream) {
  if (p < 1 || p > kMaxP || m < 1) {
    set_error("bfmm_l2p: unsupported p=%d m=%d", p, m);
    return 2;
  }
  if (max_leaves <= 0) return 0;
  Interp ip = make_interp(p, scheme, interp);
  const LeafGeom g = make_leaf_geom(geom);
  if (p >= 2 && p <= 8) {
    LeafCall a{pts4, nullptr, m, leaves, starts, counts, n_leaves, max_leaves, levels,
               per_point, ip, g, locals, phi_sorted, ref_flag, as_stream(stream)};
    return dispatch_leaf(p, false, a);
  }
  const int p3 = p * p * p;
  const int mc = std::min(m, (int)((200 * 1024) / (sizeof(double) * p3)));
  size_t smem = sizeof(double) * mc * p3;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(l2p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  l2p_kernel<<<grid_cap(max_leaves, 16), kLeafThreads, smem,
               as_stream(stream)>>>(pts4, m, mc, leaves, starts, counts, n_leaves,
                                    ip, g, locals, phi_sorted, ref_flag);
  return check_launch("l2p_kernel");
}

static Halves make_halves(int p, const double *H) {
  Halves hv{};
  for (int s = 0; s < 2; ++s)
    for (int e = 0; e < p * p; ++e) hv.H[s][e] = H[s * p * p + e];
  return hv;
}

extern "C" int bfmm_m2m(const double *child, double *parent, int64_t n_parent,
                        int p, int m, const double *H, bfmm_stream_t stream) {
  if (p < 1 || p > kMaxP) {
    set_error("bfmm_m2m: unsupported p=%d", p);
    return 2;
  }
  if (n_parent <= 0) return 0;
  if (p >= 2 && p <= 8)
    return dispatch_xfer(p, true, child, parent, n_parent, m, make_halves(p, H),
                         as_stream(stream));
  size_t smem = sizeof(double) * 4 * p * p * p;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(m2m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  m2m_kernel<<<grid_cap(n_parent * m, 16), kXferThreads, smem,
               as_stream(stream)>>>(child, parent, n_parent, p, m,
                                    make_halves(p, H));
  return check_launch("m2m_kernel");
}

extern "C" int bfmm_l2l(const double *parent, double *child, int64_t n_parent,
                        int p, int m, const double *H, bfmm_stream_t stream) {
  if (p < 1 || p > kMaxP) {
    set_error("bfmm_l2l: unsupported p=%d", p);
    return 2;
  }
  if (n_parent <= 0) return 0;
  if (p >= 2 && p <= 8)
    return dispatch_xfer(p, false, parent, child, n_parent, m, make_halves(p, H),
                         as_stream(stream));
  size_t smem = sizeof(double) * 4 * p * p * p;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(l2l_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  l2l_kernel<<<grid_cap(n_parent * m, 16), kXferThreads, smem,
               as_stream(stream)>>>(parent, child, n_parent, p, m,
                                    make_halves(p, H));
  return check_launch("l2l_kernel");
}

extern "C" int bfmm_l2p(const double *pts4, int m, const int64_t *leaves,
                        const int64_t *starts, const int64_t *counts,
                        const int64_t *n_leaves, int64_t max_leaves, int levels,
                        int p, int scheme, const double *interp,
                        const double *geom, const double *locals,
                        double *phi_sorted, int32_t *ref_flag,
                        bfmm_stream_t stream) {
  return l2p_impl(pts4, m, leaves, starts, counts, n_leaves, max_leaves, levels, p, scheme,
                  interp, geom, locals, phi_sorted, ref_flag, false, stream);
}

extern "C" int bfmm_l2p_points(const double *pts4, int m, const int64_t *leaves,
                               const int64_t *starts, const int64_t *counts,
                               const int64_t *n_leaves, int64_t max_leaves, int levels,
                               int p, int scheme, const double *interp,
                               const double *geom, const double *locals,
                               double *phi_sorted, int32_t *ref_flag,
                               bfmm_stream_t stream) {
  return l2p_impl(pts4, m, leaves, starts, counts, n_leaves, max_leaves, levels, p, scheme,
                  interp, geom, locals, phi_sorted, ref_flag, true, stream);
}

extern "C" int bfmm_p2m(const double *pts4, const double *wsorted, int m,
                        const int64_t *leaves, const int64_t *starts,
                        const int64_t *counts, const int64_t *n_leaves,
                        int64_t max_leaves, int levels, int p, int scheme,
                        const double *interp, const double *geom,
                        double *moments, int32_t *ref_flag,
                        bfmm_stream_t stream) {
  return p2m_impl(pts4, wsorted, m, leaves, starts, counts, n_leaves, max_leaves, levels, p,
                  scheme, interp, geom, moments, ref_flag, false, stream);
}

extern "C" int bfmm_p2m_cells(const double *pts4, const double *wsorted, int m,
                              const int32_t *cell_start, const int32_t *cell_count, int levels,
                              int p, int scheme, const double *interp, const double *geom,
                              double *moments, int32_t *ref_flag, bfmm_stream_t stream) {
  if (p < 2 || p > 8 || m < 1 || levels < 2) {
    set_error("bfmm_p2m_cells: unsupported p=%d m=%d levels=%d", p, m, levels);
    return 2;
  }
  const LeafGeom g = make_leaf_geom(geom);
  if (g.cell_lo < 0 || g.cell_hi > (int64_t(1) << (3 * levels)) || g.cell_lo > g.cell_hi) {
    set_error("bfmm_p2m_cells: cell range [%lld, %lld) outside level %d", (long long)g.cell_lo,
              (long long)g.cell_hi, levels);
    return 2;
  }
  LeafCall a{pts4, wsorted, m, nullptr, nullptr, nullptr, nullptr, 0, levels, false,
             make_interp(p, scheme, interp), g, nullptr, moments, ref_flag, as_stream(stream)};
  return dispatch_p2m_cells(p, a, cell_start, cell_count);
}

extern "C" int bfmm_l2p_cells(const double *pts4, int m, const int32_t *cell_start,
                              const int32_t *cell_count, int levels, int p, int scheme,
                              const double *interp, const double *geom, const double *locals,
                              double *phi_sorted, int32_t *ref_flag, bfmm_stream_t stream) {
  if (p < 2 || p > 8 || m < 1 || levels < 2) {
    set_error("bfmm_l2p_cells: unsupported p=%d m=%d levels=%d", p, m, levels);
    return 2;
  }
  const LeafGeom g = make_leaf_geom(geom);
  if (g.cell_lo < 0 || g.cell_hi > (int64_t(1) << (3 * levels)) || g.cell_lo > g.cell_hi) {
    set_error("bfmm_l2p_cells: cell range [%lld, %lld) outside level %d", (long long)g.cell_lo,
              (long long)g.cell_hi, levels);
    return 2;
  }
  LeafCall a{pts4, nullptr, m, nullptr, nullptr, nullptr, nullptr, 0, levels, true,
             make_interp(p, scheme, interp), g, locals, phi_sorted, ref_flag, as_stream(stream)};
  return dispatch_l2p_cells(p, a, cell_start, cell_count);
}

static bool pair_args_ok(const char *what, int p, int levels, const LeafGeom &g) {
  if (p < 2 || p > 8 || levels < 3) {
    set_error("%s: unsupported p=%d levels=%d", what, p, levels);
    return false;
  }
  if (g.cell_lo < 0 || g.cell_hi > (int64_t(1) << (3 * levels)) || g.cell_lo > g.cell_hi ||
      g.cell_lo % 8 || g.cell_hi % 8) {
    set_error("%s: cell range [%lld, %lld) not whole parents of level %d", what,
              (long long)g.cell_lo, (long long)g.cell_hi, levels);
    return false;
  }
  return true;
}

extern "C" int bfmm_p2m_pair(const double *pts4, const double *wsorted, const int32_t *cell_start,
                             const int32_t *cell_count, int levels, int p, int scheme,
                             const double *interp, const double *geom, double *mom_leaf,
                             double *mom_parent, int32_t *ref_flag, bfmm_stream_t stream) {
  const LeafGeom g = make_leaf_geom(geom);
  if (!pair_args_ok("bfmm_p2m_pair", p, levels, g)) return 2;
  LeafCall a{pts4, wsorted, 1, nullptr, nullptr, nullptr, nullptr, 0, levels, false,
             make_interp(p, scheme, interp), g, nullptr, mom_leaf, ref_flag, as_stream(stream)};
  return dispatch_p2m_pair(p, a, cell_start, cell_count, mom_parent);
}

extern "C" int bfmm_l2p_pair(const double *pts4, const int32_t *cell_start,
                             const int32_t *cell_count, int levels, int p, int scheme,
                             const double *interp, const double *geom, const double *loc_leaf,
                             const double *loc_parent, double *phi_sorted, int32_t *ref_flag,
                             bfmm_stream_t stream) {
  const LeafGeom g = make_leaf_geom(geom);
  if (!pair_args_ok("bfmm_l2p_pair", p, levels, g)) return 2;
  LeafCall a{pts4, nullptr, 1, nullptr, nullptr, nullptr, nullptr, 0, levels, true,
             make_interp(p, scheme, interp), g, loc_leaf, phi_sorted, ref_flag, as_stream(stream)};
  return dispatch_l2p_pair(p, a, cell_start, cell_count, loc_parent);
}

extern "C" int bfmm_p2m_sparse(const double *pts4, const double *wsorted, int m,
                               const int64_t *leaves, const int64_t *starts,
                               const int64_t *counts, const int64_t *n_leaves,
                               int64_t max_leaves, int levels, int p, int scheme,
                               const double *interp, const double *geom,
                               double *moments, int32_t *ref_flag,
                               bfmm_stream_t stream) {
  return p2m_impl(pts4, wsorted, m, leaves, starts, counts, n_leaves, max_leaves, levels, p,
                  scheme, interp, geom, moments, ref_flag, true, stream);
}
