// CTA-per-(parent, column) M2M / L2L specialised on P (included by
// interp.cu; production path for 2 <= p <= 8).  T[o] = kron(H[ox], H[oy],
// H[oz]) (interpolation.py:136-155), o = 4 ox + 2 oy + oz.  The eight child
// transforms share their factors, so M2M contracts z for the four (ox, oy)
// pairs (summing the two oz children), then y (summing oy), then x (summing
// ox): 7 P^3 outputs of 2P terms each instead of 24 P^3 of P; L2L runs the
// same three stages in reverse (x: 2, y: 4, z: 8 tensors).  Each stage is
// spread over the CTA's threads, one output element per thread-iteration,
// with the children of one parent staged contiguously in shared memory.
#pragma once

constexpr int kXferThreads2 = 128;

template <int P>
constexpr size_t xfer_smem() {
  return sizeof(double) * (2 * P * P + 14 * P * P * P);
}

// parent[q] = sum_o T[o] child[8q + o] (engine.py:187-204)
template <int P>
__global__ void __launch_bounds__(kXferThreads2)
m2m_stage_kernel(const double *__restrict__ child, double *__restrict__ parent,
                 int64_t n_parent, int m, Halves hv) {
  constexpr int P2 = P * P, P3 = P2 * P;
  extern __shared__ double smx[];
  double *sH = smx, *sc = sH + 2 * P2, *t1 = sc + 8 * P3, *t2 = t1 + 4 * P3;
  const int tid = threadIdx.x;
  for (int e = tid; e < 2 * P2; e += kXferThreads2) sH[e] = hv.H[e / P2][e % P2];
  for (int64_t w = blockIdx.x; w < n_parent * m; w += gridDim.x) {
    const int64_t q = w / m;
    const int c = (int)(w - q * m);
    for (int e = tid; e < 8 * P3; e += kXferThreads2) {
      const int o = e / P3, r = e - o * P3;
      sc[e] = child[((8 * q + o) * m + c) * (int64_t)P3 + r];
    }
    __syncthreads();
    for (int e = tid; e < 4 * P3; e += kXferThreads2) {  // z, summing oz
      const int oxy = e / P3, r = e - oxy * P3, ij = r / P, kp = r - ij * P;
      double s = 0.0;
#pragma unroll
      for (int oz = 0; oz < 2; ++oz) {
        const double *src = sc + (2 * oxy + oz) * P3 + ij * P, *h = sH + oz * P2 + kp * P;
#pragma unroll
        for (int k = 0; k < P; ++k) s = fma(h[k], src[k], s);
      }
      t1[e] = s;
    }
    __syncthreads();
    for (int e = tid; e < 2 * P3; e += kXferThreads2) {  // y, summing oy
      const int ox = e / P3, r = e - ox * P3, i = r / P2, jp = (r / P) % P, kp = r % P;
      double s = 0.0;
#pragma unroll
      for (int oy = 0; oy < 2; ++oy) {
        const double *src = t1 + (2 * ox + oy) * P3 + i * P2 + kp, *h = sH + oy * P2 + jp * P;
#pragma unroll
        for (int j = 0; j < P; ++j) s = fma(h[j], src[j * P], s);
      }
      t2[e] = s;
    }
    __syncthreads();
    double *dst = parent + (q * m + c) * (int64_t)P3;
    for (int e = tid; e < P3; e += kXferThreads2) {  // x, summing ox
      const int ip = e / P2, jk = e - ip * P2;
      double s = 0.0;
#pragma unroll
      for (int ox = 0; ox < 2; ++ox) {
        const double *src = t2 + ox * P3 + jk, *h = sH + ox * P2 + ip * P;
#pragma unroll
        for (int i = 0; i < P; ++i) s = fma(h[i], src[i * P2], s);
      }
      dst[e] = s;
    }
  }
}

// child[8q + o] += T[o]^T parent[q] (engine.py:296-311)
template <int P>
__global__ void __launch_bounds__(kXferThreads2)
l2l_stage_kernel(const double *__restrict__ parent, double *__restrict__ child,
                 int64_t n_parent, int m, Halves hv) {
  constexpr int P2 = P * P, P3 = P2 * P;
  extern __shared__ double smx[];
  double *sH = smx, *sp = sH + 2 * P2, *u = sp + P3, *t = u + 2 * P3;
  const int tid = threadIdx.x;
  for (int e = tid; e < 2 * P2; e += kXferThreads2) sH[e] = hv.H[e / P2][e % P2];
  for (int64_t w = blockIdx.x; w < n_parent * m; w += gridDim.x) {
    const int64_t q = w / m;
    const int c = (int)(w - q * m);
    const double *src0 = parent + (q * m + c) * (int64_t)P3;
    for (int e = tid; e < P3; e += kXferThreads2) sp[e] = src0[e];
    __syncthreads();
    for (int e = tid; e < 2 * P3; e += kXferThreads2) {  // x, per ox
      const int ox = e / P3, r = e - ox * P3, ip = r / P2, jk = r - ip * P2;
      const double *h = sH + ox * P2 + ip;
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < P; ++i) s = fma(h[i * P], sp[i * P2 + jk], s);
      u[e] = s;
    }
    __syncthreads();
    for (int e = tid; e < 4 * P3; e += kXferThreads2) {  // y, per (ox, oy)
      const int oxy = e / P3, r = e - oxy * P3, ip = r / P2, jp = (r / P) % P, k = r % P;
      const double *h = sH + (oxy & 1) * P2 + jp, *src = u + (oxy >> 1) * P3 + ip * P2 + k;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < P; ++j) s = fma(h[j * P], src[j * P], s);
      t[e] = s;
    }
    __syncthreads();
    for (int e = tid; e < 8 * P3; e += kXferThreads2) {  // z, per child
      const int o = e / P3, r = e - o * P3, ijp = r / P, kp = r - ijp * P;
      const double *h = sH + (o & 1) * P2 + kp, *src = t + (o >> 1) * P3 + ijp * P;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < P; ++k) s = fma(h[k * P], src[k], s);
      child[((8 * q + o) * m + c) * (int64_t)P3 + r] += s;
    }
    __syncthreads();
  }
}

// Warp per (parent, column) for large levels (C5: 2.1M parents at level 7).
// Each of the three Kronecker stages gives every lane whole 1-D lines
// (P inputs from each of the two halves -> P outputs) with the transfer
// factors H[s][a][b] read at compile-time indices from the kernel
// parameter bank (no shared-memory operand loads, unrolled on P); the
// intermediates sit in the warp's own shared slice (__syncwarp only), so
// ~20-30 parents per SM are in flight instead of one per 128-thread CTA.
// Same sums in the same order as m2m_stage_kernel / l2l_stage_kernel.
template <int P>
constexpr int xfer_warps() { return P <= 5 ? 8 : P == 6 ? 4 : 1; }

template <int P>
__global__ void __launch_bounds__(32 * xfer_warps<P>(), P <= 5 ? 4 : 2)
m2m_warp_kernel(const double *__restrict__ child, double *__restrict__ parent,
                int64_t n_parent, int m, Halves hv) {
  constexpr int P2 = P * P, P3 = P2 * P, W = xfer_warps<P>();
  __shared__ double s_t1[W][4 * P3];  // z done: [oxy][i][j][k']
  __shared__ double s_t2[W][2 * P3];  // y done: [ox][i][j'][k']
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *t1 = s_t1[wid], *t2 = s_t2[wid];
  for (int64_t w = int64_t(blockIdx.x) * W + wid; w < n_parent * m; w += int64_t(gridDim.x) * W) {
    const int64_t q = w / m;
    const int c = (int)(w - q * m);
    // z, summing oz: line (oxy, i, j)
    for (int l = lane; l < 4 * P2; l += 32) {
      const int oxy = l / P2, ij = l - oxy * P2;
      double v[2][P];
#pragma unroll
      for (int oz = 0; oz < 2; ++oz) {
        const double *src = child + ((8 * q + 2 * oxy + oz) * m + c) * (int64_t)P3 + ij * P;
#pragma unroll
        for (int k = 0; k < P; ++k) v[oz][k] = src[k];
      }
#pragma unroll
      for (int kp = 0; kp < P; ++kp) {
        double s = 0.0;
#pragma unroll
        for (int oz = 0; oz < 2; ++oz)
#pragma unroll
          for (int k = 0; k < P; ++k) s = fma(hv.H[oz][kp * P + k], v[oz][k], s);
        t1[l * P + kp] = s;
      }
    }
    __syncwarp();
    // y, summing oy: line (ox, i, k')
    for (int l = lane; l < 2 * P2; l += 32) {
      const int ox = l / P2, r = l - ox * P2, i = r / P, kp = r - i * P;
      double v[2][P];
#pragma unroll
      for (int oy = 0; oy < 2; ++oy)
#pragma unroll
        for (int j = 0; j < P; ++j) v[oy][j] = t1[(2 * ox + oy) * P3 + i * P2 + j * P + kp];
#pragma unroll
      for (int jp = 0; jp < P; ++jp) {
        double s = 0.0;
#pragma unroll
        for (int oy = 0; oy < 2; ++oy)
#pragma unroll
          for (int j = 0; j < P; ++j) s = fma(hv.H[oy][jp * P + j], v[oy][j], s);
        t2[ox * P3 + i * P2 + jp * P + kp] = s;
      }
    }
    __syncwarp();
    // x, summing ox: line (j', k')
    double *dst = parent + (q * m + c) * (int64_t)P3;
    for (int l = lane; l < P2; l += 32) {
      double v[2][P];
#pragma unroll
      for (int ox = 0; ox < 2; ++ox)
#pragma unroll
        for (int i = 0; i < P; ++i) v[ox][i] = t2[ox * P3 + i * P2 + l];
#pragma unroll
      for (int ip = 0; ip < P; ++ip) {
        double s = 0.0;
#pragma unroll
        for (int ox = 0; ox < 2; ++ox)
#pragma unroll
          for (int i = 0; i < P; ++i) s = fma(hv.H[ox][ip * P + i], v[ox][i], s);
        dst[ip * P2 + l] = s;
      }
    }
    __syncwarp();
  }
}

template <int P>
__global__ void __launch_bounds__(32 * xfer_warps<P>(), P <= 5 ? 4 : 2)
l2l_warp_kernel(const double *__restrict__ parent, double *__restrict__ child,
                int64_t n_parent, int m, Halves hv) {
  constexpr int P2 = P * P, P3 = P2 * P, W = xfer_warps<P>();
  __shared__ double s_u[W][2 * P3];  // x done: [ox][i'][j][k]
  __shared__ double s_t[W][4 * P3];  // y done: [ox oy][i'][j'][k]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *u = s_u[wid], *t = s_t[wid];
  for (int64_t w = int64_t(blockIdx.x) * W + wid; w < n_parent * m; w += int64_t(gridDim.x) * W) {
    const int64_t q = w / m;
    const int c = (int)(w - q * m);
    const double *src0 = parent + (q * m + c) * (int64_t)P3;
    // x, per ox: line (j, k)
    for (int l = lane; l < P2; l += 32) {
      double v[P];
#pragma unroll
      for (int i = 0; i < P; ++i) v[i] = src0[i * P2 + l];
#pragma unroll
      for (int ox = 0; ox < 2; ++ox)
#pragma unroll
        for (int ip = 0; ip < P; ++ip) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < P; ++i) s = fma(hv.H[ox][i * P + ip], v[i], s);
          u[ox * P3 + ip * P2 + l] = s;
        }
    }
    __syncwarp();
    // y, per (ox, oy): line (ox, i', k)
    for (int l = lane; l < 2 * P2; l += 32) {
      const int ox = l / P2, r = l - ox * P2, ip = r / P, k = r - ip * P;
      double v[P];
#pragma unroll
      for (int j = 0; j < P; ++j) v[j] = u[ox * P3 + ip * P2 + j * P + k];
#pragma unroll
      for (int oy = 0; oy < 2; ++oy)
#pragma unroll
        for (int jp = 0; jp < P; ++jp) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < P; ++j) s = fma(hv.H[oy][j * P + jp], v[j], s);
          t[(2 * ox + oy) * P3 + ip * P2 + jp * P + k] = s;
        }
    }
    __syncwarp();
    // z, per child: line (oxy, i', j') -> the two oz children
    for (int l = lane; l < 4 * P2; l += 32) {
      const int oxy = l / P2, ijp = l - oxy * P2;
      double v[P];
#pragma unroll
      for (int k = 0; k < P; ++k) v[k] = t[oxy * P3 + ijp * P + k];
#pragma unroll
      for (int oz = 0; oz < 2; ++oz) {
        double *dst = child + ((8 * q + 2 * oxy + oz) * m + c) * (int64_t)P3 + ijp * P;
#pragma unroll
        for (int kp = 0; kp < P; ++kp) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < P; ++k) s = fma(hv.H[oz][k * P + kp], v[k], s);
          dst[kp] += s;
        }
      }
    }
    __syncwarp();
  }
}

template <int P>
int launch_xfer(bool up, const double *src, double *dst, int64_t n_parent, int m,
                const Halves &hv, cudaStream_t st) {
  constexpr size_t smem = xfer_smem<P>();
  static unsigned long long attr = 0;
  if (first_on_device(&attr)) {
    cudaFuncSetAttribute(m2m_stage_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(l2l_stage_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  }
  if constexpr (P <= 6) {
    if (n_parent * m >= 4096) {  // large levels: warp per (parent, column)
      constexpr int W = xfer_warps<P>();
      const unsigned gw =
          (unsigned)std::min<int64_t>(ceil_div(n_parent * m, W), (int64_t)kNumSMs * 64);
      if (up) {
        m2m_warp_kernel<P><<<gw, 32 * W, 0, st>>>(src, dst, n_parent, m, hv);
        return check_launch("m2m_warp_kernel");
      }
      l2l_warp_kernel<P><<<gw, 32 * W, 0, st>>>(src, dst, n_parent, m, hv);
      return check_launch("l2l_warp_kernel");
    }
  }
  const unsigned grid = (unsigned)std::min<int64_t>(n_parent * m, (int64_t)kNumSMs * 16);
  if (up) {
    m2m_stage_kernel<P><<<grid, kXferThreads2, smem, st>>>(src, dst, n_parent, m, hv);
    return check_launch("m2m_stage_kernel");
  }
  l2l_stage_kernel<P><<<grid, kXferThreads2, smem, st>>>(src, dst, n_parent, m, hv);
  return check_launch("l2l_stage_kernel");
}

inline int dispatch_xfer(int p, bool up, const double *src, double *dst, int64_t n_parent,
                         int m, const Halves &hv, cudaStream_t st) {
  switch (p) {
    case 2: return launch_xfer<2>(up, src, dst, n_parent, m, hv, st);
    case 3: return launch_xfer<3>(up, src, dst, n_parent, m, hv, st);
    case 4: return launch_xfer<4>(up, src, dst, n_parent, m, hv, st);
    case 5: return launch_xfer<5>(up, src, dst, n_parent, m, hv, st);
    case 6: return launch_xfer<6>(up, src, dst, n_parent, m, hv, st);
    case 7: return launch_xfer<7>(up, src, dst, n_parent, m, hv, st);
    default: return launch_xfer<8>(up, src, dst, n_parent, m, hv, st);
  }
}
