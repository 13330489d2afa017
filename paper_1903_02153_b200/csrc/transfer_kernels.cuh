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
