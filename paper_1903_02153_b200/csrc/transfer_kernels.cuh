// Warp-per-(parent, column) M2M / L2L specialised on P (included by
// interp.cu; production path for 2 <= p <= 8).  T[o] = kron(H[ox], H[oy],
// H[oz]) (interpolation.py:136-155) is applied as three P x P contractions
// in the warp's shared slice; only __syncwarp between passes, so warps of a
// CTA never wait on each other.
#pragma once

constexpr int kXferWarps = 8;

// out = (up ? T[o] : T[o]^T) in, on P^3 tensors (index (i*P + j)*P + k).
template <int P, bool UP>
__device__ __forceinline__ void kron_warp(const Halves &hv, int o, const double *in,
                                          double *t1, double *t2, double *out,
                                          bool accumulate, int lane) {
  constexpr int P3 = P * P * P;
  const double *Hx = hv.H[(o >> 2) & 1];
  const double *Hy = hv.H[(o >> 1) & 1];
  const double *Hz = hv.H[o & 1];
  for (int e = lane; e < P3; e += 32) {  // contract z
    const int ij = e / P, k = e - ij * P;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < P; ++q) s = fma(UP ? Hz[k * P + q] : Hz[q * P + k], in[ij * P + q], s);
    t1[e] = s;
  }
  __syncwarp();
  for (int e = lane; e < P3; e += 32) {  // contract y
    const int i = e / (P * P), j = (e / P) % P, k = e % P;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < P; ++q)
      s = fma(UP ? Hy[j * P + q] : Hy[q * P + j], t1[(i * P + q) * P + k], s);
    t2[e] = s;
  }
  __syncwarp();
  for (int e = lane; e < P3; e += 32) {  // contract x
    const int i = e / (P * P), jk = e - i * P * P;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < P; ++q)
      s = fma(UP ? Hx[i * P + q] : Hx[q * P + i], t2[q * P * P + jk], s);
    out[e] = accumulate ? out[e] + s : s;
  }
  __syncwarp();
}

// parent[q] = sum_o T[o] child[8q + o] (engine.py:187-204)
template <int P>
__global__ void __launch_bounds__(32 * kXferWarps)
m2m_warp_kernel(const double *__restrict__ child, double *__restrict__ parent,
                int64_t n_parent, int m, Halves hv) {
  constexpr int P3 = P * P * P;
  extern __shared__ double smx[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *in = smx + wid * 4 * P3, *t1 = in + P3, *t2 = t1 + P3, *acc = t2 + P3;
  for (int64_t w = int64_t(blockIdx.x) * kXferWarps + wid; w < n_parent * m;
       w += int64_t(gridDim.x) * kXferWarps) {
    const int64_t q = w / m;
    const int c = (int)(w - q * m);
#pragma unroll 1
    for (int o = 0; o < 8; ++o) {
      const double *src = child + ((8 * q + o) * m + c) * (int64_t)P3;
      for (int e = lane; e < P3; e += 32) in[e] = src[e];
      __syncwarp();
      kron_warp<P, true>(hv, o, in, t1, t2, acc, o > 0, lane);
    }
    double *dst = parent + (q * m + c) * (int64_t)P3;
    for (int e = lane; e < P3; e += 32) dst[e] = acc[e];
    __syncwarp();
  }
}

// child[8q + o] += T[o]^T parent[q] (engine.py:296-311)
template <int P>
__global__ void __launch_bounds__(32 * kXferWarps)
l2l_warp_kernel(const double *__restrict__ parent, double *__restrict__ child,
                int64_t n_parent, int m, Halves hv) {
  constexpr int P3 = P * P * P;
  extern __shared__ double smx[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *in = smx + wid * 4 * P3, *t1 = in + P3, *t2 = t1 + P3, *out = t2 + P3;
  for (int64_t w = int64_t(blockIdx.x) * kXferWarps + wid; w < n_parent * m;
       w += int64_t(gridDim.x) * kXferWarps) {
    const int64_t q = w / m;
    const int c = (int)(w - q * m);
    const double *src = parent + (q * m + c) * (int64_t)P3;
    for (int e = lane; e < P3; e += 32) in[e] = src[e];
    __syncwarp();
#pragma unroll 1
    for (int o = 0; o < 8; ++o) {
      double *dst = child + ((8 * q + o) * m + c) * (int64_t)P3;
      for (int e = lane; e < P3; e += 32) out[e] = dst[e];
      __syncwarp();
      kron_warp<P, false>(hv, o, in, t1, t2, out, true, lane);
      for (int e = lane; e < P3; e += 32) dst[e] = out[e];
      __syncwarp();
    }
  }
}

template <int P>
int launch_xfer(bool up, const double *src, double *dst, int64_t n_parent, int m,
                const Halves &hv, cudaStream_t st) {
  constexpr size_t smem = sizeof(double) * 4 * P * P * P * kXferWarps;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(m2m_warp_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(l2l_warp_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  const unsigned grid = (unsigned)grid_cap(ceil_div(n_parent * m, kXferWarps), 8);
  if (up) {
    m2m_warp_kernel<P><<<grid, 32 * kXferWarps, smem, st>>>(src, dst, n_parent, m, hv);
    return check_launch("m2m_warp_kernel");
  }
  l2l_warp_kernel<P><<<grid, 32 * kXferWarps, smem, st>>>(src, dst, n_parent, m, hv);
  return check_launch("l2l_warp_kernel");
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
