// Shared helpers for the bfmm CUDA sources (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bfmm.h"

namespace bfmm {

// Thread-local message behind bfmm_last_error().
void set_error(const char *fmt, ...);

// Process-wide count of kernels this library has launched (bfmm_launch_count).
void add_launches(long long n);

inline int check_launch(const char *what) {
  add_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

inline cudaStream_t as_stream(bfmm_stream_t s) {
  return reinterpret_cast<cudaStream_t>(s);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int kNumSMs = 148;  // B200

// Per-device one-time setup (function attributes, __constant__ tables live
// in each device's context): true the first time it is called for the
// current device with this mask word.
inline bool first_on_device(unsigned long long *mask) {
  int d = 0;
  cudaGetDevice(&d);
  const unsigned long long bit = 1ull << (d & 63);
  return (__atomic_fetch_or(mask, bit, __ATOMIC_ACQ_REL) & bit) == 0;
}

// 21-bit Morton spread: bit b of v moves to bit 3b (octree.py:75-83 layout).
__host__ __device__ inline uint64_t spread3(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__host__ __device__ inline uint64_t compact3(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v | (v >> 2)) & 0x10C30C30C30C30C3ull;
  v = (v | (v >> 4)) & 0x100F00F00F00F00Full;
  v = (v | (v >> 8)) & 0x1F0000FF0000FFull;
  v = (v | (v >> 16)) & 0x1F00000000FFFFull;
  v = (v | (v >> 32)) & 0x1FFFFFull;
  return v;
}

// x in the high bit of each triple (octree.py:86-93).
__host__ __device__ inline uint64_t morton3(uint64_t ix, uint64_t iy,
                                            uint64_t iz) {
  return (spread3(ix) << 2) | (spread3(iy) << 1) | spread3(iz);
}

__host__ __device__ inline void unmorton3(uint64_t id, int &ix, int &iy,
                                          int &iz) {
  ix = (int)compact3(id >> 2);
  iy = (int)compact3(id >> 1);
  iz = (int)compact3(id);
}

// Far-field pair rule along one axis (octree.py:128-145): the source
// coordinate c + t stays inside [0, n); a +3 step needs an even target
// coordinate, a -3 step an odd one.
__host__ __device__ inline bool far_axis_ok(int n, int c, int t) {
  const int s = c + t;
  if (s < 0 || s >= n) return false;
  if (t == 3) return (c & 1) == 0;
  if (t == -3) return (c & 1) == 1;
  return true;
}

// The pair (target c, source c + t) is one of cell_pairs_for_offset(level, t)
// (octree.py:202-221) iff every axis passes.
__host__ __device__ inline bool far_pair(int n, int cx, int cy, int cz, int tx,
                                         int ty, int tz) {
  return far_axis_ok(n, cx, tx) && far_axis_ok(n, cy, ty) &&
         far_axis_ok(n, cz, tz);
}

}  // namespace bfmm
