// Tree build: leaf binning + stable radix sort + run-length segments.
//
// Replaces _Partition.build (engine.py:71-80) and Octree.leaf_index
// (octree.py:186-200).  Bit-exactness with NumPy: the leaf coordinate is
// floor((x - lo) / h) computed with IEEE subtraction and correctly rounded
// division (no reciprocal, no FMA), the same clip, and CUB's LSD radix sort
// is stable, so `perm` equals np.argsort(ids, kind="stable").
#include <cub/cub.cuh>

#include "common.cuh"

namespace bfmm {
namespace {

struct TreeGeom {
  double lo[3], hi[3], h, tol;
};

template <typename Key>
__global__ void leaf_keys_kernel(const double *__restrict__ pts, int64_t n,
                                 TreeGeom g, int levels, Key *__restrict__ keys,
                                 int64_t *__restrict__ iota,
                                 int32_t *__restrict__ domain_flag) {
  const int64_t nmax = (int64_t(1) << levels) - 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t c[3];
    bool bad = false, nonfinite = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double x = pts[3 * i + a];
      // octree.py:190-192: pts < lo - tol or pts > high + tol
      bad |= (x < __dsub_rn(g.lo[a], g.tol)) | (x > __dadd_rn(g.hi[a], g.tol));
      nonfinite |= !isfinite(x);  // engine.py:55-56
      double f = floor(__ddiv_rn(__dsub_rn(x, g.lo[a]), g.h));
      int64_t v = (int64_t)f;  // astype(int64) truncation of an integral value
      v = v < 0 ? 0 : (v > nmax ? nmax : v);
      c[a] = v;
    }
    if (bad) atomicOr(domain_flag, 1);
    if (nonfinite) atomicOr(domain_flag, 2);
    keys[i] = (Key)morton3((uint64_t)c[0], (uint64_t)c[1], (uint64_t)c[2]);
    iota[i] = i;
  }
}

template <typename Key>
__global__ void heads_kernel(const Key *__restrict__ k, int64_t n,
                             int32_t *__restrict__ head) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

template <typename Key>
__global__ void runs_kernel(const Key *__restrict__ k, const int32_t *head,
                            const int32_t *__restrict__ run, int64_t n,
                            int64_t *__restrict__ leaves,
                            int64_t *__restrict__ starts,
                            int64_t *__restrict__ n_leaves) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (head[i]) {
      leaves[run[i]] = (int64_t)k[i];
      starts[run[i]] = i;
    }
    if (i == n - 1) *n_leaves = (int64_t)run[i] + head[i];
  }
}

__global__ void counts_kernel(const int64_t *__restrict__ leaves,
                              const int64_t *__restrict__ starts,
                              const int64_t *__restrict__ n_leaves, int64_t n,
                              int64_t *__restrict__ counts,
                              int32_t *__restrict__ cell_start,
                              int32_t *__restrict__ cell_count) {
  const int64_t nl = *n_leaves;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < nl;
       r += int64_t(gridDim.x) * blockDim.x) {
    int64_t end = (r + 1 < nl) ? starts[r + 1] : n;
    int64_t c = end - starts[r];
    counts[r] = c;
    cell_start[leaves[r]] = (int32_t)starts[r];
    cell_count[leaves[r]] = (int32_t)c;
  }
}

__global__ void gather_points_kernel(const double *__restrict__ pts,
                                     const int64_t *__restrict__ perm,
                                     int64_t n, double *__restrict__ pts4) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t j = perm[i];
    double4 v;
    v.x = pts[3 * j];
    v.y = pts[3 * j + 1];
    v.z = pts[3 * j + 2];
    v.w = 0.0;
    reinterpret_cast<double4 *>(pts4)[i] = v;
  }
}

__global__ void gather_weights_kernel(const double *__restrict__ w, int64_t n,
                                      int m, const int64_t *__restrict__ perm,
                                      double *__restrict__ ws,
                                      double *__restrict__ pts4,
                                      int32_t *__restrict__ weights_flag) {
  const int64_t total = n * m;
  bool bad = false;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t i = e / m;
    int c = (int)(e - i * m);
    double v = w[perm[i] * m + c];
    bad |= !isfinite(v);
    ws[e] = v;
    if (c == 0) pts4[4 * i + 3] = v;
  }
  // "weights contain non-finite values" (engine.py:496-497), checked on the
  // device in the same pass instead of an O(N) host scan
  if (weights_flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(weights_flag, 1);
}

inline int grid_for(int64_t n, int threads) {
  int64_t b = ceil_div(n, threads);
  int64_t cap = int64_t(kNumSMs) * 32;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

struct ScratchLayout {
  size_t keys_in, keys_out, iota, head, run, cub;
  size_t total;
};

template <typename Key>
ScratchLayout layout(int64_t n) {
  ScratchLayout s{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  s.keys_in = take(sizeof(Key) * n);
  s.keys_out = take(sizeof(Key) * n);
  s.iota = take(sizeof(int64_t) * n);
  s.head = take(sizeof(int32_t) * n);
  s.run = take(sizeof(int32_t) * n);
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (Key *)nullptr,
                                  (Key *)nullptr, (int64_t *)nullptr,
                                  (int64_t *)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int32_t *)nullptr,
                                (int32_t *)nullptr, (int)n);
  s.cub = take(sort_bytes > scan_bytes ? sort_bytes : scan_bytes);
  s.total = off;
  return s;
}

template <typename Key>
int build(const double *points, int64_t n, const TreeGeom &g, int levels,
          void *scratch, size_t scratch_bytes, int64_t *perm, double *pts4,
          int64_t *leaves, int64_t *starts, int64_t *counts, int64_t *n_leaves,
          int32_t *cell_start, int32_t *cell_count, int32_t *domain_flag,
          cudaStream_t st) {
  ScratchLayout s = layout<Key>(n);
  if (scratch_bytes < s.total) {
    set_error("bfmm_tree_build: scratch too small (%zu < %zu)", scratch_bytes,
              s.total);
    return 2;
  }
  char *base = static_cast<char *>(scratch);
  Key *kin = reinterpret_cast<Key *>(base + s.keys_in);
  Key *kout = reinterpret_cast<Key *>(base + s.keys_out);
  int64_t *iota = reinterpret_cast<int64_t *>(base + s.iota);
  int32_t *head = reinterpret_cast<int32_t *>(base + s.head);
  int32_t *run = reinterpret_cast<int32_t *>(base + s.run);
  void *cub_tmp = base + s.cub;
  size_t cub_bytes = s.total - s.cub;

  const size_t ncell = size_t(1) << (3 * levels);
  if (cudaMemsetAsync(cell_count, 0, ncell * sizeof(int32_t), st) != cudaSuccess ||
      cudaMemsetAsync(n_leaves, 0, sizeof(int64_t), st) != cudaSuccess) {
    set_error("bfmm_tree_build: memset failed");
    return 1;
  }
  if (n == 0) return 0;
  const int T = 256;
  leaf_keys_kernel<Key><<<grid_for(n, T), T, 0, st>>>(points, n, g, levels,
                                                      kin, iota, domain_flag);
  if (check_launch("leaf_keys_kernel")) return 1;
  size_t sb = cub_bytes;
  if (cub::DeviceRadixSort::SortPairs(cub_tmp, sb, kin, kout, iota, perm,
                                      (int)n, 0, 3 * levels,
                                      st) != cudaSuccess) {
    set_error("bfmm_tree_build: radix sort failed");
    return 1;
  }
  add_launches(2 + (3 * levels + 7) / 8);  // CUB onesweep: histogram, scan, passes
  heads_kernel<Key><<<grid_for(n, T), T, 0, st>>>(kout, n, head);
  if (check_launch("heads_kernel")) return 1;
  sb = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, sb, head, run, (int)n, st) !=
      cudaSuccess) {
    set_error("bfmm_tree_build: scan failed");
    return 1;
  }
  add_launches(2);  // CUB scan: init + scan
  runs_kernel<Key><<<grid_for(n, T), T, 0, st>>>(kout, head, run, n, leaves,
                                                 starts, n_leaves);
  if (check_launch("runs_kernel")) return 1;
  counts_kernel<<<grid_for(n, T), T, 0, st>>>(leaves, starts, n_leaves, n,
                                              counts, cell_start, cell_count);
  if (check_launch("counts_kernel")) return 1;
  gather_points_kernel<<<grid_for(n, T), T, 0, st>>>(points, perm, n, pts4);
  return check_launch("gather_points_kernel");
}

// Active cells of a coarser level: the distinct ancestors (leaf >> shift) of
// the occupied leaves that fall in [lo, hi).  `leaves` is sorted, so an
// ancestor is new exactly where it differs from its predecessor's.
__global__ void active_flags_kernel(const int64_t *__restrict__ leaves,
                                    const int64_t *__restrict__ n_leaves,
                                    int64_t cap, int shift, int64_t lo,
                                    int64_t hi, int32_t *__restrict__ flag) {
  const int64_t nl = *n_leaves;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cap;
       i += int64_t(gridDim.x) * blockDim.x) {
    int32_t f = 0;
    if (i < nl) {
      const int64_t a = leaves[i] >> shift;
      f = (a >= lo && a < hi && (i == 0 || (leaves[i - 1] >> shift) != a)) ? 1 : 0;
    }
    flag[i] = f;
  }
}

__global__ void active_emit_kernel(const int64_t *__restrict__ leaves,
                                   int64_t cap, int shift,
                                   const int32_t *__restrict__ flag,
                                   const int32_t *__restrict__ pos,
                                   int64_t *__restrict__ list,
                                   int64_t *__restrict__ count) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cap;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (flag[i]) list[pos[i]] = leaves[i] >> shift;
    if (i == cap - 1) *count = (int64_t)pos[i] + flag[i];
  }
}

// Histogram of the octant (cell & 7) of the first *n cells.
__global__ void octant_hist_kernel(const int64_t *__restrict__ cells,
                                   const int64_t *__restrict__ n_dev,
                                   int64_t *__restrict__ hist) {
  __shared__ unsigned long long h[8];
  if (threadIdx.x < 8) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t n = *n_dev;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(&h[cells[i] & 7], 1ull);
  __syncthreads();
  if (threadIdx.x < 8 && h[threadIdx.x])
    atomicAdd(reinterpret_cast<unsigned long long *>(hist) + threadIdx.x, h[threadIdx.x]);
}

}  // namespace
}  // namespace bfmm

using namespace bfmm;

extern "C" size_t bfmm_tree_scratch_bytes(int64_t n, int levels) {
  if (n < 1) n = 1;
  return (3 * levels <= 32) ? layout<uint32_t>(n).total
                            : layout<uint64_t>(n).total;
}

extern "C" int bfmm_tree_build(const double *points, int64_t n,
                               const double *geom, int levels, void *scratch,
                               size_t scratch_bytes, int64_t *perm,
                               double *pts4, int64_t *leaves, int64_t *starts,
                               int64_t *counts, int64_t *n_leaves,
                               int32_t *cell_start, int32_t *cell_count,
                               int32_t *domain_flag, bfmm_stream_t stream) {
  if (levels < 2 || levels > 21) {
    set_error("bfmm_tree_build: levels %d outside [2, 21]", levels);
    return 2;
  }
  if (n < 0 || n > INT32_MAX) {
    set_error("bfmm_tree_build: n=%lld unsupported", (long long)n);
    return 2;
  }
  TreeGeom g;
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = geom[a];
    g.hi[a] = geom[3 + a];
  }
  g.h = geom[6];
  g.tol = geom[7];
  cudaStream_t st = as_stream(stream);
  if (3 * levels <= 32)
    return build<uint32_t>(points, n, g, levels, scratch, scratch_bytes, perm,
                           pts4, leaves, starts, counts, n_leaves, cell_start,
                           cell_count, domain_flag, st);
  return build<uint64_t>(points, n, g, levels, scratch, scratch_bytes, perm,
                         pts4, leaves, starts, counts, n_leaves, cell_start,
                         cell_count, domain_flag, st);
}

extern "C" int bfmm_gather_weights(const double *w, int64_t n, int m,
                                   const int64_t *perm, double *wsorted,
                                   double *pts4, int32_t *weights_flag,
                                   bfmm_stream_t stream) {
  if (n == 0) return 0;
  gather_weights_kernel<<<grid_for(n * m, 256), 256, 0, as_stream(stream)>>>(
      w, n, m, perm, wsorted, pts4, weights_flag);
  return check_launch("gather_weights_kernel");
}

extern "C" size_t bfmm_active_cells_scratch_bytes(int64_t max_leaves) {
  if (max_leaves < 1) max_leaves = 1;
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int32_t *)nullptr,
                                (int32_t *)nullptr, (int)max_leaves);
  return 2 * ((max_leaves * sizeof(int32_t) + 255) & ~size_t(255)) + cub_bytes;
}

extern "C" int bfmm_active_cells(const int64_t *leaves, const int64_t *n_leaves,
                                 int64_t max_leaves, int shift, int64_t lo,
                                 int64_t hi, void *scratch, size_t scratch_bytes,
                                 int64_t *list, int64_t *count,
                                 bfmm_stream_t stream) {
  if (max_leaves < 1 || max_leaves > INT32_MAX || shift < 0 || shift > 60) {
    set_error("bfmm_active_cells: max_leaves=%lld shift=%d unsupported",
              (long long)max_leaves, shift);
    return 2;
  }
  if (scratch_bytes < bfmm_active_cells_scratch_bytes(max_leaves)) {
    set_error("bfmm_active_cells: scratch too small");
    return 2;
  }
  cudaStream_t st = as_stream(stream);
  const size_t a = (max_leaves * sizeof(int32_t) + 255) & ~size_t(255);
  int32_t *flag = static_cast<int32_t *>(scratch);
  int32_t *pos = reinterpret_cast<int32_t *>(static_cast<char *>(scratch) + a);
  void *tmp = static_cast<char *>(scratch) + 2 * a;
  size_t tb = scratch_bytes - 2 * a;
  const int T = 256;
  active_flags_kernel<<<grid_for(max_leaves, T), T, 0, st>>>(leaves, n_leaves, max_leaves,
                                                            shift, lo, hi, flag);
  if (check_launch("active_flags_kernel")) return 1;
  if (cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, (int)max_leaves, st) !=
      cudaSuccess) {
    set_error("bfmm_active_cells: scan failed");
    return 1;
  }
  add_launches(2);
  active_emit_kernel<<<grid_for(max_leaves, T), T, 0, st>>>(leaves, max_leaves, shift, flag,
                                                           pos, list, count);
  return check_launch("active_emit_kernel");
}

extern "C" int bfmm_octant_histogram(const int64_t *cells, const int64_t *n_dev,
                                     int64_t max_n, int64_t *hist, bfmm_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  if (cudaMemsetAsync(hist, 0, 8 * sizeof(int64_t), st) != cudaSuccess) {
    set_error("bfmm_octant_histogram: memset failed");
    return 1;
  }
  if (max_n <= 0) return 0;
  octant_hist_kernel<<<grid_for(max_n, 256), 256, 0, st>>>(cells, n_dev, hist);
  return check_launch("octant_hist_kernel");
}

extern "C" size_t bfmm_group_by_octant_scratch_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (unsigned long long *)nullptr,
                                 (unsigned long long *)nullptr, (int)(n < 1 ? 1 : n), 0, 3);
  return bytes;
}

extern "C" int bfmm_group_by_octant(const int64_t *cells, int64_t n, int64_t *out,
                                    void *scratch, size_t scratch_bytes,
                                    bfmm_stream_t stream) {
  if (n <= 0) return 0;
  if (n > INT32_MAX || scratch_bytes < bfmm_group_by_octant_scratch_bytes(n)) {
    set_error("bfmm_group_by_octant: n=%lld or scratch too small", (long long)n);
    return 2;
  }
  // stable LSD sort on the 3 octant bits: grouped by octant, ascending within
  if (cub::DeviceRadixSort::SortKeys(scratch, scratch_bytes,
                                     reinterpret_cast<const unsigned long long *>(cells),
                                     reinterpret_cast<unsigned long long *>(out), (int)n, 0,
                                     3, as_stream(stream)) != cudaSuccess) {
    set_error("bfmm_group_by_octant: sort failed");
    return 1;
  }
  add_launches(2);
  return 0;
}
