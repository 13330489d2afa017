// Near field: built-in device functors, the NVRTC JIT for user kernels,
// launchers, the non-finite locator and the output scatter.
#include <cub/cub.cuh>
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "p2p.cuh"

namespace bfmm {
namespace {

// ---- built-in kernels (kernel.py:149-180): profile f(r) with r = |x - y| ----
// 1/r, r = 0 -> 0
// eval_fast: the hot-loop body; bodies with exp use the flagged fast exp
// (bfmm_exp_fast), the others are eval itself.
struct KLaplace {
  // cheap body: keep 5 CTAs/SM (<= 96 registers) for latency-bound sparse leaves
  static constexpr int kMinBlocks = 5;
  __device__ __forceinline__ static double eval(double dx, double dy, double dz) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    return r2 == 0.0 ? 0.0 : rsqrt(r2);
  }
  template <class F>
  __device__ __forceinline__ static double eval_fast(double dx, double dy, double dz, F &bad) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    bool b = false;
    const double v = bfmm_nf::bfmm_rsqrt_fast(r2, b);
    bfmm_nf::flag_set(bad, b && r2 != 0.0);
    return r2 == 0.0 ? 0.0 : v;
  }
  // flag-free hot-loop body (p2p.cuh, bfmm_rsqrt_raw)
  static constexpr bool kAccFlag = true;
  template <bool ZT>
  __device__ __forceinline__ static void accum_fast(double dx, double dy, double dz, double w,
                                                    double &acc) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    const double v = bfmm_nf::bfmm_rsqrt_raw(r2);
    if (!ZT || bfmm_nf::bfmm_nonzero_bits(r2)) acc = fma(v, w, acc);
  }
};
// 1/r^4, r = 0 -> 0
struct KLaplaceForce {
  __device__ __forceinline__ static double eval(double dx, double dy, double dz) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    return r2 == 0.0 ? 0.0 : 1.0 / (r2 * r2);
  }
  template <class F>
  __device__ __forceinline__ static double eval_fast(double dx, double dy, double dz, F &bad) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    bool b = false;
    const double v = bfmm_nf::bfmm_rcp_fast(r2 * r2, b);
    bfmm_nf::flag_set(bad, b && r2 != 0.0);
    return r2 == 0.0 ? 0.0 : v;
  }
  static constexpr bool kAccFlag = true;
  template <bool ZT>
  __device__ __forceinline__ static void accum_fast(double dx, double dy, double dz, double w,
                                                    double &acc) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    const double v = bfmm_nf::bfmm_rcp_raw(r2 * r2);
    if (!ZT || bfmm_nf::bfmm_nonzero_bits(r2)) acc = fma(v, w, acc);
  }
};
// exp(-r^2)
struct KGaussian {
  __device__ __forceinline__ static double eval(double dx, double dy, double dz) {
    return bfmm_nf::bfmm_exp(-(dx * dx + dy * dy + dz * dz));
  }
  template <class F>
  __device__ __forceinline__ static double eval_fast(double dx, double dy, double dz, F &bad) {
    return bfmm_nf::bfmm_exp_fast(-(dx * dx + dy * dy + dz * dz), bad);
  }
};
// exp(-r)
struct KExponential {
  __device__ __forceinline__ static double eval(double dx, double dy, double dz) {
    return bfmm_nf::bfmm_exp(-sqrt(dx * dx + dy * dy + dz * dz));
  }
  template <class F>
  __device__ __forceinline__ static double eval_fast(double dx, double dy, double dz, F &bad) {
    return bfmm_nf::bfmm_exp_fast(-bfmm_nf::bfmm_sqrt_fast(dx * dx + dy * dy + dz * dz, bad), bad);
  }
};
// log r, r = 0 -> 0
struct KLogarithm {
  __device__ __forceinline__ static double eval(double dx, double dy, double dz) {
    const double r2 = dx * dx + dy * dy + dz * dz;
    return r2 == 0.0 ? 0.0 : 0.5 * log(r2);
  }
  template <class F>
  __device__ __forceinline__ static double eval_fast(double dx, double dy, double dz, F &) {
    return eval(dx, dy, dz);
  }
};

constexpr int kMCs[5] = {1, 2, 4, 8, 16};

// ---- JIT (NVRTC + driver API loaded lazily) ---------------------------------
const char kP2PSource[] =
#include "p2p_src.inc"
    ;

struct Driver {
  bool ok = false;
  CUresult (*ModuleLoadData)(CUmodule *, const void *) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned,
                           unsigned, unsigned, unsigned, CUstream, void **,
                           void **) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char **) = nullptr;
};

Driver &driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    d.ModuleLoadData = (decltype(d.ModuleLoadData))dlsym(h, "cuModuleLoadData");
    d.ModuleGetFunction =
        (decltype(d.ModuleGetFunction))dlsym(h, "cuModuleGetFunction");
    d.LaunchKernel = (decltype(d.LaunchKernel))dlsym(h, "cuLaunchKernel");
    d.GetErrorString = (decltype(d.GetErrorString))dlsym(h, "cuGetErrorString");
    d.ok = d.ModuleLoadData && d.ModuleGetFunction && d.LaunchKernel;
  });
  return d;
}

struct JitKernel {
  CUfunction p2p[5];
  CUfunction locate;
  CUfunction sym;
  CUfunction direct;
  CUfunction block;
  CUfunction group;
  CUfunction tile;
  CUfunction tile1;
};

std::mutex g_jit_mu;
std::vector<JitKernel> g_jit;                       // handle - 6
std::unordered_map<std::string, int> g_jit_cache;  // source -> handle

constexpr int kFirstJit = 6;

std::string functor_source(int kind, const char *expr) {
  // body(fast): the prologue that defines r / r2 for the expression; the fast
  // body takes r from the branch-free bfmm_sqrt_fast
  auto body = [&](bool fast) {
    std::string b;
    if (kind == 0)
      b = std::string("const double r = ") +
          (fast ? "bfmm_sqrt_fast(dx * dx + dy * dy + dz * dz, bfmm_bad_)"
                : "sqrt(dx * dx + dy * dy + dz * dz)") +
          ";\n return (" + std::string(expr) + ");";
    else if (kind == 1)
      b = "const double r2 = dx * dx + dy * dy + dz * dz;\n return (" + std::string(expr) + ");";
    else
      b = "return (" + std::string(expr) + ");";
    return b;
  };
  // exp() in user expressions maps to the branch-free bfmm_exp (p2p.cuh);
  // eval_fast uses the flagged fast paths (bfmm_exp_fast, bfmm_sqrt_fast)
  return "#define exp(x) bfmm_exp(x)\nstruct KUser {\n __device__ __forceinline__ "
         "static double eval(double dx, double dy, double dz) {\n " +
         body(false) + "\n }\n#undef exp\n#define exp(x) bfmm_exp_fast(x, bfmm_bad_)\n"
         "#define sqrt(x) bfmm_sqrt_fast(x, bfmm_bad_)\n"
         " template <class F> __device__ __forceinline__ static double eval_fast(double dx, "
         "double dy, double dz, F &bfmm_bad_) {\n " + body(true) + "\n }\n#undef exp\n#undef sqrt\n};\n";
}

int jit_compile(int kind, const char *expr, int *handle) {
  std::lock_guard<std::mutex> lock(g_jit_mu);
  // modules are loaded into the current device's context: one per device
  int dev = 0;
  cudaGetDevice(&dev);
  std::string key = std::to_string(dev) + ":" + std::to_string(kind) + ":" + expr;
  auto it = g_jit_cache.find(key);
  if (it != g_jit_cache.end()) {
    *handle = it->second;
    return 0;
  }
  Driver &d = driver();
  if (!d.ok) {
    set_error("bfmm_kernel_compile: libcuda.so.1 not available");
    return 3;
  }
  std::string src = std::string(kP2PSource) + "\nnamespace bfmm_nf {\n" +
                    functor_source(kind, expr) + "}\n";
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "bfmm_user_p2p.cu", 0, nullptr,
                         nullptr) != NVRTC_SUCCESS) {
    set_error("bfmm_kernel_compile: nvrtcCreateProgram failed");
    return 3;
  }
  std::vector<std::string> names;
  for (int i = 0; i < 5; ++i)
    names.push_back("bfmm_nf::p2p_kernel<bfmm_nf::KUser, " +
                    std::to_string(kMCs[i]) + ">");
  names.push_back("bfmm_nf::locate_kernel<bfmm_nf::KUser>");
  names.push_back("bfmm_nf::p2p_sym_kernel<bfmm_nf::KUser>");
  names.push_back("bfmm_nf::direct_kernel<bfmm_nf::KUser>");
  names.push_back("bfmm_nf::pair_block_kernel<bfmm_nf::KUser>");
  names.push_back("bfmm_nf::p2p_group_kernel<bfmm_nf::KUser>");
  names.push_back("bfmm_nf::p2p_tile_kernel<bfmm_nf::KUser, 0>");
  names.push_back("bfmm_nf::p2p_tile_kernel<bfmm_nf::KUser, 1>");
  for (auto &n : names) nvrtcAddNameExpression(prog, n.c_str());
  std::vector<std::string> opt_s = {"--gpu-architecture=sm_100a", "--std=c++17",
                                    "-default-device", "-lineinfo"};
  // BFMM_JIT_OPTS: extra NVRTC options (tuning experiments, e.g. -D...)
  if (const char *extra = getenv("BFMM_JIT_OPTS")) {
    std::string e(extra), tok;
    for (size_t i = 0; i <= e.size(); ++i) {
      if (i == e.size() || e[i] == ' ') {
        if (!tok.empty()) opt_s.push_back(tok);
        tok.clear();
      } else {
        tok += e[i];
      }
    }
  }
  std::vector<const char *> opts;
  for (auto &o : opt_s) opts.push_back(o.c_str());
  nvrtcResult rc = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
  if (rc != NVRTC_SUCCESS) {
    size_t logn = 0;
    nvrtcGetProgramLogSize(prog, &logn);
    std::string log(logn, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    set_error("bfmm_kernel_compile: NVRTC failed for '%s': %s", expr,
              log.c_str());
    nvrtcDestroyProgram(&prog);
    return 4;
  }
  size_t cubin_n = 0;
  nvrtcGetCUBINSize(prog, &cubin_n);
  std::vector<char> cubin(cubin_n);
  nvrtcGetCUBIN(prog, cubin.data());
  std::vector<std::string> lowered;
  for (auto &n : names) {
    const char *ln = nullptr;
    nvrtcGetLoweredName(prog, n.c_str(), &ln);
    lowered.push_back(ln ? ln : "");
  }
  nvrtcDestroyProgram(&prog);
  // make sure the runtime has initialised the primary context
  cudaFree(0);
  CUmodule mod;
  CUresult cr = d.ModuleLoadData(&mod, cubin.data());
  if (cr != CUDA_SUCCESS) {
    const char *msg = "?";
    if (d.GetErrorString) d.GetErrorString(cr, &msg);
    set_error("bfmm_kernel_compile: cuModuleLoadData: %s", msg);
    return 3;
  }
  JitKernel jk;
  for (int i = 0; i < 12; ++i) {
    CUfunction f;
    if (d.ModuleGetFunction(&f, mod, lowered[i].c_str()) != CUDA_SUCCESS) {
      set_error("bfmm_kernel_compile: missing %s", names[i].c_str());
      return 3;
    }
    if (i < 5) jk.p2p[i] = f;
    else if (i == 5) jk.locate = f;
    else if (i == 6) jk.sym = f;
    else if (i == 7) jk.direct = f;
    else if (i == 8) jk.block = f;
    else if (i == 9) jk.group = f;
    else if (i == 10) jk.tile = f;
    else jk.tile1 = f;
  }
  g_jit.push_back(jk);
  *handle = kFirstJit + (int)g_jit.size() - 1;
  g_jit_cache[key] = *handle;
  return 0;
}

// ---- launch helpers ---------------------------------------------------------
template <class K>
void launch_builtin(int mci, dim3 grid, const bfmm_nf::Args &a, int c0,
                    cudaStream_t st) {
  const int T = 32 * bfmm_nf::kWarps;
  switch (mci) {
    case 0: bfmm_nf::p2p_kernel<K, 1><<<grid, T, 0, st>>>(a, c0); break;
    case 1: bfmm_nf::p2p_kernel<K, 2><<<grid, T, 0, st>>>(a, c0); break;
    case 2: bfmm_nf::p2p_kernel<K, 4><<<grid, T, 0, st>>>(a, c0); break;
    case 3: bfmm_nf::p2p_kernel<K, 8><<<grid, T, 0, st>>>(a, c0); break;
    default: bfmm_nf::p2p_kernel<K, 16><<<grid, T, 0, st>>>(a, c0); break;
  }
}

int launch_p2p(int handle, int mci, dim3 grid, const bfmm_nf::Args &a, int c0,
               cudaStream_t st) {
  switch (handle) {
    case 1: launch_builtin<KLaplace>(mci, grid, a, c0, st); break;
    case 2: launch_builtin<KLaplaceForce>(mci, grid, a, c0, st); break;
    case 3: launch_builtin<KGaussian>(mci, grid, a, c0, st); break;
    case 4: launch_builtin<KExponential>(mci, grid, a, c0, st); break;
    case 5: launch_builtin<KLogarithm>(mci, grid, a, c0, st); break;
    default: {
      JitKernel jk;
      {
        std::lock_guard<std::mutex> lock(g_jit_mu);
        if (handle < kFirstJit || handle - kFirstJit >= (int)g_jit.size()) {
          set_error("bfmm_p2p: unknown kernel handle %d", handle);
          return 2;
        }
        jk = g_jit[handle - kFirstJit];
      }
      bfmm_nf::Args args = a;
      int c = c0;
      void *params[] = {&args, &c};
      CUresult r = driver().LaunchKernel(jk.p2p[mci], grid.x, 1, 1,
                                         32 * bfmm_nf::kWarps, 1, 1, 0,
                                         (CUstream)st, params, nullptr);
      if (r != CUDA_SUCCESS) {
        set_error("bfmm_p2p: cuLaunchKernel failed (%d)", (int)r);
        return 1;
      }
      return 0;
    }
  }
  return check_launch("p2p_kernel");
}

int launch_locate(int handle, const bfmm_nf::Args &a,
                  unsigned long long *key, cudaStream_t st) {
  dim3 grid(kNumSMs * 8), block(128);
  switch (handle) {
    case 1: bfmm_nf::locate_kernel<KLaplace><<<grid, block, 0, st>>>(a, key); break;
    case 2: bfmm_nf::locate_kernel<KLaplaceForce><<<grid, block, 0, st>>>(a, key); break;
    case 3: bfmm_nf::locate_kernel<KGaussian><<<grid, block, 0, st>>>(a, key); break;
    case 4: bfmm_nf::locate_kernel<KExponential><<<grid, block, 0, st>>>(a, key); break;
    case 5: bfmm_nf::locate_kernel<KLogarithm><<<grid, block, 0, st>>>(a, key); break;
    default: {
      JitKernel jk;
      {
        std::lock_guard<std::mutex> lock(g_jit_mu);
        if (handle < kFirstJit || handle - kFirstJit >= (int)g_jit.size()) {
          set_error("bfmm_p2p_locate: unknown kernel handle %d", handle);
          return 2;
        }
        jk = g_jit[handle - kFirstJit];
      }
      bfmm_nf::Args args = a;
      unsigned long long *k = key;
      void *params[] = {&args, &k};
      if (driver().LaunchKernel(jk.locate, grid.x, 1, 1, block.x, 1, 1, 0,
                                (CUstream)st, params, nullptr) != CUDA_SUCCESS) {
        set_error("bfmm_p2p_locate: cuLaunchKernel failed");
        return 1;
      }
      return 0;
    }
  }
  return check_launch("locate_kernel");
}

// Work units per target leaf: 32-target chunks, or (wide, one weight column)
// 64-target units while the leaf has 64 left and 32-target chunks for the
// remainder (p2p_kernel decodes the same split); leaves outside
// [cell_lo, cell_hi) (other ranks' shards) get none.
__global__ void chunk_counts_kernel(const int64_t *__restrict__ counts,
                                    const int64_t *__restrict__ leaves,
                                    const int64_t *__restrict__ n_leaves,
                                    int64_t max_leaves, int64_t cell_lo,
                                    int64_t cell_hi, int small_max, int wide,
                                    int64_t *__restrict__ nch) {
  // leaves of <= small_max points go to p2p_group_kernel instead
  const int64_t nl = *n_leaves;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
       i < max_leaves; i += int64_t(gridDim.x) * blockDim.x)
    nch[i] = (i < nl && leaves[i] >= cell_lo && leaves[i] < cell_hi && counts[i] > small_max)
                 ? (wide ? (counts[i] >> 6) + (((counts[i] & 63) + 31) >> 5)
                         : (counts[i] + 31) / 32)
                 : 0;
}

// chunk -> leaf map from the inclusive chunk prefix (entries past cap are
// left to the kernel's binary search)
__global__ void chunk_map_kernel(const int64_t *__restrict__ incl,
                                 const int64_t *__restrict__ n_leaves,
                                 int64_t max_leaves, int64_t cap,
                                 int32_t *__restrict__ chunk_leaf) {
  const int64_t nl = *n_leaves;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
       i < max_leaves && i < nl; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c1 = incl[i] < cap ? incl[i] : cap;
    for (int64_t c = i ? incl[i - 1] : 0; c < c1; ++c) chunk_leaf[c] = (int32_t)i;
  }
}

__global__ void scatter_kernel(const double *__restrict__ far,
                               const double *__restrict__ near,
                               const int64_t *__restrict__ perm, int64_t n,
                               int m, double *__restrict__ phi, int32_t *flag) {
  const int64_t total = n * m;
  bool bad = false;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / m;
    const int c = (int)(e - i * m);
    const double nv = near[e];
    bad |= !isfinite(nv);
    phi[perm[i] * m + c] = (far ? far[e] : 0.0) + nv;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Near list for one neighbour offset (engine.py:401-417): per target leaf,
// the index of the source leaf at cell + t among the nonempty source leaves
// (np.searchsorted), or -1.  Same in-range rule as the P2P kernel.
__global__ void near_pairs_kernel(int levels, int t_index,
                                  const int64_t *__restrict__ tleaves,
                                  const int64_t *__restrict__ n_tleaves,
                                  const int64_t *__restrict__ sleaves,
                                  const int64_t *__restrict__ n_sleaves,
                                  int64_t *__restrict__ out) {
  const int64_t nt = *n_tleaves, ns = *n_sleaves;
  const int n = 1 << levels;
  const int dx = t_index / 9 - 1, dy = (t_index / 3) % 3 - 1, dz = t_index % 3 - 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nt;
       i += int64_t(gridDim.x) * blockDim.x) {
    int cx, cy, cz;
    unmorton3((uint64_t)tleaves[i], cx, cy, cz);
    const int sx = cx + dx, sy = cy + dy, sz = cz + dz;
    int64_t res = -1;
    if (sx >= 0 && sx < n && sy >= 0 && sy < n && sz >= 0 && sz < n) {
      const int64_t id = (int64_t)morton3(sx, sy, sz);
      int64_t lo = 0, hi = ns;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (sleaves[mid] < id) lo = mid + 1; else hi = mid;
      }
      if (lo < ns && sleaves[lo] == id) res = lo;
    }
    out[i] = res;
  }
}

// Near pair count (the "near_pairs" timing entry, engine.py:532).
__global__ void near_count_kernel(const int64_t *__restrict__ tleaves,
                                  const int64_t *__restrict__ tcounts,
                                  const int64_t *__restrict__ n_tleaves,
                                  const int32_t *__restrict__ scell_count,
                                  int levels, unsigned long long *total) {
  const int64_t nt = *n_tleaves;
  const int n = 1 << levels;
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nt;
       i += int64_t(gridDim.x) * blockDim.x) {
    int cx, cy, cz;
    unmorton3((uint64_t)tleaves[i], cx, cy, cz);
    int64_t s = 0;
    for (int nb = 0; nb < 27; ++nb) {
      const int sx = cx + nb / 9 - 1, sy = cy + (nb / 3) % 3 - 1, sz = cz + nb % 3 - 1;
      if (sx < 0 || sx >= n || sy < 0 || sy >= n || sz < 0 || sz >= n) continue;
      s += scell_count[morton3(sx, sy, sz)];
    }
    local += (unsigned long long)(s * tcounts[i]);
  }
  // one atomic per warp (a same-address atomic per thread serialises)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(total, local);
}

// Work of each level-2 subtree for balanced Morton shards: near pairs of its
// target leaves (27-neighbourhood source count x target count) plus one
// unit per target point, summed into 64 bins (leaf >> 3 (levels - 2)).
__global__ void level2_work_kernel(const int64_t *__restrict__ tleaves,
                                   const int64_t *__restrict__ tcounts,
                                   const int64_t *__restrict__ n_tleaves,
                                   const int32_t *__restrict__ scell_count, int levels,
                                   unsigned long long *__restrict__ bins) {
  __shared__ unsigned long long b[64];
  if (threadIdx.x < 64) b[threadIdx.x] = 0;
  __syncthreads();
  const int64_t nt = *n_tleaves;
  const int n = 1 << levels;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nt;
       i += int64_t(gridDim.x) * blockDim.x) {
    int cx, cy, cz;
    unmorton3((uint64_t)tleaves[i], cx, cy, cz);
    int64_t s = 0;
    for (int nb = 0; nb < 27; ++nb) {
      const int sx = cx + nb / 9 - 1, sy = cy + (nb / 3) % 3 - 1, sz = cz + nb % 3 - 1;
      if (sx < 0 || sx >= n || sy < 0 || sy >= n || sz < 0 || sz >= n) continue;
      s += scell_count[morton3(sx, sy, sz)];
    }
    atomicAdd(&b[tleaves[i] >> (3 * (levels - 2))],
              (unsigned long long)((s + 1) * tcounts[i]));
  }
  __syncthreads();
  if (threadIdx.x < 64 && b[threadIdx.x]) atomicAdd(&bins[threadIdx.x], b[threadIdx.x]);
}

// Layout: nch[max_leaves] | incl[max_leaves] | CUB temp | chunk counter
// (256 B) | chunk -> leaf map (int32, room for every chunk of n_targets
// points: at most one partial chunk per leaf plus n/32 full ones; the map is
// used only when the caller's scratch holds all of it).
size_t p2p_fixed(int64_t max_leaves, size_t *cub_off) {
  size_t cub_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, cub_bytes, (int64_t *)nullptr,
                                (int64_t *)nullptr, (int)max_leaves);
  size_t a = ((size_t)max_leaves * 2 * sizeof(int64_t) + 255) & ~size_t(255);
  *cub_off = a;
  return a + ((cub_bytes + 255) & ~size_t(255));
}
size_t p2p_scratch(int64_t max_leaves, size_t *cub_off, int64_t n_targets = 0) {
  const size_t map = n_targets > 0 ? (size_t)(max_leaves + n_targets / 32 + 1) : 0;
  return p2p_fixed(max_leaves, cub_off) + ((map * sizeof(int32_t) + 255) & ~size_t(255)) + 256;
}

bfmm_nf::Args make_args(const double *tpts4, const int64_t *tleaves,
                         const int64_t *tstarts, const int64_t *tcounts,
                         const int64_t *n_tleaves, const double *spts4,
                         const double *sw, int m, const int32_t *scs,
                         const int32_t *scc, int levels, double *out,
                         const int64_t *work) {
  bfmm_nf::Args a;
  a.tpts4 = tpts4;
  a.tleaves = reinterpret_cast<const long long *>(tleaves);
  a.tstarts = reinterpret_cast<const long long *>(tstarts);
  a.tcounts = reinterpret_cast<const long long *>(tcounts);
  a.n_tleaves = reinterpret_cast<const long long *>(n_tleaves);
  a.spts4 = spts4;
  a.sw = sw;
  a.m = m;
  a.scell_start = scs;
  a.scell_count = scc;
  a.levels = levels;
  a.out = out;
  a.work_incl = reinterpret_cast<const long long *>(work);
  a.gate = nullptr;
  a.work_ctr = nullptr;
  a.chunk_leaf = nullptr;
  a.chunk_cap = 0;
  a.wide = m == 1 ? 1 : 0;  // must match chunk_counts_kernel's unit split
  return a;
}

__global__ void too_big_kernel(const int64_t *__restrict__ counts,
                               const int64_t *__restrict__ n_leaves, int limit,
                               int *flag) {
  const int64_t nl = *n_leaves;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nl;
       i += int64_t(gridDim.x) * blockDim.x)
    if (counts[i] > limit) atomicOr(flag, 1);
}

// flag = 0 -> "not too big"; the fallback P2P is gated on flag != 0
int launch_sym(int handle, const bfmm_nf::Args &a, double *slots, int64_t nt,
               double sgn, const int *flag, int64_t lo, int64_t hi, cudaStream_t st) {
  const dim3 grid(kNumSMs * 16), block(32 * bfmm_nf::kWarps);
  const long long sl = (long long)nt;
  switch (handle) {
    case 1: bfmm_nf::p2p_sym_kernel<KLaplace><<<grid, block, 0, st>>>(a, slots, sl, sgn, flag, lo, hi); break;
    case 2: bfmm_nf::p2p_sym_kernel<KLaplaceForce><<<grid, block, 0, st>>>(a, slots, sl, sgn, flag, lo, hi); break;
    case 3: bfmm_nf::p2p_sym_kernel<KGaussian><<<grid, block, 0, st>>>(a, slots, sl, sgn, flag, lo, hi); break;
    case 4: bfmm_nf::p2p_sym_kernel<KExponential><<<grid, block, 0, st>>>(a, slots, sl, sgn, flag, lo, hi); break;
    case 5: bfmm_nf::p2p_sym_kernel<KLogarithm><<<grid, block, 0, st>>>(a, slots, sl, sgn, flag, lo, hi); break;
    default: {
      JitKernel jk;
      {
        std::lock_guard<std::mutex> lock(g_jit_mu);
        if (handle < kFirstJit || handle - kFirstJit >= (int)g_jit.size()) {
          set_error("bfmm_p2p_symmetric: unknown kernel handle %d", handle);
          return 2;
        }
        jk = g_jit[handle - kFirstJit];
      }
      bfmm_nf::Args args = a;
      double *sp = slots;
      long long n = sl, l0 = lo, h0 = hi;
      double sg = sgn;
      const int *fp = flag;
      void *params[] = {&args, &sp, &n, &sg, &fp, &l0, &h0};
      if (driver().LaunchKernel(jk.sym, grid.x, 1, 1, block.x, 1, 1, 0, (CUstream)st,
                                params, nullptr) != CUDA_SUCCESS) {
        set_error("bfmm_p2p_symmetric: cuLaunchKernel failed");
        return 1;
      }
      add_launches(1);
      return 0;
    }
  }
  return check_launch("p2p_sym_kernel");
}

}  // namespace
}  // namespace bfmm

using namespace bfmm;

// leaves of at most this many points take the one-thread-per-target kernel
constexpr int kSmallLeaf = 8;

extern "C" int bfmm_kernel_compile(int kind, const char *expr, int *handle) {
  if (kind < 0 || kind > 2 || !expr || !handle) {
    set_error("bfmm_kernel_compile: bad arguments");
    return 2;
  }
  return jit_compile(kind, expr, handle);
}

// p2p_group_kernel over the leaves of <= small_max points
static int launch_group(int handle, const double *tpts4, const int64_t *tleaves,
                        const int64_t *tstarts, const int64_t *tcounts, const int64_t *n_tleaves,
                        int64_t max_tleaves, const double *spts4, const int32_t *scell_start,
                        const int32_t *scell_count, int levels, int64_t cell_lo, int64_t cell_hi,
                        int small_max, double *out, cudaStream_t st) {
  bfmm_nf::Args a = make_args(tpts4, tleaves, tstarts, tcounts, n_tleaves, spts4, nullptr, 1,
                               scell_start, scell_count, levels, out, nullptr);
  const int64_t warps = ceil_div(max_tleaves, bfmm_nf::kGroupLeaves);
  const dim3 grid((unsigned)std::min<int64_t>(ceil_div(warps, bfmm_nf::kWarps),
                                              (int64_t)kNumSMs * 16)),
      block(32 * bfmm_nf::kWarps);
  const long long lo = cell_lo, hi = cell_hi;
  const int sm = small_max;
  switch (handle) {
    case 1: bfmm_nf::p2p_group_kernel<KLaplace><<<grid, block, 0, st>>>(a, lo, hi, sm); break;
    case 2: bfmm_nf::p2p_group_kernel<KLaplaceForce><<<grid, block, 0, st>>>(a, lo, hi, sm); break;
    case 3: bfmm_nf::p2p_group_kernel<KGaussian><<<grid, block, 0, st>>>(a, lo, hi, sm); break;
    case 4: bfmm_nf::p2p_group_kernel<KExponential><<<grid, block, 0, st>>>(a, lo, hi, sm); break;
    case 5: bfmm_nf::p2p_group_kernel<KLogarithm><<<grid, block, 0, st>>>(a, lo, hi, sm); break;
    default: {
      JitKernel jk;
      {
        std::lock_guard<std::mutex> lock(g_jit_mu);
        if (handle < kFirstJit || handle - kFirstJit >= (int)g_jit.size()) {
          set_error("p2p_group_kernel: unknown kernel handle %d", handle);
          return 2;
        }
        jk = g_jit[handle - kFirstJit];
      }
      bfmm_nf::Args args = a;
      long long l1 = lo, h1 = hi;
      int s1 = sm;
      void *params[] = {&args, &l1, &h1, &s1};
      if (driver().LaunchKernel(jk.group, grid.x, 1, 1, block.x, 1, 1, 0, (CUstream)st, params,
                                nullptr) != CUDA_SUCCESS) {
        set_error("p2p_group_kernel: cuLaunchKernel failed");
        return 1;
      }
      add_launches(1);
      return 0;
    }
  }
  return check_launch("p2p_group_kernel");
}

// p2p_tile_kernel over the target cells of <= small_max points in
// [cell_lo, cell_hi): one CTA per aligned 64-cell Morton block
static int launch_tile(int handle, const double *tpts4, const int32_t *tcell_start,
                       const int32_t *tcell_count, const double *spts4,
                       const int32_t *scell_start, const int32_t *scell_count, int levels,
                       int64_t cell_lo, int64_t cell_hi, int small_max, double *out,
                       cudaStream_t st) {
  // BFMM_TILE_MODE=0 (diagnostic): one thread per target (bitwise equal to
  // p2p_group_kernel); default 1: a warp per target cell
  const char *tm = getenv("BFMM_TILE_MODE");
  const int mode = (tm && tm[0] == '0') ? 0 : 1;
  bfmm_nf::Args a = make_args(tpts4, nullptr, nullptr, nullptr, nullptr, spts4, nullptr, 1,
                               scell_start, scell_count, levels, out, nullptr);
  const int64_t tiles = ceil_div(cell_hi, 64) - cell_lo / 64;
  if (tiles <= 0) return 0;
  static unsigned long long attr = 0;
  (void)attr;
  const dim3 grid((unsigned)std::min<int64_t>(tiles, (int64_t)kNumSMs * 5 * 8)),
      block(bfmm_nf::kTileThreads);
  long long lo = cell_lo, hi = cell_hi;
  int sm = small_max;
  const int *cs = tcell_start, *cc = tcell_count;
#define BFMM_TILE(KK)                                                                     \
  (mode == 1 ? (bfmm_nf::p2p_tile_kernel<KK, 1><<<grid, block, 0, st>>>(a, cs, cc, lo, hi, sm)) \
             : (bfmm_nf::p2p_tile_kernel<KK, 0><<<grid, block, 0, st>>>(a, cs, cc, lo, hi, sm)))
  switch (handle) {
    case 1: BFMM_TILE(KLaplace); break;
    case 2: BFMM_TILE(KLaplaceForce); break;
    case 3: BFMM_TILE(KGaussian); break;
    case 4: BFMM_TILE(KExponential); break;
    case 5: BFMM_TILE(KLogarithm); break;
#undef BFMM_TILE
    default: {
      JitKernel jk;
      {
        std::lock_guard<std::mutex> lock(g_jit_mu);
        if (handle < kFirstJit || handle - kFirstJit >= (int)g_jit.size()) {
          set_error("p2p_tile_kernel: unknown kernel handle %d", handle);
          return 2;
        }
        jk = g_jit[handle - kFirstJit];
      }
      void *params[] = {&a, &cs, &cc, &lo, &hi, &sm};
      if (driver().LaunchKernel(mode == 1 ? jk.tile1 : jk.tile, grid.x, 1, 1, block.x, 1, 1, 0, (CUstream)st, params,
                                nullptr) != CUDA_SUCCESS) {
        set_error("p2p_tile_kernel: cuLaunchKernel failed");
        return 1;
      }
      add_launches(1);
      return 0;
    }
  }
  return check_launch("p2p_tile_kernel");
}

extern "C" size_t bfmm_p2p_scratch_bytes(int64_t max_tleaves, int64_t n_targets) {
  size_t off;
  return p2p_scratch(max_tleaves < 1 ? 1 : max_tleaves, &off, n_targets);
}

static int p2p_impl(int handle, const double *tpts4, const int64_t *tleaves,
                    const int64_t *tstarts, const int64_t *tcounts,
                    const int64_t *n_tleaves, int64_t max_tleaves,
                    const int32_t *tcell_start, const int32_t *tcell_count,
                    const double *spts4, const double *swsorted, int m,
                    const int32_t *scell_start, const int32_t *scell_count,
                    int levels, int64_t cell_lo, int64_t cell_hi,
                    double *out, void *scratch, size_t scratch_bytes,
                    bfmm_stream_t stream) {
  if (max_tleaves <= 0) return 0;
  size_t cub_off;
  const size_t fixed = p2p_fixed(max_tleaves, &cub_off);
  size_t need = p2p_scratch(max_tleaves, &cub_off);
  if (scratch_bytes < need) {
    set_error("bfmm_p2p: scratch too small (%zu < %zu)", scratch_bytes, need);
    return 2;
  }
  // chunk map capacity: whatever the caller's scratch holds between the
  // fixed part and the counter (bfmm_p2p_scratch_bytes sizes it for n)
  const int64_t map_cap = (int64_t)((scratch_bytes - 256 - fixed) / sizeof(int32_t));
  auto *ctr = reinterpret_cast<unsigned long long *>(static_cast<char *>(scratch) + fixed);
  int32_t *chunk_leaf = reinterpret_cast<int32_t *>(static_cast<char *>(scratch) + fixed + 256);
  cudaStream_t st = as_stream(stream);
  int64_t *nch = static_cast<int64_t *>(scratch);
  int64_t *incl = nch + max_tleaves;
  chunk_counts_kernel<<<(unsigned)std::min<int64_t>(ceil_div(max_tleaves, 256),
                                                    kNumSMs * 16),
                        256, 0, st>>>(tcounts, tleaves, n_tleaves, max_tleaves,
                                      cell_lo, cell_hi, m == 1 ? kSmallLeaf : 0, m == 1 ? 1 : 0,
                                      nch);
  if (check_launch("chunk_counts_kernel")) return 1;
  if (m == 1) {
    // one weight column: leaves of <= kSmallLeaf points (sparse clouds: C5's
    // 3.8 per leaf, C4's sphere shell) run one thread per target
    // (p2p_group_kernel); the 32-target chunks below cover the rest
    // (tiled through shared memory when the target cell map is given)
    if (int rc = tcell_start
                     ? launch_tile(handle, tpts4, tcell_start, tcell_count, spts4, scell_start,
                                   scell_count, levels, cell_lo, cell_hi, kSmallLeaf, out, st)
                     : launch_group(handle, tpts4, tleaves, tstarts, tcounts, n_tleaves,
                                    max_tleaves, spts4, scell_start, scell_count, levels, cell_lo,
                                    cell_hi, kSmallLeaf, out, st))
      return rc;
  }
  size_t cb = fixed - cub_off;
  if (cub::DeviceScan::InclusiveSum(static_cast<char *>(scratch) + cub_off, cb,
                                    nch, incl, (int)max_tleaves,
                                    st) != cudaSuccess) {
    set_error("bfmm_p2p: scan failed");
    return 1;
  }
  add_launches(2);  // CUB scan: init + scan
  bfmm_nf::Args a = make_args(tpts4, tleaves, tstarts, tcounts, n_tleaves,
                               spts4, swsorted, m, scell_start, scell_count,
                               levels, out, incl);
  a.work_ctr = ctr;
  if (map_cap > 0) {
    chunk_map_kernel<<<(unsigned)std::min<int64_t>(ceil_div(max_tleaves, 256), kNumSMs * 16),
                       256, 0, st>>>(incl, n_tleaves, max_tleaves, map_cap, chunk_leaf);
    if (check_launch("chunk_map_kernel")) return 1;
    a.chunk_leaf = chunk_leaf;
    a.chunk_cap = map_cap;
  }
  // 16 CTAs per SM (more than fit): every resident warp claims chunks from
  // the counter until they run out, CTAs that start later find none
  dim3 grid(kNumSMs * 16);
  int c0 = 0;
  while (c0 < m) {
    const int left = m - c0;
    int mci = 0;
    if (m == 1) mci = 0;
    else if (left >= 16) mci = 4;
    else if (left >= 8) mci = 3;
    else if (left >= 4) mci = 2;
    else if (left >= 2) mci = 1;
    else mci = 0;
    if (cudaMemsetAsync(ctr, 0, sizeof(*ctr), st) != cudaSuccess) {
      set_error("bfmm_p2p: counter reset failed");
      return 1;
    }
    int rc = launch_p2p(handle, mci, grid, a, c0, st);
    if (rc) return rc;
    c0 += kMCs[mci];
  }
  return 0;
}

extern "C" int bfmm_p2p(int handle, const double *tpts4, const int64_t *tleaves,
                        const int64_t *tstarts, const int64_t *tcounts,
                        const int64_t *n_tleaves, int64_t max_tleaves,
                        const double *spts4, const double *swsorted, int m,
                        const int32_t *scell_start, const int32_t *scell_count,
                        int levels, int64_t cell_lo, int64_t cell_hi,
                        double *out, void *scratch, size_t scratch_bytes,
                        bfmm_stream_t stream) {
  return p2p_impl(handle, tpts4, tleaves, tstarts, tcounts, n_tleaves, max_tleaves, nullptr,
                  nullptr, spts4, swsorted, m, scell_start, scell_count, levels, cell_lo, cell_hi,
                  out, scratch, scratch_bytes, stream);
}

extern "C" int bfmm_p2p_cells(int handle, const double *tpts4, const int64_t *tleaves,
                              const int64_t *tstarts, const int64_t *tcounts,
                              const int64_t *n_tleaves, int64_t max_tleaves,
                              const int32_t *tcell_start, const int32_t *tcell_count,
                              const double *spts4, const double *swsorted, int m,
                              const int32_t *scell_start, const int32_t *scell_count,
                              int levels, int64_t cell_lo, int64_t cell_hi, double *out,
                              void *scratch, size_t scratch_bytes, bfmm_stream_t stream) {
  if (!tcell_start || !tcell_count) {
    set_error("bfmm_p2p_cells: target cell map required");
    return 2;
  }
  return p2p_impl(handle, tpts4, tleaves, tstarts, tcounts, n_tleaves, max_tleaves, tcell_start,
                  tcell_count, spts4, swsorted, m, scell_start, scell_count, levels, cell_lo,
                  cell_hi, out, scratch, scratch_bytes, stream);
}

// Near field for sparse clouds (p2p_group_kernel): one weight column, one
// lane per target, kGroupLeaves leaves per warp, leaves of <= small_max
// points only.
extern "C" int bfmm_p2p_grouped(int handle, const double *tpts4, const int64_t *tleaves,
                                const int64_t *tstarts, const int64_t *tcounts,
                                const int64_t *n_tleaves, int64_t max_tleaves,
                                const double *spts4, const int32_t *scell_start,
                                const int32_t *scell_count, int levels, int64_t cell_lo,
                                int64_t cell_hi, double *out, bfmm_stream_t stream) {
  if (max_tleaves <= 0) return 0;
  return launch_group(handle, tpts4, tleaves, tstarts, tcounts, n_tleaves, max_tleaves, spts4,
                      scell_start, scell_count, levels, cell_lo, cell_hi, 1 << 30, out,
                      as_stream(stream));
}

extern "C" int bfmm_p2p_locate(int handle, const double *tpts4,
                               const int64_t *tleaves, const int64_t *tstarts,
                               const int64_t *tcounts, const int64_t *n_tleaves,
                               int64_t max_tleaves, const double *spts4,
                               const int32_t *scell_start,
                               const int32_t *scell_count, int levels,
                               unsigned long long *key, bfmm_stream_t stream) {
  if (max_tleaves <= 0) return 0;
  bfmm_nf::Args a = make_args(tpts4, tleaves, tstarts, tcounts, n_tleaves,
                               spts4, nullptr, 1, scell_start, scell_count,
                               levels, nullptr, nullptr);
  return launch_locate(handle, a, key, as_stream(stream));
}

extern "C" int bfmm_near_pairs(int levels, int t_index, const int64_t *tleaves,
                               const int64_t *n_tleaves, int64_t max_tleaves,
                               const int64_t *sleaves, const int64_t *n_sleaves,
                               int64_t *out, bfmm_stream_t stream) {
  if (t_index < 0 || t_index >= 27) {
    set_error("bfmm_near_pairs: offset index %d outside [0, 27)", t_index);
    return 2;
  }
  if (max_tleaves <= 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(max_tleaves, 256), 4096);
  near_pairs_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      levels, t_index, tleaves, n_tleaves, sleaves, n_sleaves, out);
  return check_launch("near_pairs_kernel");
}

extern "C" int bfmm_near_pair_count(const int64_t *tleaves,
                                    const int64_t *tcounts,
                                    const int64_t *n_tleaves,
                                    int64_t max_tleaves,
                                    const int32_t *scell_count, int levels,
                                    int64_t *total, bfmm_stream_t stream) {
  cudaStream_t st = as_stream(stream);
  if (cudaMemsetAsync(total, 0, sizeof(int64_t), st) != cudaSuccess) {
    set_error("bfmm_near_pair_count: memset failed");
    return 1;
  }
  if (max_tleaves <= 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(max_tleaves, 256), 1024);
  near_count_kernel<<<grid, 256, 0, st>>>(tleaves, tcounts, n_tleaves,
                                          scell_count, levels,
                                          reinterpret_cast<unsigned long long *>(total));
  return check_launch("near_count_kernel");
}

extern "C" int bfmm_scatter_output(const double *far_sorted,
                                   const double *near_sorted,
                                   const int64_t *perm, int64_t n, int m,
                                   double *phi, int32_t *nonfinite_flag,
                                   bfmm_stream_t stream) {
  if (n == 0) return 0;
  const int64_t total = n * m;
  unsigned grid = (unsigned)std::min<int64_t>(ceil_div(total, 256), kNumSMs * 32);
  scatter_kernel<<<grid, 256, 0, as_stream(stream)>>>(far_sorted, near_sorted,
                                                      perm, n, m, phi,
                                                      nonfinite_flag);
  return check_launch("scatter_kernel");
}

extern "C" size_t bfmm_p2p_symmetric_scratch_bytes(int64_t nt, int64_t max_tleaves) {
  size_t off;
  const size_t chunk = (p2p_scratch(max_tleaves < 1 ? 1 : max_tleaves, &off) + 255) & ~size_t(255);
  return chunk + ((14 * (size_t)(nt < 1 ? 1 : nt) * sizeof(double) + 255) & ~size_t(255)) + 512;
}

extern "C" int bfmm_p2p_symmetric(int handle, const double *pts4,
                                  const int64_t *leaves, const int64_t *starts,
                                  const int64_t *counts, const int64_t *n_leaves,
                                  int64_t max_leaves, const int32_t *cell_start,
                                  const int32_t *cell_count, int levels,
                                  int64_t cell_lo, int64_t cell_hi, int64_t nt,
                                  double sign, double *out, void *scratch,
                                  size_t scratch_bytes, bfmm_stream_t stream) {
  if (max_leaves <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  size_t cub_off;
  const size_t chunk = (p2p_scratch(max_leaves, &cub_off) + 255) & ~size_t(255);
  const size_t slot_bytes = (14 * (size_t)nt * sizeof(double) + 255) & ~size_t(255);
  if (scratch_bytes < chunk + slot_bytes + 512) {
    set_error("bfmm_p2p_symmetric: scratch too small");
    return 2;
  }
  char *base = static_cast<char *>(scratch);
  double *slots = reinterpret_cast<double *>(base + chunk);
  int *flag = reinterpret_cast<int *>(base + chunk + slot_bytes);
  auto *ctr = reinterpret_cast<unsigned long long *>(base + chunk + slot_bytes + 256);
  if (cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess ||
      cudaMemsetAsync(ctr, 0, sizeof(*ctr), st) != cudaSuccess ||
      cudaMemsetAsync(slots, 0, 14 * (size_t)nt * sizeof(double), st) != cudaSuccess) {
    set_error("bfmm_p2p_symmetric: memset failed");
    return 1;
  }
  const unsigned g1 = (unsigned)std::min<int64_t>(ceil_div(max_leaves, 256), kNumSMs * 8);
  too_big_kernel<<<g1, 256, 0, st>>>(counts, n_leaves, bfmm_nf::kSymMax, flag);
  if (check_launch("too_big_kernel")) return 1;
  // fallback work list + gated plain P2P (runs only when a leaf is too big)
  int64_t *nch = reinterpret_cast<int64_t *>(base);
  int64_t *incl = nch + max_leaves;
  chunk_counts_kernel<<<(unsigned)std::min<int64_t>(ceil_div(max_leaves, 256), kNumSMs * 16),
                        256, 0, st>>>(counts, leaves, n_leaves, max_leaves, cell_lo, cell_hi,
                                      0, 1, nch);
  if (check_launch("chunk_counts_kernel")) return 1;
  size_t cb = chunk - cub_off;
  if (cub::DeviceScan::InclusiveSum(base + cub_off, cb, nch, incl, (int)max_leaves, st) !=
      cudaSuccess) {
    set_error("bfmm_p2p_symmetric: scan failed");
    return 1;
  }
  add_launches(2);
  bfmm_nf::Args a = make_args(pts4, leaves, starts, counts, n_leaves, pts4, nullptr, 1,
                              cell_start, cell_count, levels, out, incl);
  a.work_ctr = ctr;
  int rc = launch_sym(handle, a, slots, nt, sign, flag, cell_lo, cell_hi, st);
  if (rc) return rc;
  a.work_ctr = nullptr;
  a.gate = flag;
  rc = launch_p2p(handle, 0, dim3(kNumSMs * 16), a, 0, st);
  if (rc) return rc;
  const unsigned g2 = (unsigned)std::min<int64_t>(ceil_div(nt, 256), kNumSMs * 16);
  bfmm_nf::sym_reduce_kernel<<<g2, 256, 0, st>>>(slots, (long long)nt, out, flag);
  return check_launch("sym_reduce_kernel");
}

// ---- direct sum (engine.py:565-624) -------------------------------------------
extern "C" int bfmm_direct(int handle, const double *tpts, int64_t nt,
                           const double *spts, const double *sw, int64_t ns, int m,
                           double *out, bfmm_stream_t stream) {
  if (nt <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  const dim3 grid((unsigned)ceil_div(nt, 128)), block(128);
  const long long lnt = nt, lns = ns;
  for (int c0 = 0; c0 < m; c0 += 4) {
    switch (handle) {
      case 1: bfmm_nf::direct_kernel<KLaplace><<<grid, block, 0, st>>>(tpts, lnt, spts, sw, lns, m, c0, out); break;
      case 2: bfmm_nf::direct_kernel<KLaplaceForce><<<grid, block, 0, st>>>(tpts, lnt, spts, sw, lns, m, c0, out); break;
      case 3: bfmm_nf::direct_kernel<KGaussian><<<grid, block, 0, st>>>(tpts, lnt, spts, sw, lns, m, c0, out); break;
      case 4: bfmm_nf::direct_kernel<KExponential><<<grid, block, 0, st>>>(tpts, lnt, spts, sw, lns, m, c0, out); break;
      case 5: bfmm_nf::direct_kernel<KLogarithm><<<grid, block, 0, st>>>(tpts, lnt, spts, sw, lns, m, c0, out); break;
      default: {
        JitKernel jk;
        {
          std::lock_guard<std::mutex> lock(g_jit_mu);
          if (handle < kFirstJit || handle - kFirstJit >= (int)g_jit.size()) {
            set_error("bfmm_direct: unknown kernel handle %d", handle);
            return 2;
          }
          jk = g_jit[handle - kFirstJit];
        }
        const double *tp = tpts, *sp = spts, *wp = sw;
        double *op = out;
        long long a1 = lnt, a2 = lns;
        int mm = m, cc = c0;
        void *params[] = {&tp, &a1, &sp, &wp, &a2, &mm, &cc, &op};
        if (driver().LaunchKernel(jk.direct, grid.x, 1, 1, block.x, 1, 1, 0, (CUstream)st,
                                  params, nullptr) != CUDA_SUCCESS) {
          set_error("bfmm_direct: cuLaunchKernel failed");
          return 1;
        }
        add_launches(1);
        continue;
      }
    }
    if (check_launch("direct_kernel")) return 1;
  }
  return 0;
}

// ---- kernel values on pair grids (M2L table build, operators.py:88-108, 244-258)
extern "C" int bfmm_kernel_block(int handle, const double *xt, int64_t na, const double *ys,
                                 int64_t nb, const double *shift, int nt, double *out,
                                 int32_t *bad, bfmm_stream_t stream) {
  if (na <= 0 || nb <= 0 || nt <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  const int64_t total = na * nb * (int64_t)nt;
  const dim3 grid((unsigned)std::min<int64_t>(ceil_div(total, 256), kNumSMs * 32)), block(256);
  const long long a1 = na, a2 = nb;
  int *bp = reinterpret_cast<int *>(bad);
  switch (handle) {
    case 1: bfmm_nf::pair_block_kernel<KLaplace><<<grid, block, 0, st>>>(xt, a1, ys, a2, shift, nt, out, bp); break;
    case 2: bfmm_nf::pair_block_kernel<KLaplaceForce><<<grid, block, 0, st>>>(xt, a1, ys, a2, shift, nt, out, bp); break;
    case 3: bfmm_nf::pair_block_kernel<KGaussian><<<grid, block, 0, st>>>(xt, a1, ys, a2, shift, nt, out, bp); break;
    case 4: bfmm_nf::pair_block_kernel<KExponential><<<grid, block, 0, st>>>(xt, a1, ys, a2, shift, nt, out, bp); break;
    case 5: bfmm_nf::pair_block_kernel<KLogarithm><<<grid, block, 0, st>>>(xt, a1, ys, a2, shift, nt, out, bp); break;
    default: {
      JitKernel jk;
      {
        std::lock_guard<std::mutex> lock(g_jit_mu);
        if (handle < kFirstJit || handle - kFirstJit >= (int)g_jit.size()) {
          set_error("bfmm_kernel_block: unknown kernel handle %d", handle);
          return 2;
        }
        jk = g_jit[handle - kFirstJit];
      }
      const double *x = xt, *y = ys, *s = shift;
      long long b1 = a1, b2 = a2;
      int t = nt;
      double *o = out;
      void *params[] = {&x, &b1, &y, &b2, &s, &t, &o, &bp};
      if (driver().LaunchKernel(jk.block, grid.x, 1, 1, block.x, 1, 1, 0, (CUstream)st, params,
                                nullptr) != CUDA_SUCCESS) {
        set_error("bfmm_kernel_block: cuLaunchKernel failed");
        return 1;
      }
      add_launches(1);
      return 0;
    }
  }
  return check_launch("pair_block_kernel");
}

extern "C" int bfmm_level2_work(const int64_t *tleaves, const int64_t *tcounts,
                                const int64_t *n_tleaves, int64_t max_tleaves,
                                const int32_t *scell_count, int levels, int64_t *bins,
                                bfmm_stream_t stream) {
  if (levels < 2) {
    set_error("bfmm_level2_work: levels %d < 2", levels);
    return 2;
  }
  cudaStream_t st = as_stream(stream);
  if (cudaMemsetAsync(bins, 0, 64 * sizeof(int64_t), st) != cudaSuccess) {
    set_error("bfmm_level2_work: memset failed");
    return 1;
  }
  if (max_tleaves <= 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(max_tleaves, 256), kNumSMs * 4);
  level2_work_kernel<<<grid, 256, 0, st>>>(tleaves, tcounts, n_tleaves, scell_count, levels,
                                           reinterpret_cast<unsigned long long *>(bins));
  return check_launch("level2_work_kernel");
}
