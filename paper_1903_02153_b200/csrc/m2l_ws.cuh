// Warp-specialised implicit-GEMM M2L (included by m2l_cheb.cu).
//
// Same contraction as m2l_dmma.cuh, but no CTA-wide barrier per k-step:
//  * warp kConsumers (the last warp) is the producer: it gathers the z rows
//    and the core tile of each (offset, 8-wide rank group) step into one of
//    kS shared stages with cp.async, and signals the stage's "full" mbarrier
//    through cp.async.mbarrier.arrive (completion-tracked);
//  * the 8 consumer warps wait on "full", run the DMMAs, and arrive on the
//    stage's "empty" mbarrier; the producer waits on "empty" before refilling.
// Consumer warps thus drift independently by up to kS steps, which keeps the
// FP64 tensor pipe busy across step boundaries.
#pragma once

constexpr int kWsConsumers = 8, kWsStages = 8;

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_cp_async_arrive(uint64_t *bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

template <int NT8, int MW>
struct WsShape {
  static constexpr int TM = 8 * MW * kWsConsumers;
  static constexpr int TN = 8 * NT8;
  static constexpr int LDK = 8;  // one rank group (8 doubles) per step
  static constexpr int stage_elems = (TM + TN) * LDK;
  static constexpr size_t smem =
      sizeof(double) * kWsStages * stage_elems + 2 * kWsStages * sizeof(uint64_t);
  static constexpr int threads = 32 * (kWsConsumers + 1);
};

// Octant-grouped active target cells: cells[off[o] .. off[o + 1]) are the
// listed cells with (cell & 7) == o.
struct OctList {
  const int64_t *cells;
  int64_t off[9];
};

template <int NT8, int MW>
__global__ void __launch_bounds__(WsShape<NT8, MW>::threads, 2)
m2l_ws_kernel(const double *__restrict__ z, double *__restrict__ lt, int level,
              int m, int rp, int nsplit, int64_t q_lo, int64_t nq, OctList act,
              const double *__restrict__ cores) {
  using S = WsShape<NT8, MW>;
  constexpr int TM = S::TM, TNc = S::TN, LDK = S::LDK;
  extern __shared__ __align__(16) double sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + kWsStages * S::stage_elems);
  uint64_t *empty = full + kWsStages;
  const int o = blockIdx.z & 7;
  const int split = blockIdx.z >> 3;
  const int per = (189 + nsplit - 1) / nsplit;
  const int v_lo = split * per, v_hi = min(189, v_lo + per);
  const int n = 1 << level;
  // rows: (index q, column) of the octant-o target cells, either the children
  // 8 (q_lo + q) + o of a dense parent range (lt rows absolute), or the listed
  // active cells act.cells[act.off[o] + q] (lt rows compact, in list order)
  const int64_t *ocells = act.cells ? act.cells + act.off[o] : nullptr;
  const int64_t rows = (act.cells ? act.off[o + 1] - act.off[o] : nq) * m;
  const int64_t row0 = int64_t(blockIdx.x) * TM;
  if (row0 >= rows) return;  // octant lists differ in length (whole CTA)
  const int n0 = blockIdx.y * TNc;
  const int groups = rp >> 3;
  const int nsteps = (v_hi - v_lo) * groups;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(&full[s], 32);            // every producer lane arrives once
      mbar_init(&empty[s], kWsConsumers); // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kWsConsumers) {
    // ---------------- producer warp ----------------
    constexpr int RPL = TM / 32;  // A rows per lane
    int cx[RPL], cy[RPL], cz[RPL], colm[RPL];
    bool rok[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int64_t r = row0 + lane + 32 * i;
      rok[i] = r < rows;
      cx[i] = cy[i] = cz[i] = colm[i] = 0;
      if (rok[i]) {
        const int64_t q = r / m;
        colm[i] = (int)(r - q * m);
        const int64_t cell = ocells ? ocells[q] : 8 * (q_lo + q) + o;
        unmorton3((uint64_t)cell, cx[i], cy[i], cz[i]);
      }
    }
    int64_t srow[RPL];
    int vi = v_lo, grp = 0;
    for (int step = 0; step < nsteps; ++step) {
      const int s = step % kWsStages;
      if (step >= kWsStages) mbar_wait(&empty[s], ((step / kWsStages) - 1) & 1);
      double *As = sm + s * S::stage_elems;
      double *Bs = As + TM * LDK;
      const int t = c_valid[o][vi];
      if (grp == 0) {
        const int t0 = c_offsets[t][0], t1 = c_offsets[t][1], t2 = c_offsets[t][2];
#pragma unroll
        for (int i = 0; i < RPL; ++i)
          srow[i] = (rok[i] && far_pair(n, cx[i], cy[i], cz[i], t0, t1, t2))
                        ? ((int64_t)morton3(cx[i] + t0, cy[i] + t1, cz[i] + t2) * m +
                           colm[i]) * rp
                        : -1;
      }
      const int k0 = 8 * grp;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = lane + 32 * i;
        const bool v = srow[i] >= 0;
        const double *src = v ? z + srow[i] + k0 : z;
#pragma unroll
        for (int pc = 0; pc < 4; ++pc)
          cp_async16(As + r * LDK + 2 * (pc ^ ((r & 1) << 1)), src + 2 * pc, v);
      }
      const double *bt = cores + ((int64_t)t * rp + n0) * rp + k0;
#pragma unroll
      for (int e = lane; e < TNc * 4; e += 32) {
        const int r = e >> 2, pc = e & 3;
        const bool v = n0 + r < rp;
        cp_async16(Bs + r * LDK + 2 * (pc ^ ((r & 1) << 1)),
                   v ? bt + (int64_t)r * rp + 2 * pc : cores, v);
      }
      mbar_cp_async_arrive(&full[s]);
      if (++grp == groups) {
        grp = 0;
        ++vi;
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int g = lane >> 2, t4 = lane & 3;
  double acc[MW][NT8][2];
#pragma unroll
  for (int i = 0; i < MW; ++i)
#pragma unroll
    for (int j = 0; j < NT8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // rows are 64 B (4 pieces); odd rows XOR the piece by 2 so the two rows of
  // an 8-lane LDS.128 phase land in disjoint banks
  const int off = 2 * (t4 ^ ((g & 1) << 1));
  for (int step = 0; step < nsteps; ++step) {
    const int s = step % kWsStages;
    mbar_wait(&full[s], (step / kWsStages) & 1);
    const double *As = sm + s * S::stage_elems;
    const double *Bs = As + TM * LDK;
    const double *Aw = As + (warp * 8 * MW + g) * LDK + off;
    const double *Bw = Bs + g * LDK + off;
    double2 a[MW], b[NT8];
#pragma unroll
    for (int i = 0; i < MW; ++i) a[i] = *reinterpret_cast<const double2 *>(Aw + i * 8 * LDK);
#pragma unroll
    for (int j = 0; j < NT8; ++j) b[j] = *reinterpret_cast<const double2 *>(Bw + j * 8 * LDK);
    // both k4 halves of the step: all MW x NT8 accumulators with the first,
    // then all with the second, so consecutive DMMAs on one accumulator are
    // MW * NT8 instructions apart (back-to-back pairs stall on its latency)
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
      for (int i = 0; i < MW; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
      for (int i = 0; i < MW; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int i = 0; i < MW; ++i) {
    const int64_t r = row0 + warp * 8 * MW + i * 8 + g;
    if (r >= rows) continue;
    const int64_t q = r / m;
    const int c = (int)(r - q * m);
    const int64_t orow = ocells ? act.off[o] + q : 8 * (q_lo + q) + o;
    double *dst = lt + ((orow * m + c) * nsplit + split) * rp;
#pragma unroll
    for (int j = 0; j < NT8; ++j) {
      const int col = n0 + j * 8 + 2 * t4;
      if (col < rp)
        *reinterpret_cast<double2 *>(dst + col) =
            make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

struct M2LCall {
  const double *z;
  double *lt;
  int level, m, rp, nsplit;
  int64_t q_lo, nq;  // target parents [q_lo, q_lo + nq) at level - 1
  OctList act;       // or: listed active cells (act.cells != nullptr)
  const double *cores;
  cudaStream_t st;
};

template <int NT8, int MW>
int launch_ws(const M2LCall &a) {
  using S = WsShape<NT8, MW>;
  static unsigned long long attr_set = 0;
  if (first_on_device(&attr_set)) {
    cudaFuncSetAttribute(m2l_ws_kernel<NT8, MW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::smem);
  }
  int64_t rows = a.nq * a.m;
  if (a.act.cells) {  // the longest octant list sizes the grid
    rows = 0;
    for (int o = 0; o < 8; ++o) rows = std::max(rows, (a.act.off[o + 1] - a.act.off[o]) * a.m);
  }
  if (rows <= 0) return 0;
  dim3 grid((unsigned)ceil_div(rows, S::TM), (unsigned)ceil_div(a.rp, S::TN), 8 * a.nsplit);
  m2l_ws_kernel<NT8, MW><<<grid, S::threads, S::smem, a.st>>>(
      a.z, a.lt, a.level, a.m, a.rp, a.nsplit, a.q_lo, a.nq, a.act, a.cores);
  return check_launch("m2l_ws_kernel");
}

template <int MW>
int dispatch_ws_nt8(int nt8, const M2LCall &a) {
  switch (nt8) {
    case 1: return launch_ws<1, MW>(a);
    case 2: return launch_ws<2, MW>(a);
    case 3: return launch_ws<3, MW>(a);
    case 4: return launch_ws<4, MW>(a);
    case 5: return launch_ws<5, MW>(a);
    case 6: return launch_ws<6, MW>(a);
    case 7: return launch_ws<7, MW>(a);
    default: return launch_ws<8, MW>(a);
  }
}

// Column-tile width: the whole rank when rp <= 64, else 56- or 64-wide
// tiles, whichever pads less.  Row tiles: 128 rows, or 64 on tiny levels.
inline int m2l_nt8(int rp) {
  if (rp <= 64) return rp / 8;
  const int w7 = (int)(ceil_div(rp, 56) * 56 - rp), w8 = (int)(ceil_div(rp, 64) * 64 - rp);
  return w7 < w8 ? 7 : 8;
}
inline int m2l_mw(int64_t rows) { return rows <= 64 ? 1 : 2; }

inline int dispatch_ws(int mw, int nt8, const M2LCall &a) {
  if (mw == 1) return dispatch_ws_nt8<1>(nt8, a);
  return dispatch_ws_nt8<2>(nt8, a);
}
