// Implicit-GEMM M2L on the FP64 tensor cores (included by m2l_cheb.cu).
//
// CTA: 8 warps, each owning MW m8 row tiles (8*MW rows) x TN = 8*NT8 columns,
// i.e. MW*NT8 independent m8n8k4 accumulator chains per warp.  K advances
// over (valid offset, k-chunk) steps through a 2-stage cp.async ring; a
// chunk is G groups of 8 rank indices (compile time, so the inner loop is
// fully unrolled and branch free; a chunk past rp is zero-filled).
//
// Rank-index interleave: inside every group of 8, rank index k is stored at
// position 2*(k%4) + (k/4)%2 in BOTH z and the cores (the host permutes V's
// columns and the cores' k index identically; the contraction over k is
// unchanged).  Lane t4 of an m8n8k4 fragment then finds its k of two
// consecutive k4 steps side by side and loads both with one LDS.128.
#pragma once

constexpr int kM2LWarps = 8, kStages = 2;

template <int NT8, int MW, int G>
struct M2LShape {
  static constexpr int TM = 8 * MW * kM2LWarps;
  static constexpr int TN = 8 * NT8;
  static constexpr int LDK = 8 * G;  // doubles per shared row
  static constexpr int stage_elems = (TM + TN) * LDK;
  static constexpr size_t smem = sizeof(double) * kStages * stage_elems;
  // two CTAs per SM when both fit in the 228 KB of shared memory
  static constexpr int min_blocks = smem <= 112 * 1024 ? 2 : 1;
  // with an even G rows are 128 B multiples, so odd rows XOR their 16 B
  // piece index by 4 to keep each 8-lane LDS.128 phase conflict free
  static constexpr int swz_mask = (G % 2 == 0) ? 4 : 0;
};

// grid: (row tiles, column tiles, 8 octants x nsplit offset ranges).  Split
// s accumulates the valid offsets [s*per, (s+1)*per) and writes column block
// s of lt (layout (cells, m, nsplit, rp)); the U projection then sums the
// blocks in a fixed order, so results stay deterministic.
template <int NT8, int MW, int G>
__global__ void __launch_bounds__(32 * kM2LWarps, (M2LShape<NT8, MW, G>::min_blocks))
m2l_dmma_kernel(const double *__restrict__ z, double *__restrict__ lt,
                int level, int m, int rp, int nchunks, int nsplit,
                const double *__restrict__ cores) {
  using S = M2LShape<NT8, MW, G>;
  constexpr int TM = S::TM, TNc = S::TN, LDK = S::LDK;
  constexpr int pieces = 4 * G;  // 16-byte pieces per row chunk
  constexpr int kT = 32 * kM2LWarps;
  constexpr int tpr = kT / TM;  // loader threads per A row
  extern __shared__ __align__(16) double sm[];
  const int o = blockIdx.z & 7;
  const int split = blockIdx.z >> 3;
  const int per = (189 + nsplit - 1) / nsplit;
  const int v_lo = split * per, v_hi = min(189, v_lo + per);
  const int n = 1 << level;
  const int64_t rows = (int64_t(1) << (3 * level - 3)) * m;
  const int64_t row0 = int64_t(blockIdx.x) * TM;
  const int n0 = blockIdx.y * TNc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;

  // A loader: thread -> (row tid % TM, pieces tid / TM + k * tpr)
  const int a_row = tid % TM, a_p0 = tid / TM;
  const int a_swz = (a_row & 1) ? S::swz_mask : 0;
  const int64_t my_row = row0 + a_row;
  int cx = 0, cy = 0, cz = 0, colm = 0;
  const bool row_ok = my_row < rows;
  if (row_ok) {
    const int64_t q = my_row / m;
    colm = (int)(my_row - q * m);
    unmorton3((uint64_t)(8 * q + o), cx, cy, cz);
  }
  const int nsteps = (v_hi - v_lo) * nchunks;

  // producer position: (valid-offset index, chunk), advanced incrementally
  int p_vi = v_lo, p_ch = 0, p_slot = 0;
  auto issue_next = [&]() {
    double *As = sm + p_slot * S::stage_elems;
    double *Bs = As + TM * LDK;
    const int t = c_valid[o][p_vi];
    const int k0 = p_ch * 8 * G;
    const int t0 = c_offsets[t][0], t1 = c_offsets[t][1], t2 = c_offsets[t][2];
    const bool ok = row_ok && far_pair(n, cx, cy, cz, t0, t1, t2);
    const double *src =
        ok ? z + ((int64_t)morton3(cx + t0, cy + t1, cz + t2) * m + colm) * rp + k0
           : z;
    const int live = rp - k0;  // doubles of this row chunk inside rp
#pragma unroll
    for (int pc = a_p0; pc < pieces; pc += tpr) {
      const bool v = ok && 2 * pc < live;
      cp_async16(As + a_row * LDK + 2 * (pc ^ a_swz), v ? src + 2 * pc : z, v);
    }
    const double *bt = cores + ((int64_t)t * rp + n0) * rp + k0;
#pragma unroll
    for (int e = tid; e < TNc * pieces; e += kT) {
      const int r = e / pieces, pc = e - r * pieces;
      const bool v = (n0 + r < rp) && 2 * pc < live;
      const int sw = (r & 1) ? S::swz_mask : 0;
      cp_async16(Bs + r * LDK + 2 * (pc ^ sw), v ? bt + (int64_t)r * rp + 2 * pc : cores,
                 v);
    }
    if (++p_ch == nchunks) {
      p_ch = 0;
      ++p_vi;
    }
    p_slot ^= 1;
  };

  double acc[MW][NT8][2];
#pragma unroll
  for (int i = 0; i < MW; ++i)
#pragma unroll
    for (int j = 0; j < NT8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // fragment rows all have the parity of g, so the swizzle is per lane
  const int lane_swz = (g & 1) ? S::swz_mask : 0;
  if (nsteps > 0) issue_next();
  cp_async_commit();
  for (int step = 0; step < nsteps; ++step) {
    cp_async_wait<0>();
    __syncthreads();
    if (step + 1 < nsteps) issue_next();
    cp_async_commit();
    const double *As = sm + (step & 1) * S::stage_elems;
    const double *Bs = As + TM * LDK;
    const double *Aw = As + (warp * 8 * MW + g) * LDK;
    const double *Bw = Bs + g * LDK;
#pragma unroll
    for (int k8 = 0; k8 < G; ++k8) {
      const int off = 2 * ((4 * k8 + t4) ^ lane_swz);
      double2 a[MW], b[NT8];
#pragma unroll
      for (int i = 0; i < MW; ++i)
        a[i] = *reinterpret_cast<const double2 *>(Aw + i * 8 * LDK + off);
#pragma unroll
      for (int j = 0; j < NT8; ++j)
        b[j] = *reinterpret_cast<const double2 *>(Bw + j * 8 * LDK + off);
#pragma unroll
      for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int i = 0; i < MW; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
#pragma unroll
      for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int i = 0; i < MW; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
    }
  }
  cp_async_wait<0>();
  // epilogue: lane holds C[row g][cols 2*t4, 2*t4+1] of each 8x8 tile
#pragma unroll
  for (int i = 0; i < MW; ++i) {
    const int64_t r = row0 + warp * 8 * MW + i * 8 + g;
    if (r >= rows) continue;
    const int64_t q = r / m;
    const int c = (int)(r - q * m);
    double *dst = lt + (((8 * q + o) * m + c) * nsplit + split) * rp;
#pragma unroll
    for (int j = 0; j < NT8; ++j) {
      const int col = n0 + j * 8 + 2 * t4;
      if (col < rp)
        *reinterpret_cast<double2 *>(dst + col) =
            make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

template <int NT8, int MW, int G>
int launch_m2l(const double *z, double *lt, int level, int m, int rp, int nsplit,
               const double *cores, cudaStream_t st) {
  using S = M2LShape<NT8, MW, G>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(m2l_dmma_kernel<NT8, MW, G>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::smem);
    attr_set = true;
  }
  const int nchunks = (int)ceil_div(rp / 8, G);
  const int64_t rows = (int64_t(1) << (3 * level - 3)) * m;
  dim3 grid((unsigned)ceil_div(rows, S::TM), (unsigned)ceil_div(rp, S::TN),
            8 * nsplit);
  m2l_dmma_kernel<NT8, MW, G><<<grid, 32 * kM2LWarps, S::smem, st>>>(
      z, lt, level, m, rp, nchunks, nsplit, cores);
  return check_launch("m2l_dmma_kernel");
}

// Tile choice: rp <= 64 -> one column tile and one k chunk (NT8 = G = rp/8);
// larger ranks -> 56- or 64-wide tiles and chunks, whichever pads less.
struct M2LConfig {
  int nt8, g, mw;
};

inline M2LConfig m2l_config(int level, int m, int rp) {
  const int64_t rows = (int64_t(1) << (3 * level - 3)) * m;
  M2LConfig c;
  if (rp <= 64) {
    c.nt8 = c.g = rp / 8;
  } else {
    const int w7 = (int)(ceil_div(rp, 56) * 56 - rp), w8 = (int)(ceil_div(rp, 64) * 64 - rp);
    c.nt8 = c.g = (w7 < w8) ? 7 : 8;
  }
  // 128-row tiles when two CTAs still fit per SM, else 64-row tiles
  const size_t smem2 = sizeof(double) * kStages * (128 + 8 * c.nt8) * 8 * c.g;
  c.mw = (rows <= 64 || smem2 > 112 * 1024) ? 1 : 2;
  return c;
}

inline int m2l_tile_rows(const M2LConfig &c) { return 8 * c.mw * kM2LWarps; }

template <int MW>
int dispatch_g(int g, const double *z, double *lt, int level, int m, int rp,
               int nsplit, const double *cores, cudaStream_t st) {
  switch (g) {
    case 1: return launch_m2l<1, MW, 1>(z, lt, level, m, rp, nsplit, cores, st);
    case 2: return launch_m2l<2, MW, 2>(z, lt, level, m, rp, nsplit, cores, st);
    case 3: return launch_m2l<3, MW, 3>(z, lt, level, m, rp, nsplit, cores, st);
    case 4: return launch_m2l<4, MW, 4>(z, lt, level, m, rp, nsplit, cores, st);
    case 5: return launch_m2l<5, MW, 5>(z, lt, level, m, rp, nsplit, cores, st);
    case 6: return launch_m2l<6, MW, 6>(z, lt, level, m, rp, nsplit, cores, st);
    case 7: return launch_m2l<7, MW, 7>(z, lt, level, m, rp, nsplit, cores, st);
    default: return launch_m2l<8, MW, 8>(z, lt, level, m, rp, nsplit, cores, st);
  }
}

inline int dispatch_m2l(const M2LConfig &c, const double *z, double *lt,
                        int level, int m, int rp, int nsplit,
                        const double *cores, cudaStream_t st) {
  if (c.mw == 1) return dispatch_g<1>(c.g, z, lt, level, m, rp, nsplit, cores, st);
  return dispatch_g<2>(c.g, z, lt, level, m, rp, nsplit, cores, st);
}
