// M2L (Chebyshev, engine.py:228-256) on the int8 tensor cores (tcgen05),
// FP64-exact to ~2^-46 of the operand scales (included by m2l_cheb.cu).
//
// B200's tcgen05 has no FP64 kind, but it multiplies int8 at 4.5 POPS.  The
// translation lt[c, i] = sum_{t in valid(o)} sum_k C_t[i, k] z[c + t, k] is
// run as an error-free sum of int8 GEMMs (Ozaki-style splitting):
//   z / 2^ez      = sum_a 2^(-6-7a) Za,  Za in [-64, 64]   (per level ez)
//   C_t[i] / 2^ei = sum_b 2^(-6-7b) Cb,  Cb in [-64, 64]   (per rank row ei)
// so  lt[c, i] = 2^(ez+ei) sum_{a+b<S} 2^(-12-7(a+b)) (Za Cb^T)[c, i]  plus a
// truncation below 2^(-7S) of the scales.  Every int8 product Za Cb^T is
// accumulated EXACTLY in int32 TMEM (|digit product| <= 2^12, K <= 189 * 256
// and at most S products per accumulator stay below 2^31), pairs with the
// same a + b share one accumulator, and only the S accumulators are
// converted to FP64 at the end -- the result is bitwise independent of the
// summation order.
//
// Tile: 128 target rows (cells of one child octant, or (cell, column) rows
// when m > 1) x 64 rank rows.  Stage = one (offset, 32-wide k chunk): the
// four producer warps gather the S digit planes of the 128 source rows
// z[c + t] (zero-filled where c + t leaves the grid -- exactly the pairs
// cell_pairs_for_offset omits, octree.py:202-221) and copy the matching
// pre-sliced core block, all with cp.async into the K-major no-swizzle
// layout the MMA descriptor reads; one elected thread issues the
// S(S+1)/2 tcgen05.mma.kind::i8 per stage and releases the stage with
// tcgen05.commit.  The same four warps then drain TMEM.
#pragma once

// tcgen05.cuh is included at file scope by m2l_cheb.cu

constexpr int kI8TM = 128, kI8TN = 64;
#ifdef BFMM_I8_TRACE
__device__ long long g_i8_trace[8192];
__device__ int g_trace_n;
#endif
constexpr int kI8Threads = 160;  // warp 0: TMEM + MMA issue; warps 1-4: producers/epilogue

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mbar_spin(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nSPIN_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra SPIN_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared on the TMA engine, completing on *bar.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

template <int S>
struct I8Shape {
  static constexpr int A_SLICE = kI8TM * 32, B_SLICE = kI8TN * 32;
  static constexpr int STAGE = S * (A_SLICE + B_SLICE);
  static constexpr int NS = (S >= 8 ? 4 : (S >= 7 ? 5 : 6));
  static constexpr int LAG = NS - 3;  // cp.async groups a producer keeps in flight
  static constexpr size_t smem = (size_t)NS * STAGE + (2 * NS + 1) * 8 + 16;
};

// Scale of a weight column's z digits: 2^(ez - 12) (NaN when max|z| is not
// finite, so non-finite moments still propagate).
__device__ __forceinline__ double i8_zscale(unsigned long long bits) {
  const double amax = __longlong_as_double((long long)bits);
  if (!(amax <= 1.7976931348623157e308)) return __longlong_as_double(0x7ff8000000000000ll);
  int ez = 0;
  if (amax > 0) frexp(amax, &ez);
  return ldexp(1.0, ez - 12);
}

// One TMEM lane (tile row) of the S int32 accumulators -> FP64 lt row:
// x = sum_d 2^(-B d) acc_d (Horner, fixed order; B = 7 or 8 digit bits), times the z scale and the
// rank row's core scale.  zero: no MMA ran (write zeros).
template <int S, int W, int B>
__device__ __forceinline__ void i8_drain(uint32_t tl, double *dst, double zsc, int nt, int rp,
                                         const double *__restrict__ cpow, bool zero) {
#pragma unroll 1
  for (int c0 = 0; c0 < kI8TN; c0 += W) {  // W columns at a time: S x W registers
    uint32_t acc[S][W];
#pragma unroll
    for (int d = 0; d < S; ++d) {
      if constexpr (W == 16) bfmm::tc::ld16(tl + d * kI8TN + c0, acc[d]);
      else bfmm::tc::ld8(tl + d * kI8TN + c0, acc[d]);
    }
    bfmm::tc::wait_ld();
    const int colb = nt * kI8TN + c0;
#pragma unroll
    for (int jj = 0; jj < W; jj += 2) {
      if (!dst || colb + jj >= rp) continue;  // rp is a multiple of 8
      double x2[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        double x = (double)(int32_t)acc[S - 1][jj + u];
#pragma unroll
        constexpr double kStep = B == 8 ? 0.00390625 : 0.0078125;  // 2^-B
        for (int d = S - 2; d >= 0; --d) x = fma(x, kStep, (double)(int32_t)acc[d][jj + u]);
        x2[u] = zero ? 0.0 : x * zsc * cpow[colb + jj + u];
      }
      *reinterpret_cast<double2 *>(dst + colb + jj) = make_double2(x2[0], x2[1]);
    }
  }
}

template <int S, int B>
__global__ void __launch_bounds__(kI8Threads, 1)
m2l_i8_kernel(const int8_t *__restrict__ zs, const unsigned long long *__restrict__ zmax,
              const int8_t *__restrict__ cs, const double *__restrict__ cpow,
              double *__restrict__ lt, int level, int m, int rp, int kc_n, int ntn,
              int nsplit, int64_t q_lo, int64_t nq, OctList act, int mixed) {
  using Sh = I8Shape<S>;
  constexpr int NS = Sh::NS;
  extern __shared__ __align__(1024) uint8_t smi[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smi + NS * Sh::STAGE);
  uint64_t *empty = full + NS;
  uint64_t *done = empty + NS;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

  // mixed (coarse levels): one row per cell of all eight octants, all 316
  // offsets, the parity rule applied per row (zero rows) -- a level with a few
  // cells per octant then fills one tile instead of eight nearly empty ones
  const int o = mixed ? 0 : (blockIdx.z & 7);
  const int split = mixed ? blockIdx.z : (blockIdx.z >> 3);
  const int ntap = mixed ? 316 : 189;
  const int per = (ntap + nsplit - 1) / nsplit;
  const int v_lo = split * per, v_hi = min(ntap, v_lo + per);
  const int nt = blockIdx.y;
  const int n = 1 << level;
  const int64_t *ocells = act.cells ? act.cells + act.off[o] : nullptr;
  const int64_t rows = mixed ? 8 * nq * m : (act.cells ? act.off[o + 1] - act.off[o] : nq) * m;
  auto cell_of = [&](int64_t q) -> int64_t {  // q-th cell of this CTA's row set
    return mixed ? 8 * q_lo + q : (ocells ? ocells[q] : 8 * (q_lo + q) + o);
  };
  auto orow_of = [&](int64_t q) -> int64_t {  // its lt row
    return mixed ? 8 * q_lo + q : (ocells ? act.off[o] + q : 8 * (q_lo + q) + o);
  };
  const int64_t row0 = int64_t(blockIdx.x) * kI8TM;
  if (row0 >= rows) return;  // whole CTA
  // (cell indices are 30-bit Morton codes: levels <= 10, checked by the caller)
  const int nsteps = (v_hi - v_lo) * kc_n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (nsteps <= 0) {  // a split past the last offset: its lt block is zero
    for (int e = threadIdx.x; e < kI8TM * kI8TN; e += kI8Threads) {
      const int64_t r = row0 + e / kI8TN;
      const int col = nt * kI8TN + e % kI8TN;
      if (r >= rows || col >= rp) continue;
      const int64_t q = r / m;
      const int c = (int)(r - q * m);
      const int64_t orow = orow_of(q);
      lt[((orow * m + c) * nsplit + split) * rp + col] = 0.0;
    }
    return;
  }

  if (warp == 0) bfmm::tc::alloc(tmem_slot, 512);
  if (threadIdx.x == 32) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 5);  // one arrival per producer warp + the bulk copy's expect_tx
      mbar_init(&empty[s], 1);   // tcgen05.commit
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  bfmm::tc::fence_before();
  __syncthreads();
  bfmm::tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- MMA issue (warp 0, one elected lane) ----------------
    // The whole warp runs the loop so the descriptors stay warp-uniform
    // (uniform datapath, no per-MMA register -> uniform moves); a descriptor
    // for smem address x + d is desc(x) + d / 16, so each MMA costs one add.
    const uint64_t dbase = bfmm::tc::desc_kmajor(bfmm::tc::smem_u32(smi), 128, 256);
    int s = 0;
    uint32_t ph = 0;
    for (int step = 0; step < nsteps; ++step) {
      if (lane == 0) mbar_wait(&full[s], ph);
      __syncwarp();
#ifdef BFMM_I8_TRACE
      if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && step < 1024)
        g_i8_trace[step] = clock64();
#endif
      bfmm::tc::fence_after();
      const uint64_t dA = dbase + (uint64_t)((s * Sh::STAGE) >> 4);
      const uint64_t dB = dA + (uint64_t)((S * Sh::A_SLICE) >> 4);
      if (elect_one()) {
        // pairs (a, b) with a + b < S: for fixed a the accumulators a + b of
        // b = b0 .. b0 + nb - 1 are contiguous TMEM columns and the planes
        // B_b contiguous smem rows, so ONE MMA with N = 64 nb covers them
        // (N <= 256): 10 MMAs per stage at S = 7 instead of 28, and each A
        // plane is read from shared memory once or twice instead of S - a times
#pragma unroll
        for (int a = 0; a < S; ++a) {
#pragma unroll
          for (int b0 = 0; b0 < S - a; b0 += 4) {
            const int nb = min(4, S - a - b0);
            // accumulators a + b are first written by a = 0 in step 0
            bfmm::tc::mma_i8(tmem + (uint32_t)((a + b0) * kI8TN),
                             dA + (uint64_t)((a * Sh::A_SLICE) >> 4),
                             dB + (uint64_t)((b0 * Sh::B_SLICE) >> 4),
                             bfmm::tc::idesc_i8(kI8TM, kI8TN * nb),
                             (step > 0 || a > 0) ? 1u : 0u);
          }
        }
        bfmm::tc::commit(&empty[s]);
      }
      __syncwarp();
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
    }
    if (elect_one()) bfmm::tc::commit(done);
    __syncwarp();
  } else {
    // ---------------- producers: gather z digits + copy core digits ----------------
    // thread p computes the source row of tile row p.  Its warp copies the
    // S digit planes of its 32 rows: instruction (j, half) moves plane j
    // (32 contiguous bytes = one sector per row) of 16 rows, lanes l and
    // l + 16 taking the two 16-byte K halves -- 16 sectors per instruction and
    // conflict-free shared-memory writes (bank group = row & 7).  The core
    // block of the stage (S * 2 KB, contiguous in cs) is one bulk copy
    // (TMA engine) issued by thread 32 and tracked by the same mbarrier.
    const int p = threadIdx.x - 32;  // tile row 0..127
    const int wrow = p & ~31;        // first tile row of this warp
    const int64_t r = row0 + p;
    const bool rok = r < rows;
    int cx = 0, cy = 0, cz = 0, colm = 0;
    uint32_t cd = 0;  // the row's cell as a 30-bit Morton code
    if (rok) {
      const int64_t q = r / m;
      colm = (int)(r - q * m);
      const int64_t cell = cell_of(q);
      cd = (uint32_t)cell;
      unmorton3((uint64_t)cell, cx, cy, cz);
    }
    constexpr uint32_t MX = 0x24924924u, MY = 0x12492492u, MZ = 0x09249249u;
    const int hl = lane >> 4;  // K half of this lane
    // this lane's shared-memory slot in a stage: row wrow + (lane & 15) (+ 16)
    uint8_t *const dstA0 = smi + bfmm::tc::kmajor_off(wrow + (lane & 15), 16 * hl);
    const int64_t rowbytes = (int64_t)kc_n * S * 32;
    int s = 0, sl = 0, step = 0;
    uint32_t ph = 0;
    for (int vi = v_lo; vi < v_hi; ++vi) {
      const int t = mixed ? vi : c_valid[o][vi];
      // the octant's parity already admits t (octant mode); only the grid
      // bounds remain -- mixed rows check the full rule
      const int sx = cx + c_offsets[t][0], sy = cy + c_offsets[t][1], sz = cz + c_offsets[t][2];
      int srow = -1;
      const bool ok = mixed ? far_pair(n, cx, cy, cz, c_offsets[t][0], c_offsets[t][1],
                                       c_offsets[t][2])
                            : ((unsigned)sx < (unsigned)n && (unsigned)sy < (unsigned)n &&
                               (unsigned)sz < (unsigned)n);
      if (rok && ok) {
        const uint32_t sc = (((cd | ~MX) + c_dil[t][0]) & MX) | (((cd | ~MY) + c_dil[t][1]) & MY) |
                            (((cd | ~MZ) + c_dil[t][2]) & MZ);
        srow = (int)sc * m + colm;
      }
      const int sr0 = __shfl_sync(0xffffffffu, srow, lane & 15);
      const int sr1 = __shfl_sync(0xffffffffu, srow, 16 + (lane & 15));
      const int8_t *src0 = zs + (sr0 >= 0 ? (int64_t)sr0 * rowbytes + 16 * hl : 0);
      const int8_t *src1 = zs + (sr1 >= 0 ? (int64_t)sr1 * rowbytes + 16 * hl : 0);
      const int8_t *bsrc = cs + ((int64_t)t * ntn + nt) * kc_n * (int64_t)(S * Sh::B_SLICE);
      for (int kc = 0; kc < kc_n; ++kc, ++step) {
        if (step >= NS) {  // one waiter per warp (mbarrier ops are per thread)
          if (lane == 0) mbar_wait(&empty[s], ph ^ 1u);
          __syncwarp();
        }
        uint8_t *sA = smi + s * Sh::STAGE;
#ifdef BFMM_I8_TRACE
        if (lane == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && step < 1024)
          g_i8_trace[1024 * (1 + (p >> 5)) + step] = clock64();
#endif
        if (p == 0) {
          mbar_expect_tx(&full[s], S * Sh::B_SLICE);
          bulk_g2s(sA + S * Sh::A_SLICE, bsrc + kc * (S * Sh::B_SLICE), S * Sh::B_SLICE, &full[s]);
        }
        uint8_t *d0 = dstA0 + s * Sh::STAGE;
        const int8_t *a0 = src0 + kc * (S * 32), *a1 = src1 + kc * (S * 32);
#pragma unroll
        for (int j = 0; j < S; ++j) {
          cp_async16(d0 + j * Sh::A_SLICE, a0 + 32 * j, sr0 >= 0);
          cp_async16(d0 + j * Sh::A_SLICE + 512, a1 + 32 * j, sr1 >= 0);
        }
        // stage step - LAG has landed for this thread once at most LAG newer
        // groups are pending; the warp then arrives once (an arrival per
        // thread would serialise 128 mbarrier operations per stage).  As in
        // CUTLASS's sm100 cp.async + UMMA mainloop, the mbarrier completion
        // orders the copies before the MMA's shared-memory reads.
        cp_async_commit();
        if (step >= Sh::LAG) {
          cp_async_wait<Sh::LAG>();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[sl]);
          if (++sl == NS) sl = 0;
        }
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    cp_async_wait<0>();
    __syncwarp();
    if (lane == 0)
      for (int k = max(0, nsteps - Sh::LAG); k < nsteps; ++k) mbar_arrive(&full[k % NS]);

    // ---------------- epilogue: S int32 accumulators -> FP64 ----------------
    mbar_wait(done, 0);
    bfmm::tc::fence_after();
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
    const int er = 32 * quarter + lane;
    const int64_t orr = row0 + er;
    double *dst = nullptr;
    double zsc = 0.0;
    if (orr < rows) {
      const int64_t q = orr / m;
      const int c = (int)(orr - q * m);
      const int64_t orow = orow_of(q);
      dst = lt + ((orow * m + c) * nsplit + split) * rp;
      zsc = i8_zscale(zmax[c]);
    }
    i8_drain<S, 16, B>(tmem + ((uint32_t)(32 * quarter) << 16), dst, zsc, nt, rp, cpow, false);
  }
  bfmm::tc::fence_before();
  __syncthreads();
  if (warp == 0) bfmm::tc::dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// Plane-buffered variant for dense levels >= 4 (m2l_i8p_kernel).
//
// The gather kernel above reads, per tile, 189 shifted copies of 128 source
// rows -- 5.6x more than the distinct sources the tile touches -- and is
// L2-bandwidth bound.  Here a tile is a 1 x 16 x 8 block (x, y, z) of
// same-octant targets (stride 2 cells), tile row r = 8 y + z (2 x 8 x 8 at
// level 4, see I8PShape).  The 189
// offsets split into 28 groups by (t_x, parity of o_y + t_y, parity of
// o_z + t_z); all sources of a group lie in ONE parity plane x = x_t + t_x,
// y = 2Y' + py, z = 2Z' + pz with Y' in [16 yb - 2, 16 yb + 18) and
// Z' in [8 zb - 2, 8 zb + 10).  That 20 x 12 plane of digit rows is loaded
// once into shared memory, Z' fastest at 16 B per row, so the A operand of
// every offset of the group is a plain K-major no-swizzle descriptor into
// it: start = plane + ((dy + 2) 12 + dz + 2) 16 B, 8-row groups (y) at
// SBO = 192 B, K halves at LBO = 3840 B, where (dy, dz) = floor((o + t) / 2)
// per axis.  Out-of-grid sources are zero rows, exactly the pairs
// cell_pairs_for_offset omits (octree.py:202-221).  A traffic drops from
// 189 x 128 rows to 28 x 240 rows per tile; the int32 sums are the same
// integers as the gather kernel's (exact, any order).
//
// Warp roles (192 threads): 0 = TMEM + MMA issue, 1 = core-block bulk
// copies (B ring), 2-5 = plane loads (cp.async) then the TMEM drain.

constexpr int kI8PThreads = 192;
#ifndef BFMM_I8P_SMEM_KB
#define BFMM_I8P_SMEM_KB 227
#endif
// Tile XT x YT x 8 (x, y, z) same-octant targets, XT * YT = 16: 1 x 16 x 8
// for levels >= 5, 2 x 8 x 8 at level 4.  A plane buffer holds, per Y' row,
// the XT source x-planes of the group side by side: row (Y', x, Z'), Z'
// fastest, so the 16 row groups g = y XT + x of the A operand sit at the
// uniform stride SBO = 12 * 16 B for any XT.
template <int S, int XT>
struct I8PShape {
  static constexpr int YT = 16 / XT;
  static constexpr int ROWS = (YT + 4) * XT * 12;  // plane rows (Y' x x x Z')
  static constexpr int HALF = ROWS * 16;           // one K half of one digit plane
  static constexpr int PLANE = S * 2 * HALF;       // one plane buffer
  static constexpr int B_STAGE = S * kI8TN * 32;
  static constexpr int BUDGET = BFMM_I8P_SMEM_KB * 1024 - 512;
  // three plane buffers when a 4-deep core ring still fits (measured: three
  // plane buffers matter more than a deeper ring), else two
  static constexpr int NP = (3 * PLANE + 4 * B_STAGE <= BUDGET) ? 3 : 2;
  static constexpr int NB_FIT = (BUDGET - NP * PLANE) / B_STAGE;
  static constexpr int NB = NB_FIT > 12 ? 12 : NB_FIT;
  static constexpr size_t smem = (size_t)NP * PLANE + (size_t)NB * B_STAGE +
                                 (2 * NP + 2 * NB + 1) * 8 + 16;
};

// register cap: leaves room on the SM for near-field (P2P) CTAs running
// concurrently on another stream
template <int S, int XT, int B>
__global__ void __maxnreg__(128)
m2l_i8p_kernel(const int8_t *__restrict__ zs, const unsigned long long *__restrict__ zmax,
               const int8_t *__restrict__ cs, const double *__restrict__ cpow,
               double *__restrict__ lt, int level, int m, int rp, int kc_n, int ntn,
               int nsplit, int4 box) {
  // box: the target cells this launch covers, in same-octant (half-
  // resolution) coordinates: origin (box.x, box.y, box.z), box.w = packed
  // tile counts (x tiles << 20 | y tiles << 10 | z tiles); a whole level or
  // a Morton-aligned shard of it (a box, see i8_plane_box)
  using Sh = I8PShape<S, XT>;
  constexpr int NP = Sh::NP, NB = Sh::NB, YT = Sh::YT;
  extern __shared__ __align__(1024) uint8_t smp[];
  uint8_t *const planes = smp;
  uint8_t *const bring = smp + NP * Sh::PLANE;
  uint64_t *pfull = reinterpret_cast<uint64_t *>(bring + NB * Sh::B_STAGE);
  uint64_t *pempty = pfull + NP;
  uint64_t *bfull = pempty + NP;
  uint64_t *bempty = bfull + NB;
  uint64_t *done = bempty + NB;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

  const int n = 1 << level;  // cells per axis
  // octant fastest in the launch order: the eight octant tiles of one
  // spatial block run together and share their source parity planes in L2
  // (octant-major order re-read every plane from DRAM once per octant)
  const int o = blockIdx.x & 7, split = blockIdx.z;
  const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
  const int ybn = (box.w >> 10) & 1023, zbn = box.w & 1023;
  int tile = blockIdx.x >> 3;
  const int zb = tile % zbn + box.z / 8;
  tile /= zbn;
  const int yb = tile % ybn + box.y / YT;
  const int xb = tile / ybn + box.x / XT;
  const int col = blockIdx.y / ntn, nt = blockIdx.y - col * ntn;
  const int xs = 2 * xb * XT + ox;  // target x of the tile's first x slot (slots 2 apart)
  const int units = 28 * kc_n;
  const int per = (units + nsplit - 1) / nsplit;
  const int u_lo = split * per, u_hi = min(units, u_lo + per);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // a unit (kc, g) is live when its plane is inside the grid and the group
  // has offsets; every role walks the same live units in the same order
  auto live = [&](int u, int &kc, int &g, int &tx) {
    kc = u / 28;
    g = u - kc * 28;
    tx = g / 4 - 3;
    // some x slot's source plane inside the grid
    return xs + tx + 2 * (XT - 1) >= 0 && xs + tx < n && c_grp_off[o][g + 1] > c_grp_off[o][g];
  };
  bool any = false;
  for (int u = u_lo; u < u_hi; ++u) {
    int kc, g, tx;
    any |= live(u, kc, g, tx);
  }

  if (warp == 0) bfmm::tc::alloc(tmem_slot, 512);
  if (threadIdx.x == 32) {
    for (int i = 0; i < NP; ++i) {
      mbar_init(&pfull[i], 4);  // one arrival per plane-producer warp
      mbar_init(&pempty[i], 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  bfmm::tc::fence_before();
  __syncthreads();
  bfmm::tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- MMA issue ----------------
    const uint64_t dP = bfmm::tc::desc_kmajor(bfmm::tc::smem_u32(planes), Sh::HALF, 192);  // SBO: 12 rows
    const uint64_t dB = bfmm::tc::desc_kmajor(bfmm::tc::smem_u32(bring), 128, 256);
    int ps = 0, bs = 0;
    uint32_t pph = 0, bph = 0;
    bool first = true;
    for (int u = u_lo; u < u_hi; ++u) {
      int kc, g, tx;
      if (!live(u, kc, g, tx)) continue;
#ifdef BFMM_I8_TRACE
      const bool trc = lane == 0 && blockIdx.x == 3 && blockIdx.y == 0 && blockIdx.z == 0;
      long long tw0 = clock64();
#endif
      if (lane == 0) mbar_wait(&pfull[ps], pph);
#ifdef BFMM_I8_TRACE
      if (trc && g_trace_n < 4000) { g_i8_trace[2 * g_trace_n] = tw0; g_i8_trace[2 * g_trace_n + 1] = -clock64(); ++g_trace_n; }
#endif
      __syncwarp();
      bfmm::tc::fence_after();
      for (int e = c_grp_off[o][g]; e < c_grp_off[o][g + 1]; ++e) {
        const int t = c_grp[o][e];
        const int dy = (oy + c_offsets[t][1]) >> 1, dz = (oz + c_offsets[t][2]) >> 1;
#ifdef BFMM_I8_TRACE
        long long tb0 = clock64();
#endif
        if (lane == 0) mbar_wait(&bfull[bs], bph);
#ifdef BFMM_I8_TRACE
        if (trc && g_trace_n < 4000) { g_i8_trace[2 * g_trace_n] = tb0; g_i8_trace[2 * g_trace_n + 1] = clock64(); ++g_trace_n; }
#endif
        __syncwarp();
        bfmm::tc::fence_after();
        const uint64_t dA =
            dP + (uint64_t)((ps * Sh::PLANE + ((dy + 2) * XT * 12 + dz + 2) * 16) >> 4);
        const uint64_t dBs = dB + (uint64_t)((bs * Sh::B_STAGE) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int a = 0; a < S; ++a) {
#pragma unroll
            for (int b0 = 0; b0 < S - a; b0 += 4) {
              const int nb = min(4, S - a - b0);
              bfmm::tc::mma_i8(tmem + (uint32_t)((a + b0) * kI8TN),
                               dA + (uint64_t)((a * 2 * Sh::HALF) >> 4),
                               dBs + (uint64_t)((b0 * kI8TN * 32) >> 4),
                               bfmm::tc::idesc_i8(kI8TM, kI8TN * nb),
                               (!first || a > 0) ? 1u : 0u);
            }
          }
          bfmm::tc::commit(&bempty[bs]);
        }
        __syncwarp();
        first = false;
        if (++bs == NB) {
          bs = 0;
          bph ^= 1u;
        }
      }
      if (elect_one()) bfmm::tc::commit(&pempty[ps]);
      __syncwarp();
      if (++ps == NP) {
        ps = 0;
        pph ^= 1u;
      }
    }
    if (elect_one()) bfmm::tc::commit(done);
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- core blocks (B ring) ----------------
    if (lane == 0) {
      int bs = 0, k = 0;
      uint32_t bph = 0;
      for (int u = u_lo; u < u_hi; ++u) {
        int kc, g, tx;
        if (!live(u, kc, g, tx)) continue;
        for (int e = c_grp_off[o][g]; e < c_grp_off[o][g + 1]; ++e, ++k) {
          const int t = c_grp[o][e];
          if (k >= NB) mbar_wait(&bempty[bs], bph ^ 1u);
          mbar_expect_tx(&bfull[bs], Sh::B_STAGE);
          bulk_g2s(bring + bs * Sh::B_STAGE,
                   cs + (((int64_t)t * ntn + nt) * kc_n + kc) * (int64_t)Sh::B_STAGE,
                   Sh::B_STAGE, &bfull[bs]);
          if (++bs == NB) {
            bs = 0;
            bph ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- plane loads ----------------
    const int p = threadIdx.x - 64;  // 0..127
    const int64_t rowbytes = (int64_t)kc_n * S * 32;
    int ps = 0, k = 0, pl = 0;
    uint32_t pph = 0;
    for (int u = u_lo; u < u_hi; ++u) {
      int kc, g, tx;
      if (!live(u, kc, g, tx)) continue;
      const int py = (g >> 1) & 1, pz = g & 1;
      if (k >= NP) {
        if (lane == 0) mbar_wait(&pempty[ps], pph ^ 1u);
        __syncwarp();
      }
      uint8_t *buf = planes + ps * Sh::PLANE;
      for (int row = p; row < Sh::ROWS; row += 128) {
        const int yx = row / 12, Zp = 8 * zb - 2 + row % 12;
        const int Yp = YT * yb - 2 + yx / XT, x = xs + 2 * (yx % XT) + tx;
        const int y = 2 * Yp + py, z = 2 * Zp + pz;
        const bool v = x >= 0 && x < n && y >= 0 && y < n && z >= 0 && z < n;
        const int8_t *src =
            v ? zs + ((int64_t)morton3(x, y, z) * m + col) * rowbytes + kc * (S * 32) : zs;
        uint8_t *dst = buf + row * 16;
#pragma unroll
        for (int j = 0; j < S; ++j) {
          cp_async16(dst + j * 2 * Sh::HALF, src + 32 * j, v);
          cp_async16(dst + j * 2 * Sh::HALF + Sh::HALF, src + 32 * j + 16, v);
        }
      }
      cp_async_commit();
      if (k >= 1) {  // the previous plane has landed: publish it
        cp_async_wait<1>();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[pl]);
        if (++pl == NP) pl = 0;
      }
      ++k;
      if (++ps == NP) {
        ps = 0;
        pph ^= 1u;
      }
    }
    cp_async_wait<0>();
    __syncwarp();
    if (k >= 1 && lane == 0) mbar_arrive(&pfull[pl]);

    // ---------------- drain ----------------
    if (any) {
      mbar_wait(done, 0);
      bfmm::tc::fence_after();
    }
    const int quarter = warp & 3;
    const int er = 32 * quarter + lane;
    const int g = er >> 3, zl = er & 7;  // row group g = y XT + x
    const int64_t cell = (int64_t)morton3(xs + 2 * (g % XT), 2 * (YT * yb + g / XT) + oy,
                                          2 * (8 * zb + zl) + oz);
    double *dst = lt + ((cell * m + col) * nsplit + split) * rp;
    i8_drain<S, 8, B>(tmem + ((uint32_t)(32 * quarter) << 16), dst, i8_zscale(zmax[col]), nt, rp, cpow,
                !any);
  }
  bfmm::tc::fence_before();
  __syncthreads();
  if (warp == 0) bfmm::tc::dealloc(tmem, 512);
}

// max |z| over n doubles as the bit pattern of a non-negative double
// (order-preserving as an unsigned integer, so atomicMax is exact).
// groups (nullable): the rows are the m rows of each listed cell, compact row
// r = array row groups[r / m] * m + r % m (sparse clouds: occupied cells).
__global__ void absmax_bits_kernel(const double *__restrict__ z, int64_t rows, int rp, int m,
                                   unsigned long long *__restrict__ out,
                                   const int64_t *__restrict__ groups = nullptr) {
  // block column blockIdx.y = weight column c: rows c, c + m, c + 2m, ...
  const int c = blockIdx.y;
  const int64_t nr = (rows - c + m - 1) / m;
  const int64_t n = nr * rp;
  unsigned long long mx = 0;
  if (m == 1 && !groups) {  // one column: the whole array, no index arithmetic
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
      const unsigned long long b =
          (unsigned long long)__double_as_longlong(z[e]) & 0x7fffffffffffffffull;
      mx = b > mx ? b : mx;
    }
  } else {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
      const int64_t i = e / rp;
      const int k = (int)(e - i * rp);
      const int64_t R = groups ? groups[i] * m + c : c + i * m;
      const unsigned long long b =
          (unsigned long long)__double_as_longlong(z[R * rp + k]) & 0x7fffffffffffffffull;
      mx = b > mx ? b : mx;
    }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, mx, s);
    mx = o2 > mx ? o2 : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out + c, mx);
}

// z (rows x rp) -> S signed 7-bit digit planes, zs[row][kc][j][32]; digit j
// of x is taken from x / 2^ez exactly, ez the exponent of the row's weight
// column (row % m) -- every A row of the M2L gathers one column only, so a
// per-column scale is a per-row scale of the GEMM and each right-hand side
// is cut independently of the others (scalings by powers of two and
// x - rint(x) are exact in FP64).  k >= rp is zero padding.
template <int S, int B>
__global__ void z_slice_kernel(const double *__restrict__ z, int64_t rows, int rp, int kc_n,
                               int m, const unsigned long long *__restrict__ zmax,
                               int8_t *__restrict__ zs,
                               const int64_t *__restrict__ groups = nullptr) {
  const int64_t total = rows * kc_n * 2;
  const unsigned per_row = (unsigned)(kc_n * 2);
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    // 32-bit division when the index fits (every level up to 2^31 chunks)
    const int64_t crow = total <= 0xffffffffll ? (int64_t)((unsigned)e / per_row) : e / per_row;
    const int rem = (int)(e - crow * per_row);
    // listed cells: compact row -> the cell's row of the level's arrays
    const int64_t row = groups ? groups[crow / m] * m + crow % m : crow;
    const int kc = rem >> 1, h = rem & 1;
    const int k0 = kc * 32 + h * 16;
    const double amax = __longlong_as_double((long long)zmax[m == 1 ? 0 : row % m]);
    int ez = 0;
    if (amax > 0 && amax <= 1.7976931348623157e308) frexp(amax, &ez);
    const double inv = ldexp(1.0, 6 - ez);  // first digit: x * 2^(6 - ez) in [-64, 64]
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int k = k0 + u;
      const double v = k < rp ? z[row * rp + k] : 0.0;
      x[u] = (v == v && fabs(v) <= 1.7976931348623157e308) ? v * inv : 0.0;
    }
    int8_t *dst = zs + ((row * kc_n + kc) * S) * 32 + 16 * h;
    if constexpr (B == 8) {
      // base 2^8: X = rint(x 2^(8(S-1))) (|X| <= 2^(8S-10) with |x| <= 64)
      // as S signed bytes in [-128, 127] (digit j weight 2^(-6-8j) of x /
      // 2^6, the same leading weight as the 7-bit split); exact integer steps
      int64_t X[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) X[u] = (int64_t)rint(ldexp(x[u], 8 * (S - 1)));
      uint32_t w[S][4];
#pragma unroll
      for (int j = S - 1; j >= 0; --j) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) w[j][q4] = 0;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int8_t dg = j > 0 ? (int8_t)(X[u] & 0xff) : (int8_t)X[u];
          X[u] = (X[u] - dg) >> 8;
          w[j][u >> 2] |= ((uint32_t)(uint8_t)dg) << (8 * (u & 3));
        }
      }
#pragma unroll
      for (int j = 0; j < S; ++j)
        *reinterpret_cast<uint4 *>(dst + j * 32) = make_uint4(w[j][0], w[j][1], w[j][2], w[j][3]);
    } else {
#pragma unroll
      for (int j = 0; j < S; ++j) {
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double dg = rint(x[u]);
          x[u] = (x[u] - dg) * 128.0;
          w[u >> 2] |= ((uint32_t)(uint8_t)(int8_t)(int)dg) << (8 * (u & 3));
        }
        *reinterpret_cast<uint4 *>(dst + j * 32) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

struct I8Call {
  const int8_t *zs;
  const unsigned long long *zmax;
  const int8_t *cs;
  const double *cpow;
  double *lt;
  int level, m, rp, kc_n, ntn, nsplit;
  int64_t q_lo, nq;
  OctList act;
  cudaStream_t st;
};

// The plane kernel covers dense levels >= 4 (1 x 16 x 8 tiles from level 5,
// 2 x 8 x 8 at level 4) over a box of target cells: the whole level, or a
// Morton shard [8 q_lo, 8 (q_lo + nq)) that is an aligned power-of-two block
// -- the low b bits of the Morton id vary, i.e. z gets ceil(b/3) of them,
// y ceil((b-1)/3), x ceil((b-2)/3): always a box (the cells-balanced shards
// of 2, 4, 8, ... ranks: slabs, columns, octants).  Its same-octant extents
// must be whole tiles.  Unaligned shards and listed cells use the gather
// kernel.  BFMM_I8_GATHER (diagnostic) forces the gather kernel.
inline bool i8_plane_box(const I8Call &a, int XT, int YT, int4 *box) {
  if (a.act.cells || a.level < 4 || getenv("BFMM_I8_GATHER")) return false;
  const int64_t c0 = 8 * a.q_lo, len = 8 * a.nq;
  if (len <= 0 || (len & (len - 1)) || c0 % len) return false;
  int b = 0;
  while ((int64_t(1) << b) < len) ++b;
  const int ez = 1 << ((b + 2) / 3), ey = 1 << ((b + 1) / 3), ex = 1 << (b / 3);
  int x0, y0, z0;
  unmorton3((uint64_t)c0, x0, y0, z0);
  // same-octant (half-resolution) extents and origin
  const int hx = ex / 2, hy = ey / 2, hz = ez / 2;
  if (hx < XT || hy < YT || hz < 8 || hx % XT || hy % YT || hz % 8) return false;
  if (hx / XT > 1023 || hy / YT > 1023 || hz / 8 > 1023) return false;
  if (box) *box = make_int4(x0 / 2, y0 / 2, z0 / 2, ((hx / XT) << 20) | ((hy / YT) << 10) | (hz / 8));
  return true;
}

// coarse dense levels (<= 512 cells): one mixed-octant row set, all 316
// offsets (see m2l_i8_kernel); BFMM_I8_OCTANT (diagnostic) forces octant mode
inline bool i8_mixed_ok(const I8Call &a) {
  return !a.act.cells && a.level <= 3 && !getenv("BFMM_I8_OCTANT");
}

template <int S, int B>
int launch_i8(const I8Call &a) {
  using Sh = I8Shape<S>;
  static unsigned long long attr_set = 0;
  if (first_on_device(&attr_set)) {
    cudaFuncSetAttribute(m2l_i8_kernel<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Sh::smem);
  }
  const int mixed = i8_mixed_ok(a) ? 1 : 0;
  int64_t rows = mixed ? 8 * a.nq * a.m : a.nq * a.m;
  if (a.act.cells) {
    rows = 0;
    for (int o = 0; o < 8; ++o) rows = std::max(rows, (a.act.off[o + 1] - a.act.off[o]) * a.m);
  }
  if (rows <= 0) return 0;
  dim3 grid((unsigned)ceil_div(rows, kI8TM), (unsigned)a.ntn, (mixed ? 1 : 8) * a.nsplit);
  m2l_i8_kernel<S, B><<<grid, kI8Threads, Sh::smem, a.st>>>(
      a.zs, a.zmax, a.cs, a.cpow, a.lt, a.level, a.m, a.rp, a.kc_n, a.ntn, a.nsplit, a.q_lo,
      a.nq, a.act, mixed);
  return check_launch("m2l_i8_kernel");
}

template <int S, int XT, int B>
int launch_i8p(const I8Call &a) {
  using Sh = I8PShape<S, XT>;
  static unsigned long long attr_set = 0;
  if (first_on_device(&attr_set)) {
    cudaFuncSetAttribute(m2l_i8p_kernel<S, XT, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Sh::smem);
  }
  int4 box;
  i8_plane_box(a, XT, Sh::YT, &box);
  const int tiles = (box.w >> 20) * ((box.w >> 10) & 1023) * (box.w & 1023);
  dim3 grid((unsigned)tiles * 8, (unsigned)(a.ntn * a.m), a.nsplit);
  m2l_i8p_kernel<S, XT, B><<<grid, kI8PThreads, Sh::smem, a.st>>>(
      a.zs, a.zmax, a.cs, a.cpow, a.lt, a.level, a.m, a.rp, a.kc_n, a.ntn, a.nsplit, box);
  return check_launch("m2l_i8p_kernel");
}

inline bool i8_plane_ok(const I8Call &a) {
  return i8_plane_box(a, a.level >= 5 ? 1 : 2, a.level >= 5 ? 16 : 8, nullptr);
}

#include "m2l_i8p2.cuh"

template <int XT>
int dispatch_i8p(int S, int B, const I8Call &a) {
  if (B == 8) return launch_i8p<6, XT, 8>(a);
  switch (S) {
    case 5: return launch_i8p<5, XT, 7>(a);
    case 6: return launch_i8p<6, XT, 7>(a);
    case 7: return launch_i8p<7, XT, 7>(a);
    default: return launch_i8p<8, XT, 7>(a);
  }
}

// S digits of B bits (B = 8 only with S = 6, see i8_base256_ok)
inline int dispatch_i8(int S, int B, const I8Call &a) {
  int4 box2;
  // six 8-bit digits on dense levels >= 5: the CTA-pair plane kernel
  // (BFMM_I8_1CTA, diagnostic: the single-CTA one)
  if (B == 8 && S == 6 && i8p2_ok(a, &box2)) return launch_i8p2(a, box2);
  if (i8_plane_ok(a)) return a.level >= 5 ? dispatch_i8p<1>(S, B, a) : dispatch_i8p<2>(S, B, a);
  if (B == 8) return launch_i8<6, 8>(a);
  switch (S) {
    case 5: return launch_i8<5, 7>(a);
    case 6: return launch_i8<6, 7>(a);
    case 7: return launch_i8<7, 7>(a);
    default: return launch_i8<8, 7>(a);
  }
}
