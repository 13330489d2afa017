// CTA-pair (cta_group::2) variant of the plane-buffered int8 M2L
// (m2l_i8p_kernel, m2l_i8.cuh) for six 8-bit digits at dense levels >= 5.
//
// The single-CTA kernel is bound by shared-memory operand reads: per stage
// (one offset, K = 32) its 8 grouped MMAs read 32 KB of z planes (A) and
// 42 KB of core digit planes (B) for 672 cycles of MMA work.  Here two CTAs
// on the two SMs of a TPC run ONE M = 256 MMA stream: CTA r holds tile r of
// a pair of z-adjacent same-octant tiles (its 128 target rows: A) and half
// of every core-digit pair -- digit 2k + r of the pairs (0,1), (2,3), (4,5)
// (B rows r*64 .. r*64+63 of an N = 128 MMA).  The digit products are
// grouped as (a, pair k) for a + 2k < 6: 12 MMAs of 256 x 128 x 32 per
// stage, 24 digit products (the 21 of a + b < 6 plus (1,5), (3,3), (5,1),
// which land in accumulator 6 and are dropped), and per SM each MMA reads
// 4 KB of A + 2 KB of B for 64 cycles of tensor work (96 B/cycle instead of
// ~138).  Accumulator d = a + b keeps the single-CTA TMEM layout (64
// columns per digit sum), so the drain is the same.
//
// SPLIT (the default): the three pairs with a + 2k = 5 drop their wasted
// half instead -- they run as N = 64 MMAs of digit 2k alone, whose B half
// from CTA r is rank rows 32r .. 32r+31 of digit 2k.  Each CTA therefore
// also stages those half planes of digits 0, 2, 4 (3 KB more per stage):
// 9 MMAs of N = 128 + 3 of N = 64, exactly the 21 digit products (12.5 %
// less tensor work per stage), bitwise the same accumulators 0..5.
//
// Synchronisation: only the leader (cluster rank 0) issues MMAs.  Both CTAs'
// plane-producer warps arrive on the LEADER's plane-full barrier (count 8,
// shared::cluster addresses); each CTA's core-block loader waits for its own
// bulk copies and then arrives on the leader's core-ready barrier (count
// 2).  The leader's tcgen05.commit multicasts to the same barrier offsets
// in both CTAs (plane-empty, core-empty, done), so each CTA recycles its own
// buffers and drains its own TMEM lanes.
#pragma once

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(const void *p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(out)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// relaxed remote arrival: the forwarder only relays that a bulk copy (async
// proxy) has completed on this CTA's barrier -- no generic-proxy data of its
// own to publish, so no release fence (a release.cluster arrive costs a
// GPU-scope MEMBAR per core block)
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nWAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n"
               ::: "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this smem offset in both CTAs of the pair once
// all prior MMAs of this thread have completed
__device__ __forceinline__ void commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// warps: 0 MMA issue (leader), 1 core-block bulk copies, 2-5 plane loads
// then the TMEM drain, 6 forwards each landed core block to the leader
constexpr int kI8P2Threads = 224;

template <int NBMAX, bool SPLIT>
struct I8P2Shape {
  static constexpr int S = 6, XT = 1, YT = 16;
  static constexpr int ROWS = (YT + 4) * XT * 12;
  static constexpr int HALF = ROWS * 16;
  static constexpr int PLANE = S * 2 * HALF;
  static constexpr int B_PLANE = kI8TN * 32;  // one digit plane, 64 rank rows x 32 k
  static constexpr int B_HALF = B_PLANE / 2;   // 32 rank rows of one digit
  // this CTA's three digits (+ its halves of digits 0, 2, 4 when SPLIT)
  static constexpr int B_STAGE = 3 * B_PLANE + (SPLIT ? 3 * B_HALF : 0);
  static constexpr int BUDGET = BFMM_I8P_SMEM_KB * 1024 - 512;
  static constexpr int NP = 3;
  static constexpr int NB_FIT = (BUDGET - NP * PLANE) / B_STAGE;
  static constexpr int NB = NB_FIT > NBMAX ? NBMAX : NB_FIT;
  static constexpr size_t smem = (size_t)NP * PLANE + (size_t)NB * B_STAGE +
                                 (2 * NP + 3 * NB + 1) * 8 + 16;
};

// NBMAX = 12: the whole SM's shared memory; NBMAX = 6 (BFMM_I8_COSCHED):
// ~176 KB, leaving room for one near-field tile CTA beside it on each SM
template <int NBMAX, bool SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kI8P2Threads, 1)
m2l_i8p2_kernel(const int8_t *__restrict__ zs, const unsigned long long *__restrict__ zmax,
                const int8_t *__restrict__ cs, const double *__restrict__ cpow,
                double *__restrict__ lt, int level, int m, int rp, int kc_n, int ntn,
                int nsplit, int4 box) {
  using Sh = I8P2Shape<NBMAX, SPLIT>;
  constexpr int S = Sh::S, NP = Sh::NP, NB = Sh::NB, YT = Sh::YT, XT = Sh::XT;
  extern __shared__ __align__(1024) uint8_t smp[];
  uint8_t *const planes = smp;
  uint8_t *const bring = smp + NP * Sh::PLANE;
  uint64_t *pfull = reinterpret_cast<uint64_t *>(bring + NB * Sh::B_STAGE);  // leader: 8 arrivals
  uint64_t *pempty = pfull + NP;
  uint64_t *bfull = pempty + NP;   // this CTA's bulk copies (tx)
  uint64_t *bready = bfull + NB;   // leader: both CTAs' core halves landed (2 arrivals)
  uint64_t *bempty = bready + NB;
  uint64_t *done = bempty + NB;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n = 1 << level;
  // launch order: (tile pair, octant, rank) with the rank fastest -- the
  // two CTAs of a cluster take z-adjacent tiles of the same octant; octants
  // next, so a block's eight octant pairs share their planes in L2
  const int o = (blockIdx.x >> 1) & 7, split = blockIdx.z;
  const int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
  const int ybn = (box.w >> 10) & 1023, zbn = box.w & 1023;
  int tile = 2 * (blockIdx.x >> 4) + (int)rank;
  const int zb = tile % zbn + box.z / 8;
  tile /= zbn;
  const int yb = tile % ybn + box.y / YT;
  const int xb = tile / ybn + box.x / XT;
  const int col = blockIdx.y / ntn, nt = blockIdx.y - col * ntn;
  const int xs = 2 * xb * XT + ox;
  const int units = 28 * kc_n;
  const int per = (units + nsplit - 1) / nsplit;
  const int u_lo = split * per, u_hi = min(units, u_lo + per);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // same xb, octant and split in both CTAs: the same live units in the same
  // order, so the two plane / core rings stay in lock step
  auto live = [&](int u, int &kc, int &g, int &tx) {
    kc = u / 28;
    g = u - kc * 28;
    tx = g / 4 - 3;
    return xs + tx >= 0 && xs + tx < n && c_grp_off[o][g + 1] > c_grp_off[o][g];
  };
  bool any = false;
  for (int u = u_lo; u < u_hi; ++u) {
    int kc, g, tx;
    any |= live(u, kc, g, tx);
  }

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < NP; ++i) {
      mbar_init(&pfull[i], 8);  // 4 plane-producer warps x 2 CTAs (leader's copy used)
      mbar_init(&pempty[i], 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bready[i], 2);  // one loader per CTA (leader's copy used)
      mbar_init(&bempty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  bfmm::tc::fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrival
  bfmm::tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- MMA issue (leader only) ----------------
    if (leader) {
      const uint64_t dP = bfmm::tc::desc_kmajor(bfmm::tc::smem_u32(planes), Sh::HALF, 192);
      const uint64_t dB = bfmm::tc::desc_kmajor(bfmm::tc::smem_u32(bring), 128, 256);
      int ps = 0, bs = 0;
      uint32_t pph = 0, bph = 0;
      bool first = true;
      for (int u = u_lo; u < u_hi; ++u) {
        int kc, g, tx;
        if (!live(u, kc, g, tx)) continue;
        if (lane == 0) mbar_wait_cluster(&pfull[ps], pph);
        __syncwarp();
        bfmm::tc::fence_after();
        for (int e = c_grp_off[o][g]; e < c_grp_off[o][g + 1]; ++e) {
          const int t = c_grp[o][e];
          const int dy = (oy + c_offsets[t][1]) >> 1, dz = (oz + c_offsets[t][2]) >> 1;
          if (lane == 0) mbar_wait_cluster(&bready[bs], bph);
          __syncwarp();
          bfmm::tc::fence_after();
          const uint64_t dA =
              dP + (uint64_t)((ps * Sh::PLANE + ((dy + 2) * XT * 12 + dz + 2) * 16) >> 4);
          const uint64_t dBs = dB + (uint64_t)((bs * Sh::B_STAGE) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int a = 0; a < S; ++a) {
#pragma unroll
              for (int k = 0; 2 * k + a < S; ++k) {
                if (SPLIT && 2 * k + a == S - 1) {
                  // digit 2k alone (N = 64): rank rows 0-31 from CTA 0's
                  // half plane, 32-63 from CTA 1's -> accumulator S - 1
                  mma_i8_pair(tmem + (uint32_t)((a + 2 * k) * kI8TN),
                              dA + (uint64_t)((a * 2 * Sh::HALF) >> 4),
                              dBs + (uint64_t)((3 * Sh::B_PLANE + k * Sh::B_HALF) >> 4),
                              bfmm::tc::idesc_i8(256, 64), (!first || a > 0) ? 1u : 0u);
                  continue;
                }
                // rows 0-63 of B: digit 2k (CTA 0's plane k), rows 64-127:
                // digit 2k + 1 (CTA 1's plane k) -> accumulators a+2k, a+2k+1
                mma_i8_pair(tmem + (uint32_t)((a + 2 * k) * kI8TN),
                            dA + (uint64_t)((a * 2 * Sh::HALF) >> 4),
                            dBs + (uint64_t)((k * Sh::B_PLANE) >> 4),
                            bfmm::tc::idesc_i8(256, 128), (!first || a > 0) ? 1u : 0u);
              }
            }
            commit_pair(&bempty[bs]);
          }
          __syncwarp();
          first = false;
          if (++bs == NB) {
            bs = 0;
            bph ^= 1u;
          }
        }
        if (elect_one()) commit_pair(&pempty[ps]);
        __syncwarp();
        if (++ps == NP) {
          ps = 0;
          pph ^= 1u;
        }
      }
      if (elect_one()) commit_pair(done);
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- this CTA's core digit halves (B ring) ----------------
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
          const int8_t *blk = cs + (((int64_t)t * ntn + nt) * kc_n + kc) * (int64_t)(S * Sh::B_PLANE);
#pragma unroll
          for (int j = 0; j < 3; ++j)  // digits 2j + rank
            bulk_g2s(bring + bs * Sh::B_STAGE + j * Sh::B_PLANE,
                     blk + (2 * j + (int)rank) * Sh::B_PLANE, Sh::B_PLANE, &bfull[bs]);
          if (SPLIT) {
#pragma unroll
            for (int j = 0; j < 3; ++j)  // rank rows 32 rank .. of digit 2j
              bulk_g2s(bring + bs * Sh::B_STAGE + 3 * Sh::B_PLANE + j * Sh::B_HALF,
                       blk + 2 * j * Sh::B_PLANE + (int)rank * Sh::B_HALF, Sh::B_HALF,
                       &bfull[bs]);
          }
          if (++bs == NB) {
            bs = 0;
            bph ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 6) {
    // ---------------- forward landed core halves to the leader ----------------
    if (lane == 0) {
      const uint32_t ready = map_to_rank(bready, 0);
      int bs = 0;
      uint32_t bph = 0;
      for (int u = u_lo; u < u_hi; ++u) {
        int kc, g, tx;
        if (!live(u, kc, g, tx)) continue;
        for (int e = c_grp_off[o][g]; e < c_grp_off[o][g + 1]; ++e) {
          mbar_wait(&bfull[bs], bph);
          mbar_arrive_cluster_relaxed(ready + (uint32_t)(bs * 8));
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
    const uint32_t full0 = map_to_rank(pfull, 0);
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
      if (k >= 1) {  // the previous plane has landed: publish it to the leader
        cp_async_wait<1>();
        bfmm::tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(full0 + (uint32_t)(pl * 8));
        if (++pl == NP) pl = 0;
      }
      ++k;
      if (++ps == NP) {
        ps = 0;
        pph ^= 1u;
      }
    }
    cp_async_wait<0>();
    bfmm::tc::fence_proxy_async();
    __syncwarp();
    if (k >= 1 && lane == 0) mbar_arrive_cluster(full0 + (uint32_t)(pl * 8));

    // ---------------- drain this CTA's 128 TMEM lanes ----------------
    if (any) {
      mbar_wait_cluster(done, 0);
      bfmm::tc::fence_after();
    }
    const int quarter = warp & 3;
    const int er = 32 * quarter + lane;
    const int g2 = er >> 3, zl = er & 7;
    const int64_t cell = (int64_t)morton3(xs + 2 * (g2 % XT), 2 * (YT * yb + g2 / XT) + oy,
                                          2 * (8 * zb + zl) + oz);
    double *dst = lt + ((cell * m + col) * nsplit + split) * rp;
    i8_drain<S, 8, 8>(tmem + ((uint32_t)(32 * quarter) << 16), dst, i8_zscale(zmax[col]), nt, rp,
                      cpow, !any);
  }
  bfmm::tc::fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer is done with the shared TMEM allocation too
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// level >= 5 plane tiles (1 x 16 x 8) whose z-tile count is even: tiles
// pair up along z inside one CTA cluster
inline bool i8p2_ok(const I8Call &a, int4 *box) {
  if (a.level < 5 || getenv("BFMM_I8_1CTA")) return false;
  if (!i8_plane_box(a, 1, 16, box)) return false;
  return (box->w & 1023) % 2 == 0;
}

template <int NBMAX, bool SPLIT>
int launch_i8p2_nb(const I8Call &a, int4 box) {
  using Sh = I8P2Shape<NBMAX, SPLIT>;
  static unsigned long long attr_set = 0;
  if (first_on_device(&attr_set)) {
    cudaFuncSetAttribute(m2l_i8p2_kernel<NBMAX, SPLIT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::smem);
  }
  const int tiles = (box.w >> 20) * ((box.w >> 10) & 1023) * (box.w & 1023);
  dim3 grid((unsigned)tiles * 8, (unsigned)(a.ntn * a.m), a.nsplit);
  m2l_i8p2_kernel<NBMAX, SPLIT><<<grid, kI8P2Threads, Sh::smem, a.st>>>(
      a.zs, a.zmax, a.cs, a.cpow, a.lt, a.level, a.m, a.rp, a.kc_n, a.ntn, a.nsplit, box);
  return check_launch("m2l_i8p2_kernel");
}

// BFMM_I8P2_N128=1: the unsplit variant (24 products, 12 N = 128 MMAs)
inline int launch_i8p2(const I8Call &a, int4 box) {
  const char *cs = getenv("BFMM_I8_COSCHED");
  const char *un = getenv("BFMM_I8P2_N128");
  if (un && un[0] == '1')
    return (cs && cs[0] == '1') ? launch_i8p2_nb<6, false>(a, box)
                                : launch_i8p2_nb<12, false>(a, box);
  return (cs && cs[0] == '1') ? launch_i8p2_nb<6, true>(a, box)
                              : launch_i8p2_nb<12, true>(a, box);
}
