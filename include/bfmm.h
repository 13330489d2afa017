/*
 * bfmm.h — C ABI of the B200-native black-box FMM matvec (phi = K sigma).
 *
 * This is the drop-in boundary under the Python evaluator
 * (paper_1903_02153_b200.FmmEvaluator), which mirrors the reference's
 * FmmEvaluator.evaluate (engine.py:482-536).  The reference has no FFI of
 * its own (it is pure Python/NumPy); each entry point below
 * replaces one NumPy stage of that method and cites it.
 *
 * Conventions
 *  - Every pointer argument is DEVICE memory allocated by the caller
 *    (PyTorch in the shipped host), except where marked "host".
 *  - Every call is asynchronous on `stream` (a cudaStream_t) and returns 0
 *    on success; nonzero means a launch/config error whose text is
 *    available from bfmm_last_error().  No call synchronises except
 *    bfmm_kernel_compile (NVRTC) and bfmm_device_fp64_probe.
 *  - Internal data layouts (all float64, row-major):
 *      pts4      (N, 4)        sorted points x, y, z, weight column 0
 *      wsorted   (N, m)        sorted weights
 *      moments / locals (8^l, m, p^3)   dense over every cell of a level
 *      z / lt    (8^l, m, rp)  rank-space moments / local accumulators,
 *                              rp = rank padded to a multiple of 8
 *  - Cell ids are the reference's Morton ids (octree.py:75-107): x in the
 *    high bit of each bit triple, children of q are 8q..8q+7.
 */
#ifndef BFMM_H
#define BFMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *bfmm_stream_t; /* cudaStream_t */

/* ---- library ---------------------------------------------------------- */
const char *bfmm_last_error(void);
int bfmm_version(void);

/* ---- tree: distribute (engine.py:60-94, octree.py:186-200) ------------ */

/* Scratch bytes bfmm_tree_build needs for n points at `levels`. */
size_t bfmm_tree_scratch_bytes(int64_t n, int levels);

/* Leaf id per point (floor((x-lo)/h), clip, Morton; octree.py:186-200),
 * stable radix sort (== np.argsort(kind="stable"), engine.py:74),
 * run-length encode (== np.unique(return_index, return_counts),
 * engine.py:76-77), plus dense per-cell (start, count) maps.
 * geom (host) = {lo_x, lo_y, lo_z, hi_x, hi_y, hi_z, h, tol}.
 * domain_flag is set to 1 when a point lies outside [lo-tol, hi+tol]
 * (the DomainError of octree.py:190-196).  leaves/starts/counts have
 * capacity n; *n_leaves (device) receives the nonempty-leaf count. */
int bfmm_tree_build(const double *points, int64_t n, const double *geom,
                    int levels, void *scratch, size_t scratch_bytes,
                    int64_t *perm, double *pts4, int64_t *leaves,
                    int64_t *starts, int64_t *counts, int64_t *n_leaves,
                    int32_t *cell_start, int32_t *cell_count,
                    int32_t *domain_flag, bfmm_stream_t stream);

/* w (N, m) original order -> wsorted (N, m) and pts4[:, 3] = w[perm, 0]
 * (the weights[part.perm] of engine.py:168,528).  A non-finite weight sets
 * *weights_flag |= 1 (device; may be NULL) -- the reference's
 * ConfigurationError("weights contain non-finite values", engine.py:496-497). */
int bfmm_gather_weights(const double *w, int64_t n, int m,
                        const int64_t *perm, double *wsorted, double *pts4,
                        int32_t *weights_flag, bfmm_stream_t stream);

/* Active cells for sparse clouds: the sorted distinct ancestors
 * leaves[i] >> shift (shift = 3 * (levels - level)) of the n_leaves
 * (device) occupied leaves that lie in [lo, hi) -> list, their number ->
 * *count (device).  Only these cells' local expansions can reach a target
 * point (L2L / L2P descend from occupied cells only, engine.py:206-226), so
 * the M2L restricted to them (bfmm_m2l_cheb_list) gives the same phi. */
size_t bfmm_active_cells_scratch_bytes(int64_t max_leaves);
int bfmm_active_cells(const int64_t *leaves, const int64_t *n_leaves,
                      int64_t max_leaves, int shift, int64_t lo, int64_t hi,
                      void *scratch, size_t scratch_bytes, int64_t *list,
                      int64_t *count, bfmm_stream_t stream);
/* hist[o] (device, 8 entries) = number of the first *n_dev cells with
 * (cell & 7) == o. */
int bfmm_octant_histogram(const int64_t *cells, const int64_t *n_dev, int64_t max_n,
                          int64_t *hist, bfmm_stream_t stream);
/* out = cells stably grouped by octant (cell & 7), ascending within a group. */
size_t bfmm_group_by_octant_scratch_bytes(int64_t n);
int bfmm_group_by_octant(const int64_t *cells, int64_t n, int64_t *out, void *scratch,
                         size_t scratch_bytes, bfmm_stream_t stream);

/* ---- upward pass ------------------------------------------------------- */

/* P2M over leaf CELLS for sparse clouds (a few points per leaf): every
 * cell of the geom's range [cell_lo, cell_hi) gets its moments written,
 * zeros for empty cells (no memset of the level-L array needed); cell_start
 * / cell_count are the tree build's dense per-cell maps.  Same moments as
 * bfmm_p2m (engine.py:159-185).  2 <= p <= 8. */
int bfmm_p2m_cells(const double *pts4, const double *wsorted, int m,
                   const int32_t *cell_start, const int32_t *cell_count, int levels, int p,
                   int scheme, const double *interp, const double *geom, double *moments,
                   int32_t *ref_flag, bfmm_stream_t stream);

/* L2P over leaf CELLS for sparse clouds: the locals of a chunk of
 * consecutive cells of the geom's range are staged in shared memory, one
 * thread per point of the chunk.  Same phi as bfmm_l2p / bfmm_l2p_points
 * (engine.py:313-337; bitwise equal to bfmm_l2p_points).  2 <= p <= 8. */
int bfmm_l2p_cells(const double *pts4, int m, const int32_t *cell_start,
                   const int32_t *cell_count, int levels, int p, int scheme,
                   const double *interp, const double *geom, const double *locals,
                   double *phi_sorted, int32_t *ref_flag, bfmm_stream_t stream);

/* P2M leaf_moments (engine.py:159-185).  interp (host) holds the 1-D
 * basis: scheme 0 (Chebyshev) p*p coefficients S[n][j] = c_n T_n(x_j),
 * scheme 1 (uniform) p nodes followed by p*p inverse node differences.
 * geom (host) = {lo_x, lo_y, lo_z, h_leaf, cell_lo, cell_hi}: only leaves
 * whose Morton id lies in [cell_lo, cell_hi) are processed (a rank's shard;
 * [0, 8^L) for all).  moments must be zeroed by the caller; cells without
 * points stay zero.  ref_flag is set when a point's leaf-frame coordinate
 * exceeds 1 + 1e-9 (engine.py:339-345). */
int bfmm_p2m(const double *pts4, const double *wsorted, int m,
             const int64_t *leaves, const int64_t *starts,
             const int64_t *counts, const int64_t *n_leaves,
             int64_t max_leaves, int levels, int p, int scheme,
             const double *interp, const double *geom, double *moments,
             int32_t *ref_flag, bfmm_stream_t stream);
/* Same moments with one thread per (leaf, x-node) instead of a warp per
 * leaf: for sparse clouds of a few points per leaf (same products and
 * point order). */
int bfmm_p2m_sparse(const double *pts4, const double *wsorted, int m,
                    const int64_t *leaves, const int64_t *starts,
                    const int64_t *counts, const int64_t *n_leaves,
                    int64_t max_leaves, int levels, int p, int scheme,
                    const double *interp, const double *geom, double *moments,
                    int32_t *ref_flag, bfmm_stream_t stream);

/* M2M ascend (engine.py:187-204): parent[q] = sum_o T[o] child[8q+o] with
 * T[o] = kron(Hx, Hy, Hz) (interpolation.py:136-155).  H (host) holds the
 * two p x p half-interval matrices H[s][a][b], s = 0 lower / 1 upper half. */
int bfmm_m2m(const double *child, double *parent, int64_t n_parent, int p,
             int m, const double *H, bfmm_stream_t stream);

/* ---- far field --------------------------------------------------------- */

/* C = alpha * A @ B + beta * C for row-major A (rows, K), B (K, N),
 * C (rows, N).  A may be stored as a_splits blocks of K per row
 * (rows, a_splits, K); they are first summed in order IN PLACE into block 0
 * (A is modified).  Used for z = moments @ V and
 * locals = scale * lt @ U^T (engine.py:233, 252-255). */
int bfmm_rows_gemm(const double *A, int64_t rows, int K, const double *B,
                   int N, double *C, double alpha, double beta, int a_splits,
                   bfmm_stream_t stream);
/* bfmm_rows_gemm with beta = 0, a_splits = 1, K, N <= 128 on the persistent
 * DMMA kernel (B resident in shared memory), plus max |C| into *zmax (device,
 * zero it first; bit pattern of a non-negative double, atomicMax) -- the
 * digit scale bfmm_m2l_i8_slice_z takes with BFMM_I8_ZMAX_GIVEN for one
 * weight column (replaces its absmax pass). */
int bfmm_rows_gemm_max(const double *A, int64_t rows, int K, const double *B, int N,
                       double *C, double alpha, unsigned long long *zmax,
                       bfmm_stream_t stream);
/* C = alpha * A @ B on the int8 tensor cores (csrc/proj_i8.cuh), A (rows, K)
 * FP64 row-major, K, N <= 128: every A row is cut into six signed 8-bit
 * digits under its own power-of-two scale, B arrives pre-cut (bdig: the
 * digit image [ceil(N/64)][ceil(K/32)][6][64 x 32 K-major core matrices] of
 * B^T with one scale per column n, bpow[n] = 2^e_n -- the same layout and
 * builder as the M2L cores, engine._i8_core_slices), and the 21 digit
 * products with a + b < 6 are summed exactly in int32 TMEM (truncation
 * ~2^-46 of the row / column scales).  zmax (nullable, device): atomic max
 * of |C| as a double bit pattern (zero it first) -- the digit scale
 * bfmm_m2l_i8_slice_z needs, for one weight column.  Same C as
 * bfmm_rows_gemm with beta = 0, a_splits = 1 (engine.py:233, 252-255). */
int bfmm_rows_gemm_i8(const double *A, int64_t rows, int K, const int8_t *bdig,
                      const double *bpow, int N, double *C, double alpha,
                      unsigned long long *zmax, bfmm_stream_t stream);
/* Same, but A row r lands in C row groups[r / group_rows] * group_rows +
 * r % group_rows (compact rows of listed cells scattered to their cells). */
int bfmm_rows_gemm_scatter(const double *A, int64_t rows, int K,
                           const double *B, int N, double *C, double alpha,
                           double beta, int a_splits, const int64_t *groups,
                           int64_t group_rows, bfmm_stream_t stream);
/* Rows of listed cells only, in place in the level's arrays: for
 * r < rows, with cell row R = groups[r / group_rows] * group_rows +
 * r % group_rows, C[R] = alpha * A[R] @ B (A and C both indexed by R; the
 * other rows of C are not written).  The V projection z = M V of a sparse
 * cloud (engine.py:233): only the cells with sources below them have
 * moments, the caller zero-fills z once. */
int bfmm_rows_gemm_cells(const double *A, int64_t rows, int K, const double *B, int N,
                         double *C, double alpha, const int64_t *groups,
                         int64_t group_rows, bfmm_stream_t stream);

/* M2L Chebyshev (engine.py:228-256): for every cell c at `level` and
 * column, lt[c][i] = sum over the valid far offsets t of
 * sum_k cores[t][i][k] z[c + t][k], cores = C_t zero-padded to rp x rp.
 * The valid pairs follow octree.py:128-145 and match
 * cell_pairs_for_offset (octree.py:202-221) pair for pair.  FP64 tensor
 * cores (mma.sync m8n8k4 f64).  The 189 offsets of each cell are split into
 * nsplit contiguous ranges written to separate column blocks:
 * lt has layout (8^level, m, nsplit, rp) and the caller sums the blocks
 * (bfmm_rows_gemm with a_splits = nsplit does it while projecting).
 * Only target cells whose parent lies in [q_lo, q_lo + nq) are computed (a
 * rank's Morton shard; q_lo = 0, nq = 8^(level-1) for all); z must hold
 * every cell.  Warp-specialised: one producer warp gathers z rows and core
 * tiles with cp.async into an 8-stage mbarrier ring, 8 consumer warps run
 * the DMMAs. */
int bfmm_m2l_cheb_splits(int level, int m, int rp, int64_t nq);
int bfmm_m2l_cheb(const double *z, double *lt, int level, int m, int rp,
                  int nsplit, int64_t q_lo, int64_t nq, const double *cores,
                  bfmm_stream_t stream);
/* Same translation for listed target cells only (sparse clouds): cells
 * (device) holds the active cells grouped by octant -- cells[oct_off[o] ..
 * oct_off[o + 1]) have (cell & 7) == o -- and oct_off (host, 9 entries) the
 * group offsets (bfmm_active_cells at this level, bfmm_octant_histogram,
 * bfmm_group_by_octant).  lt is compact: row oct_off[o] + q for listed cell
 * q of octant o, layout (n_listed, m, nsplit, rp). */
int bfmm_m2l_cheb_cells(const double *z, double *lt, int level, int m, int rp,
                        int nsplit, const int64_t *cells, const int64_t *oct_off,
                        const double *cores, bfmm_stream_t stream);

/* Same translation on the int8 tensor cores (tcgen05.mma kind::i8, TMEM
 * accumulators; csrc/m2l_i8.cuh), FP64-accurate by error-free splitting:
 * z is cut into S signed 7-bit digit planes under one per-level power-of-two
 * scale, the cores into S planes under one scale per rank row i, and the
 * S(S+1)/2 digit products whose weights exceed 2^(-7S) are accumulated
 * exactly in int32.  Same lt layout and meaning as bfmm_m2l_cheb /
 * bfmm_m2l_cheb_cells (replaces engine.py:228-256, ops:217-237).
 *  - bfmm_m2l_i8_slice_z: z (rows x rp, FP64, row = cell * m + column) ->
 *    zs (bfmm_m2l_i8_zs_bytes bytes: [row][ceil(rp/32)][S][32] int8) and
 *    zmax (device, m x 8 bytes: the bit pattern of max|z| per weight column,
 *    the power-of-two scale of that column's digits).
 *  - cs: core digits, [316][ceil(rp/64)][ceil(rp/32)][S][64 x 32 K-major
 *    core-matrix image] int8; cpow: 2^(e_i) per rank row, ceil(rp/64)*64
 *    doubles (built on the host, engine._i8_core_slices).
 *  - S in 5..8, rp <= 256: S signed 7-bit digits per operand (base 2^7).
 *    S = 6 | BFMM_I8_BASE256: six signed 8-bit digits (base 2^8, 47 bits,
 *    21 digit products instead of the 28 of S = 7 at a comparable
 *    truncation), allowed while 6 K 2^14 < 2^31 for the K = offsets x 32 x
 *    ceil(rp/32) terms an accumulator sums (rp <= 96; <= 64 for the
 *    mixed-octant coarse levels). */
#define BFMM_I8_BASE256 0x100
/* S flag of bfmm_m2l_i8_slice_z: zmax holds the scales already (from
 * bfmm_m2l_i8_zmax, e.g. max-reduced over the ranks of a sharded matvec so
 * every shard cuts its digits exactly like the unsharded evaluation). */
#define BFMM_I8_ZMAX_GIVEN 0x200
size_t bfmm_m2l_i8_zs_bytes(int64_t rows, int rp, int S);
/* zmax[c] = bit pattern of max |z| over weight column c (the first half of
 * bfmm_m2l_i8_slice_z). */
int bfmm_m2l_i8_zmax(const double *z, int64_t rows, int m, int rp,
                     unsigned long long *zmax, bfmm_stream_t stream);
int bfmm_m2l_i8_slice_z(const double *z, int64_t rows, int m, int rp, int S,
                        int8_t *zs, unsigned long long *zmax, bfmm_stream_t stream);
/* Sparse clouds: the same for the m rows of each listed cell only (compact
 * row r = array row cells[r / m] * m + r % m of z and zs; rows = listed
 * cells x m).  The digit rows of the other cells are not written: the caller
 * zero-fills zs once (their z is zero).  Without BFMM_I8_ZMAX_GIVEN the scale
 * is taken over the listed rows. */
int bfmm_m2l_i8_slice_z_cells(const double *z, int64_t rows, int m, int rp, int S,
                              int8_t *zs, unsigned long long *zmax, const int64_t *cells,
                              bfmm_stream_t stream);
int bfmm_m2l_i8_splits(int level, int m, int rp, int64_t nq);
int bfmm_m2l_i8(const int8_t *zs, const unsigned long long *zmax, const int8_t *cs,
                const double *cpow, double *lt, int level, int m, int rp, int S,
                int nsplit, int64_t q_lo, int64_t nq, bfmm_stream_t stream);
int bfmm_m2l_i8_cells(const int8_t *zs, const unsigned long long *zmax,
                      const int8_t *cs, const double *cpow, double *lt, int level,
                      int m, int rp, int S, int nsplit, const int64_t *cells,
                      const int64_t *oct_off, bfmm_stream_t stream);

/* M2L uniform / FFT (engine.py:258-292): locals[c] = scale * crop(
 * irfft( sum_t S_t * rfft(pad(moments[c + t])) ) ) over the valid far
 * offsets t.  symbols (device) (316, q, q, q//2+1) complex128 interleaved
 * (the reference's rfftn symbols, ops:156-159).  Scratch for a chunk of
 * `cols` weight columns (X and Y spectra); bfmm_m2l_fft processes as many
 * columns per pass as its scratch holds. */
int bfmm_m2l_fft_scratch_bytes(int level, int cols, int p, size_t *bytes);
int bfmm_m2l_fft(const double *moments, double *locals, int level, int m,
                 int p, const double *symbols, double scale, int64_t q_lo,
                 int64_t nq, void *scratch, size_t scratch_bytes,
                 bfmm_stream_t stream);

/* ---- downward pass ----------------------------------------------------- */

/* L2L descend (engine.py:296-311): child[8q+o] += T[o]^T parent[q]. */
int bfmm_l2l(const double *parent, double *child, int64_t n_parent, int p,
             int m, const double *H, bfmm_stream_t stream);

/* L2P read_potentials (engine.py:313-337): phi_sorted[i] =
 * W(x_i) . locals[leaf(i)] (assigns; targets in sorted order).  geom as in
 * bfmm_p2m (rows of leaves outside [cell_lo, cell_hi) are left untouched). */
int bfmm_l2p(const double *pts4, int m, const int64_t *leaves,
             const int64_t *starts, const int64_t *counts,
             const int64_t *n_leaves, int64_t max_leaves, int levels, int p,
             int scheme, const double *interp, const double *geom,
             const double *locals, double *phi_sorted, int32_t *ref_flag,
             bfmm_stream_t stream);
/* Same contraction with one thread per sorted point (the point's leaf is
 * recomputed from its coordinates exactly as bfmm_tree_build bins it): for
 * sparse leaves of a few points, where a warp per leaf leaves lanes idle.
 * Bitwise-identical results to bfmm_l2p. */
int bfmm_l2p_points(const double *pts4, int m, const int64_t *leaves,
                    const int64_t *starts, const int64_t *counts,
                    const int64_t *n_leaves, int64_t max_leaves, int levels, int p,
                    int scheme, const double *interp, const double *geom,
                    const double *locals, double *phi_sorted, int32_t *ref_flag,
                    bfmm_stream_t stream);

/* Leaf-pair P2M / L2P for sparse clouds, one weight column, levels >= 3,
 * 2 <= p <= 8 (replaces engine.py:176-204 at the leaf level and
 * :296-327 below level L-1).  A warp per parent cell q of level L-1 and its
 * eight leaf children, whose points are contiguous in sorted order; the cell
 * range [cell_lo, cell_hi) of geom (whole parents) is the shard.
 *  - bfmm_p2m_pair: mom_leaf[c] (level L, every cell of the range, zeros for
 *    empty ones -- as bfmm_p2m_cells) and mom_parent[q] (level L-1) straight
 *    from the points with the parent's basis, i.e. M2M(M_L) exactly in exact
 *    arithmetic: the caller skips the L -> L-1 M2M.
 *  - bfmm_l2p_pair: phi_i = S_L(x_i) . loc_leaf[c] + S_{L-1}(x_i) .
 *    loc_parent[q], where loc_leaf holds the level-L M2L locals WITHOUT the
 *    parent's L2L part (which the second term supplies exactly): the caller
 *    skips the L-1 -> L L2L. */
int bfmm_p2m_pair(const double *pts4, const double *wsorted, const int32_t *cell_start,
                  const int32_t *cell_count, int levels, int p, int scheme,
                  const double *interp, const double *geom, double *mom_leaf,
                  double *mom_parent, int32_t *ref_flag, bfmm_stream_t stream);
int bfmm_l2p_pair(const double *pts4, const int32_t *cell_start, const int32_t *cell_count,
                  int levels, int p, int scheme, const double *interp, const double *geom,
                  const double *loc_leaf, const double *loc_parent, double *phi_sorted,
                  int32_t *ref_flag, bfmm_stream_t stream);

/* ---- near field (engine.py:349-478) ------------------------------------ */

/* Compile (NVRTC, cached by source) a P2P kernel for a device functor.
 * kind: 0 = expression in r (profile), 1 = expression in r2,
 * 2 = expression in dx, dy, dz (diff_func).  Returns a handle > 0 in
 * *handle.  Built-in handles (no JIT): 1 laplacian, 2 laplacianforce,
 * 3 gaussian, 4 exponential, 5 logarithm. */
int bfmm_kernel_compile(int kind, const char *expr, int *handle);

/* Scratch bytes bfmm_p2p needs for n_targets points in at most max_tleaves
 * occupied leaves (per-leaf chunk prefix, chunk -> leaf map, work counter).
 * n_targets = 0 gives the minimum, without the map (chunks are then located
 * by binary search). */
size_t bfmm_p2p_scratch_bytes(int64_t max_tleaves, int64_t n_targets);

/* out[i] = sum over the 27 neighbour leaves of the target leaf of
 * K(x_i - y_j) w_j, targets and sources both in sorted order; assigns the
 * rows of target leaves whose Morton id lies in [cell_lo, cell_hi) (a
 * rank's shard) and leaves the other rows untouched.  The source structure
 * is the dense per-cell (start, count) map of bfmm_tree_build. */
int bfmm_p2p(int handle, const double *tpts4, const int64_t *tleaves,
             const int64_t *tstarts, const int64_t *tcounts,
             const int64_t *n_tleaves, int64_t max_tleaves,
             const double *spts4, const double *swsorted, int m,
             const int32_t *scell_start, const int32_t *scell_count,
             int levels, int64_t cell_lo, int64_t cell_hi, double *out,
             void *scratch, size_t scratch_bytes, bfmm_stream_t stream);

/* bfmm_p2p with the target tree's dense cell map (tcell_start /
 * tcell_count of bfmm_tree_build): for one weight column the cells of <= 8
 * points run through p2p_tile_kernel -- a CTA per aligned 4 x 4 x 4 Morton
 * block of target cells with its 6 x 6 x 6 source halo staged in shared
 * memory, one thread per target, the same sums in the same order as the
 * thread-per-target path of bfmm_p2p (bitwise equal).  Same output and
 * sharding contract as bfmm_p2p (engine.py:349-478). */
int bfmm_p2p_cells(int handle, const double *tpts4, const int64_t *tleaves,
                   const int64_t *tstarts, const int64_t *tcounts,
                   const int64_t *n_tleaves, int64_t max_tleaves,
                   const int32_t *tcell_start, const int32_t *tcell_count,
                   const double *spts4, const double *swsorted, int m,
                   const int32_t *scell_start, const int32_t *scell_count,
                   int levels, int64_t cell_lo, int64_t cell_hi, double *out,
                   void *scratch, size_t scratch_bytes, bfmm_stream_t stream);

/* Symmetric near field for shared targets = sources and a kernel with
 * K(y, x) = sign K(x, y) (the reference's transpose replay,
 * engine.py:361-364, 442-457): each unordered neighbour-leaf pair is
 * evaluated once; a leaf's own points accumulate their row sums over its 14
 * half-neighbours in registers (slot 0), the partner leaf's points receive
 * the column sums in slot h of the half-neighbour offset, and the 14 slots
 * are added in a fixed order (deterministic, no atomics).  Writes
 * out (nt rows, m = 1) for every point touched; when a leaf holds more than
 * 64 points the library falls back to bfmm_p2p on the device (no host
 * synchronisation).  Leaves outside [cell_lo, cell_hi) start no pairs; the
 * pairs a shard starts may add to other shards' rows (sum across ranks). */
size_t bfmm_p2p_symmetric_scratch_bytes(int64_t nt, int64_t max_tleaves);
int bfmm_p2p_symmetric(int handle, const double *pts4, const int64_t *leaves,
                       const int64_t *starts, const int64_t *counts,
                       const int64_t *n_leaves, int64_t max_leaves,
                       const int32_t *cell_start, const int32_t *cell_count,
                       int levels, int64_t cell_lo, int64_t cell_hi, int64_t nt,
                       double sign, double *out, void *scratch,
                       size_t scratch_bytes, bfmm_stream_t stream);

/* Kernel values on point-pair grids for the M2L table build on the device
 * (replaces the host assembly of operators.py:244-258 `_dense_family` and
 * operators.py:88-108 `uniform_difference_grid`):
 *   out[t][a][b] = K(xt[a] - (ys[b] + shift[t]))   t < nt, a < na, b < nb
 * with the functor `handle` (built-in or NVRTC).  xt (na, 3), ys (nb, 3),
 * shift (nt, 3) device arrays; a non-finite value sets *bad |= 1 (device). */
int bfmm_kernel_block(int handle, const double *xt, int64_t na, const double *ys,
                      int64_t nb, const double *shift, int nt, double *out,
                      int32_t *bad, bfmm_stream_t stream);

/* Direct O(nt * ns) sum, the reference's direct_evaluate (engine.py:565-624):
 * out[i][c] = sum_j K(t_i - s_j) w[j][c] with explicit differences
 * (coincident points give r = 0 exactly) and Neumaier-compensated
 * accumulation in place of 80-bit long double.  tpts (nt, 3), spts (ns, 3),
 * w (ns, m), out (nt, m). */
int bfmm_direct(int handle, const double *tpts, int64_t nt, const double *spts,
                const double *w, int64_t ns, int m, double *out,
                bfmm_stream_t stream);

/* Near field for sparse clouds (a few points per leaf, one weight column):
 * the same sums as bfmm_p2p in the same (neighbour-order) sequence, one
 * thread per target and 8 consecutive target leaves per warp, without the
 * 32-target chunk prefix (no scratch).  Replaces engine.py:349-478 like
 * bfmm_p2p. */
int bfmm_p2p_grouped(int handle, const double *tpts4, const int64_t *tleaves,
                     const int64_t *tstarts, const int64_t *tcounts, const int64_t *n_tleaves,
                     int64_t max_tleaves, const double *spts4, const int32_t *scell_start,
                     const int32_t *scell_count, int levels, int64_t cell_lo, int64_t cell_hi,
                     double *out, bfmm_stream_t stream);

/* Locate the first non-finite kernel value in the near field in the
 * reference's enumeration order (offset, target row, source row;
 * engine.py:362-441).  *key (device, init UINT64_MAX) receives
 * (offset << 58) | (target_row << 29) | source_row. */
int bfmm_p2p_locate(int handle, const double *tpts4, const int64_t *tleaves,
                    const int64_t *tstarts, const int64_t *tcounts,
                    const int64_t *n_tleaves, int64_t max_tleaves,
                    const double *spts4, const int32_t *scell_start,
                    const int32_t *scell_count, int levels,
                    unsigned long long *key, bfmm_stream_t stream);

/* phi[perm[i]] = far_sorted[i] + near_sorted[i] (engine.py:530);
 * nonfinite_flag is set when a near-field sum is non-finite. */
int bfmm_scatter_output(const double *far_sorted, const double *near_sorted,
                        const int64_t *perm, int64_t n, int m, double *phi,
                        int32_t *nonfinite_flag, bfmm_stream_t stream);

/* ---- interaction lists (parity / diagnostics) ------------------------- */

/* Far pairs of one offset t_index (0..315, lexicographic) at `level` in
 * the reference's meshgrid order: identical to
 * Octree.cell_pairs_for_offset (octree.py:202-221).  Built from the same
 * far_pair() rule bfmm_m2l_cheb applies.  tg/sr capacity 8^level; *count
 * (device) receives the pair count. */
size_t bfmm_far_pairs_scratch_bytes(int level);
int bfmm_far_pairs(int level, int t_index, int64_t *tg, int64_t *sr,
                   int64_t *count, void *scratch, size_t scratch_bytes,
                   bfmm_stream_t stream);

/* Near list of neighbour offset t_index (0..26, lexicographic) like
 * FmmEvaluator._neighbor_segments (engine.py:401-417): out[i] = index of
 * the nonempty source leaf at tleaves[i] + t, or -1. */
int bfmm_near_pairs(int levels, int t_index, const int64_t *tleaves,
                    const int64_t *n_tleaves, int64_t max_tleaves,
                    const int64_t *sleaves, const int64_t *n_sleaves,
                    int64_t *out, bfmm_stream_t stream);

/* Ordered near-field point pairs (timings["near_pairs"], engine.py:532). */
int bfmm_near_pair_count(const int64_t *tleaves, const int64_t *tcounts,
                         const int64_t *n_tleaves, int64_t max_tleaves,
                         const int32_t *scell_count, int levels,
                         int64_t *total, bfmm_stream_t stream);

/* bins[c] (device, 64) = work of the target leaves under level-2 cell c:
 * sum over its leaves of count * (1 + sources in the 27 neighbour leaves).
 * Feeds work-balanced Morton shard boundaries (parallel.py). */
int bfmm_level2_work(const int64_t *tleaves, const int64_t *tcounts,
                     const int64_t *n_tleaves, int64_t max_tleaves,
                     const int32_t *scell_count, int levels, int64_t *bins,
                     bfmm_stream_t stream);

/* ---- diagnostics ------------------------------------------------------- */

/* Measure the FP64 FMA peak of this device (GFLOP/s) with a DFMA chain
 * kernel (synchronises). */
int bfmm_device_fp64_probe(double *gflops, bfmm_stream_t stream);

/* Same for the FP64 tensor-core MMA (mma.sync m8n8k4 f64 -> DMMA). */
int bfmm_device_dmma_probe(double *gflops, bfmm_stream_t stream);
/* tcgen05 self-test (diagnostic): D (128 x 64, int32, row-major) = A (128 x K,
 * int8, row-major) * B (64 x K, int8, row-major)^T on the 5th-gen tensor
 * cores (kind::i8, TMEM accumulator); K a multiple of 32. */
int bfmm_tc_i8_selftest(const int8_t *A, const int8_t *B, int K, int32_t *D,
                        bfmm_stream_t stream);

/* Dense int8 tensor-core throughput (tcgen05.mma kind::i8, 128 x 256 x 32
 * MMAs back to back from shared memory, one CTA per SM) in TOPS: the peak
 * the int8 M2L (bfmm_m2l_i8) is measured against. */
int bfmm_device_i8_probe(double *tops, bfmm_stream_t stream);
/* The same with 128 x N x 32 MMAs, N in {64, 128, 192, 256} (shape sweep). */
int bfmm_device_i8_probe_n(int N, double *tops, bfmm_stream_t stream);

/* DMMA throughput with warps_per_sm resident warps x `chains` independent
 * accumulator chains (microarchitecture sweep behind the M2L tiling). */
int bfmm_device_dmma_sweep(int warps_per_sm, int chains, double *gflops,
                           bfmm_stream_t stream);

/* Number of kernels this library has launched in this process (own
 * kernels plus the CUB sort/scan kernels it invokes). */
long long bfmm_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* BFMM_H */
