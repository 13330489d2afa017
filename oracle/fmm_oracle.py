"""CPU ORACLE for the black-box FMM matvec — TEST INFRASTRUCTURE ONLY.

This module is a plain-NumPy restatement of the reference algorithm
(``boxfmm`` inside ``arxiv/paper_1903_02153``; abbreviations below:
``eng`` = pkg/src/boxfmm/engine.py, ``oct`` = octree.py, ``itp`` =
interpolation.py, ``ops`` = operators.py, ``ker`` = kernel.py).  It exists
so that the CUDA product can be checked on the GPU box, where the
reference itself is not available.

Rules:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
  baseline / ``--impl reference`` arm may import this module.  The product
  package (``paper_1903_02153_b200``) never does.
* Parity of this oracle is PINNED against the real reference: the
  fixtures under ``tests/golden/`` were produced by importing the
  reference from ``/root/reference`` (script: tests/golden/make_golden.py)
  and ``tests/test_oracle_golden.py`` checks this module against them.

Kernels are passed duck-typed: any object with ``name``, ``homogen``,
``symmetry`` and one of ``profile`` / ``diff_func`` / ``pair_func``
(numpy callables), exactly the reference ``KernelSpec`` contract
(ker:53-84).
"""

from __future__ import annotations

import itertools
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

try:  # pin BLAS to one thread inside the matvec, like the reference (eng:501)
    from threadpoolctl import threadpool_limits
except Exception:  # pragma: no cover
    threadpool_limits = None


class OracleDomainError(ValueError):
    pass


class OracleKernelError(ValueError):
    def __init__(self, msg, indices=None):
        super().__init__(msg)
        self.indices = indices


# ----------------------------------------------------------------------------
# Morton geometry (oct:75-145)
# ----------------------------------------------------------------------------

_SPREAD_MASKS = ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF),
                 (8, 0x100F00F00F00F00F), (4, 0x10C30C30C30C30C3),
                 (2, 0x1249249249249249))


def spread3(v):
    """Put bit b of a 21-bit integer at bit 3b (standard magic-number
    interleave; oct:75-83)."""
    x = np.asarray(v).astype(np.uint64) & np.uint64((1 << 21) - 1)
    for shift, mask in _SPREAD_MASKS:
        x = (x | (x << np.uint64(shift))) & np.uint64(mask)
    return x


def morton(ix, iy, iz):
    """Cell id with x in the most significant bit of each triple (oct:86-93)."""
    return ((spread3(ix) << np.uint64(2)) | (spread3(iy) << np.uint64(1))
            | spread3(iz)).astype(np.int64)


def unmorton(ids, level):
    """Inverse of :func:`morton` for ``level`` bit triples (oct:96-107)."""
    ids = np.asarray(ids, dtype=np.int64)
    out = [np.zeros_like(ids) for _ in range(3)]
    for b in range(level):
        tri = (ids >> (3 * b)) & 7
        for axis in range(3):
            out[axis] |= ((tri >> (2 - axis)) & 1) << b
    return tuple(out)


def far_offsets():
    """(316, 3) lexicographic offsets of max-norm 2 or 3 (oct:110-119)."""
    rng = range(-3, 4)
    return np.array([t for t in itertools.product(rng, rng, rng)
                     if max(map(abs, t)) >= 2], dtype=np.int64)


def near_offsets():
    """(27, 3) lexicographic offsets of max-norm <= 1 (oct:122-125)."""
    rng = range(-1, 2)
    return np.array(list(itertools.product(rng, rng, rng)), dtype=np.int64)


FAR = far_offsets()
NEAR = near_offsets()


def axis_targets(n, t):
    """Target coordinates along one axis with source = target + t inside
    [0, n); a +3 step needs an even target, a -3 step an odd one
    (oct:128-145)."""
    lo, hi = max(0, -t), min(n - 1, n - 1 - t)
    if hi < lo:
        return np.zeros(0, np.int64)
    c = np.arange(lo, hi + 1, dtype=np.int64)
    if abs(t) == 3:
        c = c[(c & 1) == (0 if t > 0 else 1)]
    return c


def offset_pairs(level, t):
    """(targets, sources) for all cells at ``level`` with source = target + t,
    enumerated in meshgrid(ij) order (oct:202-221)."""
    n = 1 << level
    axes = [axis_targets(n, int(c)) for c in t]
    if min(a.size for a in axes) == 0:
        e = np.zeros(0, np.int64)
        return e, e
    gx, gy, gz = (g.ravel() for g in np.meshgrid(*axes, indexing="ij"))
    return morton(gx, gy, gz), morton(gx + t[0], gy + t[1], gz + t[2])


# ----------------------------------------------------------------------------
# Domain + leaf binning (oct:26-65, 186-200; eng:60-94)
# ----------------------------------------------------------------------------

def domain_low_high(center, length):
    c = np.asarray(center, dtype=np.float64)
    half = 0.5 * length
    return c - half, c + half


def leaf_of(points, center, length, levels):
    """Leaf id per point: floor((x - lo)/h) clipped to the grid (oct:186-200)."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    lo, hi = domain_low_high(center, length)
    tol = 1e-12 * length
    if pts.size and (np.any(pts < lo - tol) or np.any(pts > hi + tol)):
        raise OracleDomainError("point outside the domain box")
    n = 1 << levels
    g = np.floor((pts - lo) / (length / n)).astype(np.int64)
    np.clip(g, 0, n - 1, out=g)
    return morton(g[:, 0], g[:, 1], g[:, 2])


class Binned:
    """Points stably sorted by leaf id (eng:71-80)."""

    def __init__(self, points, center, length, levels):
        ids = (leaf_of(points, center, length, levels) if len(points)
               else np.zeros(0, np.int64))
        self.perm = np.argsort(ids, kind="stable")
        self.points = points[self.perm]
        self.leaves, self.starts, self.counts = np.unique(
            ids[self.perm], return_index=True, return_counts=True)
        self.grid = unmorton(self.leaves, levels)

    @property
    def n(self):
        return self.points.shape[0]


# ----------------------------------------------------------------------------
# Interpolation (itp:47-155)
# ----------------------------------------------------------------------------

def nodes(p, scheme):
    """Ascending Chebyshev roots or equispaced nodes on [-1, 1] (itp:47-56)."""
    if p == 1:
        return np.zeros(1)
    if scheme == "chebyshev":
        k = np.arange(p, 0, -1)
        return np.cos(np.pi * (2 * k - 1) / (2 * p))
    return np.linspace(-1.0, 1.0, p)


def weights_1d(x, p, scheme):
    """(n, p) interpolation weights at points x (itp:66-90)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    nd = nodes(p, scheme)
    if scheme == "chebyshev":
        deg = np.arange(p)
        tx = np.cos(np.outer(deg, np.arccos(np.clip(x, -1.0, 1.0))))
        tn = np.cos(np.outer(deg, np.arccos(np.clip(nd, -1.0, 1.0))))
        coef = np.where(deg == 0, 1.0 / p, 2.0 / p)
        return tx.T @ (coef[:, None] * tn)
    w = np.ones((x.size, p))
    for j in range(p):
        for k in range(p):
            if k != j:
                w[:, j] *= (x - nd[k]) / (nd[j] - nd[k])
    return w


def weights_3d(ref, p, scheme):
    """(n, p^3) tensor weights, z fastest: a = (i*p + j)*p + k (itp:117-133)."""
    wx, wy, wz = (weights_1d(ref[:, a], p, scheme) for a in range(3))
    return (wx[:, :, None, None] * wy[:, None, :, None]
            * wz[:, None, None, :]).reshape(ref.shape[0], p ** 3)


def node_grid(p, scheme, half_width):
    nd = nodes(p, scheme)
    g = np.meshgrid(nd, nd, nd, indexing="ij")
    return half_width * np.stack([a.ravel() for a in g], axis=1)


def child_transfers(p, scheme):
    """(8, p^3, p^3): T[o][a, b] = parent node a's weight at child o's node b
    (itp:136-155)."""
    nd = nodes(p, scheme)
    lo = weights_1d(0.5 * nd - 0.5, p, scheme).T
    hi = weights_1d(0.5 * nd + 0.5, p, scheme).T
    out = np.empty((8, p ** 3, p ** 3))
    for o in range(8):
        fx, fy, fz = (hi if (o >> s) & 1 else lo for s in (2, 1, 0))
        out[o] = np.kron(fx, np.kron(fy, fz))
    return out


# ----------------------------------------------------------------------------
# Kernel evaluation (ker:104-127; eng:105-113)
# ----------------------------------------------------------------------------

def kernel_from_diffs(kernel, dx, dy, dz):
    if kernel.profile is not None:
        return kernel.profile(np.sqrt(dx * dx + dy * dy + dz * dz))
    if kernel.diff_func is not None:
        return kernel.diff_func(dx, dy, dz)
    raise ValueError("kernel has no difference form")


def kernel_rows(kernel, a, b):
    """K(a[i], b[i]) for matched rows."""
    if kernel.profile is not None or kernel.diff_func is not None:
        return kernel_from_diffs(kernel, a[:, 0] - b[:, 0], a[:, 1] - b[:, 1],
                                 a[:, 2] - b[:, 2])
    return np.array([kernel.pair_func(x, y) for x, y in zip(a, b)])


def kernel_matrix(kernel, X, Y):
    if kernel.profile is not None or kernel.diff_func is not None:
        return kernel_from_diffs(kernel, X[:, 0, None] - Y[None, :, 0],
                                 X[:, 1, None] - Y[None, :, 1],
                                 X[:, 2, None] - Y[None, :, 2])
    return np.array([[kernel.pair_func(x, y) for y in Y] for x in X])


# ----------------------------------------------------------------------------
# M2L tables (ops:74-378)
# ----------------------------------------------------------------------------

MIRROR = np.array([{tuple(t): j for j, t in enumerate(FAR)}[tuple(-t)] for t in FAR])


def dense_translation(kernel, t, p, scheme, width):
    """D_t[a, b] = K(target node a, source node b), source cell at t*width
    (ops:74-85)."""
    tn = node_grid(p, scheme, 0.5 * width)
    d = kernel_matrix(kernel, tn, tn + np.asarray(t, np.float64) * width)
    if not np.all(np.isfinite(d)):
        raise OracleKernelError("non-finite kernel value on the node grid")
    return d


def _family(kernel, p, scheme, width):
    sym = kernel.symmetry in (-1, 1)
    mats = {j: dense_translation(kernel, FAR[j], p, scheme, width)
            for j in range(len(FAR)) if (not sym or tuple(FAR[j]) > (0, 0, 0))}

    def get(j):
        return mats[j] if j in mats else kernel.symmetry * mats[MIRROR[j]].T
    return mats, get


def _stacked_svd(blocks, p3):
    """Right singular vectors/values of a tall stack via a running R-only QR
    that flushes every max(4 p^3, 2048) rows (ops:269-293)."""
    R, pending, rows = None, [], 0
    flush = max(4 * p3, 2048)
    for b in blocks:
        pending.append(b)
        rows += b.shape[0]
        if rows >= flush:
            R = np.linalg.qr(np.vstack(([R] if R is not None else []) + pending), mode="r")
            pending, rows = [], 0
    if pending or R is None:
        R = np.linalg.qr(np.vstack(([R] if R is not None else []) + pending), mode="r")
    _, s, vt = np.linalg.svd(R, full_matrices=False)
    return vt, s


def _cut(s, eps):
    return max(1, int(np.count_nonzero(s >= eps * s[0])))


def chebyshev_block(kernel, p, width, eps):
    """U, V, cores for one width (ops:300-329)."""
    p3 = p ** 3
    mats, get = _family(kernel, p, "chebyshev", width)
    vt_u, s_u = _stacked_svd((get(j).T for j in range(len(FAR))), p3)
    if kernel.symmetry in (-1, 1):
        r = _cut(s_u, eps)
        u = np.ascontiguousarray(vt_u[:r].T)
        v = u
        cores = np.empty((len(FAR), r, r))
        for j, d in mats.items():
            cores[j] = u.T @ d @ u
            cores[MIRROR[j]] = kernel.symmetry * cores[j].T
    else:
        vt_v, s_v = _stacked_svd((get(j) for j in range(len(FAR))), p3)
        r = max(_cut(s_u, eps), _cut(s_v, eps))
        u = np.ascontiguousarray(vt_u[:r].T)
        v = np.ascontiguousarray(vt_v[:r].T)
        cores = np.stack([u.T @ get(j) @ v for j in range(len(FAR))])
    return {"kind": "chebyshev", "width": width, "u": u, "v": v, "cores": cores}


def difference_grid(kernel, t, p, width):
    """Kernel on the wrapped (2p-1)^3 node-difference grid (ops:88-108)."""
    q = 2 * p - 1
    d = np.arange(q)
    d = np.where(d < p, d, d - q).astype(np.float64)
    h = width / max(p - 1, 1)
    u = [h * d - t[a] * width for a in range(3)]
    vals = kernel_from_diffs(kernel, u[0][:, None, None], u[1][None, :, None],
                             u[2][None, None, :])
    if not np.all(np.isfinite(vals)):
        raise OracleKernelError("non-finite kernel value on the difference grid")
    return vals


def uniform_block(kernel, p, width):
    grids = np.stack([difference_grid(kernel, t, p, width) for t in FAR])
    return {"kind": "uniform", "width": width, "grids": grids,
            "symbols": np.fft.rfftn(grids, axes=(1, 2, 3))}


def build_tables(kernel, levels, order, scheme, eps, length, force_per_level=False):
    """{level or 0: block}, single-level key 0 for homogeneous kernels
    (ops:344-378).  Returns (blocks, single)."""
    single = kernel.homogen != 0.0 and not force_per_level
    widths = {0: 1.0} if single else {l: length / 2 ** l for l in range(2, levels + 1)}
    blocks = {}
    for lev, w in widths.items():
        blocks[lev] = (chebyshev_block(kernel, order, w, eps) if scheme == "chebyshev"
                       else uniform_block(kernel, order, w))
    return blocks, single


def level_scale(kernel, single, length, level):
    """width^m for single-level tables (ops:188-192)."""
    return (length / 2 ** level) ** kernel.homogen if single else 1.0


# ----------------------------------------------------------------------------
# The matvec (eng:159-536)
# ----------------------------------------------------------------------------

def _split(n, k):
    k = max(1, min(k, n))
    e = np.linspace(0, n, k + 1).astype(np.int64)
    return [(int(e[i]), int(e[i + 1])) for i in range(k) if e[i + 1] > e[i]]


def _pool_map(fn, items, threads):
    if threads <= 1 or len(items) <= 1:
        return [fn(x) for x in items]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, items))


class OracleFMM:
    """Kernel + plan parameters + tables; :meth:`matvec` is the FMM."""

    def __init__(self, kernel, levels, order, scheme="chebyshev", eps=1e-5,
                 center=(0.0, 0.0, 0.0), length=1.0, threads=1, tables=None,
                 force_per_level=False):
        self.kernel = kernel
        self.L, self.p = int(levels), int(order)
        self.scheme = str(getattr(scheme, "value", scheme)).lower()
        self.eps = eps
        self.center = tuple(float(c) for c in center)
        self.length = float(length)
        self.threads = max(1, int(threads))
        self.T = child_transfers(self.p, self.scheme)
        if tables is None:
            tables = build_tables(kernel, self.L, self.p, self.scheme, eps,
                                  self.length, force_per_level)
        self.blocks, self.single = tables
        self.disable_far = False
        self.stage = {}

    def block(self, lev):
        return self.blocks[0] if self.single else self.blocks[lev]

    def scale(self, lev):
        return level_scale(self.kernel, self.single, self.length, lev)

    def leaf_geometry(self, binned):
        h = self.length / (1 << self.L)
        lo, _ = domain_low_high(self.center, self.length)
        g = np.stack(binned.grid, axis=1).astype(np.float64)
        return lo + (g + 0.5) * h, 0.5 * h

    def ref_coords(self, binned, rows):
        """Leaf-frame coordinates of sorted rows [a, b) clipped to [-1, 1]
        after the eng:339-345 sanity bound."""
        centers, hw = self.leaf_geometry(binned)
        seg = np.repeat(np.arange(len(binned.leaves)), binned.counts)
        ref = (binned.points[rows] - centers[seg[rows]]) / hw
        if ref.size and np.max(np.abs(ref)) > 1.0 + 1e-9:
            raise OracleDomainError("point landed outside its leaf")
        return np.clip(ref, -1.0, 1.0), seg[rows]

    # P2M (eng:159-185)
    def p2m(self, src, w):
        p3, m = self.p ** 3, w.shape[1]
        M = np.zeros((8 ** self.L, p3, m))
        if src.n == 0:
            return M
        ws = w[src.perm]
        leaf_chunks = _split(len(src.leaves), self.threads * 4)

        def work(rng):
            a, b = rng
            r0, r1 = int(src.starts[a]), int(src.starts[b - 1] + src.counts[b - 1])
            ref, _ = self.ref_coords(src, slice(r0, r1))
            W = weights_3d(ref, self.p, self.scheme)
            rel = src.starts[a:b] - r0
            for c in range(m):
                M[src.leaves[a:b], :, c] = np.add.reduceat(W * ws[r0:r1, c, None], rel, axis=0)
        _pool_map(work, leaf_chunks, self.threads)
        return M

    # M2M (eng:187-204)
    def m2m(self, M_leaf):
        levels = {self.L: M_leaf}
        for lev in range(self.L, 2, -1):
            ch = levels[lev]
            n, p3, m = ch.shape
            par = np.zeros((n // 8, p3, m))
            for o in range(8):
                par += np.einsum("ab,nbc->nac", self.T[o], ch[o::8], optimize=True)
            levels[lev - 1] = par
        return levels

    # M2L (eng:208-292)
    def m2l(self, lev, M):
        blk = self.block(lev)
        n, p3, m = M.shape
        pairs = [offset_pairs(lev, t) for t in FAR]
        groups = [list(range(g, len(FAR), self.threads)) for g in range(min(self.threads, len(FAR)))]
        if blk["kind"] == "chebyshev":
            r = blk["u"].shape[1]
            Z = np.ascontiguousarray(np.einsum("ar,nac->rnc", blk["v"], M, optimize=True))

            def work(js):
                acc = np.zeros((r, n, m))
                for j in js:
                    tg, sr = pairs[j]
                    if tg.size:
                        acc[:, tg] += (blk["cores"][j] @ Z[:, sr].reshape(r, -1)).reshape(r, tg.size, m)
                return acc
            acc = sum(_pool_map(work, groups, self.threads))
            out = np.ascontiguousarray(np.einsum("ar,rnc->nac", blk["u"], acc, optimize=True))
        else:
            p, q = self.p, 2 * self.p - 1
            x = np.zeros((n, m, q, q, q))
            x[:, :, :p, :p, :p] = M.transpose(0, 2, 1).reshape(n, m, p, p, p)
            X = np.fft.rfftn(x, axes=(2, 3, 4))
            del x
            sym = blk["symbols"]

            def work(js):
                acc = np.zeros_like(X)
                for j in js:
                    tg, sr = pairs[j]
                    if tg.size:
                        acc[tg] += sym[j] * X[sr]
                return acc
            Y = sum(_pool_map(work, groups, self.threads))
            y = np.fft.irfftn(Y, s=(q, q, q), axes=(2, 3, 4))[:, :, :p, :p, :p]
            out = np.ascontiguousarray(y.reshape(n, m, p3).transpose(0, 2, 1))
        s = self.scale(lev)
        return out * s if s != 1.0 else out

    # L2L (eng:296-311)
    def l2l(self, locs):
        for lev in range(2, self.L):
            par, ch = locs[lev], locs[lev + 1]
            for o in range(8):
                ch[o::8] += np.einsum("ba,nbc->nac", self.T[o], par, optimize=True)
        return locs[self.L]

    # L2P (eng:313-337)
    def l2p(self, tgt, Lleaf, phi):
        if tgt.n == 0:
            return

        def work(rng):
            r0, r1 = rng
            ref, seg = self.ref_coords(tgt, slice(r0, r1))
            W = weights_3d(ref, self.p, self.scheme)
            phi[tgt.perm[r0:r1]] = np.einsum("na,nac->nc", W, Lleaf[tgt.leaves[seg]])
        _pool_map(work, _split(tgt.n, self.threads * 4), self.threads)

    # P2P (eng:349-478) — all 27 ordered offsets, no transpose replay
    def p2p(self, tgt, src, ws):
        out = np.zeros((tgt.n, ws.shape[1]))
        if tgt.n == 0 or src.n == 0:
            return out, 0
        nl = 1 << self.L
        ix, iy, iz = tgt.grid
        tasks = []
        for t in NEAR:
            jx, jy, jz = ix + t[0], iy + t[1], iz + t[2]
            ok = (jx >= 0) & (jx < nl) & (jy >= 0) & (jy < nl) & (jz >= 0) & (jz < nl)
            ids = morton(jx[ok], jy[ok], jz[ok])
            pos = np.minimum(np.searchsorted(src.leaves, ids), len(src.leaves) - 1)
            hit = src.leaves[pos] == ids
            tseg, sseg = np.nonzero(ok)[0][hit], pos[hit]
            sizes = tgt.counts[tseg] * src.counts[sseg]
            # ~4M point pairs per task (eng:44-45)
            cum = np.cumsum(sizes)
            a = 0
            while a < len(sizes):
                base = cum[a - 1] if a else 0
                b = min(max(int(np.searchsorted(cum, base + 4_000_000)) + 1, a + 1), len(sizes))
                tasks.append((tseg[a:b], sseg[a:b]))
                a = b

        def work(task):
            tseg, sseg = task
            tc, sc = tgt.counts[tseg], src.counts[sseg]
            sizes = tc * sc
            tot = int(sizes.sum())
            pid = np.repeat(np.arange(len(sizes)), sizes)
            within = np.arange(tot) - np.repeat(np.cumsum(sizes) - sizes, sizes)
            rt = tgt.starts[tseg][pid] + within // sc[pid]
            rs = src.starts[sseg][pid] + within % sc[pid]
            vals = kernel_rows(self.kernel, tgt.points[rt], src.points[rs])
            bad = ~np.isfinite(vals)
            if bad.any():
                i = int(np.argmax(bad))
                ti, si = int(tgt.perm[rt[i]]), int(src.perm[rs[i]])
                raise OracleKernelError(
                    f"non-finite kernel value for target {ti} and source {si}", (ti, si))
            part = np.zeros_like(out)
            for c in range(ws.shape[1]):
                part[:, c] = np.bincount(rt, weights=vals * ws[rs, c], minlength=tgt.n)
            return part, tot
        res = _pool_map(work, tasks, self.threads)
        for part, _ in res:
            out += part
        return out, int(sum(n for _, n in res))

    def _prep(self, sources, targets, weights):
        src = np.ascontiguousarray(sources, dtype=np.float64)
        shared = targets is None or targets is sources
        tgt = src if shared else np.ascontiguousarray(targets, dtype=np.float64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        squeeze = w.ndim == 1
        return src, tgt, shared, (w[:, None] if squeeze else w), squeeze

    def matvec(self, sources, targets=None, weights=None):
        src_pts, tgt_pts, shared, w, squeeze = self._prep(sources, targets, weights)
        ctx = threadpool_limits(limits=1) if threadpool_limits else _Null()
        with ctx:
            src = Binned(src_pts, self.center, self.length, self.L)
            tgt = src if shared else Binned(tgt_pts, self.center, self.length, self.L)
            phi = np.zeros((tgt_pts.shape[0], w.shape[1]))
            M = self.m2m(self.p2m(src, w))
            self.stage = {"src": src, "tgt": tgt, "M": M}
            if not self.disable_far:
                locs = {lev: self.m2l(lev, M[lev]) for lev in range(2, self.L + 1)}
                self.stage["m2l"] = {k: v.copy() for k, v in locs.items()}
                self.l2p(tgt, self.l2l(locs), phi)
                self.stage["locals"] = locs  # after L2L (eng:296-311)
            near, npairs = self.p2p(tgt, src, w[src.perm])
            phi[tgt.perm] += near
            self.stage["near_pairs"] = npairs
        return phi[:, 0] if squeeze else phi


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ----------------------------------------------------------------------------
# Direct sum (eng:565-624), extended-precision accumulation
# ----------------------------------------------------------------------------

def direct_sum(kernel, sources, targets=None, weights=None, tb=1024, sb=8192):
    shared = targets is None or targets is sources
    src = np.ascontiguousarray(sources, dtype=np.float64)
    tgt = src if shared else np.ascontiguousarray(targets, dtype=np.float64)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    squeeze = w.ndim == 1
    if squeeze:
        w = w[:, None]
    out = np.zeros((tgt.shape[0], w.shape[1]), dtype=np.longdouble)
    gemm = shared and kernel.profile is not None
    if gemm:
        s2 = np.einsum("ij,ij->i", src, src)
    for a in range(0, tgt.shape[0], tb):
        b = min(tgt.shape[0], a + tb)
        acc = np.zeros((b - a, w.shape[1]), dtype=np.longdouble)
        for c in range(0, src.shape[0], sb):
            d = min(src.shape[0], c + sb)
            if gemm:
                r2 = s2[a:b, None] + s2[None, c:d]
                r2 -= 2.0 * (tgt[a:b] @ src[c:d].T)
                np.clip(r2, 0.0, None, out=r2)
                lo, hi = max(a, c), min(b, d)
                if lo < hi:
                    k = np.arange(lo, hi)
                    r2[k - a, k - c] = 0.0
                vals = kernel.profile(np.sqrt(r2))
            else:
                vals = kernel_matrix(kernel, tgt[a:b], src[c:d])
            acc += vals @ w[c:d]
        out[a:b] = acc
    res = np.asarray(out, dtype=np.float64)
    return res[:, 0] if squeeze else res


def default_threads():
    try:
        import psutil
        return max(1, psutil.cpu_count(logical=False) or os.cpu_count() or 1)
    except Exception:  # pragma: no cover
        return max(1, os.cpu_count() or 1)
