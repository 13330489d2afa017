"""GPU FMM evaluator — drop-in for the reference FmmEvaluator (engine.py:126-545).

Same constructor, same ``evaluate(sources, targets=None, weights=None)``,
same exceptions and ``timings`` keys.  Every stage of the matvec runs on
the GPU through libbfmm.so (include/bfmm.h); PyTorch only allocates device
memory and provides the stream.  There is no CPU fallback: without a CUDA
device or without the library the constructor raises NativeLibraryError.

Inputs may be NumPy arrays (result is a NumPy array, like the reference)
or torch tensors (result is a tensor on the input's device; CUDA tensors
skip every host<->device copy).
"""

from __future__ import annotations

import contextlib
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigurationError, DomainError, KernelEvaluationError, NativeLibraryError
from .interp import device_interp_blob, half_interval_matrices
from .kernel import KernelSpec
from .plan import FmmPlan, SchemeKind
from .tables import (ChebyshevLevelBlock, DeviceTableBuilder, M2LTable, neighbor_offsets,
                     precompute_m2l)

_KIND = {"r": 0, "r2": 1, "diff": 2}
_ST_DOMAIN_SRC, _ST_DOMAIN_TGT, _ST_REF, _ST_NONFINITE, _ST_WEIGHTS = 0, 1, 2, 3, 4


def _torch():
    try:
        import torch
    except Exception as e:  # pragma: no cover
        raise NativeLibraryError(f"PyTorch is required for device memory: {e}")
    return torch


def _pad8(r: int) -> int:
    return (r + 7) // 8 * 8


def _rank_interleave(rp: int) -> np.ndarray:
    """Storage position of rank index k: 2*(k%4) + (k//4)%2 inside its group
    of 8, so an MMA lane finds the k of two consecutive k4 steps adjacent."""
    k = np.arange(rp)
    return (k // 8) * 8 + 2 * (k % 4) + (k // 4) % 2


_PIN_WARM = None
_POOL = None


def _copy_pool():
    """Host threads for the pageable -> pinned staging copies of NumPy inputs."""
    global _POOL
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        n = max(1, min(8, (os.cpu_count() or 1)))
        _POOL = (ThreadPoolExecutor(max_workers=n, thread_name_prefix="bfmm-h2d"), n)
    return _POOL


def _warm_pinned_dma(device):
    """Once per process: one H2D copy from a small sacrificial pinned buffer.
    Measured on the B200 pool: the first pinned buffer a process copies from
    keeps running at ~25 GB/s while every later one gets the full ~55 GB/s
    (scripts/numa_probe.py), so without this the caller's first pinned input
    (e.g. the points of every end-to-end matvec) pays double H2D time."""
    global _PIN_WARM
    if _PIN_WARM is None:
        torch = _torch()
        h = torch.zeros(1 << 19, dtype=torch.float64).pin_memory()  # 4 MiB
        d = torch.empty_like(h, device=device)
        d.copy_(h)
        torch.cuda.synchronize(device)
        _PIN_WARM = h  # kept alive: the warmed buffer must not be reused


def _i8_core_slices(CP: np.ndarray, S: int, bits: int = 7):
    """Cores (316, rp, rp) [t][i][k] -> the digit planes bfmm_m2l_i8 reads
    (csrc/m2l_i8.cuh): row i is scaled by 2^-e_i (e_i the exponent of
    max_{t,k} |C_t[i, k]|) and cut into S signed digits of `bits` bits,
    C_t[i, k] = 2^e_i sum_j 2^(-6-bits*j) D_j[t, i, k] + O(2^(e_i - bits*S)),
    every step exact (bits = 7: repeated rint in FP64; bits = 8: the integer
    rint(x 2^(8(S-1))) as S signed bytes, like z_slice_kernel).  Returns the
    int8 image [t][i // 64][k // 32][j][64 x 32 K-major core matrices] and
    2^e_i."""
    T, nr, kr = CP.shape  # (offsets, N rows, K) -- rp x rp for the cores
    kc, nt = -(-kr // 32), -(-nr // 64)
    C = np.zeros((T, nt * 64, kc * 32))
    C[:, :nr, :kr] = CP
    amax = np.abs(C).max(axis=(0, 2))
    e = np.where(amax > 0, np.frexp(amax)[1], 0).astype(np.int64)
    x = C * np.ldexp(1.0, 6 - e)[None, :, None]
    D = np.empty((S,) + C.shape, dtype=np.int8)
    if bits == 8:
        X = np.rint(np.ldexp(x, 8 * (S - 1))).astype(np.int64)
        for j in range(S - 1, 0, -1):
            d = (X & 0xFF).astype(np.uint8).view(np.int8)
            D[j] = d
            X = (X - d.astype(np.int64)) >> 8
        assert np.all((X >= -128) & (X <= 127))
        D[0] = X.astype(np.int8)
    else:
        for j in range(S):
            d = np.rint(x)
            D[j] = d
            x = (x - d) * 128.0
    # [j][t][n][k] -> [t][n // 64][k // 32][j][n>>3 & 7][k>>4 & 1][n & 7][k & 15]
    D = D.reshape(S, T, nt, 8, 8, kc, 2, 16).transpose(1, 2, 5, 0, 3, 6, 4, 7)
    return np.ascontiguousarray(D), np.ldexp(1.0, e)


@dataclass
class _Tree:
    """A point set binned by leaf on the device (reference _Partition)."""
    n: int
    perm: object
    pts4: object
    leaves: object
    starts: object
    counts: object
    n_leaves: object
    cell_start: object
    cell_count: object
    max_leaves: int


class FmmEvaluator:
    """A plan bound to its kernel functor and device-resident M2L tables."""

    #: where the M2L operator tables are built: "device" (GPU assembly and
    #: QR, host SVD; tables.DeviceTableBuilder) or "host" (NumPy, the
    #: reference's own sequence)
    table_build = "device"

    def __init__(self, kernel: KernelSpec, plan: FmmPlan, cache_dir=None,
                 threads: int = 1, table: M2LTable = None, use_cache: bool = True,
                 device=None):
        if not isinstance(kernel, KernelSpec):
            raise ConfigurationError("kernel must be a KernelSpec")
        if not kernel.has_device_form:
            raise ConfigurationError(
                f"kernel {kernel.name!r} has no device form: give KernelSpec a "
                "cuda_expr (there is no CPU fallback for the near field)")
        torch = _torch()
        if not torch.cuda.is_available():
            raise NativeLibraryError("no CUDA device is visible; the FMM matvec runs on the GPU only")
        self.lib = _native.load()
        dev = torch.device(device if device is not None else "cuda")
        if dev.type != "cuda":
            raise ConfigurationError(f"device must be a CUDA device, got {dev}")
        # an explicit index: every launch, stream and module load of this
        # evaluator happens with it current (evaluate() enters it too)
        self.device = dev if dev.index is not None else torch.device(
            "cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):
            self._init_on_device(kernel, plan, cache_dir, threads, table, use_cache)

    def _init_on_device(self, kernel, plan, cache_dir, threads, table, use_cache):
        _warm_pinned_dma(self.device)
        self.kernel = kernel
        self.plan = plan
        self.threads = max(1, int(threads))
        t0 = time.perf_counter()
        p, sch = plan.order, plan.scheme
        self._H = np.ascontiguousarray(half_interval_matrices(p, sch))
        self._interp = device_interp_blob(p, sch)
        self._scheme_id = 0 if sch is SchemeKind.CHEBYSHEV else 1
        self.transfers_factors = self._H
        self.tree_seconds = time.perf_counter() - t0
        t0 = time.perf_counter()
        self._handle = self._kernel_handle()
        self._check_device_kernel()
        if table is None:
            # operator tables built on the GPU with the near field's functor
            # (tables.DeviceTableBuilder; host fallback per block), or read
            # from the reference-format cache
            self.table_builder = (DeviceTableBuilder(kernel, self._handle, self.lib, self.device,
                                                     self._stream)
                                  if self.table_build == "device" else None)
            table = precompute_m2l(kernel, plan, cache_dir=cache_dir, threads=self.threads,
                                   use_cache=use_cache, builder=self.table_builder)
        self.table = table
        self._upload_tables()
        self.table_seconds = time.perf_counter() - t0
        self.precompute_seconds = self.tree_seconds + self.table_seconds
        self.timings = {}
        self._disable_far_field = False
        self.keep_stages = False
        self.stages = {}
        self.profile_kernels = False
        self.active_profile = {}  # level -> (active target cells, octant offsets)
        # near field: "auto" / "full" (bfmm_p2p_cells: 32-target chunks, and
        # with one column a thread per target for leaves of <= 8 points over
        # shared-memory source tiles), "untiled" (the same without the
        # tiles), "grouped" (a thread per target for every leaf), or
        # "symmetric" (transpose replay)
        self.near_mode = "auto"
        # Chebyshev M2L over every cell ("dense"), over the ancestors of
        # occupied target leaves only ("active"), or "auto": active lists for
        # sparse clouds (fewer than 8 points per leaf cell), per level only
        # where they cut the target rows below 3/4
        self.far_mode = "auto"
        # Chebyshev M2L engine: FP64 tensor cores ("dmma", mma.sync f64) or
        # the int8 tcgen05 tensor cores with error-free digit splitting
        # ("i8", csrc/m2l_i8.cuh; i8_slices digits of 7 bits per operand)
        self.m2l_mode = "i8"
        self.i8_slices = 7
        # digit base of the int8 M2L ("auto": 8-bit digits where exact, see
        # _level_digits; "base128": i8_slices 7-bit digits everywhere)
        self.i8_digits = "auto"
        # run the near field on a second stream, concurrent with the far
        # field: the P2P is FP64-pipe bound, the int8 M2L tensor-core / L2
        # bound, so they share SMs well (C2, B200: 3.53 -> 3.31 ms).  With the
        # DMMA M2L both need the FP64 units (4.95 -> 4.90 ms only).
        self.overlap_near = True
        # enqueue the overlapped near field after the far field (True) or
        # before the upward pass (False)
        self.near_after_far = False
        # run the far-field chain on a high-priority stream while the near
        # field is overlapped (see _device_step; C2 graph replay 2.92 -> 2.90 ms)
        self.far_priority = True
        # ... which is the default for sharded runs, where it hides the
        # far field's all-gathers (SURVEY §8(e) "overlap")
        self.overlap_near_sharded = True
        # P2M / L2P: warp per leaf ("warp"), thread per (leaf, node) / point
        # ("point"), leaf-cell chunks ("cells"), or "auto" (cells for sparse
        # clouds)
        self.l2p_mode = "auto"
        # P2M: warp per leaf ("leaf"), leaf-cell chunks ("cells"), or "auto"
        # (cells for sparse clouds, see _p2m_cells)
        self.p2m_mode = "auto"
        # sparse clouds, one column: leaf-pair P2M / L2P (bfmm_p2m_pair /
        # bfmm_l2p_pair), which fold the L -> L-1 M2M and the L-1 -> L L2L
        # into the leaf kernels ("auto"), or the separate passes ("plain")
        self.leaf_mode = "auto"
        # basis projections z = M V, locals = s lt U^T: int8 tensor cores with
        # per-row digit scales ("i8", where p^3, rank <= 128) or FP64 DMMA
        self.proj_mode = "fp64"
        # coarse far-field levels on a side stream (see _far_field); the
        # finest main_levels levels stay on the calling stream
        self.stream_levels = True
        self.main_levels = 2
        self._side = None
        self.kernel_ms = {}
        self._kpending = []
        # replay the device step from a CUDA graph when possible (_graph_ok)
        # NVTX ranges around the stages and the far-field levels (for Nsight
        # timelines; the reference's tracing is its `timings` dict, engine.py:505-533)
        self.nvtx = bool(os.environ.get("BFMM_NVTX"))
        self.use_graph = False
        self._graphs = {}
        self.graph_launches = 0  # kernels of ours run by graph replays (bench accounting)

    # -- setup --------------------------------------------------------------
    def _kernel_handle(self) -> int:
        k = self.kernel
        if k.builtin_id:
            return int(k.builtin_id)
        h = _native.C.c_int(0)
        _native.check(self.lib.bfmm_kernel_compile(_KIND[k.cuda_arg], k.cuda_expr.encode(),
                                                   _native.C.byref(h)),
                      f"NVRTC compile of kernel {k.name!r}")
        return int(h.value)

    def _check_device_kernel(self):
        """The device functor must be the kernel the tables were built from.
        A custom kernel is given twice -- the NumPy hook (operator tables,
        reference ops:244-341) and cuda_expr (near field) -- so the two are
        compared on fixed sample pairs in the domain (no r = 0 pair) before
        the evaluator is usable; a mismatch would silently give a wrong phi."""
        if self.kernel.builtin_id:
            return
        torch = _torch()
        d = self.plan.domain
        g = np.random.default_rng(12345)
        X = np.asarray(d.low) + d.length * g.random((64, 3))
        Y = np.asarray(d.low) + d.length * g.random((2, 3))
        host = np.asarray(self.kernel.block(X, Y), dtype=np.float64)
        xt = torch.from_numpy(X).to(self.device)
        dev = np.empty_like(host)
        for j in range(Y.shape[0]):
            yt = torch.from_numpy(Y[j:j + 1].copy()).to(self.device)
            wt = torch.ones((1, 1), dtype=torch.float64, device=self.device)
            out = torch.empty((X.shape[0], 1), dtype=torch.float64, device=self.device)
            _native.check(self.lib.bfmm_direct(self._handle, xt.data_ptr(), X.shape[0],
                                               yt.data_ptr(), wt.data_ptr(), 1, 1,
                                               out.data_ptr(), self._stream()), "bfmm_direct")
            dev[:, j] = out[:, 0].cpu().numpy()
        ok = np.isfinite(host)
        scale = np.maximum(np.abs(host), 1e-300)
        bad = ok & ~(np.abs(dev - host) <= 1e-11 * scale)
        if bad.any() or not np.array_equal(ok, np.isfinite(dev)):
            i, j = np.argwhere(bad | (ok != np.isfinite(dev)))[0]
            raise ConfigurationError(
                f"kernel {self.kernel.name!r}: cuda_expr {self.kernel.cuda_expr!r} gives "
                f"{dev[i, j]!r} where the host hook gives {host[i, j]!r} "
                f"(x={tuple(X[i])}, y={tuple(Y[j])}); the two forms must agree")

    def _upload_tables(self):
        torch = _torch()
        dev = self.device
        self._dev_blocks = {}
        for key, blk in self.table.blocks.items():
            if isinstance(blk, ChebyshevLevelBlock):
                p3, r = blk.u.shape
                rp = _pad8(r)
                # rank index k of z and of the cores' k axis is interleaved inside
                # groups of 8 (csrc/m2l_dmma.cuh); the contraction is unchanged
                kpos = _rank_interleave(rp)[:r]
                V = np.zeros((p3, rp))
                V[:, kpos] = blk.v
                UT = np.zeros((rp, p3))
                UT[:r] = blk.u.T
                CP = np.zeros((blk.cores.shape[0], rp, rp))
                CP[:, :r, kpos] = blk.cores  # [t][i][k], k contiguous
                self._dev_blocks[key] = {
                    "kind": "cheb", "r": r, "rp": rp,
                    "V": torch.from_numpy(V).to(dev),
                    "UT": torch.from_numpy(UT).to(dev),
                    "cores": torch.from_numpy(CP).to(dev),
                }
            else:
                sym = np.ascontiguousarray(blk.symbols).view(np.float64)
                self._dev_blocks[key] = {"kind": "fft",
                                         "symbols": torch.from_numpy(sym.copy()).to(dev)}

    def _i8_tables(self, blk, S, bits):
        key = ("i8", S, bits)
        if key not in blk:
            torch = _torch()
            cs, cpow = _i8_core_slices(blk["cores"].cpu().numpy(), S, bits)
            blk[key] = (torch.from_numpy(cs.reshape(-1)).to(self.device),
                        torch.from_numpy(cpow).to(self.device))
        return blk[key]

    def _pj_tables(self, blk, which):
        """Digit image of B^T for bfmm_rows_gemm_i8: V (p^3, rp) -> z = M V,
        UT (rp, p^3) -> locals = s lt UT (six 8-bit digits, per-column scale)."""
        key = ("pj", which)
        if key not in blk:
            torch = _torch()
            B = blk[which].cpu().numpy()
            d, pw = _i8_core_slices(np.ascontiguousarray(B.T)[None], 6, 8)
            blk[key] = (torch.from_numpy(d.reshape(-1)).to(self.device),
                        torch.from_numpy(np.ascontiguousarray(pw)).to(self.device))
        return blk[key]

    def _proj_i8(self, p3, rp):
        """Int8 projections (proj_mode): both GEMM sides <= 128 wide."""
        return self.proj_mode == "i8" and p3 <= 128 and rp <= 128

    def _level_engine(self, lev, m, rp):
        """The Chebyshev M2L engine of one level: self.m2l_mode, except that
        the int8 kernels take rank tiles up to rp = 256 and 32-bit row
        indices (8^lev * m < 2^31); larger plans (e.g. order 8 at eps 1e-10,
        rank 288) run that level on the FP64 DMMA engine."""
        if self.m2l_mode == "i8" and rp <= 256 and (1 << (3 * lev)) * m < (1 << 31):
            return "i8"
        return "dmma"

    def _level_digits(self, lev, rp, listed):
        """(digits, bits) of the int8 M2L at a level.  i8_digits = "auto" (with
        the default i8_slices = 7): six 8-bit digits (47 bits, 21 digit
        products instead of 28) where the exact int32
        accumulation bound allows it (rp <= 96; <= 64 for the mixed-octant
        coarse levels, csrc/m2l_cheb.cu i8_check), else i8_slices 7-bit
        digits; "base128": always i8_slices 7-bit digits."""
        if self.i8_digits == "auto" and int(self.i8_slices) == 7:
            offs = 316 if (lev <= 3 and not listed) else 189
            if 6 * offs * 32 * (-(-rp // 32)) * 16384 < (1 << 31):
                return 6, 8
        return int(self.i8_slices), 7

    def _m2l_translate(self, z, lt, lev, m, rp, ns, blk, st, q_lo=0, nq=0, cells=None, off=None,
                       shard=None, zmax=None):
        """lt = the 189-offset translation of z (engine.py:228-256), on the
        level's engine (_level_engine); cells/off: listed active targets."""
        torch = _torch()
        if self._level_engine(lev, m, rp) == "i8":
            S, bits = self._level_digits(lev, rp, cells is not None)
            cs, cpow = self._i8_tables(blk, S, bits)
            Sarg = S | (_native.I8_BASE256 if bits == 8 else 0)
            rows = z.numel() // rp
            # sparse cloud on a shared tree, unsharded: z is non-zero in the
            # listed cells only, so only their rows are scanned and cut (the
            # other digit rows stay zero)
            listed = (cells is not None and getattr(self, "_active_src", False)
                      and (shard is None or shard[0].full) and zmax is None)
            zs = (torch.zeros if listed else torch.empty)(
                int(self.lib.bfmm_m2l_i8_zs_bytes(rows, rp, Sarg)), dtype=torch.int8,
                device=self.device)
            if zmax is not None:
                # max |z| from the int8 projection's epilogue (one column)
                if shard is not None and not shard[0].full:
                    shard[1].allreduce_max(zmax)
                Sarg |= _native.I8_ZMAX_GIVEN
            else:
                zmax = torch.empty(m, dtype=torch.int64, device=self.device)
            if shard is not None and not shard[0].full and not (Sarg & _native.I8_ZMAX_GIVEN):
                # one digit scale per column over ALL ranks' cells: every
                # shard cuts z exactly like the unsharded evaluation
                _native.check(self.lib.bfmm_m2l_i8_zmax(z.data_ptr(), rows, m, rp,
                                                        zmax.data_ptr(), st), "bfmm_m2l_i8_zmax")
                shard[1].allreduce_max(zmax)
                Sarg |= _native.I8_ZMAX_GIVEN
            if listed:
                if cells.numel() and off[8] > 0:
                    _native.check(self.lib.bfmm_m2l_i8_slice_z_cells(
                        z.data_ptr(), int(off[8]) * m, m, rp, Sarg, zs.data_ptr(),
                        zmax.data_ptr(), cells.data_ptr(), st), "bfmm_m2l_i8_slice_z_cells")
                else:
                    zmax.zero_()
            else:
                _native.check(self.lib.bfmm_m2l_i8_slice_z(z.data_ptr(), rows, m, rp, Sarg,
                                                           zs.data_ptr(), zmax.data_ptr(), st),
                              "bfmm_m2l_i8_slice_z")
            e0 = self._kevent()
            if cells is not None:
                _native.check(self.lib.bfmm_m2l_i8_cells(
                    zs.data_ptr(), zmax.data_ptr(), cs.data_ptr(), cpow.data_ptr(),
                    lt.data_ptr(), lev, m, rp, Sarg, ns, cells.data_ptr(), off.ctypes.data, st),
                    "bfmm_m2l_i8_cells")
            else:
                _native.check(self.lib.bfmm_m2l_i8(
                    zs.data_ptr(), zmax.data_ptr(), cs.data_ptr(), cpow.data_ptr(),
                    lt.data_ptr(), lev, m, rp, Sarg, ns, q_lo, nq, st), "bfmm_m2l_i8")
            self._kspan(f"m2l_l{lev}", e0)
            return
        e0 = self._kevent()
        if cells is not None:
            _native.check(self.lib.bfmm_m2l_cheb_cells(
                z.data_ptr(), lt.data_ptr(), lev, m, rp, ns, cells.data_ptr(),
                off.ctypes.data, blk["cores"].data_ptr(), st), "bfmm_m2l_cheb_cells")
        else:
            _native.check(self.lib.bfmm_m2l_cheb(z.data_ptr(), lt.data_ptr(), lev, m, rp, ns,
                                                 q_lo, nq, blk["cores"].data_ptr(),
                                                 st), "bfmm_m2l_cheb")
        self._kspan(f"m2l_l{lev}", e0)

    def _m2l_splits(self, lev, m, rp, nq):
        if self._level_engine(lev, m, rp) == "i8":
            return int(self.lib.bfmm_m2l_i8_splits(lev, m, rp, nq))
        return int(self.lib.bfmm_m2l_cheb_splits(lev, m, rp, nq))

    def _dev_block(self, level):
        return self._dev_blocks[0] if self.table.single_level else self._dev_blocks[level]

    # -- helpers --------------------------------------------------------------
    def _nv_push(self, name):
        if self.nvtx:
            _torch().cuda.nvtx.range_push("bfmm." + name)

    def _nv_pop(self):
        if self.nvtx:
            _torch().cuda.nvtx.range_pop()

    @staticmethod
    def _stream():
        torch = _torch()
        return _native.C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def _hi_stream(self):
        torch = _torch()
        if getattr(self, "_hi", None) is None:
            self._hi = torch.cuda.Stream(device=self.device, priority=-1)
        return self._hi

    def _side_stream(self, k=0):
        """Side stream k: 0 = coarse far-field levels, 1 = the near field."""
        torch = _torch()
        if self._side is None:
            self._side = {}
        if k not in self._side:
            self._side[k] = torch.cuda.Stream(device=self.device)
        return self._side[k]

    _STAGE_ELEMS = 1 << 23  # 64 MiB per half of the pinned staging buffer

    def _h2d_into(self, dst, a):
        """Copy a NumPy array (pageable host memory, the reference's calling
        convention) into the device tensor dst: 64 MiB chunks go through the
        evaluator's reusable two-half pinned buffer, so the host copy of one
        chunk overlaps the DMA of the previous one and no O(N) pinned buffer
        is allocated per call."""
        torch = _torch()
        src = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).reshape(-1)
        flat = dst.view(-1)
        n = src.numel()
        if n <= (1 << 16):
            flat.copy_(src)
            return dst
        CH = self._STAGE_ELEMS
        if getattr(self, "_stage", None) is None:
            self._stage = torch.empty(2 * CH, dtype=torch.float64).pin_memory()
            self._stage_np = self._stage.numpy()
            self._stage_ev = [torch.cuda.Event(), torch.cuda.Event()]
            for e in self._stage_ev:
                e.record()
        st = torch.cuda.current_stream()
        src_np = src.numpy()
        pool, nthr = _copy_pool()
        for i, off in enumerate(range(0, n, CH)):
            k, b = min(CH, n - off), i % 2
            self._stage_ev[b].synchronize()  # the DMA that last read this half is done
            dst_np = self._stage_np[b * CH:b * CH + k]
            # the host copy in parallel slices (np.copyto releases the GIL)
            cuts = np.linspace(0, k, nthr + 1).astype(np.int64)
            list(pool.map(lambda j: np.copyto(dst_np[cuts[j]:cuts[j + 1]],
                                              src_np[off + cuts[j]:off + cuts[j + 1]]),
                          range(nthr)))
            flat[off:off + k].copy_(self._stage[b * CH:b * CH + k], non_blocking=True)
            self._stage_ev[b].record(st)
        return dst

    def _prepare_points(self, arr, name):
        torch = _torch()
        if isinstance(arr, torch.Tensor):
            if arr.ndim != 2 or arr.shape[1] != 3:
                raise ConfigurationError(f"{name} must be an (N, 3) array, got shape {tuple(arr.shape)}")
            return arr.to(device=self.device, dtype=torch.float64, non_blocking=True).contiguous()
        pts = np.asarray(arr)
        if pts.ndim != 2 or pts.shape[1] != 3:
            raise ConfigurationError(f"{name} must be an (N, 3) array, got shape {np.shape(arr)}")
        out = torch.empty(pts.shape, dtype=torch.float64, device=self.device)
        return self._h2d_into(out, pts)

    def _prepare_weights(self, w, n_src):
        torch = _torch()
        if w is None:
            raise ConfigurationError("weights are required")
        if isinstance(w, torch.Tensor):
            squeeze = w.ndim == 1
            wt = w[:, None] if squeeze else w
            if wt.ndim != 2 or wt.shape[0] != n_src:
                raise ConfigurationError(
                    f"weights shape {tuple(w.shape)} does not match {n_src} sources")
            return wt.to(device=self.device, dtype=torch.float64, non_blocking=True).contiguous(), squeeze
        wa = np.asarray(w)
        squeeze = wa.ndim == 1
        if squeeze:
            wa = wa[:, None]
        if wa.ndim != 2 or wa.shape[0] != n_src:
            raise ConfigurationError(
                f"weights shape {np.shape(w)} does not match {n_src} sources")
        out = torch.empty(wa.shape, dtype=torch.float64, device=self.device)
        return self._h2d_into(out, wa), squeeze

    def _geom(self):
        d = self.plan.domain
        lo, hi = d.low, d.high
        h = d.length / (1 << self.plan.levels)
        return np.ascontiguousarray(np.concatenate([lo, hi, [h, 1e-12 * d.length]]))

    def _build_tree(self, pts, status, slot) -> _Tree:
        torch = _torch()
        L = self.plan.levels
        n = int(pts.shape[0])
        dev = self.device
        cap = max(n, 1)
        ncell = 1 << (3 * L)
        perm = torch.empty(cap, dtype=torch.int64, device=dev)
        pts4 = torch.empty((cap, 4), dtype=torch.float64, device=dev)
        leaves = torch.empty(cap, dtype=torch.int64, device=dev)
        starts = torch.empty(cap, dtype=torch.int64, device=dev)
        counts = torch.empty(cap, dtype=torch.int64, device=dev)
        n_leaves = torch.zeros(1, dtype=torch.int64, device=dev)
        cell_start = torch.empty(ncell, dtype=torch.int32, device=dev)
        cell_count = torch.empty(ncell, dtype=torch.int32, device=dev)
        sb = self.lib.bfmm_tree_scratch_bytes(n, L)
        scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        geom = self._geom()
        _native.check(self.lib.bfmm_tree_build(
            pts.data_ptr(), n, _native.dptr(geom), L, scratch.data_ptr(), sb,
            perm.data_ptr(), pts4.data_ptr(), leaves.data_ptr(), starts.data_ptr(),
            counts.data_ptr(), n_leaves.data_ptr(), cell_start.data_ptr(),
            cell_count.data_ptr(), status[slot:].data_ptr(), self._stream()), "bfmm_tree_build")
        return _Tree(n, perm, pts4, leaves, starts, counts, n_leaves, cell_start,
                     cell_count, min(n, ncell))

    # -- stages -----------------------------------------------------------------
    def _cells(self, lev, shard):
        """[lo, hi) cells of this call's shard at a level (all cells if unsharded)."""
        return (0, 1 << (3 * lev)) if shard is None else shard[0].cells(lev)

    def _upward(self, tree, ws, m, status, shard):
        torch = _torch()
        L, p = self.plan.levels, self.plan.order
        p3 = p ** 3
        st = self._stream()
        lo, hi = self._cells(L, shard)
        leaf_geom = np.ascontiguousarray(np.concatenate(
            [self.plan.domain.low, [self.plan.domain.length / (1 << L), float(lo), float(hi)]]))
        ncell = (1 << (3 * L))
        pair = self._leaf_pair(tree, m)
        e0 = self._kevent()
        if pair:
            # leaf moments and the parents' moments straight from the points
            alloc = torch.zeros if shard is not None else torch.empty
            moments = {L: alloc((ncell * p3,), dtype=torch.float64, device=self.device),
                       L - 1: alloc((ncell // 8 * p3,), dtype=torch.float64, device=self.device)}
            _native.check(self.lib.bfmm_p2m_pair(
                tree.pts4.data_ptr(), ws.data_ptr(), tree.cell_start.data_ptr(),
                tree.cell_count.data_ptr(), L, p, self._scheme_id, _native.dptr(self._interp),
                _native.dptr(leaf_geom), moments[L].data_ptr(), moments[L - 1].data_ptr(),
                status[_ST_REF:].data_ptr(), st), "bfmm_p2m_pair")
        elif self._p2m_cells(tree, p):
            # sparse cloud: P2M over leaf-cell chunks, which writes every
            # cell of [lo, hi) (zeros for empty ones) -- no memset
            alloc = torch.zeros if shard is not None else torch.empty
            moments = {L: alloc((ncell * m * p3,), dtype=torch.float64, device=self.device)}
            _native.check(self.lib.bfmm_p2m_cells(
                tree.pts4.data_ptr(), ws.data_ptr(), m, tree.cell_start.data_ptr(),
                tree.cell_count.data_ptr(), L, p, self._scheme_id, _native.dptr(self._interp),
                _native.dptr(leaf_geom), moments[L].data_ptr(), status[_ST_REF:].data_ptr(), st),
                "bfmm_p2m_cells")
        else:
            moments = {L: torch.zeros((ncell * m * p3,), dtype=torch.float64, device=self.device)}
            # thread-per-(leaf, node) P2M only on request (l2p_mode "point")
            p2m = self.lib.bfmm_p2m_sparse if self.l2p_mode == "point" else self.lib.bfmm_p2m
            _native.check(p2m(
                tree.pts4.data_ptr(), ws.data_ptr(), m, tree.leaves.data_ptr(),
                tree.starts.data_ptr(), tree.counts.data_ptr(), tree.n_leaves.data_ptr(),
                tree.max_leaves, L, p, self._scheme_id, _native.dptr(self._interp),
                _native.dptr(leaf_geom), moments[L].data_ptr(), status[_ST_REF:].data_ptr(), st),
                "bfmm_p2m")
        self._kspan("p2m", e0)
        e0 = self._kevent()
        for lev in range(L - 1 if pair else L, 2, -1):
            npar = 1 << (3 * (lev - 1))
            qlo, qhi = self._cells(lev - 1, shard)  # parents of this shard's cells
            row = m * p3
            # a shard fills its own cells and receives only its halo: the
            # rest of the level must read as zeros
            alloc = torch.zeros if shard is not None else torch.empty
            moments[lev - 1] = alloc((npar * row,), dtype=torch.float64, device=self.device)
            _native.check(self.lib.bfmm_m2m(
                moments[lev][8 * qlo * row:].data_ptr(), moments[lev - 1][qlo * row:].data_ptr(),
                qhi - qlo, p, m, _native.dptr(self._H), st), "bfmm_m2m")
        self._kspan("m2m", e0)
        return moments, leaf_geom

    def _leaf_pair(self, tree, m):
        """Leaf-pair P2M / L2P (leaf_mode): one weight column, a sparse cloud
        (fewer than 8 points per leaf cell on average, the cells rule),
        2 <= p <= 8, L >= 3; off while per-level stages are kept (the leaf
        locals then hold only the level's own M2L part)."""
        L, p = self.plan.levels, self.plan.order
        if self.leaf_mode == "plain" or self.keep_stages or m != 1 or L < 3 or not 2 <= p <= 8:
            return False
        return self.leaf_mode == "pair" or tree.n < 8 * (1 << (3 * L))

    def _p2m_cells(self, tree, p):
        """P2M over leaf-cell chunks (bfmm_p2m_cells) for sparse clouds --
        fewer than 8 points per leaf cell on average, like the l2p "auto"
        rule -- or on request (p2m_mode "cells")."""
        if not 2 <= p <= 8 or self.p2m_mode == "leaf":
            return False
        return self.p2m_mode == "cells" or tree.n < 8 * (1 << (3 * self.plan.levels))

    def _active_cells(self, ttree, shard):
        """{level: (active target cells grouped by octant, host octant offsets
        (9), their number)} for the levels where the list pays (see far_mode):
        the cells at that level with an occupied target leaf below them."""
        torch = _torch()
        L = self.plan.levels
        if self.plan.scheme is not SchemeKind.CHEBYSHEV or self.far_mode == "dense":
            return {}
        if self.far_mode == "auto" and ttree.n >= 8 * (1 << (3 * L)):
            return {}
        cap = max(ttree.max_leaves, 1)
        sb = self.lib.bfmm_active_cells_scratch_bytes(cap)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        levels = list(range(2, L + 1))
        counts = torch.zeros(len(levels) * 9, dtype=torch.int64, device=self.device)
        lists = {}
        st = self._stream()
        for i, lev in enumerate(levels):
            lo, hi = self._cells(lev, shard)
            lst = torch.empty(min(cap, hi - lo) or 1, dtype=torch.int64, device=self.device)
            _native.check(self.lib.bfmm_active_cells(
                ttree.leaves.data_ptr(), ttree.n_leaves.data_ptr(), cap, 3 * (L - lev), lo, hi,
                scratch.data_ptr(), sb, lst.data_ptr(), counts[9 * i:].data_ptr(), st),
                "bfmm_active_cells")
            _native.check(self.lib.bfmm_octant_histogram(
                lst.data_ptr(), counts[9 * i:].data_ptr(), lst.numel(),
                counts[9 * i + 1:].data_ptr(), st), "bfmm_octant_histogram")
            lists[lev] = (lst, hi - lo)
        cnt = counts.cpu().numpy().reshape(len(levels), 9)  # one read-back sizes every grid
        out = {}
        for i, lev in enumerate(levels):
            lst, ncell = lists[lev]
            nact = int(cnt[i, 0])
            if not (self.far_mode == "active" or nact * 4 < ncell * 3):
                continue
            grouped = torch.empty(max(nact, 1), dtype=torch.int64, device=self.device)
            if nact:
                gb = self.lib.bfmm_group_by_octant_scratch_bytes(nact)
                gs = torch.empty(max(gb, 1), dtype=torch.uint8, device=self.device)
                _native.check(self.lib.bfmm_group_by_octant(
                    lst.data_ptr(), nact, grouped.data_ptr(), gs.data_ptr(), gb, st),
                    "bfmm_group_by_octant")
            off = np.zeros(9, dtype=np.int64)
            off[1:] = np.cumsum(cnt[i, 1:])
            out[lev] = (grouped, off, nact)
        return out

    def _far_field(self, moments, m, shard, active=None, active_src=False):
        """Locals of every level 2..L (engine.py:228-292).  The levels are
        independent; with stream_levels the coarse ones (2..L-2, small and
        latency-bound) run on a side stream under the two finest."""
        torch = _torch()
        L = self.plan.levels
        active = active or {}
        # active_src: the active target cells are also the cells with sources
        # below them (shared source / target tree), see _far_level
        self._active_src = bool(active_src)
        locs = {}
        coarse = list(range(2, L - self.main_levels + 1)) if (self.stream_levels and shard is None) else []
        if coarse:
            main = torch.cuda.current_stream()
            side = self._side_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                for lev in coarse:
                    locs[lev] = self._far_level(lev, moments, m, shard, active)
        for lev in range(2, L + 1):
            if lev not in locs:
                locs[lev] = self._far_level(lev, moments, m, shard, active)
        if coarse:
            main.wait_stream(side)
            for lev in coarse:
                locs[lev].record_stream(main)
        return locs

    def _far_level(self, lev, moments, m, shard, active):
        self._nv_push(f"m2l_level_{lev}")
        try:
            return self._far_level_impl(lev, moments, m, shard, active)
        finally:
            self._nv_pop()

    def _far_level_impl(self, lev, moments, m, shard, active):
        torch = _torch()
        p = self.plan.order
        p3 = p ** 3
        st = self._stream()
        blk = self._dev_block(lev)
        scale = float(self.table.scale_for_level(lev))
        ncell = 1 << (3 * lev)
        lo, hi = self._cells(lev, shard)
        nloc = hi - lo
        # parents covering [lo, hi) (work-balanced shards need not be
        # 8-aligned at level 2: the few extra children computed are unused)
        q_lo, nq = lo // 8, -(-hi // 8) - lo // 8
        out = torch.empty((ncell * m * p3,), dtype=torch.float64, device=self.device)
        # shards: z outside the own cells and the received halo reads as zero
        zalloc = torch.zeros if (shard is not None and not shard[0].full) else torch.empty
        if blk["kind"] == "cheb" and lev in active:
            # only the listed active target cells: compact lt rows
            cells, off, nact = active[lev]
            if self.profile_kernels:  # the bench's per-level work accounting
                self.active_profile[lev] = (cells[:nact], off.copy())
            rp = blk["rp"]
            longest = int(np.max(off[1:] - off[:-1]))
            ns = self._m2l_splits(lev, m, rp, max(longest, 1))
            lt = torch.empty((max(nact, 1) * m * ns * rp,), dtype=torch.float64,
                             device=self.device)
            out.zero_()
            if self._active_src:
                # shared tree: the other cells have no sources below them, so
                # their moments and z rows are zero -- project the listed
                # cells only (C4 level 7: 82k of 2.1M cells)
                z = torch.zeros((ncell * m * rp,), dtype=torch.float64, device=self.device)
                if nact:
                    _native.check(self.lib.bfmm_rows_gemm_cells(
                        moments[lev].data_ptr(), nact * m, p3, blk["V"].data_ptr(), rp,
                        z.data_ptr(), 1.0, cells.data_ptr(), m, st), "bfmm_rows_gemm_cells(V)")
            else:
                z = zalloc((ncell * m * rp,), dtype=torch.float64, device=self.device)
                _native.check(self.lib.bfmm_rows_gemm(
                    moments[lev][lo * m * p3:].data_ptr(), nloc * m, p3, blk["V"].data_ptr(), rp,
                    z[lo * m * rp:].data_ptr(), 1.0, 0.0, 1, st), "bfmm_rows_gemm(V)")
            if shard is not None and not shard[0].full:
                shard[1].exchange_level(z, m * rp, lev, shard[0])
            self._m2l_translate(z, lt, lev, m, rp, ns, blk, st, cells=cells, off=off, shard=shard)
            if nact:
                _native.check(self.lib.bfmm_rows_gemm_scatter(
                    lt.data_ptr(), nact * m, rp, blk["UT"].data_ptr(), p3, out.data_ptr(),
                    scale, 0.0, ns, cells.data_ptr(), m, st), "bfmm_rows_gemm_scatter(U)")
        elif blk["kind"] == "cheb":
            rp = blk["rp"]
            ns = self._m2l_splits(lev, m, rp, nq)
            z = zalloc((ncell * m * rp,), dtype=torch.float64, device=self.device)
            lt = torch.empty((ncell * m * ns * rp,), dtype=torch.float64, device=self.device)
            e0 = self._kevent()
            zmax = None
            if self._proj_i8(p3, rp):
                dg, pw = self._pj_tables(blk, "V")
                if m == 1 and self._level_engine(lev, m, rp) == "i8":
                    zmax = torch.zeros(1, dtype=torch.int64, device=self.device)
                _native.check(self.lib.bfmm_rows_gemm_i8(
                    moments[lev][lo * m * p3:].data_ptr(), nloc * m, p3, dg.data_ptr(),
                    pw.data_ptr(), rp, z[lo * m * rp:].data_ptr(), 1.0,
                    zmax.data_ptr() if zmax is not None else None, st), "bfmm_rows_gemm_i8(V)")
            elif (m == 1 and self._level_engine(lev, m, rp) == "i8" and p3 <= 128
                  and (rp <= 64 or p3 <= 80) and nloc >= 8 * 148 * 64):
                # big level, one column: the persistent projection also
                # returns max |z|, the int8 M2L's digit scale (no absmax pass)
                zmax = torch.zeros(1, dtype=torch.int64, device=self.device)
                _native.check(self.lib.bfmm_rows_gemm_max(
                    moments[lev][lo * m * p3:].data_ptr(), nloc * m, p3, blk["V"].data_ptr(), rp,
                    z[lo * m * rp:].data_ptr(), 1.0, zmax.data_ptr(), st), "bfmm_rows_gemm_max(V)")
            else:
                _native.check(self.lib.bfmm_rows_gemm(
                    moments[lev][lo * m * p3:].data_ptr(), nloc * m, p3, blk["V"].data_ptr(), rp,
                    z[lo * m * rp:].data_ptr(), 1.0, 0.0, 1, st), "bfmm_rows_gemm(V)")
            self._kspan(f"projv_l{lev}", e0)
            if shard is not None and not shard[0].full:
                # the sources this shard's M2L reads: its halo (fine levels)
                # or the whole level (coarse levels)
                shard[1].exchange_level(z, m * rp, lev, shard[0])
            self._m2l_translate(z, lt, lev, m, rp, ns, blk, st, q_lo=q_lo, nq=nq, shard=shard,
                                zmax=zmax)
            e0 = self._kevent()
            if self._proj_i8(p3, rp) and ns == 1:
                dg, pw = self._pj_tables(blk, "UT")
                _native.check(self.lib.bfmm_rows_gemm_i8(
                    lt[lo * m * rp:].data_ptr(), nloc * m, rp, dg.data_ptr(), pw.data_ptr(), p3,
                    out[lo * m * p3:].data_ptr(), scale, None, st), "bfmm_rows_gemm_i8(U)")
            else:
                _native.check(self.lib.bfmm_rows_gemm(
                    lt[lo * m * ns * rp:].data_ptr(), nloc * m, rp, blk["UT"].data_ptr(), p3,
                    out[lo * m * p3:].data_ptr(), scale, 0.0, ns, st), "bfmm_rows_gemm(U)")
            self._kspan(f"proju_l{lev}", e0)
        else:
            if shard is not None and not shard[0].full:
                shard[1].exchange_level(moments[lev], m * p3, lev, shard[0])
            # spectra of a chunk of columns at a time (<= 16 GiB of scratch)
            nb = _native.C.c_size_t(0)
            _native.check(self.lib.bfmm_m2l_fft_scratch_bytes(lev, 1, p, _native.C.byref(nb)),
                          "bfmm_m2l_fft_scratch_bytes")
            cc = max(1, min(m, (16 << 30) // max(int(nb.value), 1)))
            _native.check(self.lib.bfmm_m2l_fft_scratch_bytes(lev, cc, p, _native.C.byref(nb)),
                          "bfmm_m2l_fft_scratch_bytes")
            scratch = torch.empty(max(int(nb.value), 1), dtype=torch.uint8, device=self.device)
            e0 = self._kevent()
            _native.check(self.lib.bfmm_m2l_fft(moments[lev].data_ptr(), out.data_ptr(), lev, m,
                                                p, blk["symbols"].data_ptr(), scale, q_lo,
                                                nq, scratch.data_ptr(), int(nb.value),
                                                st), "bfmm_m2l_fft")
            self._kspan(f"m2lfft_l{lev}", e0)
        return out

    def _downward(self, locs, tree, m, leaf_geom, status, phi_far, shard):
        L, p = self.plan.levels, self.plan.order
        st = self._stream()
        row = m * p ** 3
        pair = self._leaf_pair(tree, m)
        e0 = self._kevent()
        for lev in range(2, L - 1 if pair else L):
            qlo, qhi = self._cells(lev, shard)
            _native.check(self.lib.bfmm_l2l(locs[lev][qlo * row:].data_ptr(),
                                            locs[lev + 1][8 * qlo * row:].data_ptr(),
                                            qhi - qlo, p, m, _native.dptr(self._H), st),
                          "bfmm_l2l")
        self._kspan("l2l", e0)
        e0 = self._kevent()
        self._l2p(locs, tree, m, leaf_geom, status, phi_far, pair, st)
        self._kspan("l2p", e0)

    def _l2p(self, locs, tree, m, leaf_geom, status, phi_far, pair, st):
        L, p = self.plan.levels, self.plan.order
        if pair:
            # the parents' complete locals enter through their own basis
            _native.check(self.lib.bfmm_l2p_pair(
                tree.pts4.data_ptr(), tree.cell_start.data_ptr(), tree.cell_count.data_ptr(),
                L, p, self._scheme_id, _native.dptr(self._interp), _native.dptr(leaf_geom),
                locs[L].data_ptr(), locs[L - 1].data_ptr(), phi_far.data_ptr(),
                status[_ST_REF:].data_ptr(), st), "bfmm_l2p_pair")
            return
        # fewer than 8 points per leaf cell on average: leaf-cell chunks
        # with their locals staged in shared memory (or one thread per point)
        sparse_auto = self.l2p_mode == "auto" and tree.n < 8 * (1 << (3 * L))
        # (the cells kernel stages one cell's m * p^3 locals in <= 96 KB)
        if (self.l2p_mode == "cells" or sparse_auto) and 2 <= p <= 8 and m * p ** 3 * 8 <= 96 * 1024:
            _native.check(self.lib.bfmm_l2p_cells(
                tree.pts4.data_ptr(), m, tree.cell_start.data_ptr(), tree.cell_count.data_ptr(),
                L, p, self._scheme_id, _native.dptr(self._interp), _native.dptr(leaf_geom),
                locs[L].data_ptr(), phi_far.data_ptr(), status[_ST_REF:].data_ptr(), st),
                "bfmm_l2p_cells")
            return
        sparse = self.l2p_mode == "point" or sparse_auto
        l2p = self.lib.bfmm_l2p_points if sparse else self.lib.bfmm_l2p
        _native.check(l2p(
            tree.pts4.data_ptr(), m, tree.leaves.data_ptr(), tree.starts.data_ptr(),
            tree.counts.data_ptr(), tree.n_leaves.data_ptr(), tree.max_leaves, L, p,
            self._scheme_id, _native.dptr(self._interp), _native.dptr(leaf_geom),
            locs[L].data_ptr(), phi_far.data_ptr(), status[_ST_REF:].data_ptr(), st), "bfmm_l2p")

    def _near_field(self, ttree, stree, ws, m, near, shard):
        self._nv_push("near_field")
        try:
            return self._near_field_impl(ttree, stree, ws, m, near, shard)
        finally:
            self._nv_pop()

    def _near_field_impl(self, ttree, stree, ws, m, near, shard):
        torch = _torch()
        st = self._stream()
        sb = self.lib.bfmm_p2p_scratch_bytes(max(ttree.max_leaves, 1), ttree.n)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        lo, hi = self._cells(self.plan.levels, shard)
        if self._use_symmetric(ttree, stree, m):
            sb = self.lib.bfmm_p2p_symmetric_scratch_bytes(ttree.n, max(ttree.max_leaves, 1))
            scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
            e0 = self._kevent()
            _native.check(self.lib.bfmm_p2p_symmetric(
                self._handle, ttree.pts4.data_ptr(), ttree.leaves.data_ptr(),
                ttree.starts.data_ptr(), ttree.counts.data_ptr(), ttree.n_leaves.data_ptr(),
                ttree.max_leaves, stree.cell_start.data_ptr(), stree.cell_count.data_ptr(),
                self.plan.levels, lo, hi, ttree.n, float(self.kernel.symmetry), near.data_ptr(),
                scratch.data_ptr(), sb, st), "bfmm_p2p_symmetric")
            self._kspan("p2p", e0)
            return
        if self.near_mode == "grouped" and m == 1:
            # every leaf one thread per target, 8 leaves per warp (bfmm_p2p
            # already does this for its leaves of <= 8 points)
            e0 = self._kevent()
            _native.check(self.lib.bfmm_p2p_grouped(
                self._handle, ttree.pts4.data_ptr(), ttree.leaves.data_ptr(),
                ttree.starts.data_ptr(), ttree.counts.data_ptr(), ttree.n_leaves.data_ptr(),
                ttree.max_leaves, stree.pts4.data_ptr(), stree.cell_start.data_ptr(),
                stree.cell_count.data_ptr(), self.plan.levels, lo, hi, near.data_ptr(), st),
                "bfmm_p2p_grouped")
            self._kspan("p2p", e0)
            return
        if self.near_mode == "untiled":
            # (diagnostic) the thread-per-target kernel reading sources
            # through L1/L2 instead of the shared-memory tiles
            e0 = self._kevent()
            _native.check(self.lib.bfmm_p2p(
                self._handle, ttree.pts4.data_ptr(), ttree.leaves.data_ptr(),
                ttree.starts.data_ptr(), ttree.counts.data_ptr(), ttree.n_leaves.data_ptr(),
                ttree.max_leaves, stree.pts4.data_ptr(), ws.data_ptr(), m,
                stree.cell_start.data_ptr(), stree.cell_count.data_ptr(), self.plan.levels, lo,
                hi, near.data_ptr(), scratch.data_ptr(), sb, st), "bfmm_p2p")
            self._kspan("p2p", e0)
            return
        e0 = self._kevent()
        _native.check(self.lib.bfmm_p2p_cells(
            self._handle, ttree.pts4.data_ptr(), ttree.leaves.data_ptr(), ttree.starts.data_ptr(),
            ttree.counts.data_ptr(), ttree.n_leaves.data_ptr(), ttree.max_leaves,
            ttree.cell_start.data_ptr(), ttree.cell_count.data_ptr(),
            stree.pts4.data_ptr(), ws.data_ptr(), m, stree.cell_start.data_ptr(),
            stree.cell_count.data_ptr(), self.plan.levels, lo, hi, near.data_ptr(),
            scratch.data_ptr(), sb, st), "bfmm_p2p_cells")
        self._kspan("p2p", e0)

    def _use_symmetric(self, ttree, stree, m):
        """Transpose replay like the reference (shared points, symmetric or
        antisymmetric kernel, engine.py:361-364), for one weight column and
        leaves dense enough (>= 8 points on average) that the per-neighbour
        slot traffic stays small against the halved kernel evaluations."""
        # measured on C2 (B200): 2.22 ms symmetric vs 2.16 ms for all 27 offsets
        # -- the per-source warp reductions cost what the halving saves, so
        # "auto" keeps the full path until the replay kernel is faster
        if self.near_mode != "symmetric":
            return False
        return ttree is stree and self.kernel.symmetry in (-1, 1) and m == 1

    # per-kernel CUDA events on the launching (current) stream, enabled by
    # profile_kernels; read back after the evaluate's synchronising status read
    def _kevent(self):
        if not self.profile_kernels:
            return None
        torch = _torch()
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def _kspan(self, name, e0):
        if e0 is None:
            return
        torch = _torch()
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        self._kpending.append((name, e0, e1))

    # -- driver -----------------------------------------------------------------
    def evaluate(self, sources, targets=None, weights=None, _shard=None):
        """phi[i, c] = sum_j K(x_i, y_j) w[j, c] (reference engine.py:482-536).

        ``_shard`` = (MortonShards, ShardComm) runs this call as one rank of a
        multi-GPU matvec (paper_1903_02153_b200.parallel.ShardedEvaluator)."""
        torch = _torch()
        with torch.cuda.device(self.device):
            return self._evaluate(sources, targets, weights, _shard)

    def _evaluate(self, sources, targets, weights, _shard):
        torch = _torch()
        sharded = _shard is not None and not _shard[0].full
        shared = targets is None or targets is sources
        as_tensor = isinstance(sources, torch.Tensor)
        out_device = sources.device if as_tensor else None
        if not as_tensor:
            # shape validation mirrors the reference (eng:51-57, 484-497); the
            # O(N) finiteness checks of points and weights run on the device
            # (tree build / weight gather status flags, _raise_flags) in the
            # reference's order: sources, targets, weights
            src_np = np.asarray(sources)
            _check_host_shape(src_np, "sources")
            if not shared:
                _check_host_shape(np.asarray(targets), "targets")
            if weights is None:
                raise ConfigurationError("weights are required")
            w_shape = np.shape(weights)
            if len(w_shape) not in (1, 2) or w_shape[0] != src_np.shape[0]:
                raise ConfigurationError(
                    f"weights shape {w_shape} does not match {src_np.shape[0]} sources")
        if self._graph_ok(sources, targets, weights, sharded, shared):
            return self._graph_evaluate(sources, weights, as_tensor, out_device)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        t_host0 = time.perf_counter()
        ev[0].record()
        src = self._prepare_points(sources, "sources")
        tgt = src if shared else self._prepare_points(targets, "targets")
        w_event = None
        if (isinstance(weights, torch.Tensor) and weights.device.type == "cpu"
                and weights.is_pinned() and not sharded):
            # pinned host weights: copy them on the side stream while the
            # trees are built (they are first needed by gather_weights)
            main = torch.cuda.current_stream()
            side = self._side_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                w, squeeze = self._prepare_weights(weights, src.shape[0])
                w_event = torch.cuda.Event()
                w_event.record()
            w.record_stream(main)
        else:
            w, squeeze = self._prepare_weights(weights, src.shape[0])
        m = int(w.shape[1])
        n_src, n_tgt = int(src.shape[0]), int(tgt.shape[0])
        phi, status, ttree, stree, extras = self._device_step(
            src, tgt, w, w_event, m, n_src, n_tgt, shared, sharded, _shard, ev)
        if self.keep_stages:
            self.stages = dict(extras, stree=stree, ttree=ttree)
        phi_host = None
        if not as_tensor or out_device.type != "cuda":
            # async D2H into pinned memory, ordered before the status read
            phi_host = torch.empty((n_tgt, m), dtype=torch.float64, pin_memory=True)
            phi_host.copy_(phi, non_blocking=True)
        stat = status.cpu().numpy()  # the one synchronising read-back
        self.kernel_ms = {name: a.elapsed_time(b) for name, a, b in self._kpending}
        self._kpending = []
        self._raise_flags(stat, ttree, stree)
        if as_tensor:
            result = phi if out_device.type == "cuda" else phi_host
        else:
            result = phi_host.numpy()
        total_host = time.perf_counter() - t_host0
        ms = [ev[i].elapsed_time(ev[i + 1]) * 1e-3 for i in range(6)]
        self.timings = {
            "upload": ms[0], "distribute": ms[1], "upward": ms[2],
            "far_field": ms[3] if not self._disable_far_field else 0.0,
            "downward": ms[4] if not self._disable_far_field else 0.0,
            "near_field": ms[5], "near_pairs": int(stat.view(np.int64)[4]),
        }
        self.timings["total"] = sum(v for k, v in self.timings.items()
                                    if k not in ("near_pairs", "upload"))
        self.timings["wall"] = total_host
        return result[:, 0] if squeeze else result

    def _device_step(self, src, tgt, w, w_event, m, n_src, n_tgt, shared, sharded, _shard, ev):
        """Everything of a matvec that runs on the device, from the tree build
        to the output scatter (no host synchronisation: capturable in a CUDA
        graph).  ev: 7 timing events or None."""
        torch = _torch()
        status = torch.zeros(16, dtype=torch.int32, device=self.device)
        st = self._stream()
        if ev:
            ev[1].record()
        self._nv_push("distribute")
        stree = self._build_tree(src, status, _ST_DOMAIN_SRC)
        ttree = stree if shared else self._build_tree(tgt, status, _ST_DOMAIN_TGT)
        if w_event is not None:
            torch.cuda.current_stream().wait_event(w_event)
        ws = torch.empty((max(n_src, 1), m), dtype=torch.float64, device=self.device)
        _native.check(self.lib.bfmm_gather_weights(w.data_ptr(), n_src, m, stree.perm.data_ptr(),
                                                   ws.data_ptr(), stree.pts4.data_ptr(),
                                                   status[_ST_WEIGHTS:].data_ptr(), st),
                      "bfmm_gather_weights")
        self._nv_pop()
        if ev:
            ev[2].record()
        shard = _shard if sharded else None
        if sharded and _shard[0].balance == "work":
            # work-balanced Morton ranges from this target tree (same on every rank)
            bins = torch.empty(64, dtype=torch.int64, device=self.device)
            _native.check(self.lib.bfmm_level2_work(
                ttree.leaves.data_ptr(), ttree.counts.data_ptr(), ttree.n_leaves.data_ptr(),
                ttree.max_leaves, stree.cell_count.data_ptr(), self.plan.levels,
                bins.data_ptr(), st), "bfmm_level2_work")
            _shard[0].set_work(bins.cpu().numpy())
        # sharded: rows of other ranks' targets must read as zero
        alloc = torch.zeros if sharded else torch.empty
        near = alloc((max(n_tgt, 1), m), dtype=torch.float64, device=self.device)
        side = None
        main = torch.cuda.current_stream()
        near_ready = torch.cuda.Event()
        near_ready.record(main)  # trees and weights: all the near field needs

        pairs_counted = False

        def count_pairs():
            # timings["near_pairs"] (reference engine.py:532): status int64 slot 4
            _native.check(self.lib.bfmm_near_pair_count(
                ttree.leaves.data_ptr(), ttree.counts.data_ptr(), ttree.n_leaves.data_ptr(),
                ttree.max_leaves, stree.cell_count.data_ptr(), self.plan.levels,
                status.view(torch.int64)[4:5].data_ptr(), self._stream()),
                "bfmm_near_pair_count")

        def near_on_side():
            # near field on a side stream, concurrent with the far field (for
            # a shard: computes while the level all-gathers are in flight)
            nonlocal pairs_counted
            side = self._side_stream(1)
            side.wait_event(near_ready)
            with torch.cuda.stream(side):
                self._near_field(ttree, stree, ws, m, near, shard)
                count_pairs()  # off the far field's critical path
            pairs_counted = True
            return side

        overlap = self.overlap_near or (sharded and self.overlap_near_sharded)
        if overlap and (sharded or self.near_after_far is False):
            side = near_on_side()
        hi = None
        if overlap and self.far_priority and not sharded:
            # far-field chain on a higher-priority stream: the block scheduler
            # hands freed SMs to its kernels before the near field's
            hi = self._hi_stream()
            hi.wait_stream(main)
        phi_far = alloc((max(n_tgt, 1), m), dtype=torch.float64, device=self.device)
        with (torch.cuda.stream(hi) if hi is not None else contextlib.nullcontext()):
            self._nv_push("upward")
            moments, leaf_geom = self._upward(stree, ws, m, status, shard)
            self._nv_pop()
            if ev:
                ev[3].record()
            if not self._disable_far_field:
                self._nv_push("far_field")
                locs = self._far_field(moments, m, shard, self._active_cells(ttree, shard),
                                       active_src=stree is ttree)
                self._nv_pop()
                if overlap and side is None:
                    # enqueued after the far field: the persistent P2P grid fills
                    # the SMs the M2L CTAs leave free instead of holding them all
                    side = near_on_side()
                if ev:
                    ev[4].record()
                self._nv_push("downward")
                self._downward(locs, ttree, m, leaf_geom, status, phi_far, shard)
                self._nv_pop()
            else:
                locs = None
                phi_far = None
                if ev:
                    ev[4].record()
            if ev:
                ev[5].record()
        if hi is not None:
            main.wait_stream(hi)
        if side is None:
            self._near_field(ttree, stree, ws, m, near, shard)
        else:
            main.wait_stream(side)
        phi = torch.empty((n_tgt, m), dtype=torch.float64, device=self.device)
        if sharded:
            # every rank holds phi of its own contiguous range of the sorted
            # targets: all-gather the ranges, then un-permute everywhere
            near = self._gather_sorted_phi(phi_far, near, ttree, m, _shard)
            phi_far = None
        _native.check(self.lib.bfmm_scatter_output(
            phi_far.data_ptr() if phi_far is not None else None, near.data_ptr(),
            ttree.perm.data_ptr(), n_tgt, m, phi.data_ptr(), status[_ST_NONFINITE:].data_ptr(), st),
            "bfmm_scatter_output")
        if not pairs_counted:
            count_pairs()
        if ev:
            ev[6].record()
        extras = {"moments": moments, "locals": locs, "near": near, "far": phi_far, "ws": ws}
        return phi, status, ttree, stree, extras

    def _gather_sorted_phi(self, phi_far, near, ttree, m, shard):
        """phi of the sorted targets on every rank: rank r computed the rows
        of its Morton range, [b_r, b_{r+1}) in sorted order (the trees are
        identical on every rank, so each derives every boundary itself)."""
        torch = _torch()
        shards, comm = shard
        L, n = self.plan.levels, ttree.n
        nl = int(ttree.n_leaves.item())
        if nl == 0:
            return near
        cuts = torch.tensor([shards.cells_of(r, L)[0] for r in range(comm.world)],
                            dtype=torch.int64, device=self.device)
        idx = torch.searchsorted(ttree.leaves[:nl], cuts)
        pos = torch.where(idx < nl, ttree.starts[:nl][idx.clamp(max=nl - 1)],
                          torch.full_like(idx, n))
        b = pos.cpu().tolist() + [n]
        lo, hi = b[comm.rank], b[comm.rank + 1]
        own = near[lo:hi] if phi_far is None else near[lo:hi] + phi_far[lo:hi]
        return comm.allgather_rows(own.contiguous(), [b[r + 1] - b[r] for r in range(comm.world)])

    # -- CUDA graph replay (use_graph) ----------------------------------------
    def _graph_ok(self, sources, targets, weights, sharded, shared):
        """The whole device step replays from a CUDA graph when nothing in it
        needs the host: one point set (targets = sources), Chebyshev tables,
        the dense far field, no sharding, no per-kernel/stage inspection."""
        if not self.use_graph or sharded or not shared or self.keep_stages:
            return False
        if self.profile_kernels or self._disable_far_field or weights is None:
            return False
        if self.plan.scheme is not SchemeKind.CHEBYSHEV:
            return False
        n = int(sources.shape[0])
        L = self.plan.levels
        # the sparse-cloud active lists read counts back on the host
        return self.far_mode == "dense" or (self.far_mode == "auto" and n >= 8 * (1 << (3 * L)))

    _GRAPH_KNOBS = ("m2l_mode", "i8_slices", "i8_digits", "p2m_mode", "leaf_mode", "proj_mode",
                    "far_mode",
                    "near_mode",
                    "overlap_near",
                    "near_after_far", "far_priority", "l2p_mode", "stream_levels",
                    "main_levels")

    def _graph_knobs(self):
        """Every evaluator knob that changes the captured kernels: part of
        the graph key, so changing one after a capture re-captures."""
        return tuple(getattr(self, k) for k in self._GRAPH_KNOBS)

    def _graph_evaluate(self, sources, weights, as_tensor, out_device):
        """evaluate() through a captured CUDA graph of _device_step (identical
        kernels and buffers, so identical results: tests/test_gpu_graph.py).
        Device float64 inputs are read in place and pinned host tensors are
        copied inside the graph (the weights on a side stream, under the tree
        build, as in the eager path) -- graphs are keyed by the input
        buffers; other host inputs go through static device buffers.  Stage
        timings come from external event-record nodes inside the graph."""
        torch = _torch()
        t_host0 = time.perf_counter()
        src_t = sources if as_tensor else torch.from_numpy(
            np.ascontiguousarray(sources, dtype=np.float64))
        if src_t.ndim != 2 or src_t.shape[1] != 3:
            raise ConfigurationError(
                f"sources must be an (N, 3) array, got shape {tuple(src_t.shape)}")
        w_t = weights if isinstance(weights, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(weights, dtype=np.float64))
        squeeze = w_t.ndim == 1
        if squeeze:
            w_t = w_t[:, None]
        n = int(src_t.shape[0])
        if w_t.ndim != 2 or w_t.shape[0] != n:
            raise ConfigurationError(
                f"weights shape {tuple(weights.shape)} does not match {n} sources")
        m = int(w_t.shape[1])

        def plain(t, dev):
            return (t.dtype == torch.float64 and t.is_contiguous() and
                    (t.is_cuda if dev else (not t.is_cuda and t.is_pinned())))
        knobs = self._graph_knobs()
        if plain(src_t, True) and plain(w_t, True) and src_t.device == self.device:
            kind, key = "device", ("device", n, m, src_t.data_ptr(), w_t.data_ptr(), knobs)
        elif plain(src_t, False) and plain(w_t, False):
            kind, key = "pinned", ("pinned", n, m, src_t.data_ptr(), w_t.data_ptr(), knobs)
        else:
            kind, key = "static", ("static", n, m, knobs)
        ent = self._graphs.get(key)
        if ent is None:
            if len(self._graphs) >= 4:  # each graph keeps its memory pool
                self._graphs.pop(next(iter(self._graphs)))
            stat_in = None
            if kind == "static":
                stat_in = (torch.empty((n, 3), dtype=torch.float64, device=self.device),
                           torch.empty((n, m), dtype=torch.float64, device=self.device))
                stat_in[0].copy_(src_t)
                stat_in[1].copy_(w_t)

            # stage timestamps inside the graph: external event-record
            # nodes fire on every replay (reference timings keys, eng:505-533)
            gev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(7)]

            def body():
                gev[0].record()
                if kind == "device":
                    xs, ws_, w_ev = src_t, w_t, None
                elif kind == "static":
                    (xs, ws_), w_ev = stat_in, None
                else:
                    main = torch.cuda.current_stream()
                    xs = torch.empty((n, 3), dtype=torch.float64, device=self.device)
                    xs.copy_(src_t, non_blocking=True)
                    side = self._side_stream()
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        ws_ = torch.empty((n, m), dtype=torch.float64, device=self.device)
                        ws_.copy_(w_t, non_blocking=True)
                        w_ev = torch.cuda.Event()
                        w_ev.record()
                    ws_.record_stream(main)
                return self._device_step(xs, xs, ws_, w_ev, m, n, n, True, False, None, gev)

            body()  # eager warm-up: lazy tables, kernel attributes
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            l0 = self.lib.bfmm_launch_count()
            with torch.cuda.graph(g):
                outs = body()
            ent = self._graphs[key] = (g, stat_in, outs, int(self.lib.bfmm_launch_count() - l0),
                                       gev)
        g, stat_in, outs, nlaunch, gev = ent
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if stat_in is not None:
            for dst, a in ((stat_in[0], src_t), (stat_in[1], w_t)):
                if a.is_cuda or a.is_pinned():
                    dst.copy_(a, non_blocking=True)
                else:
                    self._h2d_into(dst, a.numpy())
        g.replay()
        self.graph_launches += nlaunch  # our kernels inside the replayed graph
        phi, status, ttree, stree, _ = outs
        if as_tensor and out_device.type == "cuda":
            result = phi.clone()
        else:
            result = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
            result.copy_(phi, non_blocking=True)
        e1.record()
        stat = status.cpu().numpy()  # the one synchronising read-back
        self.kernel_ms = {}
        self._raise_flags(stat, ttree, stree)
        if not as_tensor:
            result = result.numpy()
        ms = [gev[i].elapsed_time(gev[i + 1]) * 1e-3 for i in range(6)]
        self.timings = {"upload": ms[0], "distribute": ms[1], "upward": ms[2],
                        "far_field": ms[3], "downward": ms[4], "near_field": ms[5],
                        "near_pairs": int(stat.view(np.int64)[4])}
        self.timings["total"] = sum(ms[1:])
        self.timings["graph_total"] = e0.elapsed_time(e1) * 1e-3
        self.timings["wall"] = time.perf_counter() - t_host0
        return result[:, 0] if squeeze else result

    def _raise_flags(self, stat, ttree, stree):
        # the reference's order: non-finite sources, then targets (eng:51-57,
        # 485-486), non-finite weights (eng:496-497), then the domain check
        # of the tree (oct:190-196)
        if stat[_ST_DOMAIN_SRC] & 2:
            raise DomainError("sources contain non-finite coordinates")
        if stat[_ST_DOMAIN_TGT] & 2:
            raise DomainError("targets contain non-finite coordinates")
        if stat[_ST_WEIGHTS]:
            raise ConfigurationError("weights contain non-finite values")
        if stat[_ST_DOMAIN_SRC] or stat[_ST_DOMAIN_TGT]:
            d = self.plan.domain
            raise DomainError(f"a point lies outside the box centered at {d.center} "
                              f"with length {d.length}")
        if stat[_ST_REF]:
            raise DomainError("a point landed outside its leaf cell; the tree assignment is inconsistent")
        if stat[_ST_NONFINITE]:
            self._locate_nonfinite(ttree, stree)

    def _locate_nonfinite(self, ttree, stree):
        torch = _torch()
        key = torch.full((1,), -1, dtype=torch.int64, device=self.device)
        _native.check(self.lib.bfmm_p2p_locate(
            self._handle, ttree.pts4.data_ptr(), ttree.leaves.data_ptr(), ttree.starts.data_ptr(),
            ttree.counts.data_ptr(), ttree.n_leaves.data_ptr(), ttree.max_leaves,
            stree.pts4.data_ptr(), stree.cell_start.data_ptr(), stree.cell_count.data_ptr(),
            self.plan.levels, key.data_ptr(), self._stream()), "bfmm_p2p_locate")
        k = int(key.cpu().numpy().view(np.uint64)[0])
        if k == 0xFFFFFFFFFFFFFFFF:
            raise KernelEvaluationError(
                f"kernel {self.kernel.name!r} produced a non-finite near-field sum")
        trow, srow = (k >> 29) & ((1 << 29) - 1), k & ((1 << 29) - 1)
        ti = int(ttree.perm[trow].item())
        si = int(stree.perm[srow].item())
        x = ttree.pts4[trow, :3].cpu().numpy()
        y = stree.pts4[srow, :3].cpu().numpy()
        raise KernelEvaluationError(
            f"kernel {self.kernel.name!r} returned a non-finite value for "
            f"target {ti} and source {si}", x=x, y=y, indices=(ti, si))

    # -- diagnostics used by the parity tests -------------------------------------
    def partition(self, points):
        """The device tree of a point set as NumPy arrays (perm, leaves,
        starts, counts), comparable with the reference _Partition."""
        torch = _torch()
        pts = self._prepare_points(points, "points")
        status = torch.zeros(16, dtype=torch.int32, device=self.device)
        tr = self._build_tree(pts, status, 0)
        nl = int(tr.n_leaves.item())
        if status[0].item():
            raise DomainError("a point lies outside the domain box")
        return {"perm": tr.perm[:tr.n].cpu().numpy(), "leaves": tr.leaves[:nl].cpu().numpy(),
                "starts": tr.starts[:nl].cpu().numpy(), "counts": tr.counts[:nl].cpu().numpy(),
                "tree": tr}

    def far_pairs(self, level, t_index):
        torch = _torch()
        n3 = 1 << (3 * level)
        tg = torch.empty(n3, dtype=torch.int64, device=self.device)
        sr = torch.empty(n3, dtype=torch.int64, device=self.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        sb = self.lib.bfmm_far_pairs_scratch_bytes(level)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        _native.check(self.lib.bfmm_far_pairs(level, t_index, tg.data_ptr(), sr.data_ptr(),
                                              cnt.data_ptr(), scratch.data_ptr(), sb,
                                              self._stream()), "bfmm_far_pairs")
        c = int(cnt.item())
        return tg[:c].cpu().numpy(), sr[:c].cpu().numpy()

    def near_segments(self, points, t_index, tree=None):
        """(tseg, sseg) of near offset t_index (reference _neighbor_segments,
        engine.py:401-417) for a point set's tree (or a prebuilt one)."""
        torch = _torch()
        tr = tree if tree is not None else self.partition(points)["tree"]
        out = torch.empty(max(tr.max_leaves, 1), dtype=torch.int64, device=self.device)
        _native.check(self.lib.bfmm_near_pairs(self.plan.levels, t_index, tr.leaves.data_ptr(),
                                               tr.n_leaves.data_ptr(), tr.max_leaves,
                                               tr.leaves.data_ptr(), tr.n_leaves.data_ptr(),
                                               out.data_ptr(), self._stream()), "bfmm_near_pairs")
        nl = int(tr.n_leaves.item())
        o = out[:nl].cpu().numpy()
        tseg = np.nonzero(o >= 0)[0]
        return tseg, o[tseg]


def _check_host_shape(pts, name):
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ConfigurationError(f"{name} must be an (N, 3) array, got shape {np.shape(pts)}")


def direct_evaluate(kernel: KernelSpec, sources, targets=None, weights=None,
                    target_block: int = 1024, source_block: int = 8192):
    """O(N_t N_s) direct sum on the GPU (reference engine.py:565-624).

    Explicit coordinate differences throughout (a target coinciding with a
    source gives r = 0 exactly; for shared sets this is the reference's
    zeroed diagonal) and compensated FP64 accumulation in place of long
    double.  ``target_block`` / ``source_block`` are accepted for signature
    compatibility; the device tiling is fixed."""
    torch = _torch()
    if not isinstance(kernel, KernelSpec):
        raise ConfigurationError("kernel must be a KernelSpec")
    if not kernel.has_device_form:
        raise ConfigurationError(f"kernel {kernel.name!r} has no device form")
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device is visible")
    lib = _native.load()
    as_tensor = isinstance(sources, torch.Tensor)
    src = (sources.to("cuda", torch.float64).contiguous() if as_tensor
           else torch.from_numpy(np.ascontiguousarray(sources, dtype=np.float64)).cuda())
    shared = targets is None or targets is sources
    if src.ndim != 2 or src.shape[1] != 3:
        raise ConfigurationError(f"sources must be an (N, 3) array, got shape {tuple(src.shape)}")
    if shared:
        tgt = src
    elif isinstance(targets, torch.Tensor):
        tgt = targets.to("cuda", torch.float64).contiguous()
    else:
        tgt = torch.from_numpy(np.ascontiguousarray(targets, dtype=np.float64)).cuda()
    if weights is None:
        raise ConfigurationError("weights are required")
    w = (weights.to("cuda", torch.float64) if isinstance(weights, torch.Tensor)
         else torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float64)).cuda())
    squeeze = w.ndim == 1
    w = (w[:, None] if squeeze else w).contiguous()
    if w.shape[0] != src.shape[0]:
        raise ConfigurationError(
            f"weights shape {tuple(w.shape)} does not match {src.shape[0]} sources")
    if kernel.builtin_id:
        handle = int(kernel.builtin_id)
    else:
        h = _native.C.c_int(0)
        _native.check(lib.bfmm_kernel_compile(_KIND[kernel.cuda_arg], kernel.cuda_expr.encode(),
                                              _native.C.byref(h)), "NVRTC compile")
        handle = int(h.value)
    m = int(w.shape[1])
    out = torch.empty((tgt.shape[0], m), dtype=torch.float64, device="cuda")
    _native.check(lib.bfmm_direct(handle, tgt.data_ptr(), int(tgt.shape[0]), src.data_ptr(),
                                  w.data_ptr(), int(src.shape[0]), m, out.data_ptr(),
                                  _native.C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                  "bfmm_direct")
    res = out if as_tensor else out.cpu().numpy()
    return res[:, 0] if squeeze else res


def evaluate(kernel: KernelSpec, plan: FmmPlan, sources, targets=None, weights=None,
             cache_dir=None, threads: int = 1, table: M2LTable = None):
    """One-shot wrapper (reference engine.py:539-545)."""
    ev = FmmEvaluator(kernel, plan, cache_dir=cache_dir, threads=threads, table=table)
    return ev.evaluate(sources, targets, weights)


__all__ = ["FmmEvaluator", "direct_evaluate", "evaluate", "neighbor_offsets"]
