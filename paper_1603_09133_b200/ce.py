"""Host-side mirror of the reference interface for the CE hot path.

Reference names kept (proj/include/ce/):
  CompressionStrategy    compression.hpp:15-38
  FactorOptions          factorization.hpp:74-77
  ce_factorize           factorization.hpp:121-123
  CEFactorization.solve  factorization.hpp:90   (preconditioner apply)
  CEFactorization.apply_q / apply_q_transpose / apply_operator   factorization.hpp:92-96
  BreakdownError(level, block)   types.hpp:26-36
  SolveReport            minres.hpp:25-31
  pcg                    the minres contract (minres.hpp:46-47) with PCG, SURVEY.md §8b
  minres / MinresOptions minres.hpp:34-47 (minres.cpp:22-115) on the device
Vectors are numpy float64 arrays (host) or torch float64 CUDA tensors (device).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import lib

CE_OK, CE_EUSAGE, CE_EBREAKDOWN, CE_ENOCONV = 0, 1, 2, 3


class BreakdownError(RuntimeError):
    """Pivot failure that survived the diagonal-shift retry (types.hpp:26-36)."""

    def __init__(self, level: int, block: int, what: str):
        super().__init__(what)
        self.level = level
        self.block = block


def _check(rc: int):
    if rc != CE_OK:
        raise RuntimeError(L.last_error() or f"libce_gpu error {rc}")


def device_count() -> int:
    return int(lib.ce_device_count())


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class Context:
    """One GPU (ce_ctx).  Default per device via Context.get()."""

    _default = {}

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.ce_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    @classmethod
    def get(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def __del__(self):
        if getattr(self, "handle", None):
            lib.ce_ctx_destroy(self.handle)
            self.handle = None


@dataclass
class CompressionStrategy:
    """CE(eps) / CE(r) rule (compression.hpp:15-38)."""

    mode: str = "eps"  # "eps" | "rank"
    eps: float = 1e-6
    absolute: bool = False
    rank: int = 0

    @staticmethod
    def adaptive(eps: float, absolute: bool = False) -> "CompressionStrategy":
        return CompressionStrategy("eps", eps, absolute, 0)

    @staticmethod
    def fixed_rank(rank: int) -> "CompressionStrategy":
        return CompressionStrategy("rank", 0.0, False, rank)

    def _c(self) -> L.Strategy:
        return L.Strategy(1 if self.mode == "rank" else 0, float(self.eps), int(self.absolute), int(self.rank))

    def describe(self) -> str:
        """CompressionStrategy::describe (compression.cpp:10-18)."""
        return _text(lambda buf, cap: lib.ce_strategy_describe(C.byref(self._c()), buf, cap))


@dataclass
class FactorOptions:
    dense_threshold: int = 2048
    max_levels: int = 64
    forced_ranks: List[Sequence[int]] = field(default_factory=list)  # parity hook, -1 = free


@dataclass
class PcgOptions:
    tol: float = 1e-10
    maxit: int = 1000
    track_true_residual: bool = False


@dataclass
class MinresOptions:  # proj/include/ce/minres.hpp:34-38
    tol: float = 1e-10
    maxit: int = 1000
    track_true_residual: bool = True


@dataclass
class SolveReport:
    converged: bool
    iterations: int
    final_recurrence_residual: float
    final_true_residual: float
    seconds: float
    # IterationTrace (minres.hpp:12-23): (iter, recurrence_resid, true_resid or -1, seconds) per iteration
    trace: List[tuple] = field(default_factory=list)


class CoarseningPlan:
    """Per-level block -> group assignments (problems.hpp:51-65 / plan text format)."""

    def __init__(self, assigns: Sequence[Sequence[int]], join: int = 2):
        self.assigns = [_i64(a) for a in assigns]
        self.join = int(join)
        self._blocks = _i64([len(a) for a in self.assigns])
        self._flat = _i64(np.concatenate(self.assigns)) if self.assigns else _i64([0])

    @staticmethod
    def trivial() -> "CoarseningPlan":
        return CoarseningPlan([], 2)

    def _c(self) -> L.PlanHost:
        return L.PlanHost(self.join, len(self.assigns), _ptr(self._blocks, C.c_int64), _ptr(self._flat, C.c_int64))


class BlockSparseMatrix:
    """Host CSB (block_matrix.hpp:23-63): both triangles, row-major blocks."""

    def __init__(self, offsets, row_ptr, col_idx, val_ptr, values):
        self.offsets = _i64(offsets)
        self.row_ptr = _i64(row_ptr)
        self.col_idx = _i64(col_idx)
        self.val_ptr = _i64(val_ptr)
        self.values = _f64(values)
        self.n = int(self.offsets[-1])
        self.m = len(self.offsets) - 1

    def _c(self) -> L.CsbHost:
        return L.CsbHost(self.n, self.m, _ptr(self.offsets, C.c_int64), _ptr(self.row_ptr, C.c_int64),
                         _ptr(self.col_idx, C.c_int64), _ptr(self.val_ptr, C.c_int64),
                         _ptr(self.values, C.c_double))

    @staticmethod
    def from_dense(a: np.ndarray, offsets: Sequence[int]) -> "BlockSparseMatrix":
        """Blocks on the nonzero block pattern (+ full diagonal), like from_triplets (block_matrix.cpp:48-90)."""
        a = np.asarray(a, dtype=np.float64)
        offsets = _i64(offsets)
        m = len(offsets) - 1
        row_ptr, col_idx, val_ptr, vals = [0], [], [0], []
        for i in range(m):
            for j in range(m):
                blk = a[offsets[i]:offsets[i + 1], offsets[j]:offsets[j + 1]]
                if i == j or np.any(blk != 0) or np.any(a[offsets[j]:offsets[j + 1], offsets[i]:offsets[i + 1]] != 0):
                    col_idx.append(j)
                    vals.append(blk.ravel())
                    val_ptr.append(val_ptr[-1] + blk.size)
            row_ptr.append(len(col_idx))
        return BlockSparseMatrix(offsets, row_ptr, col_idx, val_ptr, np.concatenate(vals))


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _stream_ptr(x):
    import torch
    return C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)


def _check_tensor(x, n: int, ctx: "Context", what: str):
    """A torch vector handed to the device path must be a contiguous float64 CUDA tensor of n
    entries on the context's device (its data_ptr is used as a device pointer)."""
    import torch
    if not x.is_cuda:
        raise ValueError(f"{what}: torch tensors must be CUDA tensors (pass numpy arrays for host data)")
    if x.device.index != ctx.device:
        raise ValueError(f"{what}: tensor on cuda:{x.device.index}, library context on cuda:{ctx.device}")
    if x.dtype != torch.float64:
        raise TypeError(f"{what}: tensor dtype must be torch.float64, got {x.dtype}")
    if not x.is_contiguous():
        raise ValueError(f"{what}: tensor must be contiguous")
    if x.numel() != n:
        raise ValueError(f"{what} dimension mismatch: {x.numel()} != {n}")


class DeviceMatrix:
    """Device-resident operator A (ce_matrix); matvec replaces BlockSparseMatrix::matvec."""

    def __init__(self, a: BlockSparseMatrix, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.get()
        self.host = a
        h = C.c_void_p()
        _check(lib.ce_matrix_upload(self.ctx.handle, C.byref(a._c()), C.byref(h)))
        self.handle = h
        self.n = a.n

    def __del__(self):
        if getattr(self, "handle", None):
            lib.ce_matrix_free(self.handle)
            self.handle = None

    @classmethod
    def from_triplets(cls, n: int, rows, cols, vals, offsets, mirror_lower: bool = False,
                      ctx: Optional[Context] = None) -> "DeviceMatrix":
        """BlockSparseMatrix::from_triplets (block_matrix.cpp:48-90) built on the GPU
        (ce_matrix_from_triplets); numpy arrays or CUDA tensors (int64 rows / cols, float64 vals)."""
        ctx = ctx or Context.get()
        offsets = _i64(offsets)
        if _is_torch(vals):
            import torch
            rows = rows.to(torch.int64).contiguous()
            cols = cols.to(torch.int64).contiguous()
            vals = vals.to(torch.float64).contiguous()
            nnz, dev = vals.numel(), 1
            ptrs = [C.c_void_p(t.data_ptr()) for t in (rows, cols, vals)]
        else:
            rows, cols, vals = _i64(rows), _i64(cols), _f64(vals)
            nnz, dev = vals.size, 0
            ptrs = [C.c_void_p(x.ctypes.data) for x in (rows, cols, vals)]
        h = C.c_void_p()
        _check(lib.ce_matrix_from_triplets(ctx.handle, int(n), int(nnz), *ptrs, len(offsets) - 1,
                                           _ptr(offsets, C.c_int64), int(mirror_lower), dev, C.byref(h)))
        self = cls.__new__(cls)
        self.ctx, self.handle, self.n = ctx, h, int(n)
        self.host = self.csb(values=False)
        return self

    def csb(self, values: bool = True) -> BlockSparseMatrix:
        """The CSB of this device matrix (ce_matrix_csb): structure, and the block values copied
        back when `values` (else zeros of the right size)."""
        v = L.CsbHost()
        _check(lib.ce_matrix_csb(self.handle, C.byref(v), None))
        m = v.m
        nnzb = int(np.ctypeslib.as_array(v.row_ptr, (m + 1,))[-1])
        val_ptr = np.ctypeslib.as_array(v.val_ptr, (nnzb + 1,)).copy()
        vals = np.zeros(int(val_ptr[-1]))
        if values:
            _check(lib.ce_matrix_csb(self.handle, C.byref(v), _ptr(vals, C.c_double)))
        return BlockSparseMatrix(np.ctypeslib.as_array(v.offsets, (m + 1,)).copy(),
                                 np.ctypeslib.as_array(v.row_ptr, (m + 1,)).copy(),
                                 np.ctypeslib.as_array(v.col_idx, (nnzb,)).copy(), val_ptr, vals)

    def matvec(self, x):
        if _is_torch(x):
            import torch
            _check_tensor(x, self.n, self.ctx, "matvec")
            y = torch.empty_like(x)
            _check(lib.ce_matvec(self.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), self.n, 1,
                                 _stream_ptr(x)))
            return y
        x = _f64(x)
        if x.size != self.n:
            raise ValueError("matvec dimension mismatch")
        y = np.empty(self.n)
        _check(lib.ce_matvec(self.handle, x.ctypes.data, y.ctypes.data, self.n, 0, None))
        return y

    __call__ = matvec


class CEFactorization:
    """Device-resident CE factor A ~ Q^T L L^T Q (factorization.hpp:81-102)."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        self.n = int(lib.ce_factor_dim(handle))

    def __del__(self):
        if getattr(self, "handle", None):
            lib.ce_factor_free(self.handle)
            self.handle = None

    def solve(self, b):
        """x = Q^T L^-T L^-1 Q b (factorization.cpp:140-168)."""
        if _is_torch(b):
            import torch
            _check_tensor(b, self.n, self.ctx, "solve")
            x = torch.empty_like(b)
            _check(lib.ce_apply_precond(self.handle, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), self.n, 1,
                                        _stream_ptr(b)))
            return x
        b = _f64(b)
        if b.size != self.n:
            raise ValueError("solve dimension mismatch")
        x = np.empty(self.n)
        _check(lib.ce_apply_precond(self.handle, b.ctypes.data, x.ctypes.data, self.n, 0, None))
        return x

    __call__ = solve

    def _tool(self, which: int, x) -> np.ndarray:
        x = _f64(x)
        if x.size != self.n:
            raise ValueError("dimension mismatch")
        y = np.empty(self.n)
        _check(lib.ce_factor_apply_tool(self.handle, which, x.ctypes.data, y.ctypes.data, self.n))
        return y

    def apply_operator(self, x) -> np.ndarray:
        return self._tool(0, x)

    def apply_q(self, x) -> np.ndarray:
        return self._tool(1, x)

    def apply_q_transpose(self, y) -> np.ndarray:
        return self._tool(2, y)

    @property
    def stats(self) -> dict:
        s = L.FactorStats()
        _check(lib.ce_factor_get_stats(self.handle, C.byref(s)))
        return {k: getattr(s, k) for k, _ in L.FactorStats._fields_}

    def level_stats(self) -> List[dict]:
        out = []
        for lvl in range(self.stats["n_levels"]):
            s = L.LevelStats()
            _check(lib.ce_factor_get_level_stats(self.handle, lvl, C.byref(s)))
            out.append({k: getattr(s, k) for k, _ in L.LevelStats._fields_})
        return out

    def level_rows(self, level: int):
        """(sizes, retained, fcols, nsigma) of every row of `level` (0-based)."""
        m = int(self.level_stats()[level]["block_count"])
        arrs = [np.empty(m, np.int64) for _ in range(4)]
        _check(lib.ce_factor_level_rows(self.handle, level, *[_ptr(a, C.c_int64) for a in arrs]))
        return tuple(arrs)

    def row_sigma(self, level: int, row: int, cap: int = 4096) -> np.ndarray:
        out = np.empty(cap)
        k = int(lib.ce_factor_row_sigma(self.handle, level, row, _ptr(out, C.c_double), cap))
        if k < 0:
            _check(CE_EUSAGE)
        return out[:min(k, cap)].copy()

    def dump(self, path: str):
        _check(lib.ce_factor_dump(self.handle, path.encode()))


def ce_factorize(a, plan: Optional[CoarseningPlan], strategy: CompressionStrategy,
                 opts: Optional[FactorOptions] = None, ctx: Optional[Context] = None) -> CEFactorization:
    """Multilevel CE factorization on the GPU (factorization.cpp:336-461)."""
    opts = opts or FactorOptions()
    if isinstance(a, BlockSparseMatrix):
        a = DeviceMatrix(a, ctx)
    ctx = a.ctx
    plan = plan or CoarseningPlan.trivial()
    counts = _i64([len(f) for f in opts.forced_ranks]) if opts.forced_ranks else _i64([0])
    flat = _i64(np.concatenate([_i64(f) for f in opts.forced_ranks])) if opts.forced_ranks else _i64([0])
    copts = L.FactorOpts(int(opts.dense_threshold), int(opts.max_levels), len(opts.forced_ranks),
                         _ptr(counts, C.c_int64), _ptr(flat, C.c_int64))
    st = L.Status()
    h = C.c_void_p()
    rc = lib.ce_factorize(ctx.handle, a.handle, C.byref(plan._c()), C.byref(strategy._c()), C.byref(copts),
                          C.byref(h), C.byref(st))
    if rc == CE_EBREAKDOWN:
        raise BreakdownError(st.level, st.block, st.message.decode())
    _check(rc)
    f = CEFactorization(h, ctx)
    f.shift_retries = st.shift_retries
    return f


class _DeviceBytes:
    """A raw device byte range, viewed zero-copy as a torch tensor (__cuda_array_interface__)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class ShardComm:
    """torch.distributed plumbing for ce_factorize_sharded (include/ce_gpu.h ce_bcast_fn).

    One process per GPU.  The library calls `bcast(dev_ptr, bytes, root)` in the same order on
    every rank; it becomes dist.broadcast -- straight on the device buffer under NCCL (NVLink /
    NVSwitch), staged through host memory under gloo (the multi-process test backend)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
        self.device = torch.device(device)
        self.calls, self.bytes, self.error = 0, 0, None
        self.fn = L.BcastFn(self._bcast)  # kept alive with the object

    def _bcast(self, user, ptr, nbytes, root):
        try:
            import torch
            if self.device.type == "cpu":  # host buffers (the CPU test of this plumbing)
                t = torch.frombuffer((C.c_uint8 * int(nbytes)).from_address(int(ptr)), dtype=torch.uint8)
                self.dist.broadcast(t, src=root if self.group is None else self.dist.get_global_rank(self.group, root),
                                    group=self.group)
                self.calls += 1
                self.bytes += int(nbytes)
                return 0
            t = torch.as_tensor(_DeviceBytes(ptr, nbytes), device=self.device)
            src = root if self.group is None else self.dist.get_global_rank(self.group, root)
            if self.backend == "nccl":
                self.dist.broadcast(t, src=src, group=self.group)
                torch.cuda.current_stream(self.device).synchronize()
            else:
                h = t.cpu() if self.rank == root else torch.empty(int(nbytes), dtype=torch.uint8)
                self.dist.broadcast(h, src=src, group=self.group)
                if self.rank != root:
                    t.copy_(h)
                    torch.cuda.synchronize(self.device)
            self.calls += 1
            self.bytes += int(nbytes)
            return 0
        except Exception as e:  # noqa: BLE001 -- reported through the library's error path
            self.error = e
            return 1


class LocalShardComm:
    """The one-rank communicator: ce_factorize_sharded on a single GPU (every box owned here,
    every broadcast a no-op) -- the 1-GPU point of a sharded scaling series."""

    def __init__(self):
        self.rank, self.world, self.error, self.calls, self.bytes = 0, 1, None, 0, 0

        def _b(user, ptr, nbytes, root):
            self.calls += 1
            return 0
        self.fn = L.BcastFn(_b)


def ce_factorize_sharded(a, plan: CoarseningPlan, strategy: CompressionStrategy, box_of_block, comm: ShardComm,
                         opts: Optional[FactorOptions] = None, n_boxes: int = 8,
                         ctx: Optional[Context] = None) -> CEFactorization:
    """This rank's part of the subdomain-sharded factorization (ce_factorize_sharded,
    DESIGN.md §7): every rank passes the same matrix / plan / labels; the returned factor is
    complete on every rank and identical to ce_factorize of the same plan on one GPU."""
    opts = opts or FactorOptions()
    if isinstance(a, BlockSparseMatrix):
        a = DeviceMatrix(a, ctx)
    ctx = a.ctx
    labels = _i64(box_of_block)
    if labels.size != a.host.m:
        raise ValueError("box_of_block must label every level-1 block")
    counts = _i64([len(f) for f in opts.forced_ranks]) if opts.forced_ranks else _i64([0])
    flat = _i64(np.concatenate([_i64(f) for f in opts.forced_ranks])) if opts.forced_ranks else _i64([0])
    copts = L.FactorOpts(int(opts.dense_threshold), int(opts.max_levels), len(opts.forced_ranks),
                         _ptr(counts, C.c_int64), _ptr(flat, C.c_int64))
    sh = L.Shard(comm.rank, comm.world, int(n_boxes), _ptr(labels, C.c_int64), comm.fn, None)
    st = L.Status()
    h = C.c_void_p()
    rc = lib.ce_factorize_sharded(ctx.handle, a.handle, C.byref(plan._c()), C.byref(strategy._c()), C.byref(copts),
                                  C.byref(sh), C.byref(h), C.byref(st))
    if rc == CE_EBREAKDOWN:
        raise BreakdownError(st.level, st.block, st.message.decode())
    if rc != CE_OK and comm.error is not None:
        raise RuntimeError(f"sharded factorization: exchange failed: {comm.error!r}")
    _check(rc)
    f = CEFactorization(h, ctx)
    f.shift_retries = st.shift_retries
    return f


def _pattern_call(fn, rows_out: int, row_ptr, cols, *extra, square: bool = True, ctx: Optional[Context] = None):
    ctx = ctx or Context.get()
    row_ptr, cols = _i64(row_ptr), _i64(cols)
    m = len(row_ptr) - 1
    # output bound: the candidate count (square: sum of deg(k) over the entries; coarsen: nnz)
    cap = max(1, int(np.sum(np.diff(row_ptr)[cols])) if square else len(cols))
    optr, ocol, nnz = np.zeros(rows_out + 1, np.int64), np.zeros(cap, np.int64), C.c_int64()
    _check(fn(ctx.handle, m, _ptr(row_ptr, C.c_int64), _ptr(cols, C.c_int64), *extra, _ptr(optr, C.c_int64),
              _ptr(ocol, C.c_int64), cap, C.byref(nnz)))
    return optr, ocol[:nnz.value].copy()


def pattern_square(row_ptr, cols, ctx: Optional[Context] = None):
    """pattern_square (proj/src/pattern.cpp:64-86) on the GPU: CSR (sorted rows) -> CSR of P^2."""
    return _pattern_call(lib.ce_pattern_square, len(row_ptr) - 1, row_ptr, cols, ctx=ctx)


def pattern_coarsen(row_ptr, cols, group_of, ng: int, ctx: Optional[Context] = None):
    """coarsen_pattern (pattern.cpp:97-118) on the GPU; group_of[b] = -1 drops block b."""
    g = _i64(group_of)
    return _pattern_call(lib.ce_pattern_coarsen, int(ng), row_ptr, cols, int(ng), _ptr(g, C.c_int64), square=False,
                         ctx=ctx)


def shard_plan_summary(problem: "Problem", n_ranks: int, max_levels: int = 64) -> List[dict]:
    """Symbolic phase split of a "sharded"-plan problem over n_ranks (host only, no GPU):
    per level the block count, the box-interior (phase-1) rows and the rows each rank sweeps
    alone (ce_shard_plan_summary)."""
    out = np.zeros(max_levels * (2 + n_ranks), np.int64)
    nl = C.c_int64()
    _check(lib.ce_shard_plan_summary(problem.handle, int(n_ranks), int(max_levels), _ptr(out, C.c_int64), C.byref(nl)))
    rows = out[:nl.value * (2 + n_ranks)].reshape(nl.value, 2 + n_ranks)
    return [dict(blocks=int(r[0]), interior=int(r[1]), own=[int(x) for x in r[2:]]) for r in rows]


def _krylov(entry, what, a, n, b, precond, opts):
    if not isinstance(a, DeviceMatrix):
        raise TypeError(f"{what} runs on the device: `a` must be a DeviceMatrix")
    if precond is not None and not isinstance(precond, CEFactorization):
        raise TypeError("precond must be a CEFactorization or None")
    co = L.PcgOpts(float(opts.tol), int(opts.maxit), int(opts.track_true_residual))
    rep = L.Report()
    ph = precond.handle if precond is not None else None
    if _is_torch(b):
        import torch
        _check_tensor(b, n, a.ctx, what)
        x = torch.empty_like(b)
        # the solve runs on torch's current stream: b's producers and x's consumers are ordered
        rc = entry(a.ctx.handle, a.handle, ph, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), n, 1,
                   C.byref(co), C.byref(rep), _stream_ptr(b))
    else:
        b = _f64(b)
        if b.size != n:
            raise ValueError(f"{what} dimension mismatch")
        x = np.empty(n)
        rc = entry(a.ctx.handle, a.handle, ph, b.ctypes.data, x.ctypes.data, n, 0, C.byref(co), C.byref(rep), None)
    if rc not in (CE_OK, CE_ENOCONV):
        _check(rc)
    k = int(lib.ce_ctx_last_trace(a.ctx.handle, None, None, None, None, 0))
    it, rec, tru, sec = np.empty(k, np.int64), np.empty(k), np.empty(k), np.empty(k)
    lib.ce_ctx_last_trace(a.ctx.handle, _ptr(it, C.c_int64), _ptr(rec, C.c_double), _ptr(tru, C.c_double),
                          _ptr(sec, C.c_double), k)
    return SolveReport(bool(rep.converged), int(rep.iterations), rep.final_recurrence_residual,
                       rep.final_true_residual, rep.seconds,
                       [(int(i), float(r), float(t), float(q)) for i, r, t, q in zip(it, rec, tru, sec)]), x


def pcg(a: DeviceMatrix, n: int, b, precond: Optional[CEFactorization], opts: Optional[PcgOptions] = None):
    """Preconditioned CG with the minres contract; returns (SolveReport, x).

    `a` must be a DeviceMatrix and `precond` a CEFactorization or None (the
    device loop has no host callbacks).  Non-convergence is reported in the
    SolveReport, not raised, as in the reference."""
    return _krylov(lib.ce_pcg, "pcg", a, n, b, precond, opts or PcgOptions())


def minres(a: DeviceMatrix, n: int, b, precond: Optional[CEFactorization], opts: Optional[MinresOptions] = None):
    """MINRES (proj/src/minres.cpp:22-115, the paper's solver) on the device; returns
    (SolveReport, x).  Same contract as pcg: x0 = 0, recurrence stopping rule relative to
    the starting preconditioned residual, non-convergence reported, not raised."""
    return _krylov(lib.ce_minres, "minres", a, n, b, precond, opts or MinresOptions())


# ---- CSV reports of the reference CLI (proj/src/csv.cpp, proj/src/cli.cpp:60-80,153-247) ----
def _text(call) -> str:
    """Run a C text builder (buf, cap) -> length twice: size, then fill."""
    n = int(call(None, 0))
    if n < 0:
        _check(CE_EUSAGE)
    buf = C.create_string_buffer(n + 1)
    call(buf, n + 1)
    return buf.value.decode()


def fmt_double(v: float) -> str:
    """Shortest text that round-trips (csv.cpp:84-88, std::to_chars)."""
    return _text(lambda buf, cap: lib.ce_fmt_double(float(v), buf, cap))


def fmt_index(v: int) -> str:
    return str(int(v))


@dataclass
class CsvTable:
    """Comma-separated table with a header row, no quoting (csv.hpp:11-24): parse followed by
    to_string reproduces the input bytes."""

    header: List[str] = field(default_factory=list)
    rows: List[List[str]] = field(default_factory=list)

    def to_string(self) -> str:
        return "".join(",".join(r) + "\n" for r in [self.header] + self.rows)

    @staticmethod
    def parse(text: str) -> "CsvTable":
        if not text:
            raise ValueError("csv text has no header row")
        lines = text.split("\n")
        if text.endswith("\n"):
            lines.pop()
        return CsvTable(lines[0].split(","), [ln.split(",") for ln in lines[1:]])

    def write(self, path: str) -> None:
        try:
            with open(path, "wb") as fh:
                fh.write(self.to_string().encode())
        except OSError as e:
            raise OSError(f"cannot open {path} for writing") from e

    @staticmethod
    def load(path: str) -> "CsvTable":
        try:
            with open(path, "rb") as fh:
                return CsvTable.parse(fh.read().decode())
        except OSError as e:
            raise OSError(f"cannot open {path}") from e


def factor_stats_table(f: "CEFactorization") -> CsvTable:
    """factor_stats.csv (factor_stats_table, cli.cpp:60-71)."""
    return CsvTable.parse(_text(lambda buf, cap: lib.ce_factor_stats_csv(f.handle, buf, cap)))


def factor_summary_table(f: "CEFactorization", block: int, strategy: CompressionStrategy, seconds: float,
                         recon_error: str = "") -> CsvTable:
    """factor_summary.csv (run_factor, cli.cpp:167-182)."""
    return CsvTable.parse(_text(lambda buf, cap: lib.ce_factor_summary_csv(
        f.handle, int(block), C.byref(strategy._c()), float(seconds), recon_error.encode(), buf, cap)))


def trace_table(rep: SolveReport) -> CsvTable:
    """trace.csv (trace_table, cli.cpp:73-80)."""
    k = len(rep.trace)
    it = _i64([t[0] for t in rep.trace] or [0])
    cols = [np.ascontiguousarray([t[j] for t in rep.trace] or [0.0], np.float64) for j in (1, 2, 3)]
    return CsvTable.parse(_text(lambda buf, cap: lib.ce_trace_csv(
        k, _ptr(it, C.c_int64), *[_ptr(c, C.c_double) for c in cols], buf, cap)))


def solve_report_table(n: int, mode: str, strategy: Optional[CompressionStrategy], preconditioned: bool,
                       rep: SolveReport, factor_seconds: float, solve_seconds: float) -> CsvTable:
    """solve_report.csv (run_solve, cli.cpp:233-247); strategy None = "none" (no factorization)."""
    r = L.Report(int(rep.converged), int(rep.iterations), rep.final_recurrence_residual, rep.final_true_residual,
                 rep.seconds)
    sp = C.byref(strategy._c()) if strategy is not None else None
    return CsvTable.parse(_text(lambda buf, cap: lib.ce_solve_report_csv(
        int(n), mode.encode(), sp, int(preconditioned), C.byref(r), float(factor_seconds), float(solve_seconds),
        buf, cap)))


class Problem:
    """A BASELINE.json configuration generated on the host."""

    PLANS = {"reference": 0, "merge_all_axes": 1, "merge_all_colored": 2, "sharded": 3}

    def __init__(self, cfg: int, nx: int = 0, ny: int = 0, nz: int = 0, _handle=None, plan: str = "reference"):
        """plan: "reference" = geometric_block_ordering(grid, block, 2) (problems.cpp:195-258);
        "merge_all_axes" = every non-exhausted axis merges by 2 per level (J = 2^d);
        "merge_all_colored" = the same with each level's cells in mod-3 colour-major order;
        "sharded" = merge_all_colored with 8 spatial boxes, box-interior cells first."""
        if _handle is None:
            h = C.c_void_p()
            if plan not in self.PLANS:
                raise ValueError(f"plan must be one of {sorted(self.PLANS)}")
            _check(lib.ce_problem_create_plan(int(cfg), int(nx), int(ny), int(nz), self.PLANS[plan], C.byref(h)))
        else:
            h = _handle
        self.handle = h
        self.cfg = cfg
        csb = L.CsbHost()
        lib.ce_problem_csb(h, C.byref(csb))
        self.n, self.m = csb.n, csb.m
        nnzb = np.ctypeslib.as_array(csb.row_ptr, (self.m + 1,))[-1]
        self.offsets = np.ctypeslib.as_array(csb.offsets, (self.m + 1,)).copy()
        self.row_ptr = np.ctypeslib.as_array(csb.row_ptr, (self.m + 1,)).copy()
        self.col_idx = np.ctypeslib.as_array(csb.col_idx, (nnzb,)).copy()
        self.val_ptr = np.ctypeslib.as_array(csb.val_ptr, (nnzb + 1,)).copy()
        self.values = np.ctypeslib.as_array(csb.values, (int(self.val_ptr[-1]),)).copy()
        self.rhs = np.ctypeslib.as_array(lib.ce_problem_rhs(h), (self.n,)).copy()
        self.perm = np.ctypeslib.as_array(lib.ce_problem_perm(h), (self.n,)).copy()
        plan = L.PlanHost()
        lib.ce_problem_plan(h, C.byref(plan))
        blocks = np.ctypeslib.as_array(plan.level_blocks, (plan.n_levels,)).copy() if plan.n_levels else []
        flat = np.ctypeslib.as_array(plan.assign, (int(np.sum(blocks)),)).copy() if plan.n_levels else []
        assigns, at = [], 0
        for nb in blocks:
            assigns.append(flat[at:at + nb])
            at += nb
        self.plan = CoarseningPlan(assigns, plan.join)
        bp, nb = C.POINTER(C.c_int64)(), C.c_int64()
        lib.ce_problem_boxes(h, C.byref(bp), C.byref(nb))
        # CE_PLAN_SHARDED: subdomain label of every level-1 block (None for the other families)
        self.box_of_block = np.ctypeslib.as_array(bp, (self.m,)).copy() if nb.value else None
        self.n_boxes = int(nb.value)
        eps, tol, blk = C.c_double(), C.c_double(), C.c_int64()
        lib.ce_problem_params(h, C.byref(eps), C.byref(tol), C.byref(blk))
        self.eps, self.tol, self.block = eps.value, tol.value, blk.value

    def __del__(self):
        if getattr(self, "handle", None):
            lib.ce_problem_free(self.handle)
            self.handle = None

    @classmethod
    def load(cls, matrix: str, plan: Optional[str] = None, rhs: Optional[str] = None, block: int = 8) -> "Problem":
        """The reference CLI's `file` problem (cli.cpp:114-133): Matrix Market matrix, optional
        plan file (else the trivial plan with `block`), optional rhs file (else ones)."""
        h = C.c_void_p()
        enc = lambda x: None if x is None else os.fsencode(x)  # noqa: E731
        _check(lib.ce_problem_load(enc(matrix), enc(plan), enc(rhs), int(block), C.byref(h)))
        return cls(0, _handle=h)

    def save(self, matrix: Optional[str] = None, plan: Optional[str] = None, rhs: Optional[str] = None) -> None:
        """run_gen's files (cli.cpp:136-150): natural-order matrix.mtx, plan.txt, rhs.txt."""
        enc = lambda x: None if x is None else os.fsencode(x)  # noqa: E731
        _check(lib.ce_problem_save(self.handle, enc(matrix), enc(plan), enc(rhs)))

    def matrix(self) -> BlockSparseMatrix:
        return BlockSparseMatrix(self.offsets, self.row_ptr, self.col_idx, self.val_ptr, self.values)

    def strategy(self) -> CompressionStrategy:
        return CompressionStrategy.adaptive(self.eps)
