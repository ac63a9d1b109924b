"""ctypes binding of the CPU oracle (oracle/liboracle.so) — TEST INFRASTRUCTURE ONLY.

The oracle restates the reference (/root/reference/proj) on the CPU; tests use
it as the checker of the GPU library, never as the thing measured.
"""

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "liboracle.so")

vp = C.c_void_p
i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)


def _build():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", ORACLE_DIR, "-j8"], check=True, capture_output=True)


_build()
lib = C.CDLL(LIB)
_sig = {
    "oracle_last_error": (C.c_char_p, []),
    "oracle_problem_config": (C.c_int, [C.c_int, i64, i64, i64, C.POINTER(vp)]),
    "oracle_problem_config_plan": (C.c_int, [C.c_int, i64, i64, i64, C.c_int, C.POINTER(vp)]),
    "oracle_problem_reference": (C.c_int, [C.c_int, i64, i64, i64, i64, C.POINTER(vp)]),
    "oracle_problem_triplets": (C.c_int, [i64, i64, i64p, i64p, dblp, i64, i64p, C.c_int, C.POINTER(vp)]),
    "oracle_problem_free": (None, [vp]),
    "oracle_problem_n": (i64, [vp]),
    "oracle_problem_m": (i64, [vp]),
    "oracle_problem_nnzb": (i64, [vp]),
    "oracle_problem_values": (i64, [vp]),
    "oracle_problem_csb": (None, [vp, i64p, i64p, i64p, i64p, dblp]),
    "oracle_problem_rhs": (None, [vp, dblp]),
    "oracle_problem_perm": (None, [vp, i64p]),
    "oracle_plan_levels": (i64, [vp]),
    "oracle_plan_join": (i64, [vp]),
    "oracle_plan_level_blocks": (i64, [vp, i64]),
    "oracle_plan_level_assign": (None, [vp, i64, i64p]),
    "oracle_matvec": (C.c_int, [vp, dblp, dblp]),
    "oracle_problem_dense": (None, [vp, dblp]),
    "oracle_factorize": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, i64, i64, i64, i64p, i64p, C.POINTER(vp),
                                   i64p, i64p]),
    "oracle_factor_free": (None, [vp]),
    "oracle_factor_solve": (C.c_int, [vp, dblp, dblp]),
    "oracle_factor_apply": (C.c_int, [vp, C.c_int, dblp, dblp]),
    "oracle_factor_reconstruct": (C.c_int, [vp, dblp]),
    "oracle_factor_dump": (C.c_int, [vp, C.c_char_p]),
    "oracle_factor_levels": (i64, [vp]),
    "oracle_factor_tail_dim": (i64, [vp]),
    "oracle_factor_summary": (None, [vp, dblp]),
    "oracle_factor_level_stats": (None, [vp, i64, dblp]),
    "oracle_factor_level_m": (i64, [vp, i64]),
    "oracle_factor_level_structure": (None, [vp, i64, i64p, i64p, i64p]),
    "oracle_factor_row_sigma": (i64, [vp, i64, i64, dblp, i64]),
    "oracle_problem_perturb": (None, [vp, C.c_double, C.c_ulonglong]),
    "oracle_krylov": (C.c_int, [vp, vp, C.c_int, dblp, dblp, C.c_double, i64, C.c_int, i64p, dblp, dblp,
                                C.POINTER(C.c_int), dblp]),
    "oracle_compress": (C.c_int, [i64, i64, dblp, C.c_int, C.c_double, C.c_int, i64, i64p, C.POINTER(C.c_int),
                                  dblp, dblp, i64p]),
    "oracle_pattern_op": (i64, [C.c_int, i64, i64p, i64p, i64, i64p, i64p, i64p, i64]),
}
for _n, (_r, _a) in _sig.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


class OracleError(RuntimeError):
    pass


class OracleBreakdown(OracleError):
    def __init__(self, level, block, msg):
        super().__init__(msg)
        self.level, self.block = level, block


def _check(rc):
    if rc != 0:
        raise OracleError(lib.oracle_last_error().decode())


class OProblem:
    def __init__(self, handle):
        self.h = handle
        self.n = int(lib.oracle_problem_n(handle))
        self.m = int(lib.oracle_problem_m(handle))

    @staticmethod
    def config(cfg, nx=0, ny=0, nz=0, plan="reference"):
        h = vp()
        _check(lib.oracle_problem_config_plan(cfg, nx, ny, nz, {"reference": 0, "merge_all_axes": 1, "merge_all_colored": 2, "sharded": 3}[plan], C.byref(h)))
        return OProblem(h)

    @staticmethod
    def reference(kind, nx, ny, nz, block):
        h = vp()
        _check(lib.oracle_problem_reference(kind, nx, ny, nz, block, C.byref(h)))
        return OProblem(h)

    @staticmethod
    def triplets(n, rows, cols, vals, offsets, mirror_lower=False):
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        offsets = np.ascontiguousarray(offsets, np.int64)
        h = vp()
        _check(lib.oracle_problem_triplets(n, len(rows), _p(rows, C.c_int64), _p(cols, C.c_int64), _p(vals),
                                           len(offsets) - 1, _p(offsets, C.c_int64), int(mirror_lower), C.byref(h)))
        return OProblem(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib.oracle_problem_free(self.h)
            self.h = None

    def csb(self):
        nnzb = int(lib.oracle_problem_nnzb(self.h))
        nv = int(lib.oracle_problem_values(self.h))
        off = np.empty(self.m + 1, np.int64)
        rp = np.empty(self.m + 1, np.int64)
        ci = np.empty(nnzb, np.int64)
        vptr = np.empty(nnzb + 1, np.int64)
        vals = np.empty(nv)
        lib.oracle_problem_csb(self.h, _p(off, C.c_int64), _p(rp, C.c_int64), _p(ci, C.c_int64), _p(vptr, C.c_int64),
                               _p(vals))
        return off, rp, ci, vptr, vals

    def rhs(self):
        out = np.empty(self.n)
        lib.oracle_problem_rhs(self.h, _p(out))
        return out

    def perm(self):
        out = np.empty(self.n, np.int64)
        lib.oracle_problem_perm(self.h, _p(out, C.c_int64))
        return out

    def plan_assigns(self):
        out = []
        for lvl in range(int(lib.oracle_plan_levels(self.h))):
            a = np.empty(int(lib.oracle_plan_level_blocks(self.h, lvl)), np.int64)
            lib.oracle_plan_level_assign(self.h, lvl, _p(a, C.c_int64))
            out.append(a)
        return out, int(lib.oracle_plan_join(self.h))

    def matvec(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.n)
        _check(lib.oracle_matvec(self.h, _p(x), _p(y)))
        return y

    def dense(self):
        out = np.empty((self.n, self.n))
        lib.oracle_problem_dense(self.h, _p(out))
        return out

    def factorize(self, eps=1e-6, mode=0, absolute=False, rank=0, dense_threshold=2048, forced=None):
        forced = forced or []
        counts = np.array([len(f) for f in forced] or [0], np.int64)
        flat = np.concatenate([np.asarray(f, np.int64) for f in forced]) if forced else np.zeros(1, np.int64)
        h = vp()
        lvl, blk = C.c_int64(), C.c_int64()
        rc = lib.oracle_factorize(self.h, mode, eps, int(absolute), rank, dense_threshold, len(forced),
                                  _p(counts, C.c_int64), _p(flat, C.c_int64), C.byref(h), C.byref(lvl), C.byref(blk))
        if rc == 2:
            raise OracleBreakdown(lvl.value, blk.value, lib.oracle_last_error().decode())
        _check(rc)
        return OFactor(h, self.n)

    def krylov(self, b, factor=None, method="pcg", tol=1e-10, maxit=1000, track_true=False):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(self.n)
        it, rr, tr, sec = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
        conv = C.c_int()
        _check(lib.oracle_krylov(self.h, factor.h if factor else None, 0 if method == "pcg" else 1, _p(b), _p(x), tol,
                                 maxit, int(track_true), C.byref(it), C.byref(rr), C.byref(tr), C.byref(conv),
                                 C.byref(sec)))
        return dict(iterations=it.value, recurrence=rr.value, true_resid=tr.value, converged=bool(conv.value),
                    seconds=sec.value), x


class OFactor:
    def __init__(self, h, n):
        self.h, self.n = h, n

    def __del__(self):
        if getattr(self, "h", None):
            lib.oracle_factor_free(self.h)
            self.h = None

    def solve(self, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(self.n)
        _check(lib.oracle_factor_solve(self.h, _p(b), _p(x)))
        return x

    def _apply(self, which, v):
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(self.n)
        _check(lib.oracle_factor_apply(self.h, which, _p(v), _p(out)))
        return out

    def apply_operator(self, x):
        return self._apply(0, x)

    def apply_q(self, x):
        return self._apply(1, x)

    def apply_q_transpose(self, y):
        return self._apply(2, y)

    def reconstruct(self):
        out = np.empty((self.n, self.n))
        _check(lib.oracle_factor_reconstruct(self.h, _p(out)))
        return out

    def dump(self, path):
        _check(lib.oracle_factor_dump(self.h, path.encode()))

    @property
    def levels(self):
        return int(lib.oracle_factor_levels(self.h))

    @property
    def tail_dim(self):
        return int(lib.oracle_factor_tail_dim(self.h))

    def summary(self):
        out = np.empty(8)
        lib.oracle_factor_summary(self.h, _p(out))
        keys = ["factor_blocks", "predicted_factor_blocks", "l_scalar_nnz", "l_payload_bytes", "q_payload_bytes",
                "tail_bytes", "total_seconds", "tail_seconds"]
        return dict(zip(keys, out.tolist()))

    def level_structure(self, lvl):
        m = int(lib.oracle_factor_level_m(self.h, lvl))
        sizes, ret, fc = (np.empty(m, np.int64) for _ in range(3))
        lib.oracle_factor_level_structure(self.h, lvl, _p(sizes, C.c_int64), _p(ret, C.c_int64), _p(fc, C.c_int64))
        return sizes, ret, fc

    def row_sigma(self, lvl, b, cap=4096):
        out = np.empty(cap)
        k = int(lib.oracle_factor_row_sigma(self.h, lvl, b, _p(out), cap))
        return out[:min(k, cap)].copy()

    def level_stats(self):
        keys = ["block_count", "pattern_blocks", "factor_blocks", "eliminated", "retained", "max_rank", "mean_rank",
                "seconds", "l_bytes", "q_bytes", "shift_retries", "predicted_edge"]
        out = []
        for lvl in range(self.levels):
            row = np.empty(12)
            lib.oracle_factor_level_stats(self.h, lvl, _p(row))
            out.append(dict(zip(keys, row.tolist())))
        return out


def compress(F, mode=0, eps=1e-6, absolute=False, rank=0):
    F = np.ascontiguousarray(F, np.float64)
    b, f = F.shape
    r = C.c_int64()
    hb = C.c_int()
    U = np.zeros((b, b))
    sig = np.zeros(max(min(b, f), 1))
    ns = C.c_int64()
    _check(lib.oracle_compress(b, f, _p(F), mode, eps, int(absolute), rank, C.byref(r), C.byref(hb), _p(U), _p(sig),
                               C.byref(ns)))
    return r.value, (U if hb.value else None), sig[:ns.value]


def pattern_op(op, rows, ngroups=0, assign=None):
    """rows: list of sorted column lists.  op 0 square, 1 far, 2 coarsen."""
    m = len(rows)
    rp = np.zeros(m + 1, np.int64)
    for i, r in enumerate(rows):
        rp[i + 1] = rp[i] + len(r)
    cols = np.array([c for r in rows for c in r] or [0], np.int64)
    assign = np.asarray(assign if assign is not None else [0], np.int64)
    cap = max(m, ngroups, 1) ** 2 + 1
    orp = np.zeros(max(m, ngroups) + 1, np.int64)
    oc = np.zeros(cap, np.int64)
    nnz = lib.oracle_pattern_op(op, m, _p(rp, C.c_int64), _p(cols, C.c_int64), ngroups, _p(assign, C.c_int64),
                                _p(orp, C.c_int64), _p(oc, C.c_int64), cap)
    if nnz < 0:
        raise OracleError(lib.oracle_last_error().decode())
    mo = ngroups if op == 2 else m
    return [oc[orp[i]:orp[i + 1]].tolist() for i in range(mo)]
