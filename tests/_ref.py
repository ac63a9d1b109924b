"""ctypes binding of the REFERENCE itself (oracle/_ref/libceref.so: /root/reference/proj/src
compiled unmodified against the Eigen stand-in oracle/ref/eigen_subset) — TEST INFRASTRUCTURE
ONLY: it pins the oracle restatement (tests/_oracle.py) against the reference's own code.
`available()` is False where the library was not built (it needs /root/reference to build)."""

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_ref", "libceref.so")
vp, i64 = C.c_void_p, C.c_int64
i64p, dblp = C.POINTER(C.c_int64), C.POINTER(C.c_double)
_lib = None


def build():
    if not os.path.exists(LIB) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle", "ref"), "-j8"], check=True, capture_output=True)


def available():
    build()
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB)
        sig = {
            "ceref_last_error": (C.c_char_p, []),
            "ceref_problem": (C.c_int, [i64, i64, i64p, i64p, i64p, i64p, dblp, i64, i64, i64p, i64p, C.POINTER(vp)]),
            "ceref_problem_free": (None, [vp]),
            "ceref_matvec": (C.c_int, [vp, dblp, dblp]),
            "ceref_factorize": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, i64, i64, C.POINTER(vp), i64p, i64p, dblp]),
            "ceref_factor_free": (None, [vp]),
            "ceref_apply": (C.c_int, [vp, C.c_int, dblp, dblp]),
            "ceref_levels": (i64, [vp]),
            "ceref_tail_dim": (i64, [vp]),
            "ceref_level_m": (i64, [vp, i64]),
            "ceref_level_structure": (None, [vp, i64, i64p, i64p, i64p, i64p]),
            "ceref_level_stats": (None, [vp, i64, dblp]),
            "ceref_factor_summary": (None, [vp, dblp]),
            "ceref_krylov": (C.c_int, [vp, vp, C.c_int, dblp, dblp, C.c_double, i64, C.c_int, i64p, dblp, dblp,
                                       C.POINTER(C.c_int), dblp]),
        }
        for k, (r, a) in sig.items():
            f = getattr(_lib, k)
            f.restype, f.argtypes = r, a
    return _lib


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


class RefBreakdown(RuntimeError):
    def __init__(self, level, block, msg):
        super().__init__(msg)
        self.level, self.block = level, block


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().ceref_last_error().decode())


class RefProblem:
    """Built from a CSB + plan (e.g. the oracle's or the product generator's arrays)."""

    def __init__(self, offsets, row_ptr, col_idx, val_ptr, values, assigns, join=2):
        L = lib()
        a = [np.ascontiguousarray(x, np.int64) for x in (offsets, row_ptr, col_idx, val_ptr)]
        vals = np.ascontiguousarray(values, np.float64)
        blocks = np.array([len(x) for x in assigns] or [0], np.int64)
        flat = np.ascontiguousarray(np.concatenate(assigns) if assigns else np.zeros(1), np.int64)
        self.n, self.m = int(a[0][-1]), len(a[0]) - 1
        h = vp()
        _check(L.ceref_problem(self.n, self.m, *[_p(x, C.c_int64) for x in a], _p(vals), join, len(assigns),
                               _p(blocks, C.c_int64), _p(flat, C.c_int64), C.byref(h)))
        self.h = h

    @staticmethod
    def from_oracle(op):
        assigns, join = op.plan_assigns()
        return RefProblem(*op.csb(), assigns, join)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ceref_problem_free(self.h)
            self.h = None

    def matvec(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.n)
        _check(lib().ceref_matvec(self.h, _p(x), _p(y)))
        return y

    def factorize(self, eps=1e-6, mode=0, absolute=False, rank=0, dense_threshold=2048):
        h, lvl, blk, sec = vp(), i64(), i64(), C.c_double()
        rc = lib().ceref_factorize(self.h, mode, eps, int(absolute), rank, dense_threshold, C.byref(h), C.byref(lvl),
                                   C.byref(blk), C.byref(sec))
        if rc == 2:
            raise RefBreakdown(lvl.value, blk.value, lib().ceref_last_error().decode())
        _check(rc)
        f = RefFactor(h, self.n)
        f.seconds = sec.value
        return f

    def krylov(self, b, factor=None, method="pcg", tol=1e-10, maxit=1000, track_true=False):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(self.n)
        it, rr, tr, sec, conv = i64(), C.c_double(), C.c_double(), C.c_double(), C.c_int()
        _check(lib().ceref_krylov(self.h, factor.h if factor else None, 0 if method == "pcg" else 1, _p(b), _p(x), tol,
                                  maxit, int(track_true), C.byref(it), C.byref(rr), C.byref(tr), C.byref(conv),
                                  C.byref(sec)))
        return dict(iterations=it.value, recurrence=rr.value, true_resid=tr.value, converged=bool(conv.value),
                    seconds=sec.value), x


class RefFactor:
    def __init__(self, h, n):
        self.h, self.n = h, n

    def __del__(self):
        if getattr(self, "h", None):
            lib().ceref_factor_free(self.h)
            self.h = None

    def _apply(self, which, v):
        v = np.ascontiguousarray(v, np.float64)
        o = np.empty(self.n)
        _check(lib().ceref_apply(self.h, which, _p(v), _p(o)))
        return o

    def solve(self, b):
        return self._apply(0, b)

    def apply_operator(self, x):
        return self._apply(1, x)

    def apply_q(self, x):
        return self._apply(2, x)

    def apply_q_transpose(self, y):
        return self._apply(3, y)

    @property
    def levels(self):
        return int(lib().ceref_levels(self.h))

    @property
    def tail_dim(self):
        return int(lib().ceref_tail_dim(self.h))

    def level_structure(self, lvl):
        m = int(lib().ceref_level_m(self.h, lvl))
        arrs = [np.empty(m, np.int64) for _ in range(4)]
        lib().ceref_level_structure(self.h, lvl, *[_p(a, C.c_int64) for a in arrs])
        return dict(sizes=arrs[0], retained=arrs[1], has_basis=arrs[2], width=arrs[3])

    def level_stats(self):
        keys = ["block_count", "pattern_blocks", "factor_blocks", "eliminated", "retained", "max_rank", "mean_rank",
                "seconds", "l_bytes", "q_bytes", "shift_retries"]
        out = []
        for lvl in range(self.levels):
            row = np.empty(11)
            lib().ceref_level_stats(self.h, lvl, _p(row))
            out.append(dict(zip(keys, row.tolist())))
        return out

    def summary(self):
        o = np.empty(7)
        lib().ceref_factor_summary(self.h, _p(o))
        return dict(zip(["factor_blocks", "predicted_factor_blocks", "l_scalar_nnz", "l_payload_bytes",
                         "q_payload_bytes", "tail_bytes", "total_seconds"], o.tolist()))
