"""Reader of the binary factor dump shared by the oracle (oracle/factor.cpp
write_factor_dump) and the GPU library (ce_factor_dump).  DESIGN.md "Dump format"."""

import numpy as np


class _R:
    def __init__(self, path):
        self.b = open(path, "rb").read()
        self.o = 0

    def i64(self, n=None):
        k = 1 if n is None else n
        v = np.frombuffer(self.b, np.int64, k, self.o)
        self.o += 8 * k
        return int(v[0]) if n is None else v.copy()

    def f64(self, n):
        v = np.frombuffer(self.b, np.float64, n, self.o)
        self.o += 8 * n
        return v.copy()


def read_dump(path):
    r = _R(path)
    assert r.b[:4] == b"CEFD"
    r.o = 4
    ver = r.i64()
    assert ver == 1
    n, nlev, tail = r.i64(), r.i64(), r.i64()
    levels = []
    for _ in range(nlev):
        m = r.i64()
        offsets = r.i64(m + 1)
        bs = np.diff(offsets)
        retained = r.i64(m)
        has_basis = r.i64(m)
        basis = [None] * m
        for b in range(m):
            if has_basis[b]:
                basis[b] = r.f64(int(bs[b] ** 2)).reshape(bs[b], bs[b])
        fcols = r.i64(m)
        nsig = r.i64(m)
        sigma = [r.f64(int(k)) for k in nsig]
        rows = []
        for b in range(m):
            w = r.i64()
            if w == 0:
                rows.append(None)
                continue
            rk = int(retained[b])
            chol = r.f64(w * w).reshape(w, w)
            coupling = r.f64(rk * w).reshape(rk, w)
            nnb = r.i64()
            nbs = []
            for _ in range(nnb):
                t = r.i64()
                nbs.append((t, r.f64(int(bs[t]) * w).reshape(int(bs[t]), w)))
            rows.append(dict(width=w, chol=chol, coupling=coupling, neighbors=nbs))
        ng = r.i64()
        groups = []
        for _ in range(ng):
            k = r.i64()
            groups.append(r.i64(k).tolist())
        levels.append(dict(m=m, offsets=offsets, sizes=bs, retained=retained, has_basis=has_basis, basis=basis,
                           fcols=fcols, sigma=sigma, rows=rows, groups=groups))
    tail_chol = r.f64(tail * tail).reshape(tail, tail) if tail else np.zeros((0, 0))
    assert r.o == len(r.b), "trailing bytes in dump"
    return dict(n=n, levels=levels, tail_dim=tail, tail_chol=tail_chol)
