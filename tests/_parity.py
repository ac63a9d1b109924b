"""GPU-vs-oracle comparison of factor dumps (SURVEY.md §8c parity contract).

1. structure (exact): partitions, retained ranks, basis flags, groups, far widths;
2. singular values of every F_i within 1e-13 * sigma_1 (absolute);
3. factor blocks in the canonical gauge: per-row relative Frobenius error of
   [U | chol | coupling | neighbours] reported; rows whose retained spectrum has
   a relative gap below 1e-6 (gauge ill-conditioned) are reported separately.
"""

import numpy as np


def _rel(a, b):
    nb = np.linalg.norm(b)
    d = np.linalg.norm(a - b)
    return d / nb if nb > 0 else d


def compare(g, o, sigma_atol=1e-13):
    rep = dict(structure_ok=True, mismatch=None, sigma_max=0.0, row_err=[], row_err_illcond=[], tail_err=0.0,
               levels=len(o["levels"]), rank_mismatch=[])
    if g["n"] != o["n"] or len(g["levels"]) != len(o["levels"]) or g["tail_dim"] != o["tail_dim"]:
        rep["structure_ok"] = False
        rep["mismatch"] = ("levels", len(g["levels"]), len(o["levels"]), g["tail_dim"], o["tail_dim"])
        return rep
    for li, (G, O) in enumerate(zip(g["levels"], o["levels"])):
        if not np.array_equal(G["offsets"], O["offsets"]):
            rep["structure_ok"] = False
            rep["mismatch"] = ("offsets", li)
            return rep
        if not np.array_equal(G["retained"], O["retained"]):
            bad = np.nonzero(G["retained"] != O["retained"])[0]
            rep["rank_mismatch"].append((li, bad[:10].tolist()))
            rep["structure_ok"] = False
            rep["mismatch"] = ("retained", li, bad[:5].tolist())
            return rep
        for key in ("has_basis", "fcols"):
            if not np.array_equal(G[key], O[key]):
                rep["structure_ok"] = False
                rep["mismatch"] = (key, li, np.nonzero(G[key] != O[key])[0][:5].tolist())
                return rep
        if G["groups"] != O["groups"]:
            rep["structure_ok"] = False
            rep["mismatch"] = ("groups", li)
            return rep
        for b in range(O["m"]):
            so, sg = O["sigma"][b], G["sigma"][b]
            if len(so) != len(sg):
                rep["structure_ok"] = False
                rep["mismatch"] = ("nsigma", li, b)
                return rep
            if len(so):
                rep["sigma_max"] = max(rep["sigma_max"], float(np.max(np.abs(so - sg)) / so[0]))
            r = int(O["retained"][b])
            ill = False
            if len(so) > 1 and r > 1:
                gaps = (so[:r - 1] - so[1:r]) / so[0]
                ill = bool(np.any(gaps < 1e-6))
            parts_g, parts_o = [], []
            if O["basis"][b] is not None:
                parts_g.append(G["basis"][b].ravel())
                parts_o.append(O["basis"][b].ravel())
            rg, ro = G["rows"][b], O["rows"][b]
            if (rg is None) != (ro is None):
                rep["structure_ok"] = False
                rep["mismatch"] = ("width", li, b)
                return rep
            if ro is not None:
                parts_g += [rg["chol"].ravel(), rg["coupling"].ravel()] + [x.ravel() for _, x in rg["neighbors"]]
                parts_o += [ro["chol"].ravel(), ro["coupling"].ravel()] + [x.ravel() for _, x in ro["neighbors"]]
                if [t for t, _ in rg["neighbors"]] != [t for t, _ in ro["neighbors"]]:
                    rep["structure_ok"] = False
                    rep["mismatch"] = ("neighbors", li, b)
                    return rep
            if parts_o:
                e = _rel(np.concatenate(parts_g), np.concatenate(parts_o))
                (rep["row_err_illcond"] if ill else rep["row_err"]).append((e, li, b))
    if o["tail_dim"]:
        rep["tail_err"] = _rel(g["tail_chol"], o["tail_chol"])
    return rep


def summarize(rep):
    errs = np.array([e for e, _, _ in rep["row_err"]] or [0.0])
    ill = np.array([e for e, _, _ in rep["row_err_illcond"]] or [0.0])
    return dict(structure_ok=rep["structure_ok"], mismatch=rep["mismatch"], sigma_max=rep["sigma_max"],
                rows=len(rep["row_err"]), row_err_max=float(errs.max()), row_err_p99=float(np.quantile(errs, 0.99)),
                frac_le_1e10=float(np.mean(errs <= 1e-10)), illcond_rows=len(rep["row_err_illcond"]),
                illcond_err_max=float(ill.max()), tail_err=rep["tail_err"],
                worst=sorted(rep["row_err"], reverse=True)[:3])
