"""Who is closer to the exact answer when the GPU and the oracle differ at the ~1e-12 level?

The VP law amplifies strain rounding by P/Delta, so two correct FP64 evaluations of
one subcycle can differ by ~1e-12 (the oracle's plain and FMA builds do).  This script evaluates S
after ONE subcycle exactly (40-digit mpmath, the oracle's definitions: O4 strain projection,
Listing 2, projection with the diagonal box mass; inputs are the float64 test inputs taken as exact)
at the elements where the GPU and the oracle disagree most, and reports each side's distance from
it, normalised like tests/parity.py (by max |S| of the oracle over the group).

    python scripts/exact_stress.py [nx ny ns lx ly kind]      (needs the GPU for the CUDA side)
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np

import oracle
from paper_2402_00466_b200 import nxsdg
from tests.exact_mp import exact_S
from tests.parity import case, ora_mesh, ora_params


def main():
    a = sys.argv[1:]
    nxe, nye, ns = (int(a[0]), int(a[1]), int(a[2])) if a else (70, 75, 8)
    lx, ly = (float(a[3]), float(a[4])) if len(a) > 4 else (nxe * 2000.0, nye * 2000.0)
    kind = a[5] if len(a) > 5 else "warm"
    na = 6
    st = case(nxe, nye, 2, ns, na, kind, lx, ly)
    prm = nxsdg.PhysParams()
    with nxsdg.Mesh(nxe, nye, lx, ly, 2, ns, na, params=prm) as m:
        m.load(st)
        m.mevp_substeps(1, begin_step=True)
        gpu = m.state(("S11", "S12", "S22"))
    om, op = ora_mesh(nxe, nye, 2, ns, na, lx, ly), ora_params(prm)
    res = {v: oracle.Oracle(v).subcycles(om, op, 1, st) for v in ("plain", "fma")}
    G = lambda d: np.stack([d["S11"], d["S12"], d["S22"]], 1)          # (N, 3, ns)
    g, p, f = G(gpu), G(res["plain"]), G(res["fma"])
    scale = np.abs(p).max()
    worst = np.argsort(-np.abs(g - p).max(axis=(1, 2)))[:12]
    worst = np.unique(np.r_[worst, np.argsort(-np.abs(f - p).max(axis=(1, 2)))[:4]])
    rows = []
    for e in worst:
        x = exact_S(st, nxe, lx, ly, nye, ns, na, int(e), prm)
        rows.append({"elem": int(e), "gpu": float(np.abs(g[e] - x).max() / scale),
                     "oracle_plain": float(np.abs(p[e] - x).max() / scale),
                     "oracle_fma": float(np.abs(f[e] - x).max() / scale),
                     "gpu_vs_plain": float(np.abs(g[e] - p[e]).max() / scale)})
    summ = {k: max(r[k] for r in rows) for k in ("gpu", "oracle_plain", "oracle_fma", "gpu_vs_plain")}
    print(json.dumps({"case": [nxe, nye, ns, lx, ly, kind], "max_over_checked_elements": summ, "rows": rows}))


if __name__ == "__main__":
    main()
