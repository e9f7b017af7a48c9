"""NEXT-2 drift study: is the growth of the oracle's own plain-vs-FMA floor over the
paper's 30-outer-step protocol physical sensitivity or an unstable mEVP iteration?

The oracle alone (CPU), the 40 x 36 warm box at 2 km with the moving cyclone (the protocol of
tests/test_gpu_parity.py::test_paper_protocol_30_outer_steps_drift), 30 x (advect + 100 subcycles),
for alpha = beta in a list: after every outer step, the group-normalised relative max difference between
the plain (-ffp-contract=off) and FMA builds - two equally valid FP64 evaluations of the same method.
If the floor stays small at large alpha * beta (>> the stability estimate gamma ~ 9e6 at 2 km, SURVEY
§8(d).2), the growth at alpha = 1500 is the mEVP iteration amplifying rounding, not the physics.

    python scripts/drift_alpha.py [--alphas 1500 25000 100000] [--steps 30]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
from paper_2402_00466_b200 import inputs


def group_err(a, b, keys):
    num = max(float(np.abs(a[k] - b[k]).max()) for k in keys)
    den = max(float(np.abs(b[k]).max()) for k in keys)
    return num / den if den > 0 else num


def run(alpha, steps, nxe=40, nye=36, h=2e3):
    lx, ly = nxe * h, nye * h
    st = inputs.make_case(nxe, nye, 2, 6, 6, kind="warm", lx=lx, ly=ly)
    X, Y = np.meshgrid(np.arange(2 * nxe + 1) * (lx / nxe / 2), np.arange(2 * nye + 1) * (ly / nye / 2))
    om = oracle.Mesh(nxe, nye, lx=lx, ly=ly)
    prm = oracle.Params(alpha=alpha, beta=alpha)
    a, b = {k: v.copy() for k, v in st.items()}, {k: v.copy() for k, v in st.items()}
    oa, ob = oracle.Oracle("plain"), oracle.Oracle("fma")
    floor, vmax = [], []
    for k in range(steps):
        t = k * prm.dt
        f = [np.ascontiguousarray(x) for x in inputs.cyclone_forcing(X, Y, lx, ly, t)]
        for d in (a, b):
            d["ox"], d["oy"], d["ax"], d["ay"] = f
        a = oa.outer_step(om, prm, 100, a, do_advect=True)
        b = ob.outer_step(om, prm, 100, b, do_advect=True)
        e = 0.0
        for g in (("S11", "S12", "S22"), ("vx", "vy"), ("A",), ("H",)):
            e = max(e, group_err(b, a, g))
            gi = {kk: b[kk] - st[kk] for kk in g}
            ri = {kk: a[kk] - st[kk] for kk in g}
            if max(float(np.abs(v).max()) for v in ri.values()) > 0:
                e = max(e, group_err(gi, ri, g))
        floor.append(e)
        vmax.append(float(np.hypot(a["vx"], a["vy"]).max()))
    return floor, vmax


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alphas", type=float, nargs="+", default=[1500.0, 25000.0, 100000.0])
    ap.add_argument("--steps", type=int, default=30)
    a = ap.parse_args()
    res = {}
    for al in a.alphas:
        floor, vmax = run(al, a.steps)
        res[al] = floor
        print(f"alpha = beta = {al:>8g}: plain-vs-FMA floor per outer step: " + " ".join(f"{x:.1e}" for x in floor))
        print(f"{'':>24s}max |v| per outer step [m/s]:       " + " ".join(f"{x:.3f}" for x in vmax), flush=True)
    print(json.dumps({str(k): v for k, v in res.items()}))


if __name__ == "__main__":
    main()
