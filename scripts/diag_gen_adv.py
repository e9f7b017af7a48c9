"""Diagnose GPU vs oracle on general-quad advection at C4 resolution: a C4 window (global coordinates,
distorted vertices) run as its own mesh on both sides; advection only, then + subcycles."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle
from paper_2402_00466_b200 import inputs, nxsdg
from tests.parity import group_err, parity
cfg = inputs.CONFIGS["C4"]
V = inputs.distorted_vertices(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 0.25)
ix0, iy0, w, h = 3400, 1800, 96, 80
sub = inputs.make_config_case(cfg, window=(ix0, iy0, w, h))
hx, hy = cfg.lx / cfg.nx, cfg.ly / cfg.ny
for mode in ("box", "general"):
    verts = np.ascontiguousarray(V[iy0:iy0 + h + 1, ix0:ix0 + w + 1]) if mode == "general" else None
    for dt in (120.0, 30.0, 7.5):
        prm = nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha, dt=dt)
        with nxsdg.Mesh(w, h, w * hx, h * hy, 2, 6, 6, params=prm) as m:
            if verts is not None:
                m.set_vertices(verts)
            m.load(sub)
            m.advect(dt)
            got = m.state(("A", "H"))
        om = oracle.Mesh(w, h, lx=w * hx, ly=h * hy, p=2, ns=6, na=6, verts=verts)
        A, H = oracle.Oracle().advect(om, dt, sub["vx"], sub["vy"], sub["A"], sub["H"])
        dA = np.abs(got["A"] - A)
        e = np.unravel_index(np.argmax(dA), dA.shape)
        print(json.dumps({"mode": mode, "dt": dt, "A": group_err(got, {"A": A, "H": H}, ("A",)),
                          "H": group_err(got, {"A": A, "H": H}, ("H",)), "worst_elem": int(e[0]), "worst_coef": int(e[1]),
                          "dA_coef_max": [float(x) for x in dA.max(axis=0)]}), flush=True)
