"""Oracle self-consistency floor (plain vs FMA builds) on the cyclone-centre window of a config after its
outer step (advection + 100 subcycles), for several alpha = beta (R#13): a config is a valid 1e-10 target
only where two equally valid FP64 evaluations agree to ~1e-11.
    python scripts/floor_alpha.py C5 25000 100000 400000"""
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle
from paper_2402_00466_b200 import inputs


def group_err(a, b, keys):
    return max(float(np.abs(a[k] - b[k]).max()) for k in keys) / max(float(np.abs(b[k]).max()) for k in keys)


name = sys.argv[1]
cfg = inputs.CONFIGS[name]
core, nsub = 12, cfg.nsub
cx, cy = cfg.nx // 2 - core // 2, cfg.ny // 2 - core // 2
if os.environ.get("WIN"):   # "cx,cy" of the window's core (default: the cyclone centre)
    cx, cy = map(int, os.environ["WIN"].split(","))
ring = nsub + 5
ix0, iy0 = max(0, cx - ring), max(0, cy - ring)
w, h = min(cfg.nx, cx + core + ring) - ix0, min(cfg.ny, cy + core + ring) - iy0
ox, oy = cx - ix0, cy - iy0
sub = inputs.make_config_case(cfg, window=(ix0, iy0, w, h))
om = oracle.Mesh(w, h, lx=w * cfg.lx / cfg.nx, ly=h * cfg.ly / cfg.ny)
for al in map(float, sys.argv[2:]):
    prm = oracle.Params(alpha=al, beta=al)
    a = oracle.Oracle("plain").outer_step(om, prm, nsub, sub, do_advect=True)
    b = oracle.Oracle("fma").outer_step(om, prm, nsub, sub, do_advect=True)
    sl = lambda d: {k: (v[2 * oy:2 * (oy + core) + 1, 2 * ox:2 * (ox + core) + 1] if k in ("vx", "vy") else
                        v.reshape(h, w, -1)[oy:oy + core, ox:ox + core].reshape(-1, v.shape[1]))
                    for k, v in d.items() if k in ("vx", "vy", "S11", "S12", "S22")}
    A, B = sl(a), sl(b)
    print(json.dumps({"config": name, "window": [cx, cy], "alpha": al, "floor_S": group_err(B, A, ("S11", "S12", "S22")),
                      "floor_v": group_err(B, A, ("vx", "vy"))}), flush=True)
