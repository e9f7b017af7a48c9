"""Debug C5 parity: which step diverges from the oracle at 8192^2 (advection alone; prep + 1 subcycle)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import numpy as np
import oracle
from paper_2402_00466_b200 import inputs, nxsdg
from tests.parity import group_err
cfg = inputs.CONFIGS[os.environ.get("CFG", "C5")]
st = inputs.make_config_case(cfg)
prm = nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha)
opts = json.loads(os.environ.get("OPTS", "{}"))
CORE = 8
wins = [(0, 0), (cfg.nx // 2, cfg.ny // 2), (cfg.nx - 40, cfg.ny - 40), (5000, 7000), (7000, 300)]


def cut(arrs, ix0, iy0, w, h):
    p, nx, ny = cfg.p, cfg.nx, cfg.ny
    out = {}
    for k, a in arrs.items():
        if a.ndim == 2 and a.shape == (p * ny + 1, p * nx + 1):
            out[k] = np.ascontiguousarray(a[p * iy0:p * (iy0 + h) + 1, p * ix0:p * (ix0 + w) + 1])
        else:
            out[k] = np.ascontiguousarray(a.reshape(ny, nx, a.shape[1])[iy0:iy0 + h, ix0:ix0 + w].reshape(-1, a.shape[1]))
    return out


def check(tag, got, nsub, adv):
    res = []
    for (cx, cy) in wins:
        ring = nsub + (5 if adv else 2)
        ix0, iy0 = max(0, cx - ring), max(0, cy - ring)
        w, h = min(cfg.nx, cx + CORE + ring) - ix0, min(cfg.ny, cy + CORE + ring) - iy0
        sub = cut(st, ix0, iy0, w, h)
        om = oracle.Mesh(w, h, lx=w * cfg.lx / cfg.nx, ly=h * cfg.ly / cfg.ny)
        o = oracle.Oracle()
        if nsub == 0:
            A, H = o.advect(om, prm.dt, sub["vx"], sub["vy"], sub["A"], sub["H"])
            rf = dict(sub, A=A, H=H)
        else:
            rf = o.outer_step(om, oracle.Params(alpha=cfg.alpha, beta=cfg.alpha), nsub, sub, do_advect=adv)
        g = cut(got, cx, cy, CORE, CORE)
        p = cfg.p; ex, ey = cx - ix0, cy - iy0
        rc = {}
        for k, a in rf.items():
            if k not in g:
                continue
            if k in ("vx", "vy"):
                rc[k] = a[p * ey:p * (ey + CORE) + 1, p * ex:p * (ex + CORE) + 1]
            else:
                rc[k] = a.reshape(h, w, -1)[ey:ey + CORE, ex:ex + CORE].reshape(-1, a.shape[1])
        e = {n: group_err(g, rc, grp) for n, grp in (("S", ("S11", "S12", "S22")), ("v", ("vx", "vy")), ("A", ("A",)), ("H", ("H",)))}
        res.append(((cx, cy), {k: float(f"{v:.2e}") for k, v in e.items()}))
    print(tag, json.dumps(res), flush=True)


with nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, cfg.p, cfg.ns, cfg.na, params=prm) as m:
    for k, v in opts.items():
        m.set_option(getattr(nxsdg, k), v)
    m.load(st)
    m.advect(prm.dt)
    got = m.state()
    check("advect only", got, 0, True)
    m.load(st)
    m.mevp_substeps(1, begin_step=True)
    check("prep + 1 subcycle (no advect)", m.state(), 1, False)
    m.load(st)
    m.mevp_substeps(10, begin_step=True)
    check("prep + 10 subcycles (no advect)", m.state(), 10, False)
