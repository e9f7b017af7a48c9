"""Full-size parity at BASELINE.json's configurations, each at its full count, checked against the
oracle on windows (the paper's "comparing to the CPU version" protocol):

- C4 (4096^2 CG2/DG2, 125 m): one outer step = advection + BEGIN_STEP prep + 100 fused subcycles,
  exactly the launch configuration bench.py times ("box"); the same for the n_S = 8 space ("ns8") and
  for a distorted C4 mesh through the fused general-quad kernel ("general");
- C4 as 8 row strips of 4096 x 512 (the 8-GPU partition), one process per rank under torchrun on the one
  GPU (the deployment's topology: CUDA IPC P2P with fused peer stores, the device flag handshake and the
  multi-rank subcycle graph; scripts/strips8_full.py): windows centred on each of the 7 strip interfaces
  against the oracle, and every rank's rows bitwise equal to one context;
- C3 (2048^2, 250 m) and C5 (8192^2, 62.5 m, the weak-scaling per-GPU size), advection + 100.

Light cone: one subcycle moves information by at most one element (node v -> adjacent
elements' strain/stress -> their nodes), each RK stage of the advection by one element, the prep's
nodal means by one.  So the oracle run on a window padded by a ring of n_sub + 3 + 2 elements, with
the window's own (wrong) boundary conditions on the ring's outside, reproduces the global solution
exactly in the window's centre.  Windows: the four domain corners (the true boundary is inside them),
the cyclone centre, seeded random positions; for the strips, the interfaces.

Bar (north_star): relative max-norm error <= 1e-10 on S and v (fields and increments) after the full
count, <= 1e-12 on the A, H fields.  Unconditional for C3 and C4 (box and general quads), but not where
two equally valid FP64 evaluations of the method already disagree by more: for the n_S = 8 space at
125 m and for C5 at 62.5 m the oracle's own plain and FMA builds differ by 0.9e-10 ... 2.5e-10 in S after
one outer step at some windows (R#13; raising alpha does not reduce it at 62.5 m:
scripts/floor_alpha.py), so there the bar is max(1e-10, 4 x that floor), computed per window.  Every
window's errors are printed (they appear in the -m gpu log)."""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2402_00466_b200 import inputs
from tests.parity import group_err

pytestmark = pytest.mark.gpu
CORE = 12
PARAMS = ["box", "ns8", "general", "C3", "C5"]


def _cfg(kind):
    if kind == "C3":
        return inputs.CONFIGS["C3"]
    if kind == "C5":
        return inputs.CONFIGS["C5"]
    cfg = inputs.CONFIGS["C4"]
    return dataclasses.replace(cfg, ns=8) if kind == "ns8" else cfg


def _load_local(m, st, nxe):
    er0, ern, nr0, nrn = m.elem_row0, m.elem_rows, m.node_row0, m.node_rows
    loc = {k: np.ascontiguousarray(st[k][nr0:nr0 + nrn]) for k in ("vx", "vy", "ox", "oy", "ax", "ay")}
    for k in ("S11", "S12", "S22", "A", "H"):
        loc[k] = np.ascontiguousarray(st[k][er0 * nxe:(er0 + ern) * nxe])
    m.load(loc)


@pytest.fixture(scope="module", params=PARAMS)
def full_result(request):
    """Each: advection + prep + 100 fused subcycles at full size through the C ABI."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2402_00466_b200 import build
    build.build()
    from paper_2402_00466_b200 import nxsdg
    kind = request.param
    cfg = _cfg(kind)
    st = inputs.make_config_case(cfg)
    V = inputs.distorted_vertices(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 0.25) if kind == "general" else None
    prm = nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha)
    extra = {}
    with nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, cfg.p, cfg.ns, cfg.na, params=prm) as m:
        if V is not None:
            m.set_vertices(V)
        m.load(st)
        m.advect(prm.dt)
        m.mevp_substeps(cfg.nsub, begin_step=True)
        got = m.state()
    return kind, cfg, st, got, V, extra


def _cut(cfg, arrs, ix0, iy0, w, h):
    p, nx, ny = cfg.p, cfg.nx, cfg.ny
    out = {}
    for k, a in arrs.items():
        if a.ndim == 2 and a.shape == (p * ny + 1, p * nx + 1):
            out[k] = np.ascontiguousarray(a[p * iy0:p * (iy0 + h) + 1, p * ix0:p * (ix0 + w) + 1])
        else:
            n = a.shape[1]
            out[k] = np.ascontiguousarray(a.reshape(ny, nx, n)[iy0:iy0 + h, ix0:ix0 + w].reshape(-1, n))
    return out


def _windows(kind, cfg, extra):
    rng = np.random.default_rng(inputs.SEED_BASE + 4)
    nx, ny = cfg.nx, cfg.ny
    ws = [(0, 0), (nx - CORE, 0), (0, ny - CORE), (nx - CORE, ny - CORE), (nx // 2 - CORE // 2, ny // 2 - CORE // 2)]
    ws += [(int(rng.integers(0, nx - CORE)), int(rng.integers(0, ny - CORE))) for _ in range(3)]
    return ws


def _window_errors(kind, cfg, st, got, V, cx, cy):
    ring = cfg.nsub + 3 + 2
    ix0, iy0 = max(0, cx - ring), max(0, cy - ring)
    ix1, iy1 = min(cfg.nx, cx + CORE + ring), min(cfg.ny, cy + CORE + ring)
    w, h = ix1 - ix0, iy1 - iy0
    hx, hy = cfg.lx / cfg.nx, cfg.ly / cfg.ny
    sub = _cut(cfg, st, ix0, iy0, w, h)
    verts = None if V is None else np.ascontiguousarray(V[iy0:iy0 + h + 1, ix0:ix0 + w + 1])
    mesh = oracle.Mesh(w, h, lx=w * hx, ly=h * hy, p=cfg.p, ns=cfg.ns, na=cfg.na, verts=verts)
    oprm = oracle.Params(alpha=cfg.alpha, beta=cfg.alpha)
    p = cfg.p

    def core_of(res):
        out = {}
        for k, a in res.items():
            if k not in got:
                continue
            if a.ndim == 2 and a.shape == (p * h + 1, p * w + 1):
                out[k] = a[p * (cy - iy0):p * (cy - iy0 + CORE) + 1, p * (cx - ix0):p * (cx - ix0 + CORE) + 1]
            else:
                out[k] = a.reshape(h, w, a.shape[1])[cy - iy0:cy - iy0 + CORE, cx - ix0:cx - ix0 + CORE].reshape(-1, a.shape[1])
        return out

    rc = core_of(oracle.Oracle().outer_step(mesh, oprm, cfg.nsub, sub, do_advect=True))
    g = _cut(cfg, got, cx, cy, CORE, CORE)
    init = _cut(cfg, st, cx, cy, CORE, CORE)
    err, raw = {}, {}
    for name, grp in (("S", ("S11", "S12", "S22")), ("v", ("vx", "vy"))):
        err[name] = group_err(g, rc, grp)
        err["d" + name] = group_err({k: g[k] - init[k] for k in grp}, {k: rc[k] - init[k] for k in grp}, grp)
        # numerators and oracle magnitudes for the field-norm error (test below)
        raw[name] = (max(float(np.abs(g[k] - rc[k]).max()) for k in grp), max(float(np.abs(rc[k]).max()) for k in grp))
        raw["d" + name] = (max(float(np.abs((g[k] - init[k]) - (rc[k] - init[k])).max()) for k in grp),
                           max(float(np.abs(rc[k] - init[k]).max()) for k in grp))
    for name in ("A", "H"):
        err[name] = group_err(g, rc, (name,))
    err["_raw"] = raw
    bar = 1e-10
    if kind in ("ns8", "C5") and max(err["S"], err["dS"], err["v"], err["dv"]) > bar:
        fm = core_of(oracle.Oracle("fma").outer_step(mesh, oprm, cfg.nsub, sub, do_advect=True))
        floor = 0.0
        for grp in (("S11", "S12", "S22"), ("vx", "vy")):
            floor = max(floor, group_err(fm, rc, grp),
                        group_err({k: fm[k] - init[k] for k in grp}, {k: rc[k] - init[k] for k in grp}, grp))
        err["floor"] = floor
        bar = max(bar, 4 * floor)
    err["bar"] = bar
    return err


def test_full_size_window_parity(full_result, capsys):
    """Two measures, both asserted.  (1) north_star's relative max-norm error of each field,
    ||X_gpu - X_ora||_inf / ||X_ora||_inf (R#27): the numerator's max over every sampled window,
    the denominator the max of |X_ora| over the same windows (a lower bound of the field's norm, since the
    windows include the cyclone centre: conservative), <= 1e-10 unconditionally for every config.  (2) The
    stricter window-local ratio (each window's own max |X_ora| as denominator), <= 1e-10 except where the
    oracle's own plain and FMA builds already disagree by more (n_S = 8, C5: 4 x that floor)."""
    kind, cfg, st, got, V, extra = full_result
    rows, bad, raws = [], [], []
    for (cx, cy) in _windows(kind, cfg, extra):
        e = _window_errors(kind, cfg, st, got, V, cx, cy)
        raws.append(e.pop("_raw"))
        rows.append(f"  {kind:8s} ({cx:5d},{cy:5d})  " + "  ".join(f"{k}={v:.1e}" for k, v in e.items()))
        # S, v fields and increments at the bar; A, H fields at 1e-12.  One advection step at these
        # resolutions changes the high coefficients by ~1e-11 of the field while the DG volume and edge
        # terms cancel to ~11 digits, so the A, H increments carry no parity information.
        if max(e["S"], e["dS"], e["v"], e["dv"]) > e["bar"] or max(e["A"], e["H"]) > 1e-12:
            bad.append((cx, cy, e))
    norm = {k: max(r[k][0] for r in raws) / max(r[k][1] for r in raws) for k in raws[0]}
    with capsys.disabled():
        print(f"\nfull-size parity {kind} ({cfg.nx}x{cfg.ny}, n_S={cfg.ns}, advect + {cfg.nsub} subcycles, "
              f"alpha=beta={cfg.alpha:g}):")
        print("\n".join(rows))
        print(f"  {kind:8s} field-norm relative error over the windows: " +
              "  ".join(f"{k}={v:.1e}" for k, v in norm.items()) + "  bar=1.0e-10")
    assert max(norm.values()) <= 1e-10, norm
    assert not bad, bad


def test_c4_eight_strips_interfaces_and_bitwise(capsys):
    """C4 as 8 row strips in 8 processes (torchrun, IPC P2P, subcycle graph): the 7 interface windows
    against the oracle at the north_star bar, every rank's rows bitwise equal to one context."""
    import json
    import os
    import subprocess
    import sys
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "8",
                        "scripts/strips8_full.py"], cwd=root, env=env, capture_output=True, text=True, timeout=1800)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads(lines[-1])
    with capsys.disabled():
        print("\nC4 8 strips (8 processes, IPC P2P):")
        for e in d["interface_windows"]:
            print("  interface window", e["window"], "  ".join(f"{k}={v:.1e}" for k, v in e.items() if k != "window"))
        print("  " + "\n  ".join(d["transport"]))
    assert d["bitwise_equal_single"], d["bitwise_bad"]
    assert d["parity_ok"] and len(d["interface_windows"]) == 7, d["interface_windows"]
