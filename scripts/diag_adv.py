import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import oracle
from paper_2402_00466_b200 import inputs, nxsdg
from tests.parity import group_err
cfg = inputs.CONFIGS["C4"]
w = 256
for (ix0, iy0) in [(1000, 1300), (2042 - 128, 2042 - 128)]:
    st = inputs.make_config_case(cfg, window=(ix0, iy0, w, w))
    hx = cfg.lx / cfg.nx
    with nxsdg.Mesh(w, w, w * hx, w * hx, 2, 6, 6) as m:
        m.load(st); m.advect(120.0); g = m.state(("A", "H"))
    mesh = oracle.Mesh(w, w, lx=w * hx, ly=w * hx)
    A1, H1 = oracle.Oracle("plain").advect(mesh, 120.0, st["vx"], st["vy"], st["A"], st["H"])
    A2, H2 = oracle.Oracle("fma").advect(mesh, 120.0, st["vx"], st["vy"], st["A"], st["H"])
    c = slice(None)
    for name, a, b in (("gpu-plain", g["A"], A1), ("fma-plain", A2, A1)):
        d = np.abs(a - b).reshape(w, w, 6)[8:-8, 8:-8]
        print(name, "per-coef max abs err", d.reshape(-1, 6).max(0), "A max", np.abs(A1).max())
    dA = (A1 - st["A"]).reshape(w, w, 6)[8:-8, 8:-8]
    print("max |dA| per coef", np.abs(dA).reshape(-1, 6).max(0))
