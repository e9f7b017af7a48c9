#!/usr/bin/env python
"""NEXT-1 / the paper's Table 2 on B200: the Listing 2 stress update on a distorted
4096^2 CG2/DG2 quad mesh, per-element inverse maps pre-assembled and stored vs recomputed
on the fly from the four vertices.  Prints one JSON line per variant.

Algorithmic bytes per element-update (FP64): E 18 + H, A 12 + S read/write 36 = 66 doubles,
+ iMJwPSI 54 doubles when stored (120 doubles = 960 B), + the element's vertices (~2 doubles,
each vertex shared by 4 elements) on the fly (68 doubles = 544 B)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2402_00466_b200 import inputs, nxsdg

n = int(os.environ.get("N", "4096"))
lx = ly = 512e3
V = inputs.distorted_vertices(n, n, lx, ly, 0.25)
r = np.random.default_rng(3)
N = n * n
st = {k: np.ascontiguousarray(r.normal(0, 1e-6, (N, 6))) for k in ("E11", "E12", "E22")}
for k in ("H", "A"):
    st[k] = np.ascontiguousarray(r.uniform(-0.05, 0.05, (N, 6))); st[k][:, 0] = r.uniform(0.5, 1.0, N)
for k in ("S11", "S12", "S22"):
    st[k] = np.ascontiguousarray(r.uniform(-1e3, 1e3, (N, 6)))
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
m = nxsdg.Mesh(n, n, lx, ly, 2, 6, 6)
m.set_vertices(V)
for k, v in st.items():
    m.write_state(k, v)
s = torch.cuda.ExternalStream(m.stream)
for mode, name, bpe in ((0, "pre-assembled iMJwPSI per element (P:172)", 960.0), (1, "on-the-fly map from 4 vertices (P:260-265)", 544.0)):
    m.set_option(nxsdg.OPT_MAP_MODE, mode)
    for _ in range(3):
        m.run_step("stress")
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        m.run_step("stress")
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gbs = bpe * N / (ms * 1e-3) / 1e9
    print(json.dumps({"experiment": "Table 2 analog: stress update on distorted quads", "variant": name,
                      "map_mode": mode, "elements": N, "ms_per_update": ms, "element_updates_per_s": N / (ms * 1e-3),
                      "algorithmic_bytes_per_element": bpe, "achieved_GBs": gbs, "hbm_frac": gbs / peak}), flush=True)
m.destroy()
