#!/usr/bin/env python
"""NEXT-1 whole subcycle on a distorted 4096^2 CG2/DG2 quad mesh (C4 workload, vertices moved by up to
0.25 h/2): fused k_subcycle_gen (one TMA-staged pass, geometry on the fly from the vertices) vs the
unfused general step kernels (strain, stress on the fly, divergence contributions + gather, velocity).
Prints one JSON line per variant; algorithmic bytes of the fused pass = the box kernel's 680 B/element
+ one vertex (16 B) + four lumped node masses (32 B) = 728 B."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2402_00466_b200 import inputs, nxsdg

cfg = inputs.CONFIGS[os.environ.get("CFG", "C4")]
st = inputs.make_config_case(cfg)
V = inputs.distorted_vertices(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 0.25)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 2, 6, 6, params=nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha))
m.set_vertices(V)
m.load(st)
if "L2" in os.environ:   # NXSDG_OPT_L2_POLICY (default 2: evict-first stores)
    m.set_option(nxsdg.OPT_L2_POLICY, int(os.environ["L2"]))
s = torch.cuda.ExternalStream(m.stream)
N = cfg.nx * cfg.ny
bpe = m.bytes_per_element_subcycle
sweep = os.environ.get("SWEEP")
if sweep:   # fused-kernel tuning: CTAs per SM x pipeline stages
    for ctas, stages in [(2, 2), (3, 2), (2, 3), (3, 3), (0, 2)]:
        m.set_option(nxsdg.OPT_CTAS_PER_SM, ctas); m.set_option(nxsdg.OPT_STAGES, stages)
        m.mevp_substeps(2, begin_step=True); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); m.mevp_substeps(20, begin_step=False); e1.record(s); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(json.dumps({"ctas": ctas, "stages": stages, "ms_per_subcycle": ms,
                          "hbm_frac": bpe * N / (ms * 1e-3) / 1e9 / peak}), flush=True)
    m.set_option(nxsdg.OPT_CTAS_PER_SM, -1); m.set_option(nxsdg.OPT_STAGES, 2)
for unfused in (False, True, False):
    n = 20 if not unfused else 5
    m.mevp_substeps(2, begin_step=True, unfused=unfused)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); m.mevp_substeps(n, begin_step=False, unfused=unfused); e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    line = {"experiment": "NEXT-1 whole subcycle on distorted quads (C4 size)", "variant": "unfused step kernels" if unfused
            else "fused k_subcycle_gen (on-the-fly geometry)", "elements": N, "ms_per_subcycle": ms,
            "element_updates_per_s": N / (ms * 1e-3)}
    if not unfused:
        gbs = bpe * N / (ms * 1e-3) / 1e9
        line.update({"algorithmic_bytes_per_element": bpe, "achieved_GBs": gbs, "hbm_frac": gbs / peak})
    print(json.dumps(line), flush=True)
m.destroy()
