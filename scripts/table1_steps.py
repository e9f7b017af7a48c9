#!/usr/bin/env python
"""The paper's Table 1 (time per hot-path step, CPU) as a GPU analog on the C4 workload:
each step alone through the unfused debug kernels (nxsdg_run_step: strain, stress, divergence,
velocity; E and F materialised in HBM), the fused subcycle (one pass), and one advection.  CUDA events
over 20 repetitions after warm-up; prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2402_00466_b200 import inputs, nxsdg

cfg = inputs.CONFIGS[os.environ.get("CFG", "C4")]
st = inputs.make_config_case(cfg)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, cfg.p, cfg.ns, cfg.na, params=nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha))
m.load(st)
m.mevp_substeps(0, begin_step=True)
s = torch.cuda.ExternalStream(m.stream)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"workload": f"{cfg.name} {cfg.nx}x{cfg.ny} CG{cfg.p}/DG{cfg.p}", "elements": cfg.nx * cfg.ny, "ms": {}}
for step in ("strain", "stress", "divergence", "velocity"):
    out["ms"][step] = timed(lambda: m.run_step(step))
out["ms"]["sum_of_steps"] = sum(out["ms"][k] for k in ("strain", "stress", "divergence", "velocity"))
out["ms"]["fused_subcycle"] = timed(lambda: m.mevp_substeps(1, begin_step=False))
out["ms"]["advection"] = timed(lambda: m.advect(cfg.dt if hasattr(cfg, "dt") else 120.0), reps=5)
out["fused_speedup_over_steps"] = out["ms"]["sum_of_steps"] / out["ms"]["fused_subcycle"]
out["share_of_steps"] = {k: out["ms"][k] / out["ms"]["sum_of_steps"] for k in ("strain", "stress", "divergence", "velocity")}
print(json.dumps(out), flush=True)
m.destroy()
