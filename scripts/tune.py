"""Sweep fused-kernel options on C4; prints ms per subcycle (CUDA events over a 20-launch graph)."""
import sys, os, json, itertools
sys.path.insert(0, os.getcwd())
import torch
from paper_2402_00466_b200 import inputs, nxsdg
cfg = inputs.CONFIGS[os.environ.get("CFG", "C4")]
st = inputs.make_config_case(cfg)
prm = nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 2, 6, 6, params=prm)
m.load(st)
prec = int(os.environ.get("PREC", "0"))
if prec:
    m.set_option(nxsdg.OPT_PRECISION, prec)
bpe = m.bytes_per_element_subcycle
s = torch.cuda.ExternalStream(m.stream)
n = 20
res = []
CT = [int(x) for x in os.environ.get("CTAS", "2,3").split(",")]
DY = [int(x) for x in os.environ.get("DYN", "0,1").split(",")]
combos = [(0, ty, c, st, dyn) for rep in range(2) for dyn in DY for st in (2, 3) for c in CT for ty in (32,)]
for var, ty, c, stg, dyn in combos:
    m.set_option(nxsdg.OPT_DYNAMIC, dyn)
    m.set_option(nxsdg.OPT_FUSED_KERNEL, var); m.set_option(nxsdg.OPT_CHUNK_ROWS, ty); m.set_option(nxsdg.OPT_CTAS_PER_SM, c)
    try:
        m.set_option(nxsdg.OPT_STAGES, stg)
    except Exception as e:
        print("skip", stg, e); continue
    m.mevp_substeps(0, begin_step=True)
    m.mevp_substeps(n, begin_step=False); m.mevp_substeps(n, begin_step=False)
    torch.cuda.synchronize()
    t = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); m.mevp_substeps(n, begin_step=False); e1.record(s); torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) / n)
    ms = min(t)
    gbs = bpe * cfg.nx * cfg.ny / (ms * 1e-3) / 1e9
    print(json.dumps({"prec": prec, "variant": var, "ty": ty, "ctas": c, "stages": stg, "dyn": dyn, "ms": ms, "alg_GBs": gbs, "frac": gbs / 6545.6}), flush=True)
