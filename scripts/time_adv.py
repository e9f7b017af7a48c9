import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2402_00466_b200 import inputs, nxsdg
cfg = inputs.CONFIGS["C4"]
st = inputs.make_config_case(cfg)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 2, 6, 6, params=nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha))
m.load(st)
s = torch.cuda.ExternalStream(m.stream)
for rep in range(2):
    for _ in range(3): m.advect(120.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5): m.advect(120.0)
    e1.record(s); torch.cuda.synchronize()
    print(json.dumps({"advect_ms": e0.elapsed_time(e1) / 5}))
    m.mevp_substeps(0, begin_step=True); torch.cuda.synchronize()
    e0.record(s); m.mevp_substeps(0, begin_step=True); e1.record(s); torch.cuda.synchronize()
    print(json.dumps({"prep_ms": e0.elapsed_time(e1)}))
