"""NEXT-3: deviation of the FP32-storage (precision 1) and FP32-stress-arithmetic (precision 2)
subcycles from the FP64 oracle, and C4 timing."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import oracle
from paper_2402_00466_b200 import inputs, nxsdg
from tests.parity import parity, ora_mesh, ora_params
for (nxe, nye, h, al, nsub) in [(64, 56, 2000.0, 1500.0, 1), (64, 56, 2000.0, 1500.0, 20), (64, 56, 2000.0, 1500.0, 100),
                                (96, 80, 250.0, 25000.0, 1), (96, 80, 250.0, 25000.0, 20)]:
    lx, ly = nxe * h, nye * h
    st = inputs.make_case(nxe, nye, 2, 6, 6, "warm", lx=lx, ly=ly)
    prm = nxsdg.PhysParams(alpha=al, beta=al)
    res = {}
    for prec in (0, 1, 2):
        with nxsdg.Mesh(nxe, nye, lx, ly, params=prm) as m:
            m.set_option(nxsdg.OPT_PRECISION, prec)
            m.load(st); m.mevp_substeps(nsub, begin_step=True)
            res[prec] = m.state()
    ref = oracle.Oracle().subcycles(ora_mesh(nxe, nye, 2, 6, 6, lx, ly), ora_params(prm), nsub, st)
    print(json.dumps({"h": h, "alpha": al, "nsub": nsub, "fp64_vs_oracle": parity(res[0], ref, st),
                      "fp32storage_vs_oracle": parity(res[1], ref, st),
                      "fp32arith_vs_oracle": parity(res[2], ref, st)}), flush=True)
cfg = inputs.CONFIGS["C4"]
st = inputs.make_config_case(cfg)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, params=nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha))
m.load(st)
s = torch.cuda.ExternalStream(m.stream)
for prec in (0, 1, 2, 0, 1, 2):
    m.set_option(nxsdg.OPT_PRECISION, prec)
    m.mevp_substeps(20, begin_step=True); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); m.mevp_substeps(100, begin_step=False); e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 100
    bpe = m.bytes_per_element_subcycle
    print(json.dumps({"precision": ["fp64", "fp32-storage", "fp32-arith"][prec], "ms_per_subcycle": ms, "bytes_per_elem": bpe,
                      "el_upd_per_s": cfg.nx * cfg.ny / (ms * 1e-3),
                      "hbm_frac": bpe * cfg.nx * cfg.ny / (ms * 1e-3) / 1e9 / 6545.6}), flush=True)
