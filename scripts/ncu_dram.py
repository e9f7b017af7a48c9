"""A few C4 fused-subcycle launches with the options in the environment (CL, CTAS, STAGES, TY), for
`ncu --metrics dram__bytes_read.sum,...` DRAM-traffic comparisons of launch configurations."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2402_00466_b200 import inputs, nxsdg
cfg = inputs.CONFIGS["C4"]
st = inputs.make_config_case(cfg)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 2, 6, 6, params=nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha))
m.load(st)
for opt, env in ((nxsdg.OPT_CONST_STAGING, "CL"), (nxsdg.OPT_CTAS_PER_SM, "CTAS"), (nxsdg.OPT_STAGES, "STAGES"),
                 (nxsdg.OPT_CHUNK_ROWS, "TY"), (nxsdg.OPT_V_ROW_CARRY, "VCARRY"),
                 (nxsdg.OPT_L2_POLICY, "L2POL"), (nxsdg.OPT_DYNAMIC, "DYN"), (nxsdg.OPT_TAIL_SPLIT, "SPLIT")):
    if env in os.environ:
        m.set_option(opt, int(os.environ[env]))
m.mevp_substeps(0, begin_step=True)
m.mevp_substeps(4, begin_step=False)
torch.cuda.synchronize()
print("ok")
