import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import oracle
from paper_2402_00466_b200 import inputs, nxsdg
from tests.parity import case, ora_mesh, ora_params, parity
for (nxe, nye, lx, ly) in [(40, 36, 40e3, 36e3), (70, 75, 140e3, 150e3)]:
    st = case(nxe, nye, 2, 6, 6, "warm", lx, ly)
    for var in (1, 0):
        try:
            with nxsdg.Mesh(nxe, nye, lx, ly) as m:
                m.set_option(nxsdg.OPT_FUSED_KERNEL, var)
                m.load(st); m.mevp_substeps(1); got = m.state()
            ref = oracle.Oracle().subcycles(ora_mesh(nxe, nye, 2, 6, 6, lx, ly), oracle.Params(), 1, st)
            print(nxe, nye, "variant", var, parity(got, ref, st), flush=True)
        except Exception as e:
            print(nxe, nye, "variant", var, "ERROR", e, flush=True)
            raise
