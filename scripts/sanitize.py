"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2402_00466_b200 import inputs, nxsdg
for (nxe, nye, p, ns, na) in [(37, 29, 2, 6, 6), (16, 16, 1, 3, 3), (9, 70, 2, 6, 3)]:
    st = inputs.make_case(nxe, nye, p, ns, na, kind="random", lx=nxe * 1e3, ly=nye * 1e3)
    for variant in (0, 1):
        with nxsdg.Mesh(nxe, nye, nxe * 1e3, nye * 1e3, p, ns, na) as m:
            m.set_option(nxsdg.OPT_FUSED_KERNEL, variant)
            m.set_option(nxsdg.OPT_CHUNK_ROWS, 8)
            m.load(st)
            m.advect(120.0)
            m.mevp_substeps(3, begin_step=True)
            m.mevp_substeps(2, begin_step=False, unfused=True)
            m.state()
print("sanitize run ok")
