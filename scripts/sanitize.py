"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the box
kernels (TMA structured + table-driven, n_S = 3 / 6 / 8; with the round-2 TMA advection, row-marching
prep and fused P_g on the default path), the fused general-quad kernel, the sphere
kernels, the FP32 variants and the P2P transport (fused peer stores, in-process ranks on their own
streams)."""
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2402_00466_b200 import inputs, nxsdg


def run(m, st, nsub=3):
    m.load(st)
    m.advect(120.0)
    m.mevp_substeps(nsub, begin_step=True)
    m.mevp_substeps(2, begin_step=False, unfused=True)
    m.state()


for (nxe, nye, p, ns, na) in [(37, 29, 2, 6, 6), (16, 16, 1, 3, 3), (9, 70, 2, 6, 3), (33, 20, 2, 8, 6)]:
    st = inputs.make_case(nxe, nye, p, ns, na, kind="random", lx=nxe * 1e3, ly=nye * 1e3)
    for variant in (0, 1):
        with nxsdg.Mesh(nxe, nye, nxe * 1e3, nye * 1e3, p, ns, na) as m:
            m.set_option(nxsdg.OPT_FUSED_KERNEL, variant)
            m.set_option(nxsdg.OPT_CHUNK_ROWS, 8)
            run(m, st)
# default TMA path at a 32-row chunk height on a taller box: tail split (8-row sub-units), v row carry,
# node constants in registers (1) and TMA-staged (0)
nxe, nye = 40, 140
st = inputs.make_case(nxe, nye, 2, 6, 6, kind="random", lx=nxe * 1e3, ly=nye * 1e3)
for cl in (1, 0):
    with nxsdg.Mesh(nxe, nye, nxe * 1e3, nye * 1e3, 2, 6, 6) as m:
        m.set_option(nxsdg.OPT_CONST_STAGING, cl)
        m.set_option(nxsdg.OPT_CTAS_PER_SM, 1)
        run(m, st)
# session 3: the node pass inside the first subcycle (NXSDG_OPT_PREP_KERNEL 2, the PREP instantiation) and the
# batched-load row-marching prep (0) on the same tall box
for pk in (2, 0):
    with nxsdg.Mesh(nxe, nye, nxe * 1e3, nye * 1e3, 2, 6, 6) as m:
        m.set_option(nxsdg.OPT_PREP_KERNEL, pk)
        run(m, st)
# fused general quads
nxe, nye = 37, 33
st = inputs.make_case(nxe, nye, 2, 6, 6, kind="random", lx=nxe * 1e3, ly=nye * 1e3)
with nxsdg.Mesh(nxe, nye, nxe * 1e3, nye * 1e3, 2, 6, 6) as m:
    m.set_vertices(inputs.distorted_vertices(nxe, nye, nxe * 1e3, nye * 1e3, 0.25))
    run(m, st)
# sphere (R#26): the SPH instantiation of the fused TMA kernel and k_advect_q2<true>
with nxsdg.Mesh(nxe, nye, 1.0, 1.0, 2, 6, 6) as m:
    m.set_sphere(6371e3, 1.05, 0.3, 0.2)
    m.load(st)
    m.advect(120.0)
    m.mevp_substeps(3, begin_step=True)
    m.state()
# FP32 storage / arithmetic
for prec in (1, 2):
    with nxsdg.Mesh(nxe, nye, nxe * 1e3, nye * 1e3, 2, 6, 6) as m:
        m.set_option(nxsdg.OPT_PRECISION, prec)
        m.load(st)
        m.mevp_substeps(3, begin_step=True)
        m.state()
# P2P transport, 3 ranks in this process, fused peer stores, overlap path (ty = 4).  Skipped under
# initcheck (SANITIZE_P2P=0): that tool serialises launches, and ranks on separate streams that wait on
# the device for each other's flags then deadlock the host thread.
if os.environ.get("SANITIZE_P2P", "1") == "0":
    print("sanitize run ok (P2P section skipped)")
    sys.exit(0)
ms = [nxsdg.Mesh(nxe, nye, nxe * 1e3, nye * 1e3, rank=r, nranks=3, transport=nxsdg.TRANSPORT_P2P) for r in range(3)]
nxsdg.p2p_connect_local(ms)
for m in ms:
    m.set_option(nxsdg.OPT_CHUNK_ROWS, 4)
    er0, ern, nr0, nrn = m.elem_row0, m.elem_rows, m.node_row0, m.node_rows
    loc = {k: st[k][nr0:nr0 + nrn].copy() for k in ("vx", "vy", "ox", "oy", "ax", "ay")}
    for k in ("S11", "S12", "S22", "A", "H"):
        loc[k] = st[k][er0 * nxe:(er0 + ern) * nxe].copy()
    m.load(loc)
for m in ms:
    m.advect(120.0)
for m in ms:
    m.mevp_substeps(4, begin_step=True)
for m in ms:
    m.synchronize()
for m in ms:
    m.destroy()
print("sanitize run ok")
