"""The P2P transport across PROCESSES: each rank exports CUDA IPC handles of its exchanged buffers
(nxsdg_p2p_export), the blobs travel through torch.distributed (gloo), and every rank maps its
neighbours' buffers (nxsdg_p2p_connect) - the one-process-per-GPU deployment.  On one GPU the ranks
share the device (IPC between processes on the same device is allowed); rank 0 compares the gathered
strips with a single-context run, bitwise.  Launch: torchrun --nproc-per-node N scripts/p2p_two_rank.py"""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import torch.distributed as dist
from paper_2402_00466_b200 import inputs, nxsdg

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
nxe, nye = int(os.environ.get("NXE", "64")), int(os.environ.get("NYE", "61"))
ty, ns = int(os.environ.get("TY", "4")), int(os.environ.get("NS", "6"))
lx, ly = nxe * 2e3, nye * 2e3
st = inputs.make_case(nxe, nye, 2, ns, 6, kind="random", lx=lx, ly=ly)
prm = nxsdg.PhysParams()
m = nxsdg.Mesh(nxe, nye, lx, ly, 2, ns, 6, rank=rank, nranks=world, transport=nxsdg.TRANSPORT_P2P, device=dev)
nxsdg.p2p_connect_group(m, rank, world, dist.all_gather_object)
m.set_option(nxsdg.OPT_CHUNK_ROWS, ty)
m.set_option(nxsdg.OPT_MULTIRANK_GRAPH, int(os.environ.get("MR_GRAPH", "-1")))
er0, ern, nr0, nrn = m.elem_row0, m.elem_rows, m.node_row0, m.node_rows
loc = {k: np.ascontiguousarray(st[k][nr0:nr0 + nrn]) for k in ("vx", "vy", "ox", "oy", "ax", "ay")}
for k in ("S11", "S12", "S22", "A", "H"):
    loc[k] = np.ascontiguousarray(st[k][er0 * nxe:(er0 + ern) * nxe])
m.load(loc)
dist.barrier()
m.advect(prm.dt)
m.mevp_substeps(7, begin_step=True)
m.mevp_substeps(4, begin_step=False)
m.mevp_substeps(3, begin_step=False, unfused=True)
m.synchronize()
mine = m.state()
info = m.transport_info
parts = [None] * world
dist.all_gather_object(parts, mine)
dist.barrier()       # nobody unmaps / frees while a neighbour could still touch its buffers
m.destroy()
if rank == 0:
    got = {k: np.concatenate([p[k] for p in parts]) for k in mine}
    with nxsdg.Mesh(nxe, nye, lx, ly, 2, ns, 6, device=dev) as ref:
        ref.load(st); ref.advect(prm.dt); ref.mevp_substeps(7, begin_step=True)
        ref.mevp_substeps(4, begin_step=False); ref.mevp_substeps(3, begin_step=False, unfused=True)
        want = ref.state()
    # the gathered strips against the oracle (advection + 14 subcycles, SURVEY §8(c).5 bar)
    import oracle
    ns_ = want["S11"].shape[1]
    ora = oracle.Oracle().outer_step(oracle.Mesh(nxe, nye, lx=lx, ly=ly, p=2, ns=ns_, na=6), oracle.Params(), 14, st)
    oerr = max(max(float(np.abs(got[k] - ora[k]).max()) for k in g) / max(float(np.abs(ora[k]).max()) for k in g)
               for g in (("S11", "S12", "S22"), ("vx", "vy"), ("A",), ("H",)))
    bad = {k: float(np.abs(got[k] - want[k]).max()) for k in want if not np.array_equal(got[k], want[k])}
    print(json.dumps({"p2p_ranks": world, "chunk_rows": ty, "n_S": ns, "bitwise_equal": not bad, "max_diff": bad,
                      "oracle_err": oerr, "transport": info}), flush=True)
    sys.exit(0 if not bad else 3)
