"""Exercise the NCCL transport (packed halo messages, boundary/interior overlap) with several ranks
on ONE GPU: each rank gets its own NCCL_HOSTID, so NCCL treats them as separate hosts and uses its
socket transport over 127.0.0.1 (P2P/SHM off).  Rank 0 compares the gathered strips with a
single-context run, bitwise.  Launch: torchrun --nproc-per-node N scripts/nccl_two_rank.py"""
import os, sys, json
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
os.environ["NCCL_HOSTID"] = f"nxsdg-rank{rank}"
os.environ.setdefault("NCCL_P2P_DISABLE", "1"); os.environ.setdefault("NCCL_SHM_DISABLE", "1")
os.environ.setdefault("NCCL_IB_DISABLE", "1"); os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
os.environ.setdefault("NCCL_NET_GDR_LEVEL", "0")
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import torch.distributed as dist
from paper_2402_00466_b200 import inputs, nxsdg

dist.init_process_group("gloo")
nxe, nye = int(os.environ.get("NXE", "64")), int(os.environ.get("NYE", "61"))
ty = int(os.environ.get("TY", "4"))
lx, ly = nxe * 2e3, nye * 2e3
st = inputs.make_case(nxe, nye, 2, 6, 6, kind="random", lx=lx, ly=ly)
prm = nxsdg.PhysParams()
nid = nxsdg.nccl_unique_id() if rank == 0 else bytes(128)
t = torch.frombuffer(bytearray(nid), dtype=torch.uint8).clone()
dist.broadcast(t, 0)
m = nxsdg.Mesh(nxe, nye, lx, ly, rank=rank, nranks=world, transport=nxsdg.TRANSPORT_NCCL,
               nccl_id=bytes(t.numpy()), device=0)
m.set_option(nxsdg.OPT_CHUNK_ROWS, ty)
m.set_option(nxsdg.OPT_MULTIRANK_GRAPH, int(os.environ.get("MR_GRAPH", "-1")))
er0, ern, nr0, nrn = m.elem_row0, m.elem_rows, m.node_row0, m.node_rows
loc = {k: np.ascontiguousarray(st[k][nr0:nr0 + nrn]) for k in ("vx", "vy", "ox", "oy", "ax", "ay")}
for k in ("S11", "S12", "S22", "A", "H"):
    loc[k] = np.ascontiguousarray(st[k][er0 * nxe:(er0 + ern) * nxe])
m.load(loc)
m.advect(prm.dt)
m.mevp_substeps(7, begin_step=True)
m.mevp_substeps(4, begin_step=False)
m.mevp_substeps(3, begin_step=False, unfused=True)
m.synchronize()
mine = m.state()
info = m.transport_info
parts = [None] * world
dist.all_gather_object(parts, mine)
m.destroy()
if rank == 0:
    got = {k: np.concatenate([p[k] for p in parts]) for k in mine}
    with nxsdg.Mesh(nxe, nye, lx, ly) as ref:
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
    print(json.dumps({"nccl_ranks": world, "chunk_rows": ty, "bitwise_equal": not bad, "max_diff": bad,
                      "oracle_err": oerr, "transport": info}), flush=True)
    sys.exit(0 if not bad else 3)
