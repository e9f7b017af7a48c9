"""C4 (4096^2 CG2/DG2, 125 m) as N row strips, one PROCESS per rank (the one-process-per-GPU deployment's
topology; on one GPU here), P2P transport through CUDA IPC with fused peer stores, the device flag
handshake and the multi-rank subcycle graph: one outer step (advection + prep + 100 fused subcycles).

Checks: every strip interface against the oracle on a window centred on it
(light-cone ring n_sub + 5; rank r >= 1 computes the window of the interface below its strip from the
rows the two ranks own), and every rank's rows bitwise equal to a single context's run of the whole mesh
(rank 0 runs it and shares the result through /dev/shm).  Prints one JSON line on rank 0.

    torchrun --nproc-per-node 8 scripts/strips8_full.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import numpy as np
import torch
import torch.distributed as dist

import oracle
from paper_2402_00466_b200 import inputs, nxsdg
from tests.parity import group_err

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
cfg = inputs.CONFIGS[os.environ.get("CFG", "C4")]
prm = nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha)
CORE = 12
shm = os.environ.get("SHM", "/dev/shm/nxsdg_strips8")
keys = ("vx", "vy", "S11", "S12", "S22", "A", "H")

# ---- the strips
r0, er, n0, nr = nxsdg.partition(cfg.ny, cfg.p, world, rank)
st = inputs.make_config_case(cfg, window=(0, r0, cfg.nx, er))
for k in ("vx", "vy", "ox", "oy", "ax", "ay"):
    st[k] = np.ascontiguousarray(st[k][:nr])
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, cfg.p, cfg.ns, cfg.na, params=prm, rank=rank, nranks=world,
               transport=nxsdg.TRANSPORT_P2P, device=0)
nxsdg.p2p_connect_group(m, rank, world, dist.all_gather_object)
m.load(st)
dist.barrier()
t0 = time.time()
m.advect(prm.dt)
m.mevp_substeps(cfg.nsub, begin_step=True)
m.synchronize()
mine = m.state(keys)
info = m.transport_info
dist.barrier()
m.destroy()

# ---- the single context (rank 0) -> /dev/shm
if rank == 0:
    os.makedirs(shm, exist_ok=True)
    full = inputs.make_config_case(cfg)
    with nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, cfg.p, cfg.ns, cfg.na, params=prm) as ref:
        ref.set_option(nxsdg.OPT_FUSE_PREP_PG, 0)   # P_g by the prep pass, as row strips compute it
        ref.load(full)
        ref.advect(prm.dt)
        ref.mevp_substeps(cfg.nsub, begin_step=True)
        for k in keys:
            np.save(os.path.join(shm, k + ".npy"), ref.read_state(k))
    del full
dist.barrier()
bad = []
for k in keys:
    ref = np.load(os.path.join(shm, k + ".npy"), mmap_mode="r")
    if k in ("vx", "vy"):
        part = ref[n0:n0 + nr]
    else:
        part = ref[r0 * cfg.nx:(r0 + er) * cfg.nx]
    if not np.array_equal(np.asarray(part), mine[k]):
        bad.append(k)

# ---- interface windows: rank r >= 1, the interface at its first element row r0
p = cfg.p
rows = {}
cy = r0 - CORE // 2
rng = np.random.default_rng(inputs.SEED_BASE + 4 + rank)
cx = int(rng.integers(0, cfg.nx - CORE))
want = {}   # what each rank needs from each other rank: (k, global row) ranges around every interface
parts = [None] * world
mine_rows = {}
for q in range(1, world):
    qr0 = nxsdg.partition(cfg.ny, p, world, q)[0]
    qcy = qr0 - CORE // 2
    for k in ("S11", "S12", "S22", "A", "H"):
        a = mine[k].reshape(er, cfg.nx, -1)
        for gy in range(max(qcy, r0), min(qcy + CORE, r0 + er)):
            mine_rows[(q, k, gy)] = a[gy - r0].copy()
    for k in ("vx", "vy"):
        for gj in range(max(p * qcy, n0), min(p * (qcy + CORE) + 1, n0 + nr)):
            mine_rows[(q, k, gj)] = mine[k][gj - n0].copy()
dist.all_gather_object(parts, mine_rows)
err = None
if rank >= 1:
    for d in parts:
        for (q, k, g), v in d.items():
            if q == rank:
                rows[(k, g)] = v
    g = {k: np.stack([rows[(k, gy)][cx:cx + CORE] for gy in range(cy, cy + CORE)]).reshape(-1, rows[(k, cy)].shape[-1])
         for k in ("S11", "S12", "S22", "A", "H")}
    for k in ("vx", "vy"):
        g[k] = np.stack([rows[(k, gj)][p * cx:p * (cx + CORE) + 1] for gj in range(p * cy, p * (cy + CORE) + 1)])
    ring = cfg.nsub + 5
    ix0, iy0 = max(0, cx - ring), max(0, cy - ring)
    w, h = min(cfg.nx, cx + CORE + ring) - ix0, min(cfg.ny, cy + CORE + ring) - iy0
    sub = inputs.make_config_case(cfg, window=(ix0, iy0, w, h))
    om = oracle.Mesh(w, h, lx=w * cfg.lx / cfg.nx, ly=h * cfg.ly / cfg.ny, p=p, ns=cfg.ns, na=cfg.na)
    o = oracle.Oracle(threads=max(1, (os.cpu_count() or 8) // max(1, world - 1)))
    rf = o.outer_step(om, oracle.Params(alpha=cfg.alpha, beta=cfg.alpha), cfg.nsub, sub, do_advect=True)
    init = inputs.make_config_case(cfg, window=(cx, cy, CORE, CORE))
    ex, ey = cx - ix0, cy - iy0
    rc = {}
    for k, a in rf.items():
        if k in ("vx", "vy"):
            rc[k] = a[p * ey:p * (ey + CORE) + 1, p * ex:p * (ex + CORE) + 1]
        elif k in g:
            rc[k] = a.reshape(h, w, -1)[ey:ey + CORE, ex:ex + CORE].reshape(-1, a.shape[1])
    err = {}
    for name, grp in (("S", ("S11", "S12", "S22")), ("v", ("vx", "vy"))):
        err[name] = group_err(g, rc, grp)
        err["d" + name] = group_err({k: g[k] - init[k] for k in grp}, {k: rc[k] - init[k] for k in grp}, grp)
    for name in ("A", "H"):
        err[name] = group_err(g, rc, (name,))
    err["window"] = (cx, cy)
res = [None] * world
dist.all_gather_object(res, {"rank": rank, "bitwise_bad": bad, "err": err, "info": info})
if rank == 0:
    ok_bits = all(not d["bitwise_bad"] for d in res)
    errs = [d["err"] for d in res if d["err"]]
    ok_par = all(max(e["S"], e["dS"], e["v"], e["dv"]) <= 1e-10 and max(e["A"], e["H"]) <= 1e-12 for e in errs)
    print(json.dumps({"config": cfg.name, "ranks": world, "bitwise_equal_single": ok_bits,
                      "bitwise_bad": {d["rank"]: d["bitwise_bad"] for d in res if d["bitwise_bad"]},
                      "interface_windows": errs, "parity_ok": ok_par, "transport": [d["info"] for d in res],
                      "wall_s": time.time() - t0}), flush=True)
    import shutil
    shutil.rmtree(shm, ignore_errors=True)
dist.barrier()
dist.destroy_process_group()
