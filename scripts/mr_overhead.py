"""Per-subcycle overhead of the multi-rank (row-strip) path, measured on ONE GPU.

All ranks live in this process, each context on its own stream, connected by the P2P transport
(nxsdg_p2p_connect_local): the same kernels, fused peer stores, flag handshake and multi-rank subcycle
graph as the one-process-per-GPU deployment, only the peers are on the same device.

(a) C4 as 8 strips (4096 x 512 each) running concurrently vs one context on the whole C4: the 8 ranks
    share the GPU, so (T_8 - T_1) / n_sub is the extra device work per subcycle the partition adds
    (boundary/interior split, ring rows, the handshake's memops), not the latency a real 8-GPU run sees.
(b) Latency floor: 8 ranks with a few element rows each (compute ~ nothing), so the time per subcycle
    is the chain boundary kernel -> flag write -> peer wait -> interior kernel -> join, with and
    without the subcycle graph (host-issued: ~8 API calls per subcycle per rank).
(c) Host time per nxsdg_mevp_substeps call (graph replay vs host-issued), from the host's clock.

    python scripts/mr_overhead.py [--nsub 100] [--ranks 8]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2402_00466_b200 import inputs, nxsdg


def make(nx, ny, nranks, graph, prm, st):
    ms = [nxsdg.Mesh(nx, ny, 512e3, 512e3 * ny / nx, params=prm, rank=r, nranks=nranks,
                     transport=nxsdg.TRANSPORT_P2P) for r in range(nranks)]
    nxsdg.p2p_connect_local(ms)
    for m in ms:
        m.set_option(nxsdg.OPT_MULTIRANK_GRAPH, graph)
        er0, ern, nr0, nrn = m.elem_row0, m.elem_rows, m.node_row0, m.node_rows
        loc = {k: np.ascontiguousarray(st[k][nr0:nr0 + nrn]) for k in ("vx", "vy", "ox", "oy", "ax", "ay")}
        for k in ("S11", "S12", "S22", "A", "H"):
            loc[k] = np.ascontiguousarray(st[k][er0 * nx:(er0 + ern) * nx])
        m.load(loc)
    for m in ms:
        m.mevp_substeps(0, begin_step=True)
    for m in ms:
        m.synchronize()
    return ms


def timed(ms, nsub, reps):
    """Device time of `reps` calls of nsub subcycles on every rank (first rank's stream waits for all)."""
    for m in ms:
        m.mevp_substeps(nsub, begin_step=False)   # warm-up / capture
    for m in ms:
        m.synchronize()
    streams = [torch.cuda.ExternalStream(m.stream) for m in ms]
    e0 = [torch.cuda.Event(enable_timing=True) for _ in ms]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in ms]
    host = 0.0
    for ev, s in zip(e0, streams):
        ev.record(s)
    for _ in range(reps):
        for m in ms:
            t = time.perf_counter()
            m.mevp_substeps(nsub, begin_step=False)
            host += time.perf_counter() - t
    for ev, s in zip(e1, streams):
        ev.record(s)
    for m in ms:
        m.synchronize()
    dev = max(a.elapsed_time(b) for a, b in zip(e0, e1)) / (reps * nsub)
    return dev * 1e3, host / (reps * len(ms)) * 1e6     # us per subcycle, us per host call per rank


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nsub", type=int, default=100)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    prm = nxsdg.PhysParams(alpha=25000.0, beta=25000.0)
    out = {}
    # (a) C4 strips vs one context
    cfg = inputs.CONFIGS["C4"]
    st = inputs.make_config_case(cfg)
    with nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, params=prm) as m:
        m.load(st)
        m.mevp_substeps(0, begin_step=True)
        t1, h1 = timed([m], a.nsub, a.reps)
    out["c4_single_us_per_subcycle"] = t1
    for graph in (1, 0):
        ms = make(cfg.nx, cfg.ny, a.ranks, graph, prm, st)
        t8, h8 = timed(ms, a.nsub, a.reps)
        out[f"c4_{a.ranks}strips_graph{graph}_us_per_subcycle"] = t8
        out[f"c4_{a.ranks}strips_graph{graph}_extra_us_per_subcycle"] = t8 - t1
        out[f"c4_{a.ranks}strips_graph{graph}_host_us_per_call"] = h8
        out["transport"] = ms[0].transport_info
        for m in ms:
            m.destroy()
    del st
    # (b) latency floor: a few rows per rank
    for rows in (2, 8):
        nx, ny = 4096, rows * a.ranks
        stl = inputs.make_case(nx, ny, 2, 6, 6, kind="warm", lx=512e3, ly=512e3 * ny / nx)
        for graph in (1, 0):
            ms = make(nx, ny, a.ranks, graph, prm, stl)
            t, h = timed(ms, a.nsub, a.reps)
            out[f"latency_{rows}rows_graph{graph}_us_per_subcycle"] = t
            out[f"latency_{rows}rows_graph{graph}_host_us_per_call"] = h
            for m in ms:
                m.destroy()
        with nxsdg.Mesh(nx, rows, 512e3, 512e3 * rows / nx, params=prm) as m:   # one strip alone, no exchange
            m.load(inputs.make_case(nx, rows, 2, 6, 6, kind="warm", lx=512e3, ly=512e3 * rows / nx))
            m.mevp_substeps(0, begin_step=True)
            out[f"latency_{rows}rows_single_strip_us_per_subcycle"] = timed([m], a.nsub, a.reps)[0]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
