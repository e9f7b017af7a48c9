"""Fused-kernel options on C4 under SUSTAINED load (the bench's regime: 100-subcycle graphs back to
back until the power cap has settled), unlike scripts/tune.py's short bursts.  Prints ms per
subcycle and the median SM clock seen while timing (pynvml)."""
import sys, os, json, threading, time, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2402_00466_b200 import inputs, nxsdg

try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:                                  # clocks are context only
    _h = None


def sample_clocks(stop, out):
    while not stop.is_set():
        if _h is not None:
            out.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.02)


cfg = inputs.CONFIGS[os.environ.get("CFG", "C4")]
NS = int(os.environ.get("NS", "6"))
if "NY" in os.environ:   # a row strip of the config (e.g. C4 per GPU at 8 GPUs: NY=512), same resolution
    ny = int(os.environ["NY"])
    cfg = inputs.Config(cfg.name, cfg.nx, ny, cfg.p, cfg.ns, cfg.na, cfg.nsub, cfg.lx, cfg.ly * ny / cfg.ny, cfg.kind,
                        cfg.advect, cfg.alpha)
if NS != cfg.ns:
    cfg = inputs.Config(cfg.name, cfg.nx, cfg.ny, cfg.p, NS, cfg.na, cfg.nsub, cfg.lx, cfg.ly, cfg.kind, cfg.advect,
                        cfg.alpha)
st = inputs.make_config_case(cfg)
prm = nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 2, NS, 6, params=prm)
if os.environ.get("GENERAL"):   # distorted quads (NEXT-1): the fused general-quad kernel, 728 B/element
    m.set_vertices(inputs.distorted_vertices(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 0.25))
m.load(st)
prec = int(os.environ.get("PREC", "0"))
if prec:
    m.set_option(nxsdg.OPT_PRECISION, prec)
bpe = m.bytes_per_element_subcycle
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6545.6
s = torch.cuda.ExternalStream(m.stream)
n = 100
# COMBOS = "cl:ctas:stages[:ty[:split[:l2[:vc]]]],..." (cl = NXSDG_OPT_CONST_STAGING, ty = chunk rows, default 32,
# split = NXSDG_OPT_TAIL_SPLIT, default 1, l2 = NXSDG_OPT_L2_POLICY, default 2, vc = NXSDG_OPT_V_ROW_CARRY,
# default 1, pair = NXSDG_OPT_PAIR_STRIPS, default 0),
# measured REPS times, interleaved
COMBOS = [tuple(int(v) for v in x.split(":")) for x in os.environ.get("COMBOS", "0:2:2,0:3:2,1:4:2,1:3:2").split(",")]
REPS = int(os.environ.get("REPS", "2"))
m.set_option(nxsdg.OPT_DYNAMIC, int(os.environ.get("DYN", "1")))
for rep in range(REPS):
    for combo in COMBOS:
        cl, c, stg = combo[:3]
        ty = combo[3] if len(combo) > 3 else 32
        split = combo[4] if len(combo) > 4 else 1
        m.set_option(nxsdg.OPT_CHUNK_ROWS, ty)
        m.set_option(nxsdg.OPT_TAIL_SPLIT, split)
        l2 = combo[5] if len(combo) > 5 else 2
        m.set_option(nxsdg.OPT_L2_POLICY, l2)
        vc = combo[6] if len(combo) > 6 else 1
        m.set_option(nxsdg.OPT_V_ROW_CARRY, vc)
        pair = combo[7] if len(combo) > 7 else 0   # round-2 pair-strip experiment (option removed; must be 0)
        assert pair == 0, "NXSDG_OPT_PAIR_STRIPS was removed after its A/B (profiles/tune_pair_r02.log)"
        m.set_option(nxsdg.OPT_CONST_STAGING, cl)
        m.set_option(nxsdg.OPT_CTAS_PER_SM, c)
        m.set_option(nxsdg.OPT_STAGES, stg)
        m.mevp_substeps(0, begin_step=True)
        for _ in range(8):                      # ~1.6 s: let the power cap settle
            m.mevp_substeps(n, begin_step=False)
        torch.cuda.synchronize()
        clk, stop = [], threading.Event()
        th = threading.Thread(target=sample_clocks, args=(stop, clk)); th.start()
        t = []
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); m.mevp_substeps(n, begin_step=False); e1.record(s); torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1) / n)
        stop.set(); th.join()
        ms = statistics.median(t)
        gbs = bpe * cfg.nx * cfg.ny / (ms * 1e-3) / 1e9
        print(json.dumps({"prec": prec, "rep": rep, "const_regs": cl, "ctas": c, "stages": stg, "ty": ty, "split": split, "l2": l2, "vcarry": vc, "pair": pair, "ms_median": ms,
                          "ms_min": min(t), "alg_GBs": gbs, "frac": gbs / peak,
                          "sm_mhz": statistics.median(clk) if clk else None}), flush=True)
