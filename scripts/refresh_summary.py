#!/usr/bin/env python
"""Rebuild profiles/ncu_summary.json from a GPU pass (scripts/gpu_round.sh): the fused-kernel capture
(gpurun_out/prof_tma.ncu-rep), the bench command's launch list (gpurun_out/launches_r01.csv) and the
bench line (gpurun_out/bench.log).  bench.py reads k_subcycle.dram_bytes_per_launch for roofline.traffic."""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import ncu_summary as n

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "profiles", "ncu_summary.json")
old = json.load(open(out)) if os.path.exists(out) else {}
full = n.full(os.path.join(root, "gpurun_out", "prof_tma.ncu-rep"))
k = next(x for x in full if "k_subcycle" in x)
m = full[k]
rd = float(m["dram__bytes_read.sum"].split()[0]); wr = float(m["dram__bytes_write.sum"].split()[0])
scale = 1e9 if "Gbyte" in m["dram__bytes_read.sum"] else 1e6
alg = 680.0 * 4096 * 4096
bench = [json.loads(l) for l in open(os.path.join(root, "gpurun_out", "bench.log")) if l.startswith("{")][-1]
s = dict(old)
s["k_subcycle"] = dict(m, kernel=k, dram_bytes_per_launch=(rd + wr) * scale, algorithmic_bytes_per_launch=alg,
                       traffic_over_algorithmic=(rd + wr) * scale / alg)
s["launch_list"] = n.launches(os.path.join(root, "gpurun_out", "launches_r01.csv"))
s["bench_line"] = {key: bench.get(key) for key in ("value", "ms_per_step", "breakdown_ms", "roofline", "clocks",
                                                     "gpu_launches", "e2e", "cpu_baseline")}
json.dump(s, open(out, "w"), indent=1)
print(json.dumps({"kernel": k, "traffic_over_algorithmic": s["k_subcycle"]["traffic_over_algorithmic"],
                  "shares": {a: round(b["share"], 4) for a, b in s["launch_list"].items()}}, indent=1))

# Per-kernel roofline table of the other step kernels (advection stage, outer-step prep) from
# gpurun_out/prof_other.ncu-rep: DRAM bytes / duration against the measured HBM peak, FP64 pipe.
other = os.path.join(root, "gpurun_out", "prof_other.ncu-rep")
if os.path.exists(other):
    peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(root, "MEASURED_PEAKS.json")) else 6545.6

    def num(v):
        x, u = v.split()[:2]
        return float(x) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
                           "ns": 1e-9}.get(u, 1.0)

    tab = {}
    for name, mm in list(n.full(other).items()) + [(k, m)]:
        t = num(mm["gpu__time_duration.sum"])
        b = num(mm["dram__bytes_read.sum"]) + num(mm["dram__bytes_write.sum"])
        tab[name] = {"ms": t * 1e3, "dram_GB": b / 1e9, "dram_GBs": b / t / 1e9, "hbm_frac": b / t / 1e9 / peak,
                     "fp64_pipe_pct": float(mm["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"].split()[0]),
                     "warps_active_pct": float(mm["sm__warps_active.avg.pct_of_peak_sustained_active"].split()[0]),
                     "registers": mm["launch__registers_per_thread"]}
    s["per_kernel"] = tab
    json.dump(s, open(out, "w"), indent=1)
    print(json.dumps(tab, indent=1))
