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
