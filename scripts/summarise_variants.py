#!/usr/bin/env python
"""profiles/ncu_ns8_r01.json and ncu_gen_r01.json from gpurun_out/prof_ns8.ncu-rep / prof_gen.ncu-rep
(scripts/gpu_ncu_variants.sh), with the traffic ratio against the algorithmic bytes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as n

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for tag, bpe, cfg in (("ns8", 776.0, "C4 4096^2 CG2/DG2 n_S = 8, one fused subcycle launch (bench.py --ns 8 --nsub 10, "
                                     "6th launch), defaults: node constants TMA-loaded late into the consumed S region, 4 CTAs/SM"),
                      ("gen", 728.0, "C4-size distorted CG2/DG2 (delta 0.25), one fused general subcycle, defaults "
                                     "(late node constants, 4 CTAs/SM, tail split, evict-first stores)")):
    rep = os.path.join(root, "gpurun_out", f"prof_{tag}.ncu-rep")
    if not os.path.exists(rep):
        continue
    full = n.full(rep)
    k = next(iter(full))
    m = full[k]
    rd = float(m["dram__bytes_read.sum"].split()[0]); wr = float(m["dram__bytes_write.sum"].split()[0])
    scale = 1e9 if "Gbyte" in m["dram__bytes_read.sum"] else 1e6
    alg = bpe * 4096 * 4096
    out = {"kernel": k, "config": cfg, "metrics": m, "dram_bytes_per_launch": (rd + wr) * scale,
           "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": (rd + wr) * scale / alg}
    json.dump(out, open(os.path.join(root, "profiles", f"ncu_{tag}_r01.json"), "w"), indent=1)
    print(tag, k, m["gpu__time_duration.sum"], out["traffic_over_algorithmic"])
