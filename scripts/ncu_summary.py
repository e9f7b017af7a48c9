#!/usr/bin/env python
"""Summarise ncu outputs into profiles/: launch list shares (gpu__time_duration) and the
key metrics of a --set full capture.  Usage: ncu_summary.py launches.csv [prof.ncu-rep] out_prefix"""
import collections
import csv
import json
import re
import subprocess
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    tot = collections.defaultdict(float); cnt = collections.Counter()
    for r in rows:
        name = re.sub(r"\(.*", "", r[4]).strip()
        tot[name] += float(r[14]); cnt[name] += 1
    T = sum(tot.values())
    return {k: {"launches": cnt[k], "total_ms": tot[k] / 1e6, "mean_us": tot[k] / cnt[k] / 1e3, "share": tot[k] / T}
            for k in sorted(tot, key=lambda k: -tot[k])}


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "launch__occupancy_limit_registers",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
           "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
           "sm__sass_inst_executed_op_global_ld.sum", "achieved_occupancy", "sm__maximum_warps_per_active_cycle_pct"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {}
    for d in data:
        name = re.sub(r"\(.*", "", d[hdr.index("Kernel Name")]).strip()
        m = {}
        for k in METRICS:
            if k in hdr:
                m[k] = d[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        res[name] = m
    return res


if __name__ == "__main__":
    lc, rep, pre = sys.argv[1], (sys.argv[2] if len(sys.argv) > 3 else None), sys.argv[-1]
    s = {"launch_list": launches(lc)}
    if rep:
        s["full"] = full(rep)
    json.dump(s, open(pre + ".json", "w"), indent=1)
    print(json.dumps(s, indent=1))
