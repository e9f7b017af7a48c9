mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
: > gpurun_out/ncu_hints.log
for H in 0 1 3 5 7 2; do
  echo "== hints=$H" >> gpurun_out/ncu_hints.log
  NXSDG_L2_HINTS=$H timeout 300 ncu --metrics $M --clock-control none -k regex:k_subcycle -s 2 -c 1 --csv python scripts/ncu_dram.py 2>&1 | grep -E '"(gpu__|dram__|lts__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/ncu_hints.log
done
for H in 0 1 3 5 7 0; do
  NXSDG_L2_HINTS=$H COMBOS=1:4:2 REPS=1 timeout 300 python scripts/tune_sustained.py | sed "s/^/hints=$H /" >> gpurun_out/tune_hints.log 2>&1
done
