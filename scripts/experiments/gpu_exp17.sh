mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
: > gpurun_out/tune_promo2.log
for r in 1 2; do for P in 3 0 2; do
  NXSDG_TMA_L2_PROMOTION=$P COMBOS=1:4:2 REPS=1 timeout 300 python scripts/tune_sustained.py | sed "s/^/promo=$P /" >> gpurun_out/tune_promo2.log 2>&1
done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for P in 3 0 2; do
  echo "== promo=$P" >> gpurun_out/tune_promo2.log
  NXSDG_TMA_L2_PROMOTION=$P timeout 300 ncu --metrics $M --clock-control none -k regex:k_subcycle -s 2 -c 1 --csv python scripts/ncu_dram.py 2>&1 | grep -E '"(gpu__|dram__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/tune_promo2.log
done
