mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
: > gpurun_out/tune_promo3.log
for r in 1 2; do for P in 2 1; do
  NXSDG_TMA_L2_PROMOTION=$P COMBOS=1:4:2 REPS=1 timeout 300 python scripts/tune_sustained.py | sed "s/^/promo=$P /" >> gpurun_out/tune_promo3.log 2>&1
done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for P in 2 1; do
  echo "== promo=$P" >> gpurun_out/tune_promo3.log
  NXSDG_TMA_L2_PROMOTION=$P timeout 300 ncu --metrics $M --clock-control none -k regex:k_subcycle -s 2 -c 1 --csv python scripts/ncu_dram.py 2>&1 | grep -E '"(gpu__|dram__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/tune_promo3.log
done
PREC=2 COMBOS=0:4:2 REPS=1 timeout 300 python scripts/tune_sustained.py > gpurun_out/tune_p2_final.log 2>&1
NXSDG_TMA_L2_PROMOTION=3 PREC=2 COMBOS=0:4:2 REPS=1 timeout 300 python scripts/tune_sustained.py >> gpurun_out/tune_p2_final.log 2>&1
