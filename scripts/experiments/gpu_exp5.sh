mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum
: > gpurun_out/ncu_dram.log
for P in 3 2 0; do for C in "1 4 2" "0 2 2" "0 3 2"; do set -- $C
  echo "== promo=$P cl=$1 ctas=$2 stages=$3" >> gpurun_out/ncu_dram.log
  NXSDG_TMA_L2_PROMOTION=$P CL=$1 CTAS=$2 STAGES=$3 timeout 300 ncu --metrics $M --clock-control none -k regex:k_subcycle -s 2 -c 1 --csv python scripts/ncu_dram.py 2>&1 | grep -E '"(gpu__|dram__|lts__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/ncu_dram.log
done; done
for P in 3 2 0; do
NXSDG_TMA_L2_PROMOTION=$P COMBOS=1:4:2,0:3:2 REPS=1 timeout 600 python scripts/tune_sustained.py > gpurun_out/tune_promo$P.log 2>&1
done
COMBOS=1:4:2:16,1:4:2:24,1:4:2:32,1:4:2:48,1:4:2:64 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_ty.log 2>&1
