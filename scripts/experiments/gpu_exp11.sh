mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "v_row_carry or const_staging or tail_split or one_subcycle or full_subcycle or p2p_local or loopback or fp32" -p no:cacheprovider > gpurun_out/pytest_vc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vc.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
: > gpurun_out/ncu_vc.log
for C in "1 4 1" "1 4 0" "0 2 1" "0 2 0"; do set -- $C
  echo "== cl=$1 ctas=$2 vcarry=$3" >> gpurun_out/ncu_vc.log
  CL=$1 CTAS=$2 VCARRY=$3 timeout 300 ncu --metrics $M --clock-control none -k regex:k_subcycle -s 2 -c 1 --csv python scripts/ncu_dram.py 2>&1 | grep -E '"(gpu__|dram__|lts__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/ncu_vc.log
done
COMBOS=1:4:2:32:1:2:1,1:4:2:32:1:2:0,0:3:2:32:1:2:1,0:2:2:32:1:2:1 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_vc.log 2>&1
NS=8 COMBOS=0:2:2:32:1:2:1,0:2:2:32:1:2:0,1:4:2:32:1:2:1 REPS=1 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_vc_ns8.log 2>&1
PREC=2 COMBOS=0:4:2:32:1:2:1,0:4:2:32:1:2:0 REPS=1 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_vc_p2.log 2>&1
