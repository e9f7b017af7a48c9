mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
: > gpurun_out/ncu_skew.log
for C in "1 1 32" "0 0 32" "1 1 8" "1 1 16" "0 1 32"; do set -- $C
  echo "== dyn=$1 split=$2 ty=$3" >> gpurun_out/ncu_skew.log
  DYN=$1 SPLIT=$2 TY=$3 timeout 300 ncu --metrics $M --clock-control none -k regex:k_subcycle -s 2 -c 1 --csv python scripts/ncu_dram.py 2>&1 | grep -E '"(gpu__|dram__|lts__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/ncu_skew.log
done
