# TMA L2 promotion (NXSDG_TMA_L2_PROMOTION 0 none / 1 64 B / 2 128 B default / 3 256 B): sustained time and ncu DRAM bytes
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
for rep in 1 2; do for pr in 2 1 0; do
  NXSDG_TMA_L2_PROMOTION=$pr COMBOS="1:4:2" REPS=1 timeout 300 python scripts/tune_sustained.py 2>&1 | tail -1 | sed "s/^/promo$pr /" >> gpurun_out/ab_promo.log
done; done
for pr in 2 1 0; do
  NXSDG_TMA_L2_PROMOTION=$pr timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_subcycle_tma -s 3 -c 1 --csv \
    python bench.py --steps 1 --warmup 0 --nsub 5 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_promo$pr.csv 2>&1
done
