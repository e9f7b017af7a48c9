# TMA L2 promotion 128 B vs 64 B on the whole step (bench, advection, prep) and the general-quad kernel, + ncu DRAM
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
for rep in 1 2; do for pr in 2 1; do
  NXSDG_TMA_L2_PROMOTION=$pr timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/promo$pr /" >> gpurun_out/ab_promo_bench.log
  NXSDG_TMA_L2_PROMOTION=$pr GENERAL=1 COMBOS="1:4:2" REPS=1 timeout 300 python scripts/tune_sustained.py 2>&1 | tail -1 | sed "s/^/promo$pr /" >> gpurun_out/ab_promo_gen.log
done; done
for rep in 1 2; do for pr in 2 1; do
  NXSDG_TMA_L2_PROMOTION=$pr timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:k_subcycle_tma|k_advect_tma" -s 2 -c 3 --csv \
    python bench.py --steps 1 --warmup 0 --nsub 5 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_promo_b${pr}_$rep.csv 2>&1
done; done
