# round 2: perf pass - new advection / prep kernels and pair strips: tests, bench breakdown, ncu
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -p no:cacheprovider -k "advect_tma or prep or pair or p2p_local or loopback or protocol" > gpurun_out/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.log
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/bench_b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_b.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_launches_b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_advect_tma -s 3 -c 1 \
    -o gpurun_out/prof_adv_tma python bench.py --steps 1 --warmup 3 --nsub 2 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_adv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_prep_nodes -s 1 -c 1 \
    -o gpurun_out/prof_prep python bench.py --steps 1 --warmup 3 --nsub 2 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_prep.log 2>&1
for PAIR in 0 1; do
  PAIR=$PAIR timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:k_subcycle_tma -s 2 -c 2 --csv \
     python scripts/ncu_dram.py > gpurun_out/ncu_pair$PAIR.csv 2>&1
done
COMBOS="1:4:2:32:1:2:1:0,1:4:2:32:1:2:1:1" REPS=3 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_pair.log 2>&1
timeout 600 python bench.py --sphere --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_sphere.log 2>&1
