# ncu evidence for the current default kernels + variant bench lines
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle -s 5 -c 1 \
    -o gpurun_out/prof_tma python bench.py --steps 1 --warmup 3 --nsub 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_advect_q2|k_prep" -c 4 \
    -o gpurun_out/prof_other python bench.py --steps 1 --warmup 0 --nsub 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_other.log 2>&1
echo "ncu other rc=$?" >> gpurun_out/ncu_other.log
timeout 900 python bench.py --ns 8 --no-cpu-baseline > gpurun_out/bench_ns8.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ns8.log
timeout 900 python bench.py --weak --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
