mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 600 python bench.py --ns 8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ns8.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_ns8.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle -s 5 -c 1 \
    -o gpurun_out/prof_ns8 python bench.py --ns 8 --steps 1 --warmup 3 --nsub 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_ns8.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_ns8.log
