mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle -s 5 -c 1 \
    -o gpurun_out/prof_tma python bench.py --steps 1 --warmup 3 --nsub 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
