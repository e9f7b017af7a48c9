mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 600 python scripts/table1_steps.py > gpurun_out/table1.log 2>&1; echo "rc=$?" >> gpurun_out/table1.log
timeout 1200 python bench.py --weak --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
