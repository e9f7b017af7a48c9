mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py --weak --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 900 python bench.py --limiter --no-cpu-baseline > gpurun_out/bench_limiter.log 2>&1; echo "rc=$?" >> gpurun_out/bench_limiter.log
timeout 900 python bench.py --fp32-storage --no-cpu-baseline > gpurun_out/bench_fp32s.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fp32s.log
