# bench lines for the other BASELINE.json configs (C2 L2-resident, C3 2048^2) on one B200
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 900 python bench.py --config C2 --no-cpu-baseline --steps 20 > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
