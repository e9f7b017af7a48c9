mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "limit or advection" --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest_lim.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_lim.log
timeout 600 python bench.py --limiter --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_lim.log 2>&1
