mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fp32 or variants or one_subcycle" --timeout 300 -p no:cacheprovider > gpurun_out/pytest_fp32.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_fp32.log
timeout 600 python scripts/fp32_study.py > gpurun_out/fp32_study.log 2>&1
echo "study rc=$?" >> gpurun_out/fp32_study.log
for f in "" --fp32-storage --fp32-stress; do timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline $f; done > gpurun_out/bench_fp32.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_fp32.log
