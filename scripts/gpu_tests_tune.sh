mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python scripts/tune.py > gpurun_out/tune.log 2>&1; echo "tune rc=$?" >> gpurun_out/tune.log
