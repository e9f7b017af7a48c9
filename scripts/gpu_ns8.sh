mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "ns8 or k0 or debug_steps" --timeout 600 -p no:cacheprovider > gpurun_out/pytest_ns8.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_ns8.log
