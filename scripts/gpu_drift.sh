mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "drift or multi_outer or graph or roundtrip" --timeout 800 -p no:cacheprovider > gpurun_out/pytest_drift.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_drift.log
