mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_nccl.py -m gpu -q --timeout 400 -p no:cacheprovider -rf > gpurun_out/pytest_p2p.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_p2p.log
