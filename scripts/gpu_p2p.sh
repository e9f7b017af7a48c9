mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "p2p or loopback" --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest_p2p.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_p2p.log
timeout 900 python -m pytest tests/test_gpu_nccl.py -m gpu -q --timeout 400 -p no:cacheprovider -rf >> gpurun_out/pytest_p2p.log 2>&1
echo "pytest ipc rc=$?" >> gpurun_out/pytest_p2p.log
