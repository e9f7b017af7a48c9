mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests/test_gpu_full_size.py tests/test_gpu_parity.py -m gpu -q --timeout 1200 -p no:cacheprovider -rf -k "window or general" > gpurun_out/pytest_fullsize.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_fullsize.log
timeout 600 python scripts/diag_gen_adv.py > gpurun_out/diag_gen_adv.log 2>&1
