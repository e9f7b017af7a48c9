mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "const_staging or general_late or general_four or late_constants" -p no:cacheprovider > gpurun_out/pytest_lc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lc.log
