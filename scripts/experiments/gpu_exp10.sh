mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "l2_policy or ns8" -p no:cacheprovider > gpurun_out/pytest_l2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_l2.log
NS=8 COMBOS=1:4:2,0:2:2,0:3:2,1:3:2 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_ns8.log 2>&1
