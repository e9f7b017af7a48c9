mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "const_staging or general_late or general_four or late_constants or general_quads" -p no:cacheprovider > gpurun_out/pytest_lc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lc.log
COMBOS=1:4:2,2:4:2 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_box_lc2.log 2>&1
NS=8 COMBOS=0:2:2,2:4:2 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_box_lc2_ns8.log 2>&1
