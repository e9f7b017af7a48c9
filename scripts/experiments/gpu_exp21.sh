mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "general" -p no:cacheprovider > gpurun_out/pytest_genlc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_genlc.log
GENERAL=1 COMBOS=1:4:2,0:3:2,1:3:2,1:4:3 REPS=2 timeout 1200 python scripts/tune_sustained.py > gpurun_out/tune_gen_lc.log 2>&1
