mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "const_staging or fused_variants or one_subcycle or p2p_local" -p no:cacheprovider > gpurun_out/pytest_cl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cl.log
COMBOS=0:2:2,0:3:2,1:4:2,1:3:2,1:3:3 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_cl.log 2>&1
PREC=2 COMBOS=0:4:2,1:4:2,1:5:2 REPS=2 timeout 600 python scripts/tune_sustained.py > gpurun_out/tune_cl_p2.log 2>&1
