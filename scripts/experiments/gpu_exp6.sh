mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tail_split or const_staging or fused_variants or general_quads_fused or p2p_local or loopback" -p no:cacheprovider > gpurun_out/pytest_tail.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tail.log
COMBOS=1:4:2:32:0,1:4:2:32:1,1:4:2:16:0,1:4:2:16:1,1:4:2:24:1 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_tail.log 2>&1
