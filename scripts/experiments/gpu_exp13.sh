mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
COMBOS=1:4:2:32,1:4:2:8,1:4:2:12,1:4:2:16,1:4:2:24 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_ty2.log 2>&1
