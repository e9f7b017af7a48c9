mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
GENERAL=1 COMBOS=0:3:2,0:2:2,0:3:2:32:0,0:3:3,0:1:2 REPS=2 timeout 1200 python scripts/tune_sustained.py > gpurun_out/tune_gen_sustained.log 2>&1
