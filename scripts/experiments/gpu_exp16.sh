mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
NY=512 COMBOS=1:4:2:32,1:4:2:16,1:4:2:12,1:4:2:8,1:4:2:24 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_strip512.log 2>&1
NY=1024 COMBOS=1:4:2:32,1:4:2:16,1:4:2:12 REPS=1 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_strip1024.log 2>&1
CFG=C3 COMBOS=1:4:2:32,1:4:2:24,1:4:2:16 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_c3.log 2>&1
