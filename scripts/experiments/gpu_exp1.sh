mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/copy_sustained.py > gpurun_out/copy_sustained.log 2>&1
CTAS=2,3 STAGES=2,3 DYN=1 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_sustained.log 2>&1; echo rc=$? >> gpurun_out/tune_sustained.log
