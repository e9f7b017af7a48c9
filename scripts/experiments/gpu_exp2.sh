mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
NS=8 CTAS=2,3 STAGES=2,3 timeout 600 python scripts/tune_sustained.py > gpurun_out/tune_sustained_ns8.log 2>&1
PREC=1 CTAS=3,4 STAGES=2 timeout 600 python scripts/tune_sustained.py > gpurun_out/tune_sustained_p1.log 2>&1
PREC=2 CTAS=3,4 STAGES=2 timeout 600 python scripts/tune_sustained.py > gpurun_out/tune_sustained_p2.log 2>&1
CTAS=3,2 STAGES=2 DYN=1,0 timeout 600 python scripts/tune_sustained.py > gpurun_out/tune_sustained_b.log 2>&1
