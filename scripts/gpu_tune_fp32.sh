mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
for p in 0 1 2; do PREC=$p CTAS=2,3,4,6 DYN=1 timeout 600 python scripts/tune.py; done > gpurun_out/tune_fp32.log 2>&1
echo "rc=$?" >> gpurun_out/tune_fp32.log
