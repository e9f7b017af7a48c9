mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
COMBOS=1:4:2,0:3:2,0:2:2,1:4:3 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_trim.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
