mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
COMBOS=1:4:2:32:1:2,1:4:2:32:1:0,0:3:2:32:1:2,0:2:2:32:1:2,1:3:2:32:1:2 REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_l2.log 2>&1
PREC=2 COMBOS=0:4:2:32:1:2,0:4:2:32:1:0,1:4:2:32:1:2 REPS=1 timeout 600 python scripts/tune_sustained.py > gpurun_out/tune_l2_p2.log 2>&1
PREC=1 COMBOS=0:4:2:32:1:2,0:4:2:32:1:0,1:4:2:32:1:2 REPS=1 timeout 600 python scripts/tune_sustained.py > gpurun_out/tune_l2_p1.log 2>&1
for L in 2 0; do L2=$L timeout 600 python scripts/bench_general.py | sed "s/^/l2=$L /" >> gpurun_out/bench_gen_l2.log 2>&1; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
