mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 900 python scripts/tune.py > gpurun_out/tune.log 2>&1; echo "tune rc=$?" >> gpurun_out/tune.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launches.log
