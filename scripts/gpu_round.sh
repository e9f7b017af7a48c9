# full GPU pass: smoke, every -m gpu test, the default bench line, the reference arm, ncu evidence
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/gpu_state.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle -s 5 -c 1 \
    -o gpurun_out/prof_tma python bench.py --steps 1 --warmup 3 --nsub 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_advect_q2|k_prep" -c 4 \
    -o gpurun_out/prof_other python bench.py --steps 1 --warmup 0 --nsub 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_other.log 2>&1
echo "ncu other rc=$?" >> gpurun_out/ncu_other.log
timeout 900 python bench.py --ns 8 --no-cpu-baseline > gpurun_out/bench_ns8.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ns8.log
timeout 900 python bench.py --fp32-stress --no-cpu-baseline > gpurun_out/bench_fp32.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fp32.log
timeout 600 python scripts/bench_general.py > gpurun_out/bench_general.log 2>&1; echo "rc=$?" >> gpurun_out/bench_general.log
for tool in memcheck racecheck; do
  SANITIZE_P2P=1 timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
