# bench line + ncu launch list of the bench command + one full capture of the fused subcycle kernel
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/gpu_state.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle -s 5 -c 1 \
    -o gpurun_out/prof_tma python bench.py --steps 1 --warmup 3 --nsub 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_advect -s 3 -c 1 \
    -o gpurun_out/prof_adv python bench.py --steps 1 --warmup 3 --nsub 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_adv.log 2>&1
