# ncu --set full captures of the n_S = 8 box kernel and the fused general-quad kernel (current defaults)
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle_tma -s 5 -c 1 \
    -o gpurun_out/prof_ns8 python bench.py --ns 8 --steps 1 --warmup 3 --nsub 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_ns8.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_ns8.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle_gen -s 3 -c 1 \
    -o gpurun_out/prof_gen python scripts/bench_general.py > gpurun_out/ncu_gen.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_gen.log
