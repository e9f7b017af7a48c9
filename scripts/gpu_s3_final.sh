# round 2 (session 3) round-end evidence: smoke, -m gpu suite, full-size windows, bench lines (C4 default with
# e2e / cpu_baseline / parity, reference arm, C1 C2 C3 C5, sphere, n_S = 8, FP32 stress, general quads), the
# 8-rank code path on the one GPU, ncu launch list + --set full captures (fused subcycle; advection + prep)
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 2400 python -m pytest tests/test_gpu_full_size.py -m gpu -q -s --timeout 1500 -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
for C in C1 C2 C3; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$C.log 2>&1; done
timeout 900 python bench.py --weak --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_C5.log 2>&1
timeout 600 python bench.py --sphere --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_sphere.log 2>&1
timeout 600 python bench.py --ns 8 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_ns8.log 2>&1
timeout 600 python bench.py --fp32-stress --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_fp32.log 2>&1
timeout 600 python scripts/bench_general.py > gpurun_out/bench_general.log 2>&1
GENERAL=1 COMBOS="1:4:2" REPS=2 timeout 300 python scripts/tune_sustained.py > gpurun_out/tune_gen_sustained.log 2>&1
ENVN="NCCL_P2P_DISABLE=1 NCCL_SHM_DISABLE=1 NCCL_IB_DISABLE=1 NCCL_SOCKET_IFNAME=lo NXSDG_NCCL_HOSTID_PER_RANK=1"
env $ENVN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 8 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/bench_8ranks_1gpu.log 2>&1; echo "rc=$?" >> gpurun_out/bench_8ranks_1gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_launches.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle_tma -s 5 -c 1 \
    -o gpurun_out/prof_tma python bench.py --steps 1 --warmup 3 --nsub 10 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_advect_tma|k_prep_nodes_march" -c 4 \
    -o gpurun_out/prof_other python bench.py --steps 1 --warmup 0 --nsub 2 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_other.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_other.log
