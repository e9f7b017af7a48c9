# round 2 evidence: smoke, the -m gpu suite (full-size windows run separately: gpu_r02_full.sh), the bench line
# (N=1 with parity / cpu_baseline / e2e), the reference arm, the config table, 8 ranks on the one GPU under
# torchrun (the N = 8 code path with IPC P2P + subcycle graph), ncu launch list + full capture of the fused kernel
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
export CUDA_MODULE_LOADING=EAGER
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python -m pytest tests/test_gpu_full_size.py -m gpu -q --timeout 1100 -p no:cacheprovider -k "C5" > gpurun_out/pytest_full_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full_c5.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
for C in C1 C2 C3; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$C.log 2>&1; done
timeout 900 python bench.py --weak --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_C5.log 2>&1
timeout 600 python bench.py --sphere --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_sphere.log 2>&1
ENVN="NCCL_P2P_DISABLE=1 NCCL_SHM_DISABLE=1 NCCL_IB_DISABLE=1 NCCL_SOCKET_IFNAME=lo NXSDG_NCCL_HOSTID_PER_RANK=1"
env $ENVN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 8 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/bench_8ranks_1gpu.log 2>&1; echo "rc=$?" >> gpurun_out/bench_8ranks_1gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle_tma -s 5 -c 1 \
    -o gpurun_out/prof_subcycle python bench.py --steps 1 --warmup 3 --nsub 10 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_full.log 2>&1
