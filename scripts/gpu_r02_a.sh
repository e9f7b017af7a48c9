# round 2, first GPU pass: full GPU suite (new full-size C3/C5/strips8 windows, multi-rank graphs, oracle
# parity of the NCCL / P2P multi-process strips), bench N=1 with parity + cpu_baseline, bench under
# torchrun with 8 ranks on the one GPU (the N = 8 code path), multi-rank overhead
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import torch; print(torch.cuda.get_device_properties(0))" >> gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "p2p or graph" > gpurun_out/pytest_mr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mr.log
timeout 900 python -m pytest tests/test_gpu_nccl.py -m gpu -q --timeout 600 -p no:cacheprovider -s > gpurun_out/pytest_nccl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nccl.log
timeout 2400 python -m pytest tests/test_gpu_full_size.py -m gpu -q --timeout 1800 -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
ENVN="NCCL_P2P_DISABLE=1 NCCL_SHM_DISABLE=1 NCCL_IB_DISABLE=1 NCCL_SOCKET_IFNAME=lo NXSDG_NCCL_HOSTID_PER_RANK=1"
env $ENVN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 8 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/bench_8ranks_1gpu.log 2>&1; echo "rc=$?" >> gpurun_out/bench_8ranks_1gpu.log
env $ENVN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 --weak --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/bench_weak2_1gpu.log 2>&1; echo "rc=$?" >> gpurun_out/bench_weak2_1gpu.log
timeout 900 python scripts/mr_overhead.py > gpurun_out/mr_overhead.log 2>&1; echo "rc=$?" >> gpurun_out/mr_overhead.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
