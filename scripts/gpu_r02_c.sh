# round 2: GPU tests for the new paths (advection TMA, fused P_g, pair strips, sphere, multi-rank P2P / NCCL)
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
export CUDA_MODULE_LOADING=EAGER
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 200 -p no:cacheprovider -k "advect_tma or fused_prep or pair or graph or p2p or loopback" > gpurun_out/pytest_c1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c1.log
timeout 600 python -m pytest tests/test_gpu_sphere.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_sphere.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sphere.log
timeout 900 python -m pytest tests/test_gpu_nccl.py -m gpu -q --timeout 240 -p no:cacheprovider -s > gpurun_out/pytest_nccl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nccl.log
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c.log
