# session-3 re-entry check: smoke, the -m gpu suite (full-size windows separately), the bench line
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
export CUDA_MODULE_LOADING=EAGER
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_advect_tma|k_prep_nodes_march" -c 4 \
    -o gpurun_out/prof_adv_prep python bench.py --steps 1 --warmup 0 --nsub 2 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_adv.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_adv.log
