mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
export CUDA_MODULE_LOADING=EAGER
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -p no:cacheprovider -k "prep or bytes_model or general_quads_stress" > gpurun_out/pytest_e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e.log
timeout 1200 python -m pytest tests/test_gpu_full_size.py -m gpu -q --timeout 1100 -p no:cacheprovider -k "C5" > gpurun_out/pytest_full_c5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full_c5.log
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/bench_e.log 2>&1
bash scripts/gpu_sanitize.sh
