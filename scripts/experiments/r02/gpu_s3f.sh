# validation after the session-3 changes: smoke, the -m gpu suite, sphere bench, the default bench line
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3f.log
timeout 600 python bench.py --sphere --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_sphere.log 2>&1
timeout 600 python scripts/bench_general.py > gpurun_out/bench_general.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
