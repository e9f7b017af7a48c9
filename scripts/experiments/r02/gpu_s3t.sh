# programmatic dependent launch of the subcycle graph: tests (full -m gpu suite) and the C4 bench A/B (PDL 0 / 1)
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for rep in 1 2 3; do for p in 0 1; do
  timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity --pdl $p 2>&1 | tail -1 | sed "s/^/pdl$p /" >> gpurun_out/ab_pdl.log
done; done
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
