# sphere: pre-scaled row blocks + raw Gauss sums (1297 -> 1226 FP64, 40 B spill) vs 5e96bad; sphere tests
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 600 python -m pytest tests/test_gpu_sphere.py -m gpu -q --timeout 500 -p no:cacheprovider -rf > gpurun_out/pytest_s3n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3n.log
for rep in 1 2; do for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib timeout 300 python bench.py --sphere --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_sphere2.log
done; done
