# first fused subcycle forming the node constants (NXSDG_OPT_PREP_KERNEL 2): full -m gpu suite, bench A/B vs a7aef46
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3d.log
for rep in 1 2; do for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib timeout 300 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_bench2.log
done; done
