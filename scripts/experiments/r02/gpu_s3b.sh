# A/B of the session-3 kernel changes (sparse LDL^T general-quad subcycle, batched-load prep march, early c0
# loads in the advection) against the previous commit's build (libnxsdg_prev.so), interleaved
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rf -k "general or prep or advect or smoke or c4_window" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3b.log
for rep in 1 2; do for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib GENERAL=1 COMBOS="1:4:2" REPS=2 timeout 300 python scripts/tune_sustained.py 2>&1 | sed "s/^/$lib /" >> gpurun_out/ab_gen.log
  NXSDG_LIB_AB=$lib timeout 300 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_bench.log
done; done
