# separate D2H stream for HOST_ASYNC read-backs: async pipeline tests, e2e bench (vs a7... prev = a23f4ed)
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 600 python -m pytest tests -m gpu -q --timeout 500 -p no:cacheprovider -rf -k "async or forcing or read or smoke or checkpoint" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3o.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3o.log
for rep in 1 2; do for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib timeout 400 python bench.py --steps 3 --warmup 3 --e2e-steps 30 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_e2e.log
done; done
