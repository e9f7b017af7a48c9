# default kernel back at 236 registers: pair / partition tests and the C4 bench A/B vs 5e96bad
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rf -k "pair or tail or c4_window or smoke or v_row or late_const or fused" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3m.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3m.log
for rep in 1 2 3; do for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_bench6.log
done; done
