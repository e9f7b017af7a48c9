# general-quad kernel: u/w Listing 2, staged -1/m, 1D Lagrange contractions by sums/differences vs a7aef46
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rf -k "general or smoke" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3c.log
for rep in 1 2; do for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib GENERAL=1 COMBOS="1:4:2" REPS=2 timeout 300 python scripts/tune_sustained.py 2>&1 | sed "s/^/$lib /" >> gpurun_out/ab_gen2.log
done; done
timeout 900 python -m pytest tests/test_gpu_full_size.py -m gpu -q --timeout 800 -p no:cacheprovider -rf -k general > gpurun_out/pytest_full_general.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full_general.log
