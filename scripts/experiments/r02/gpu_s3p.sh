# advection with folded moment coefficients (839 -> 689 FP64 SASS) vs f4a74af: tests + C4 bench A/B
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rf -k "advect or c4_window or smoke or outer or prep or limiter or protocol or moving or strips" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3p.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3p.log
for rep in 1 2; do for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_adv_fold.log
done; done
timeout 600 ncu --set full --clock-control none -k "regex:k_advect_tma" -c 3 -o gpurun_out/prof_adv_fold python bench.py --steps 1 --warmup 0 --nsub 2 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_adv_fold.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_adv_fold.log
