# advection: RK combine input TMA-staged per warp (c0 buffer) vs 11f63d4; sphere cos/half folds
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rf -k "advect or sphere or prep or smoke or c4_window or limiter or multi_outer or protocol" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3g.log
for rep in 1 2; do for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_bench4.log
done; done
for lib in libnxsdg_prev.so libnxsdg.so; do
  NXSDG_LIB_AB=$lib timeout 300 python bench.py --sphere --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity 2>&1 | tail -1 | sed "s/^/$lib /" >> gpurun_out/ab_sphere.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_advect_tma" -c 3 \
    -o gpurun_out/prof_adv2 python bench.py --steps 1 --warmup 0 --nsub 2 --e2e-steps 0 --no-cpu-baseline --no-parity > gpurun_out/ncu_adv2.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_adv2.log
