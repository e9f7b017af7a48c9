# automatic chunk height for small single-rank meshes (C1, C2) + bench parity bar with the oracle FMA floor (C5)
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rf -k "auto_chunk or advect or prep or tail or c2 or full_subcycle or one_subcycle or smoke or loopback" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3i.log
for C in C1 C2; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_${C}_auto.log 2>&1; done
timeout 900 python bench.py --weak --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_C5_floor.log 2>&1
