# A/B: advection CTA shape (2 warps x 4 CTAs = 8/SM, 3 x 3 = 9/SM (default build), 10 x 1 = 10/SM) and the
# node pass inside the first subcycle (--prep-kernel 2) vs the row-marching kernel (0), interleaved on one box
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 600 python -m pytest tests -m gpu -q --timeout 500 -p no:cacheprovider -rf -k "prep or advect or smoke" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3e.log
for rep in 1 2; do
  for v in "libnxsdg_w2.so 0" "libnxsdg.so 0" "libnxsdg_w10.so 0" "libnxsdg.so 2"; do set -- $v
    NXSDG_LIB_AB=$1 timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity --prep-kernel $2 2>&1 | tail -1 | sed "s/^/$1 prep$2 /" >> gpurun_out/ab_bench3.log
  done
done
