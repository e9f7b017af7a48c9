# round 2: full-size window parity (C4 box / n_S = 8 / general, 8-strip interfaces, C3, C5)
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
export CUDA_MODULE_LOADING=EAGER
timeout 3300 python -m pytest tests/test_gpu_full_size.py -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
