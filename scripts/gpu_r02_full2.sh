# round 2: 8-process C4 strips (interfaces vs oracle, bitwise vs one context), then C3 / C5 full-size windows
mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
export CUDA_MODULE_LOADING=EAGER
timeout 1500 python -m pytest tests/test_gpu_full_size.py -m gpu -q --timeout 1400 -p no:cacheprovider -k "eight_strips" > gpurun_out/pytest_strips8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strips8.log
timeout 1900 python -m pytest tests/test_gpu_full_size.py -m gpu -q --timeout 1800 -p no:cacheprovider -k "C3 or C5" > gpurun_out/pytest_full35.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full35.log
