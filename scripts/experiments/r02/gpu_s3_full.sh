# round 2 (session 3) evidence: full-size window parity (C4 box / n_S = 8 / general, C3, C5, the 8-strip
# interfaces) with the field-norm bar, then compute-sanitizer over the kernel paths (incl. the PREP variant)
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 3000 python -m pytest tests/test_gpu_full_size.py -m gpu -q -s --timeout 1500 -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
for tool in memcheck racecheck synccheck initcheck; do
  P2P=1; [ "$tool" = initcheck ] && P2P=0
  SANITIZE_P2P=$P2P timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
