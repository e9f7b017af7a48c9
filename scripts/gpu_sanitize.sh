mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
export CUDA_MODULE_LOADING=EAGER
for tool in memcheck racecheck synccheck initcheck; do
  P2P=1; [ "$tool" = initcheck ] && P2P=0
  SANITIZE_P2P=$P2P timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
