mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
SANITIZE_P2P=0 timeout 1500 compute-sanitizer --tool initcheck --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_initcheck.log 2>&1
echo "initcheck rc=$?" >> gpurun_out/sanitize_initcheck.log
