mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
rm -f gpurun_out/dbg_c5.log
timeout 900 python scripts/debug_c5.py >> gpurun_out/dbg_c5.log 2>&1
OPTS='{"OPT_ADVECT_KERNEL": 1, "OPT_PREP_KERNEL": 1, "OPT_FUSE_PREP_PG": 0}' timeout 900 python scripts/debug_c5.py >> gpurun_out/dbg_c5.log 2>&1
