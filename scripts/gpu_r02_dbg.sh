mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
rm -f gpurun_out/dbg.log
export CUDA_MODULE_LOADING=EAGER
for v in "NXSDG_DEBUG_ADV_TMA=4" "NXSDG_DEBUG_ADV_TMA=5" "NXSDG_DEBUG_ADV_TMA=2 CUDA_DEVICE_MAX_CONNECTIONS=32" "NXSDG_DEBUG_ADV_TMA=2 NXSDG_P2P_GEQ=1" "NXSDG_DEBUG_ADV_TMA=2 CUDA_MODULE_LOADING=LAZY"; do
echo "=== $v" >> gpurun_out/dbg.log
env NR=2 GRAPH=0 ADVECT=1 ADVK=0 $v timeout 40 python scripts/debug_mr_graph.py >> gpurun_out/dbg.log 2>&1; echo "rc=$?" >> gpurun_out/dbg.log
done
