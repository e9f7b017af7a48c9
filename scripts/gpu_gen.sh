mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "general" --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest_gen.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gen.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_subcycle_gen -s 3 -c 1 \
    -o gpurun_out/prof_gen python scripts/bench_general.py > gpurun_out/ncu_gen.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_gen.log
