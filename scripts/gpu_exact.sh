mkdir -p gpurun_out
cd "$GRAFT_REPO_ROOT"
( timeout 900 python scripts/exact_stress.py 70 75 8 140e3 150e3 warm
  timeout 900 python scripts/exact_stress.py 37 29 8 512e3 512e3 warm
  timeout 900 python scripts/exact_stress.py 70 75 6 140e3 150e3 warm ) > gpurun_out/exact_stress.log 2>&1
echo "rc=$?" >> gpurun_out/exact_stress.log
