# general-quad kernel configurations after the FP64 cuts (const staging : CTAs/SM : stages [: chunk rows]), sustained
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
GENERAL=1 COMBOS="1:4:2,0:3:2,1:3:2,1:4:3,1:4:2:16,1:4:2:64" REPS=2 timeout 900 python scripts/tune_sustained.py > gpurun_out/tune_gen_s3.log 2>&1
