# advection: 3-slot late ring (10 warps / SM) vs the 4-slot ring (8 warps), interleaved, sustained bench
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rf -k "advect or smoke or c4_window or prep" --deselect tests/test_gpu_full_size.py > gpurun_out/pytest_s3h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3h.log
cat > /tmp/advab.py <<'PY'
import sys, os, json, time, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2402_00466_b200 import inputs, nxsdg
cfg = inputs.CONFIGS["C4"]
st = inputs.make_config_case(cfg)
prm = nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 2, 6, 6, params=prm)
m.load(st)
s = torch.cuda.ExternalStream(m.stream)
for rep in range(3):
    for stg in (4, 3):
        m.set_option(nxsdg.OPT_ADVECT_STAGES, stg)
        for _ in range(3):                       # settle: outer steps as in the bench
            m.advect(prm.dt); m.mevp_substeps(100, begin_step=True)
        t = []
        for _ in range(3):
            m.mevp_substeps(60, begin_step=False)   # keep the power cap engaged between advection timings
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); m.advect(prm.dt); e1.record(s); torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1))
            m.mevp_substeps(0, begin_step=True)
        print(json.dumps({"rep": rep, "adv_stages": stg, "advect_ms": statistics.median(t), "all": t}), flush=True)
PY
timeout 900 python /tmp/advab.py > gpurun_out/ab_adv3.log 2>&1
for rep in 1 2; do for stg in 4 3; do
  timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-parity --adv-stages $stg 2>&1 | tail -1 | sed "s/^/stages$stg /" >> gpurun_out/ab_adv3_bench.log
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_advect_tma" -c 3 \
    -o gpurun_out/prof_adv3 python bench.py --steps 1 --warmup 0 --nsub 2 --e2e-steps 0 --no-cpu-baseline --no-parity --adv-stages 3 > gpurun_out/ncu_adv3.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_adv3.log
