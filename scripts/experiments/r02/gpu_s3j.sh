# pair mode (two subcycles per launch): bitwise tests, then the sustained A/B on C4
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 500 -p no:cacheprovider -rf -x -k "pair_subcycles" > gpurun_out/pytest_s3j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3j.log
cat > /tmp/pairab.py <<'PY'
import sys, os, json, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2402_00466_b200 import inputs, nxsdg
cfg = inputs.CONFIGS["C4"]
st = inputs.make_config_case(cfg)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 2, 6, 6, params=nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha))
m.load(st)
s = torch.cuda.ExternalStream(m.stream)
m.mevp_substeps(0, begin_step=True)
for rep in range(3):
    for pair in (0, 1):
        m.set_option(nxsdg.OPT_PAIR_SUBCYCLES, pair)
        for _ in range(6): m.mevp_substeps(100, begin_step=False)
        torch.cuda.synchronize()
        t = []
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); m.mevp_substeps(100, begin_step=False); e1.record(s); torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1) / 100)
        print(json.dumps({"rep": rep, "pair": pair, "ms_per_subcycle": statistics.median(t), "all": t}), flush=True)
PY
timeout 900 python /tmp/pairab.py > gpurun_out/ab_pair.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_subcycle_tma" -s 3 -c 1 \
    -o gpurun_out/prof_pair python -c "
import sys, os; sys.path.insert(0, os.getcwd())
from paper_2402_00466_b200 import inputs, nxsdg
cfg = inputs.CONFIGS['C4']; st = inputs.make_config_case(cfg)
m = nxsdg.Mesh(cfg.nx, cfg.ny, cfg.lx, cfg.ly, 2, 6, 6, params=nxsdg.PhysParams(alpha=cfg.alpha, beta=cfg.alpha))
m.load(st); m.set_option(nxsdg.OPT_PAIR_SUBCYCLES, 1); m.mevp_substeps(10, begin_step=True); m.synchronize()
" > gpurun_out/ncu_pair.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_pair.log
