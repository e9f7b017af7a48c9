# pair mode with the pass gap: bitwise tests; A/B over chunk heights (the scratch must stay in L2)
mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"; export CUDA_MODULE_LOADING=EAGER
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 500 -p no:cacheprovider -rf -x -k "pair_subcycles" > gpurun_out/pytest_s3k.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3k.log
cat > /tmp/pairab2.py <<'PY'
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
for rep in range(2):
    for pair, ty in ((0, 32), (1, 4), (1, 8), (1, 16), (0, 8)):
        m.set_option(nxsdg.OPT_PAIR_SUBCYCLES, pair); m.set_option(nxsdg.OPT_CHUNK_ROWS, ty)
        for _ in range(5): m.mevp_substeps(100, begin_step=False)
        torch.cuda.synchronize()
        t = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); m.mevp_substeps(100, begin_step=False); e1.record(s); torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1) / 100)
        print(json.dumps({"rep": rep, "pair": pair, "ty": ty, "ms_per_subcycle": statistics.median(t)}), flush=True)
PY
timeout 900 python /tmp/pairab2.py > gpurun_out/ab_pair2.log 2>&1
