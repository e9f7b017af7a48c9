"""The NCCL transport end to end on ONE GPU: every rank gets its own NCCL_HOSTID, so NCCL treats the
ranks as separate hosts and moves the halo rows over its socket transport (127.0.0.1, P2P/SHM off).
This runs the exact multi-rank code path of the GPU box - packed messages, boundary/interior
overlap on the halo stream, unfused-path and advection halos - and checks it bitwise against a
single context; and bench.py's torchrun path (nccl process group, max-over-ranks timing)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ENV = dict(os.environ, CUDA_MODULE_LOADING="EAGER", NCCL_P2P_DISABLE="1", NCCL_SHM_DISABLE="1", NCCL_IB_DISABLE="1",
           NCCL_SOCKET_IFNAME="lo", NCCL_NET_GDR_LEVEL="0", NXSDG_NCCL_HOSTID_PER_RANK="1")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _torchrun(n, args, extra_env=None, timeout=600):
    env = dict(ENV, **(extra_env or {}))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(n), *args]
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("n,ty,graph", [(2, 4, -1), (3, 4, -1), (2, 32, -1)])
def test_nccl_strips_bitwise_equal_single(n, ty, graph):
    """NCCL row strips: bitwise equal to one context, and the gathered strips within the north_star
    bar of the oracle (advection + 14 subcycles); host-issued subcycles (the NCCL default)."""
    r = _torchrun(n, ["scripts/nccl_two_rank.py"], {"TY": str(ty), "MR_GRAPH": str(graph)})
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-3000:]
    d = json.loads(lines[-1])
    assert d["bitwise_equal"] and d["oracle_err"] <= 1e-10, d
    print(d["transport"])


@pytest.mark.parametrize("n,ty,ns,graph", [(2, 4, 6, 1), (3, 4, 6, 1), (2, 32, 8, 1), (3, 4, 6, 0)])
def test_p2p_ipc_strips_bitwise_equal_single(n, ty, ns, graph):
    """P2P transport across processes (CUDA IPC mappings exchanged through torch.distributed); bitwise
    equal to one context and within the bar of the oracle; with and without the subcycle graph."""
    r = _torchrun(n, ["scripts/p2p_two_rank.py"], {"TY": str(ty), "NS": str(ns), "MR_GRAPH": str(graph)})
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-3000:]
    d = json.loads(lines[-1])
    assert d["bitwise_equal"] and d["oracle_err"] <= 1e-10, d
    if graph:
        assert "subcycle_graph=1" in d["transport"], d["transport"]


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_bench_torchrun_two_ranks(transport):
    r = _torchrun(2, ["bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "C2",
                      "--e2e-steps", "1", "--transport", transport])
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0


def test_bench_p2p_falls_back_to_nccl():
    """If any rank cannot map its neighbours (no CUDA IPC / peer access), all ranks agree and bench.py
    runs over NCCL instead, saying so in the JSON line."""
    r = _torchrun(2, ["bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "C2",
                      "--e2e-steps", "1", "--no-cpu-baseline"], {"NXSDG_TEST_P2P_FAIL": "1"})
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-3000:]
    d = json.loads(lines[0])
    assert "nccl (p2p unavailable" in d["config"]["parallelism"] and d["value"] > 0, d["config"]

