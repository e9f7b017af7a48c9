"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/nxsdg.h declares, and its pure-host entry points behave."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nxsdg.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nxsdg_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def nx():
    from paper_2402_00466_b200 import build
    build.build()
    from paper_2402_00466_b200 import nxsdg
    return nxsdg


def test_header_declares_the_north_star_calls():
    names = _declared()
    for f in ("nxsdg_create_mesh", "nxsdg_set_forcing", "nxsdg_mevp_substeps", "nxsdg_advect", "nxsdg_read_state"):
        assert f in names


def test_library_exports_every_declared_symbol(nx):
    lib = C.CDLL(nx.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(nx.EXPORTED)


def test_library_is_sm100a_cubin(nx):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", nx.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version(nx):
    assert nx.lib.nxsdg_abi_version() == 1


@pytest.mark.parametrize("ny,p,nr", [(16, 1, 1), (16, 1, 3), (4096, 2, 8), (7, 2, 7), (10, 2, 4)])
def test_partition_covers_rows_once(nx, ny, p, nr):
    """Row strips: contiguous, balanced (remainder to low ranks), every
    element row and node row owned exactly once, the top rank also owns node row p*ny."""
    erows, nrows = [], []
    for r in range(nr):
        r0, er, n0, nrw = nx.partition(ny, p, nr, r)
        erows += list(range(r0, r0 + er))
        nrows += list(range(n0, n0 + nrw))
        assert er in (ny // nr, ny // nr + 1)
    assert erows == list(range(ny))
    assert nrows == list(range(p * ny + 1))


def test_partition_rejects_bad_args(nx):
    with pytest.raises(nx.NxsdgError):
        nx.partition(4, 2, 5, 0)
    with pytest.raises(nx.NxsdgError):
        nx.partition(4, 3, 1, 0)
    with pytest.raises(nx.NxsdgError):
        nx.partition(4, 2, 2, 2)


def test_create_mesh_argument_errors(nx):
    """Invalid arguments are rejected before any device work (no GPU needed)."""
    with pytest.raises(nx.NxsdgError) as e:
        nx.Mesh(0, 4)
    assert e.value.status == nx.ERR_INVALID_ARG
    with pytest.raises(nx.NxsdgError) as e:
        nx.Mesh(4, 4, p=2, ns=3)
    assert e.value.status == nx.ERR_UNSUPPORTED
    with pytest.raises(nx.NxsdgError) as e:
        nx.Mesh(4, 4, p=1, ns=3, na=6)
    assert e.value.status == nx.ERR_UNSUPPORTED
    with pytest.raises(nx.NxsdgError) as e:
        nx.Mesh(4, 4, params=nx.PhysParams(alpha=1.0))
    assert e.value.status == nx.ERR_INVALID_ARG
    with pytest.raises(nx.NxsdgError) as e:
        nx.Mesh(4, 4, bc=nx.BC_PERIODIC, nranks=2, rank=0, transport=nx.TRANSPORT_LOOPBACK)
    assert e.value.status == nx.ERR_UNSUPPORTED


def test_no_cpu_fallback_without_gpu(nx):
    """On a machine without a CUDA device, create_mesh fails loudly with NXSDG_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(nx.NxsdgError) as e:
        nx.Mesh(8, 8)
    assert e.value.status == nx.ERR_CUDA


def test_product_never_imports_oracle():
    """The product package shares no code with the oracle and never loads it."""
    pkg = os.path.join(ROOT, "paper_2402_00466_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
                assert "oracle.h" not in txt, f


def test_binding_option_ids_match_header():
    """The binding's OPT_* ids are the header's NXSDG_OPT_* enum values (no drift between the two)."""
    from paper_2402_00466_b200 import nxsdg
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    hdr = {m.group(1): int(m.group(2)) for m in re.finditer(r"NXSDG_OPT_([A-Z0-9_]+)\s*=\s*(\d+)", txt)}
    assert hdr, "no NXSDG_OPT_* enum in the header"
    for name, val in hdr.items():
        assert getattr(nxsdg, "OPT_" + name) == val, name
    py = {k[4:] for k in dir(nxsdg) if k.startswith("OPT_")}
    assert py == set(hdr), sorted(py ^ set(hdr))
