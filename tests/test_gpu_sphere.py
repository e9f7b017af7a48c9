"""NEXT-4 sphere (R#26; "quadrilateral meshes in spherical coordinates"): the fused TMA
subcycle kernel and the structured advection on a longitude-latitude mesh through the C ABI
(nxsdg_set_sphere) against the oracle's spherical discretisation, element by element.

Bars as everywhere (north_star): <= 1e-12 after one subcycle, <= 1e-10 after a full count, on the fields
and their increments; A, H after an advection step <= 1e-12.  Meshes: an Arctic-like patch (60 N ...
75 N, 30 degrees of longitude) at several resolutions with ragged sizes spanning several warp strips
and chunks; inputs are the warm-box / cyclone recipe evaluated on the patch's local east-north
coordinates."""
import math

import numpy as np
import pytest

import oracle
from paper_2402_00466_b200 import inputs
from tests.parity import parity

pytestmark = pytest.mark.gpu
R = 6371e3
LAT0, DLAT, DLON = math.radians(60.0), math.radians(15.0), math.radians(30.0)


@pytest.fixture(scope="module")
def nx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2402_00466_b200 import build
    build.build()
    from paper_2402_00466_b200 import nxsdg
    return nxsdg


def _case(nxe, nye, kind="warm", lat0=LAT0, dlat=DLAT, dlon=DLON):
    """Inputs on the patch's local coordinates x = R cos(mid-latitude) lon, y = R (lat - lat0)."""
    lx = R * math.cos(lat0 + 0.5 * dlat) * dlon
    ly = R * dlat
    return inputs.make_case(nxe, nye, 2, 6, 6, kind=kind, lx=lx, ly=ly)


def _omesh(nxe, nye, lat0=LAT0, dlat=DLAT, dlon=DLON, bc=0):
    return oracle.Mesh(nxe, nye, lx=dlon, ly=dlat, p=2, ns=6, na=6, bc=bc, radius=R, lat0=lat0)


def _gpu(nx, st, nxe, nye, nsub, advect=False, prm=None, lat0=LAT0, dlat=DLAT, dlon=DLON, options=None, bc=0):
    prm = prm or nx.PhysParams()
    with nx.Mesh(nxe, nye, 1.0, 1.0, 2, 6, 6, bc=bc, params=prm) as m:
        m.set_sphere(R, lat0, dlon, dlat)
        for k, v in (options or {}).items():
            m.set_option(k, v)
        m.load(st)
        if advect:
            m.advect(prm.dt)
        if nsub or bc == 0:
            m.mevp_substeps(nsub, begin_step=True)
        return m.state()


def _opar(prm):
    from dataclasses import asdict
    return oracle.Params(**asdict(prm))


@pytest.mark.parametrize("shape,kind", [((70, 45), "warm"), ((37, 29), "random"), ((1, 5), "random"),
                                        ((6, 1), "random"), ((100, 67), "warm")])
def test_sphere_one_subcycle(nx, shape, kind):
    nxe, nye = shape
    st = _case(nxe, nye, kind)
    got = _gpu(nx, st, nxe, nye, 1)
    ref = oracle.Oracle().subcycles(_omesh(nxe, nye), _opar(nx.PhysParams()), 1, st)
    e = parity(got, ref, st, ("S", "v"))
    assert max(e.values()) <= 1e-12, e


@pytest.mark.parametrize("shape,nsub", [((70, 45), 100), ((37, 29), 30)])
def test_sphere_outer_step_full_count(nx, shape, nsub):
    """advection + prep + nsub fused subcycles (the paper's outer step) on the sphere."""
    nxe, nye = shape
    st = _case(nxe, nye)
    got = _gpu(nx, st, nxe, nye, nsub, advect=True)
    ref = oracle.Oracle().outer_step(_omesh(nxe, nye), _opar(nx.PhysParams()), nsub, st, do_advect=True)
    e = parity(got, ref, st, ("S", "v"))
    assert max(e.values()) <= 1e-10, e
    ea = parity(got, ref, None, ("A", "H"))
    assert max(ea.values()) <= 1e-12, ea


@pytest.mark.parametrize("bc", [0, 1])
def test_sphere_advection(nx, bc):
    """One SSP-RK3 advection step alone (closed and periodic) against the oracle; closed: the
    cos-weighted total mass sum_K (M_K c_K)_0 is conserved (the parallel-arc fluxes cancel bitwise)."""
    nxe, nye = 48, 40
    st = _case(nxe, nye, "random")
    vx, vy = st["vx"].copy(), st["vy"].copy()
    if bc == 1:
        for v in (vx, vy):
            v[-1, :] = v[0, :]; v[:, -1] = v[:, 0]
        st = dict(st, vx=vx, vy=vy)
    prm = nx.PhysParams(dt=3000.0)
    with nx.Mesh(nxe, nye, 1.0, 1.0, 2, 6, 6, bc=bc, params=prm) as m:
        m.set_sphere(R, LAT0, DLON, DLAT)
        m.load(st)
        m.advect(prm.dt)
        got = m.state()
    A, H = oracle.Oracle().advect(_omesh(nxe, nye, bc=bc), prm.dt, st["vx"], st["vy"], st["A"], st["H"])
    e = parity(got, {"A": A, "H": H}, st, ("A", "H"))
    assert max(e.values()) <= 1e-12, e
    if bc == 0:   # mass: the cos-weighted element integral of c0 + its T^2 part's share (discrete, 3-point)
        ka = math.sqrt(0.6) / 2
        w = np.array([5, 8, 5]) / 18.0
        tg = np.array([0.5 - ka, 0.5, 0.5 + ka])

        def mass(c):
            tot = 0.0
            for iy in range(nye):
                cw = np.cos(LAT0 + (iy + tg) * DLAT / nye)
                row = c.reshape(nye, nxe, 6)[iy]
                T = tg - 0.5
                # int psi_k cos over the element for k = 0 (1), 2 (T), 4 (T^2 - 1/12); S-modes integrate to 0
                tot += (row[:, 0] * (w @ cw) + row[:, 2] * (w @ (T * cw)) + row[:, 4] * (w @ ((T * T - 1 / 12) * cw))).sum()
            return tot
        for k in ("A", "H"):
            assert abs(mass(got[k]) - mass(st[k])) <= 1e-13 * abs(mass(st[k])), k


def test_sphere_p2p_strips_bitwise(nx):
    """Row strips on the sphere (3 P2P ranks in one process, own streams, fused peer stores, the
    multi-rank subcycle graph): each rank's row tables start at its global row; bitwise = one context."""
    nxe, nye = 50, 47
    st = _case(nxe, nye, "random")
    prm = nx.PhysParams()
    ref = _gpu(nx, st, nxe, nye, 6, advect=True)
    ms = [nx.Mesh(nxe, nye, 1.0, 1.0, 2, 6, 6, params=prm, rank=r, nranks=3, transport=nx.TRANSPORT_P2P)
          for r in range(3)]
    nx.p2p_connect_local(ms)
    for m in ms:
        m.set_sphere(R, LAT0, DLON, DLAT)
        m.set_option(nx.OPT_CHUNK_ROWS, 4)
        er0, ern, nr0, nrn = m.elem_row0, m.elem_rows, m.node_row0, m.node_rows
        loc = {k: st[k][nr0:nr0 + nrn].copy() for k in ("vx", "vy", "ox", "oy", "ax", "ay")}
        for k in ("S11", "S12", "S22", "A", "H"):
            loc[k] = st[k][er0 * nxe:(er0 + ern) * nxe].copy()
        m.load(loc)
    for m in ms:
        m.advect(prm.dt)
    for m in ms:
        m.mevp_substeps(6, begin_step=True)
    for m in ms:
        m.synchronize()
    got = {k: np.concatenate([m.read_state(k) for m in ms]) for k in ref}
    for m in ms:
        m.destroy()
    for k in ref:
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)


def test_sphere_unsupported_combinations(nx):
    with nx.Mesh(8, 8, 1.0, 1.0, 2, 6, 6) as m:
        with pytest.raises(nx.NxsdgError) as e:
            m.set_sphere(R, math.radians(80.0), DLON, math.radians(15.0))   # reaches past the pole
        assert e.value.status == nx.ERR_INVALID_ARG
        m.set_sphere(R, LAT0, DLON, DLAT)
        m.load(_case(8, 8, "random"))
        with pytest.raises(nx.NxsdgError) as e:
            m.mevp_substeps(1, begin_step=True, unfused=True)
        assert e.value.status == nx.ERR_UNSUPPORTED
        with pytest.raises(nx.NxsdgError) as e:
            m.set_option(nx.OPT_PRECISION, 1)
        assert e.value.status == nx.ERR_UNSUPPORTED
    with nx.Mesh(8, 8, 1.0, 1.0, 1, 3, 3) as m:
        with pytest.raises(nx.NxsdgError) as e:
            m.set_sphere(R, LAT0, DLON, DLAT)
        assert e.value.status == nx.ERR_UNSUPPORTED
