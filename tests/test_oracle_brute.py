"""Round-2 oracle pins (``-m "not gpu"``): the parts VERDICT r01 found unpinned by mutation.

- O10 prep's nodal mean (R#17): element-wise constant data with a distinct value per element
  (closed form: mean of 4 / 2 / 1 by node type) and random DG data against a scatter-and-count
  brute force;
- O8 velocity's Jacobi (x, y) coupling (R#11): Eq. (2) is a vector equation, so the update commutes
  with rotations of the plane; and with drag off it is the complex scaling v <- (beta - i dt f) v /
  (1 + beta), whose modulus ratio is the same at every node;
- the distorted-mesh geometry of NEXT-1 (R#23): lumped mass (sum = area, per node), strain and
  divergence against assembled brute-force operators, their adjointness, advection's constant
  preservation, closed-box conservation and the whole edge/volume operator with independent normals;
- SURVEY §8(c).4 "whole subcycle": assembled global operators on 2x2 ... 4x4 meshes, both degrees,
  box and distorted, against the element-loop oracle.

The brute force lives in ``tests/brute.py`` (numpy Gauss rules, Vandermonde Lagrange bases, sympy DG
family and derivatives, adjugate geometry, normals from vertex differences).
"""
import math

import numpy as np
import pytest

from tests import brute
from oracle import Mesh, Params
from paper_2402_00466_b200 import inputs


R_EARTH = 6371e3
LAT0 = math.radians(60.0)


def _sphere_pair(nx, ny, p, ns, na, dlon=0.05, dlat=0.04, lat0=LAT0, bc=0, radius=R_EARTH):
    """lon-lat patch of nx x ny elements, each dlon x dlat [rad], southern edge lat0 (R#26)."""
    return (Mesh(nx, ny, lx=nx * dlon, ly=ny * dlat, p=p, ns=ns, na=na, bc=bc, radius=radius, lat0=lat0),
            brute.BMesh(nx, ny, nx * dlon, ny * dlat, p, ns, na, bc=bc, radius=radius, lat0=lat0))


def _pair(nx, ny, p, ns, na, lx, ly, distorted, bc=0, delta=0.28, seed=None):
    if distorted == "sphere":
        return _sphere_pair(nx, ny, p, ns, na, bc=bc)
    V = None
    if distorted:
        V = inputs.distorted_vertices(nx, ny, lx, ly, delta, **({} if seed is None else {"seed": seed}))
    return (Mesh(nx, ny, lx=lx, ly=ly, p=p, ns=ns, na=na, bc=bc, verts=V),
            brute.BMesh(nx, ny, lx, ly, p, ns, na, bc=bc, verts=V))


def _rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


# ---------------------------------------------------------------- O10 prep: nodal mean (R#17)
@pytest.mark.parametrize("p,ns,na", [(1, 3, 1), (1, 3, 3), (2, 6, 6), (2, 6, 1)])
def test_prep_elementwise_constant_mean_by_node_type(ora, p, ns, na):
    """Element-wise constant H, A with a distinct value per element: an interior vertex node is the
    mean of its 4 elements, a node on an interior element edge (vertex on the box side, or the Q2 edge
    midpoint) the mean of 2, a Q2 element-centre node its own element, a box corner its single one."""
    nx, ny = 5, 4
    mesh = Mesh(nx, ny, lx=5e3, ly=4e3, p=p, ns=ns, na=na)
    N = nx * ny
    hval = 0.5 + 0.1 * np.arange(N) + 0.013 * np.arange(N) ** 2      # all distinct
    aval = 0.05 + 0.04 * ((7 * np.arange(N)) % N)                       # distinct, inside [0, 1]
    H = np.zeros((N, na)); A = np.zeros((N, na)); H[:, 0] = hval; A[:, 0] = aval
    Hn, An = ora.prep(mesh, H, A)
    NY, NX = mesh.node_shape
    for J in range(NY):
        for I in range(NX):
            # elements whose closed square contains node (I, J): reference position x = I / p
            exs = [ix for ix in range(nx) if ix <= I / p <= ix + 1]
            eys = [iy for iy in range(ny) if iy <= J / p <= iy + 1]
            adj = [iy * nx + ix for iy in eys for ix in exs]
            assert len(adj) in (1, 2, 4)
            assert abs(Hn[J, I] - np.mean(hval[adj])) <= 1e-15 * hval.max(), (I, J, adj)
            assert abs(An[J, I] - np.mean(aval[adj])) <= 1e-15, (I, J, adj)
    if p == 2:   # the three named node kinds of Q2 explicitly
        e = lambda ix, iy: iy * nx + ix
        assert Hn[2, 2] == pytest.approx(np.mean(hval[[e(0, 0), e(1, 0), e(0, 1), e(1, 1)]]), rel=1e-15)
        assert Hn[1, 2] == pytest.approx(np.mean(hval[[e(0, 0), e(1, 0)]]), rel=1e-15)
        assert Hn[3, 3] == hval[e(1, 1)]
    assert Hn[0, 0] == hval[0] and Hn[-1, -1] == hval[-1]


@pytest.mark.parametrize("p,ns,na", [(1, 3, 3), (2, 6, 6), (2, 8, 6), (2, 6, 3)])
def test_prep_random_dg_against_scatter_count(ora, p, ns, na):
    """Random DG data (no clamps active): the oracle's gather-and-average equals an independent
    scatter-and-count of the DG polynomial (sympy family) at every node."""
    nx, ny = 4, 3
    mesh, bm = _pair(nx, ny, p, ns, na, 4e3, 3e3, distorted=False)
    r = np.random.default_rng(41)
    H = r.uniform(-0.1, 0.1, (nx * ny, na)); H[:, 0] = r.uniform(1.0, 2.0, nx * ny)
    A = r.uniform(-0.05, 0.05, (nx * ny, na)); A[:, 0] = r.uniform(0.4, 0.6, nx * ny)
    Hn, An = ora.prep(mesh, H, A)
    bh, ba = brute.prep(bm, H, A)
    np.testing.assert_allclose(Hn.ravel(), bh, rtol=1e-14)
    np.testing.assert_allclose(An.ravel(), ba, rtol=1e-14)


# ---------------------------------------------------------------- O8 velocity: Jacobi coupling (R#11)
def _vel_inputs(mesh, seed):
    r = np.random.default_rng(seed)
    shp = mesh.node_shape
    d = dict(Fx=r.normal(0, 50, shp), Fy=r.normal(0, 50, shp), mass=r.uniform(1e5, 2e5, shp),
             Hn=r.uniform(0.5, 2, shp), An=r.uniform(0.5, 1, shp),
             vnx=r.uniform(-0.2, 0.2, shp), vny=r.uniform(-0.2, 0.2, shp),
             ox=r.uniform(-0.1, 0.1, shp), oy=r.uniform(-0.1, 0.1, shp),
             ax=r.uniform(-15, 15, shp), ay=r.uniform(-15, 15, shp),
             vx=r.uniform(-0.3, 0.3, shp), vy=r.uniform(-0.3, 0.3, shp))
    return d


def _vel(ora, mesh, prm, d):
    return ora.velocity(mesh, prm, d["Fx"], d["Fy"], d["mass"], d["Hn"], d["An"], d["vnx"], d["vny"],
                        d["ox"], d["oy"], d["ax"], d["ay"], d["vx"], d["vy"])


@pytest.mark.parametrize("theta", [math.pi / 2, 0.7, -2.1])
def test_velocity_commutes_with_rotations(ora, theta):
    """Eq. (2) is a vector equation - drag, Coriolis k x v, stress force, relaxation - so the
    discrete update must commute with rotating every vector input (v^(p-1), v^n, o, a, F) by any angle:
    R(update(x)) = update(R x).  Coriolis on, drag on, beta and f dt large enough that a Gauss-Seidel
    ordering of the (x, y) pair (vy from the new vx) breaks it by many orders above rounding."""
    mesh = Mesh(3, 3, lx=3e4, ly=3e4, p=2, ns=6, na=6)
    prm = Params(beta=0.7, f_c=1e-3, dt=600.0)
    d = _vel_inputs(mesh, 17)
    c, s = math.cos(theta), math.sin(theta)
    rot = lambda x, y: (c * x - s * y, s * x + c * y)
    vx, vy = _vel(ora, mesh, prm, d)
    e = dict(d)
    for kx, ky in (("Fx", "Fy"), ("vnx", "vny"), ("ox", "oy"), ("ax", "ay"), ("vx", "vy")):
        e[kx], e[ky] = rot(d[kx], d[ky])
    wx, wy = _vel(ora, mesh, prm, e)
    rx, ry = rot(vx, vy)
    scale = np.abs(np.stack([vx, vy])).max()
    assert np.abs(wx - rx).max() < 1e-14 * scale and np.abs(wy - ry).max() < 1e-14 * scale


def test_velocity_coriolis_is_a_complex_scaling(ora):
    """Drag, stress, forcing, o and v^n off: Eq. (2) with the mEVP relaxation (R#11) reduces to
    (1 + beta) v^(p) = beta v^(p-1) + dt f v^(p-1) x k, i.e. with z = vx + i vy,
    z^(p) = (beta - i dt f) / (1 + beta) z^(p-1) (v x k is the rotation by -90 degrees): every interior
    node is scaled by the SAME complex factor, whatever its v.  Gauss-Seidel in (x, y) would make it
    node-dependent."""
    mesh = Mesh(3, 3, lx=3e4, ly=3e4, p=2, ns=6, na=6)
    beta, f, dt = 0.4, 1e-3, 600.0
    prm = Params(beta=beta, f_c=f, dt=dt, rho_atm=0.0, rho_ocean=0.0)
    d = _vel_inputs(mesh, 23)
    Z = np.zeros(mesh.node_shape)
    for k in ("Fx", "Fy", "vnx", "vny", "ox", "oy", "ax", "ay"):
        d[k] = Z
    vx, vy = _vel(ora, mesh, prm, d)
    z0 = (d["vx"] + 1j * d["vy"])[1:-1, 1:-1]
    z1 = (vx + 1j * vy)[1:-1, 1:-1]
    ratio = z1 / z0
    expect = (beta - 1j * dt * f) / (1.0 + beta)
    assert np.abs(ratio - expect).max() < 1e-14
    assert (vx[0] == 0).all() and (vx[:, 0] == 0).all() and (vy[-1] == 0).all()


def test_velocity_update_matches_vector_form(ora):
    """The whole O8 update against the vector-form brute force (Coriolis as (v - o) x k, all drag terms
    on), box and random data: also pins the Jacobi coupling with every term present."""
    mesh = Mesh(3, 3, lx=3e4, ly=3e4, p=2, ns=6, na=6)
    bm = brute.BMesh(3, 3, 3e4, 3e4, 2, 6, 6)
    prm = Params(beta=0.9, f_c=1e-3, dt=600.0)
    d = _vel_inputs(mesh, 29)
    vx, vy = _vel(ora, mesh, prm, d)
    st = lambda a, b: np.stack([d[a].ravel(), d[b].ravel()], axis=1)
    out = brute.velocity(bm, prm, d["Fx"].ravel(), d["Fy"].ravel(), d["mass"].ravel(), d["Hn"].ravel(),
                         d["An"].ravel(), st("vnx", "vny"), st("ox", "oy"), st("ax", "ay"), st("vx", "vy"))
    np.testing.assert_allclose(vx.ravel(), out[:, 0], rtol=0, atol=1e-14 * np.abs(out).max())
    np.testing.assert_allclose(vy.ravel(), out[:, 1], rtol=0, atol=1e-14 * np.abs(out).max())


# ---------------------------------------------------------------- distorted meshes (NEXT-1, R#23)
@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6)])
def test_distorted_lumped_mass(ora, p, ns):
    """O7 on a distorted mesh: sum_j m_j = Lx Ly, and every node's m_j equals an independent 8-point
    integral of phi_j |J| (exact: Q_p times a bilinear |J|)."""
    mesh, bm = _pair(5, 4, p, ns, min(ns, 6), 5e3, 4e3, distorted=True)
    m = ora.lumped_mass(mesh)
    assert abs(m.sum() - 5e3 * 4e3) < 1e-12 * 2e7
    np.testing.assert_allclose(m.ravel(), brute.lumped_mass(bm), rtol=1e-13)


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_distorted_strain_brute_force(ora, p, ns):
    """O4 on a distorted mesh against the assembled brute-force strain operator (|J|-weighted L2
    projection, 8-point rule, adjugate gradients)."""
    mesh, bm = _pair(4, 3, p, ns, min(ns, 6), 4e3, 3e3, distorted=True)
    r = np.random.default_rng(5)
    vx = r.uniform(-0.2, 0.2, mesh.node_shape); vy = r.uniform(-0.2, 0.2, mesh.node_shape)
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    G = brute.strain_matrices(bm)
    ref = ((G["11"] @ vx.ravel() + G["11y"] @ vy.ravel()).reshape(-1, ns), (G["12x"] @ vx.ravel() + G["12y"] @ vy.ravel()).reshape(-1, ns),
           (G["22"] @ vy.ravel()).reshape(-1, ns))
    scale = max(np.abs(x).max() for x in ref)
    for g, x in zip((E11, E12, E22), ref):
        assert np.abs(g - x).max() < 1e-12 * scale


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_distorted_divergence_brute_force(ora, p, ns):
    """O6 on a distorted mesh against the assembled brute-force divergence F = -D sigma."""
    mesh, bm = _pair(4, 3, p, ns, min(ns, 6), 4e3, 3e3, distorted=True)
    r = np.random.default_rng(6)
    S = [r.uniform(-1e4, 1e4, (12, ns)) for _ in range(3)]
    Fx, Fy = ora.divergence(mesh, *S)
    Dx, Dy, K = brute.divergence_matrices(bm)
    s11, s12, s22 = (x.ravel() for x in S)
    rx, ry = -(Dx @ s11 + Dy @ s12 + K @ s12), -(Dx @ s12 + Dy @ s22 - K @ s11)
    scale = max(np.abs(rx).max(), np.abs(ry).max())
    assert np.abs(Fx.ravel() - rx).max() < 1e-12 * scale and np.abs(Fy.ravel() - ry).max() < 1e-12 * scale


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_distorted_strain_divergence_adjointness(ora, p, ns):
    """Weak-form identity on a distorted mesh: sum_j v_j . F_j = -sum_K int_K sigma : eps(v) dx
    = -sum_K (S11^T M_K E11 + 2 S12^T M_K E12 + S22^T M_K E22), with M_K the |J|-weighted DG mass
    from an independent 8-point rule.  Both sides come from the oracle's strain and divergence; a
    wrong |J|, a transposed J^-1 or a sign anywhere in either breaks it."""
    mesh, bm = _pair(4, 3, p, ns, min(ns, 6), 4e3, 3e3, distorted=True)
    r = np.random.default_rng(8)
    vx = r.uniform(-1, 1, mesh.node_shape); vy = r.uniform(-1, 1, mesh.node_shape)
    S = [r.uniform(-1, 1, (12, ns)) for _ in range(3)]
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    Fx, Fy = ora.divergence(mesh, *S)
    lhs = (vx * Fx + vy * Fy).sum()
    rhs = 0.0
    for iy in range(3):
        for ix in range(4):
            e = iy * 4 + ix
            M = brute.elem_mass(bm, ix, iy, ns)
            rhs -= S[0][e] @ M @ E11[e] + 2 * S[1][e] @ M @ E12[e] + S[2][e] @ M @ E22[e]
    assert abs(lhs - rhs) < 1e-12 * max(abs(lhs), 1.0) * 10


@pytest.mark.parametrize("p,ns,na", [(1, 3, 3), (2, 6, 6), (2, 6, 1)])
def test_distorted_advection_preserves_constant_in_uniform_flow(ora, p, ns, na):
    """Divergence theorem: a constant tracer in a uniform flow (exactly representable in any CG space
    on any mesh) has zero right-hand side at every element whose neighbours all exist - the volume term
    int c v.grad psi and the edge term oint c (v.n) psi cancel (both integrands polynomial; the edge is
    straight).  Needs the true edge length and normal on distorted elements."""
    mesh, _ = _pair(5, 4, p, ns, na, 5e3, 4e3, distorted=True)
    vx = np.full(mesh.node_shape, 0.13); vy = np.full(mesh.node_shape, -0.07)
    c = np.zeros((20, na)); c[:, 0] = 0.8
    rhs = ora.advect_rhs(mesh, vx, vy, c).reshape(4, 5, na)
    assert np.abs(rhs[1:-1, 1:-1]).max() < 1e-17


def test_distorted_advection_closed_box_conserves_mass(ora):
    """Closed box (v = 0 on the boundary, no boundary flux): the semi-discrete total mass
    sum_K int_K c |J| = sum_K (M_K c_K)_0 has zero time derivative; M_K from an independent rule."""
    for p, ns, na in ((1, 3, 3), (2, 6, 6)):
        mesh, bm = _pair(5, 4, p, ns, na, 5e3, 4e3, distorted=True)
        r = np.random.default_rng(12)
        vx = r.uniform(-0.1, 0.1, mesh.node_shape); vy = r.uniform(-0.1, 0.1, mesh.node_shape)
        for v in (vx, vy):
            v[0, :] = v[-1, :] = v[:, 0] = v[:, -1] = 0.0
        c = r.uniform(-0.2, 0.2, (20, na)); c[:, 0] = r.uniform(0.5, 1.0, 20)
        rhs = ora.advect_rhs(mesh, vx, vy, c)
        tot = sum((brute.elem_mass(bm, e % 5, e // 5, na) @ rhs[e])[0] for e in range(20))
        scale = sum(abs((brute.elem_mass(bm, e % 5, e // 5, na) @ rhs[e])[0]) for e in range(20))
        assert abs(tot) < 1e-13 * scale


@pytest.mark.parametrize("p,ns,na,bc", [(1, 3, 3, 0), (2, 6, 6, 0), (2, 6, 6, 1), (2, 6, 3, 1), (1, 3, 1, 0)])
def test_distorted_advection_operator_brute_force(ora, p, ns, na, bc):
    """O11's whole operator on a distorted mesh against the brute force: volume term through the
    adjugate, edge fluxes with N = outward normal x length from the edge's end vertices, upwind trace,
    ngp-point rules, M_K solve."""
    mesh, bm = _pair(4, 4, p, ns, na, 4e3, 4e3, distorted=True, bc=bc)
    r = np.random.default_rng(31)
    vx = r.uniform(-0.1, 0.1, mesh.node_shape); vy = r.uniform(-0.1, 0.1, mesh.node_shape)
    if bc == 1:
        for v in (vx, vy):
            v[-1, :] = v[0, :]; v[:, -1] = v[:, 0]
    c = r.uniform(-0.3, 0.3, (16, na)); c[:, 0] = r.uniform(0.3, 1.0, 16)
    got = ora.advect_rhs(mesh, vx, vy, c)
    ref = brute.advect_rhs(bm, vx, vy, c)
    assert _rel(got, ref) < 1e-12


def test_box_advection_operator_brute_force(ora):
    """The same brute force on the box (closed and periodic), CG2/DG2."""
    for bc in (0, 1):
        mesh, bm = _pair(4, 3, 2, 6, 6, 4e3, 3e3, distorted=False, bc=bc)
        r = np.random.default_rng(33)
        vx = r.uniform(-0.1, 0.1, mesh.node_shape); vy = r.uniform(-0.1, 0.1, mesh.node_shape)
        if bc == 1:
            for v in (vx, vy):
                v[-1, :] = v[0, :]; v[:, -1] = v[:, 0]
        c = r.uniform(-0.3, 0.3, (12, 6)); c[:, 0] = r.uniform(0.3, 1.0, 12)
        assert _rel(ora.advect_rhs(mesh, vx, vy, c), brute.advect_rhs(bm, vx, vy, c)) < 1e-12


# ---------------------------------------------------------------- whole subcycle, assembled operators
@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("p,ns,na", [(1, 3, 3), (2, 6, 6), (2, 8, 6)])
@pytest.mark.parametrize("distorted", [False, True, "sphere"])
def test_whole_subcycle_assembled_operators(ora, n, p, ns, na, distorted):
    """n x n meshes, 3 subcycles (strain -> stress -> divergence -> velocity)
    computed with globally assembled operators (tests/brute.py) vs the element-loop oracle, on seeded
    random data (clamps active, S^0 != 0); box, distorted quads (R#23) and the lon-lat sphere (R#26)."""
    lx = ly = n * 1e3
    mesh, bm = _pair(n, n, p, ns, na, lx, ly, distorted=distorted, seed=inputs.SEED_BASE + n)
    st = inputs.make_case(n, n, p, ns, na, kind="random", lx=lx, ly=ly, seed=inputs.SEED_BASE + 10 * n + p)
    prm = Params(alpha=5.0, beta=3.0)
    got = ora.subcycles(mesh, prm, 3, st)
    ref = brute.subcycles(bm, prm, 3, st)
    for grp in (("S11", "S12", "S22"), ("vx", "vy")):
        num = max(np.abs(got[k] - ref[k]).max() for k in grp)
        den = max(np.abs(ref[k]).max() for k in grp)
        assert num <= 1e-12 * den, (grp, num / den)


# ---------------------------------------------------------------- R#4 replacement pressure
def test_replacement_pressure_scales_the_plastic_stress(ora):
    """R#4 (P_r = P Delta_raw / Delta in place of P in the -P/2 term): then
    sigma = P/(2 Delta) L(e) - P_r/2 I = (Delta_raw / Delta) [P/(2 Delta_raw) L(e) - P/2 I], i.e. exactly
    Delta_raw / Delta times the plastic-limit (Delta_min -> 0) stress of the paper's law - the stress
    vanishes with the strain rate and sits on the yield curve scaled by Delta_raw / Delta.  alpha = 1 and
    element-constant fields make one update return the projection of sigma exactly."""
    mesh = Mesh(6, 6, lx=6e3, ly=6e3, p=2, ns=6, na=6)
    N = mesh.n_elem
    r = np.random.default_rng(19)
    e11, e12, e22 = (r.normal(0, 1e-8, N) * r.choice([1e-2, 1.0, 1e2], N) for _ in range(3))
    E = [np.zeros((N, 6)) for _ in range(3)]
    E[0][:, 0], E[1][:, 0], E[2][:, 0] = e11, e12, e22
    H = np.zeros((N, 6)); H[:, 0] = r.uniform(0.5, 2.0, N)
    A = np.zeros((N, 6)); A[:, 0] = r.uniform(0.8, 1.0, N)
    Z = [np.zeros((N, 6))] * 3
    dmin = 2e-9
    rp = [o[:, 0] for o in ora.stress(mesh, Params(alpha=1.0, DeltaMin=dmin, replacement_pressure=1), *E, H, A, *Z)]
    pl = [o[:, 0] for o in ora.stress(mesh, Params(alpha=1.0, DeltaMin=0.0), *E, H, A, *Z)]
    draw = np.sqrt(1.25 * (e11**2 + e22**2) + 1.5 * e11 * e22 + e12**2)
    ratio = draw / np.sqrt(dmin**2 + draw**2)
    assert ratio.min() < 0.5 and ratio.max() > 0.99          # both regimes present
    for a, b in zip(rp, pl):
        np.testing.assert_allclose(a, ratio * b, rtol=1e-12, atol=1e-12 * np.abs(b).max())
    # zero strain rate: zero stress (the defining property of the replacement pressure)
    z = ora.stress(mesh, Params(alpha=1.0, replacement_pressure=1), *Z, H, A, *Z)
    assert max(np.abs(x).max() for x in z) == 0.0


# ---------------------------------------------------------------- sphere (NEXT-4, R#26)
def test_sphere_element_areas_closed_form(ora):
    """The Gauss integral of |J| over a lon-lat element approximates its exact spherical area
    R^2 dlon (sin lat1 - sin lat0) within the 3-point rule's error bound (|err| <= dlat^7 / 2016000 x
    |cos^(6)| x R^2 dlon ~ 1e-16 relative here), per element and in total."""
    mesh, _ = _sphere_pair(4, 5, 2, 6, 6)
    x, w = ora.gauss(3)
    tot = 0.0
    for iy in range(5):
        la, lb = LAT0 + iy * 0.04, LAT0 + (iy + 1) * 0.04
        exact = R_EARTH**2 * 0.05 * (math.sin(lb) - math.sin(la))
        for ix in range(4):
            area = sum(w[a] * w[b] * ora.jacobian(mesh, ix, iy, x[a], x[b])[0] for a in range(3) for b in range(3))
            assert abs(area - exact) < 1e-13 * exact
            tot += area
    exact_tot = R_EARTH**2 * 0.2 * (math.sin(LAT0 + 0.2) - math.sin(LAT0))
    assert abs(tot - exact_tot) < 1e-13 * exact_tot
    m = ora.lumped_mass(mesh)
    assert abs(m.sum() - tot) < 1e-12 * tot


def test_sphere_reduces_to_the_box_near_the_equator(ora):
    """Special case: a patch at the equator on a sphere of radius 1e12 m with the box's physical sizes
    (dlon = hx / R, dlat = hy / R) is the plane box up to O((L/R)^2) ~ 1e-17: one outer step (advection +
    3 subcycles) agrees with the box oracle to rounding.  Catches a swapped dlon / dlat, a missing R or
    cos in the sphere's metric."""
    nx, ny, hx, hy = 5, 4, 1.2e3, 0.9e3
    R = 1e12
    st = inputs.make_case(nx, ny, 2, 6, 6, kind="random", lx=nx * hx, ly=ny * hy)
    box = ora.outer_step(Mesh(nx, ny, lx=nx * hx, ly=ny * hy), Params(), 3, st)
    sph = ora.outer_step(Mesh(nx, ny, lx=nx * hx / R, ly=ny * hy / R, radius=R, lat0=-0.5 * ny * hy / R),
                         Params(), 3, st)
    for grp in (("S11", "S12", "S22"), ("vx", "vy"), ("A",), ("H",)):
        num = max(np.abs(box[k] - sph[k]).max() for k in grp)
        den = max(np.abs(box[k]).max() for k in grp)
        assert num <= 1e-12 * den, (grp, num / den)


@pytest.mark.parametrize("p,ns,na", [(1, 3, 3), (2, 6, 6), (2, 6, 1)])
def test_sphere_zonal_flow_preserves_constant(ora, p, ns, na):
    """A constant tracer in any zonal flow u(lat), v = 0 (divergence-free on the sphere:
    div v = (1/(R cos lat)) du/dlon = 0) is a steady state at every interior element: the volume term's
    longitude integral of d(psi)/ds is exact and the meridian-edge fluxes use the same latitude points,
    so they cancel to rounding.  Needs the sphere's edge lengths / normals and |J|."""
    mesh, _ = _sphere_pair(5, 4, p, ns, na)
    NY, NX = mesh.node_shape
    r = np.random.default_rng(3)
    u_row = r.uniform(-0.2, 0.2, NY)
    vx = np.repeat(u_row[:, None], NX, axis=1); vy = np.zeros((NY, NX))
    c = np.zeros((20, na)); c[:, 0] = 0.7
    rhs = ora.advect_rhs(mesh, vx, vy, c).reshape(4, 5, na)
    assert np.abs(rhs[1:-1, 1:-1]).max() < 1e-13 * 0.2 / (R_EARTH * 0.04)


def test_sphere_rigid_rotation_has_no_strain(ora):
    """A rigid rotation about the polar axis, u = w R cos(lat), v = 0, has zero strain rate on the
    sphere - only because of the metric term: (1/R) du/dlat + u tan(lat)/R = w (-sin + cos tan) = 0.
    Its CG2 interpolant differs from cos by O(dlat^3), so the DG strain is bounded by ~ w dlat^2;
    without the metric term E12 would be -w sin(lat)/2 ~ 0.45 w."""
    mesh, _ = _sphere_pair(6, 5, 2, 6, 6)
    NY, NX = mesh.node_shape
    om = 1e-6
    lat = LAT0 + np.arange(NY) * 0.02
    vx = np.repeat((om * R_EARTH * np.cos(lat))[:, None], NX, axis=1); vy = np.zeros((NY, NX))
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    for E in (E11, E12, E22):
        assert np.abs(E).max() < 5e-3 * om
    # the same field on the plane (no metric term) is strained: the term is what cancels it
    flat = Mesh(6, 5, lx=6 * 0.05 * R_EARTH * math.cos(LAT0), ly=5 * 0.04 * R_EARTH)
    assert np.abs(ora.strain(flat, vx, vy)[1][:, 0]).max() > 0.3 * om


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_sphere_strain_divergence_adjointness(ora, p, ns):
    """Weak-form identity on the sphere: sum_j v_j . F_j = -sum_K (S11 M_K E11 + 2 S12 M_K E12 +
    S22 M_K E22) with M_K the cos(lat)-weighted DG mass of an independent rule (the method's 3-point
    rule: the projection is the discrete L2 projection of that rule, so the identity is exact).  A sign
    or a missing factor of the metric term in either the strain or the divergence breaks it."""
    mesh, bm = _sphere_pair(4, 3, p, ns, min(ns, 6))
    r = np.random.default_rng(8)
    vx = r.uniform(-1, 1, mesh.node_shape); vy = r.uniform(-1, 1, mesh.node_shape)
    S = [r.uniform(-1, 1, (12, ns)) for _ in range(3)]
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    Fx, Fy = ora.divergence(mesh, *S)
    lhs = (vx * Fx + vy * Fy).sum()
    rhs = 0.0
    for iy in range(3):
        for ix in range(4):
            e = iy * 4 + ix
            M = brute.elem_mass(bm, ix, iy, ns)
            rhs -= S[0][e] @ M @ E11[e] + 2 * S[1][e] @ M @ E12[e] + S[2][e] @ M @ E22[e]
    assert abs(lhs - rhs) < 1e-12 * max(abs(lhs), 1.0) * 10


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_sphere_strain_and_divergence_brute_force(ora, p, ns):
    """O4 / O6 on the sphere against the assembled brute-force operators (metric from the line
    element, tan(lat)/R terms, the method's rule)."""
    mesh, bm = _sphere_pair(4, 3, p, ns, min(ns, 6))
    r = np.random.default_rng(5)
    vx = r.uniform(-0.2, 0.2, mesh.node_shape); vy = r.uniform(-0.2, 0.2, mesh.node_shape)
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    G = brute.strain_matrices(bm)
    ref = ((G["11"] @ vx.ravel() + G["11y"] @ vy.ravel()).reshape(-1, ns),
           (G["12x"] @ vx.ravel() + G["12y"] @ vy.ravel()).reshape(-1, ns), (G["22"] @ vy.ravel()).reshape(-1, ns))
    scale = max(np.abs(x).max() for x in ref)
    for g, x in zip((E11, E12, E22), ref):
        assert np.abs(g - x).max() < 1e-12 * scale
    S = [r.uniform(-1e4, 1e4, (12, ns)) for _ in range(3)]
    Fx, Fy = ora.divergence(mesh, *S)
    Dx, Dy, K = brute.divergence_matrices(bm)
    s11, s12, s22 = (x.ravel() for x in S)
    rx, ry = -(Dx @ s11 + Dy @ s12 + K @ s12), -(Dx @ s12 + Dy @ s22 - K @ s11)
    sc = max(np.abs(rx).max(), np.abs(ry).max())
    assert np.abs(Fx.ravel() - rx).max() < 1e-12 * sc and np.abs(Fy.ravel() - ry).max() < 1e-12 * sc
    np.testing.assert_allclose(ora.lumped_mass(mesh).ravel(), brute.lumped_mass(bm), rtol=1e-13)


@pytest.mark.parametrize("p,ns,na,bc", [(1, 3, 3, 0), (2, 6, 6, 0), (2, 6, 6, 1), (2, 6, 1, 0)])
def test_sphere_advection_operator_brute_force(ora, p, ns, na, bc):
    """O11 on the sphere against the brute force (meridian / parallel arc normals and lengths,
    cos(lat)-weighted mass), closed and periodic; and closed-box conservation of sum_K int_K c dA."""
    mesh, bm = _sphere_pair(4, 4, p, ns, na, bc=bc)
    r = np.random.default_rng(31)
    vx = r.uniform(-0.1, 0.1, mesh.node_shape); vy = r.uniform(-0.1, 0.1, mesh.node_shape)
    if bc == 1:
        for v in (vx, vy):
            v[-1, :] = v[0, :]; v[:, -1] = v[:, 0]
    else:
        for v in (vx, vy):
            v[0, :] = v[-1, :] = v[:, 0] = v[:, -1] = 0.0
    c = r.uniform(-0.3, 0.3, (16, na)); c[:, 0] = r.uniform(0.3, 1.0, 16)
    got = ora.advect_rhs(mesh, vx, vy, c)
    assert _rel(got, brute.advect_rhs(bm, vx, vy, c)) < 1e-12
    if bc == 0:
        d = [(brute.elem_mass(bm, e % 4, e // 4, na) @ got[e])[0] for e in range(16)]
        assert abs(sum(d)) < 1e-13 * sum(abs(x) for x in d)
