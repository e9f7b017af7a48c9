"""Pins for the oracle (``-m "not gpu"``).

Every test checks the oracle against something other than itself: a closed
form, a value printed in the paper, an invariant of the mathematics, a
textbook special case, or an independent brute-force computation written here
with different building blocks (numpy's Gauss-Legendre rule of another order,
Vandermonde-built Lagrange bases, sympy exact integration).  Each docstring
names the passage or DESIGN.md reading it pins.
"""
import math

import numpy as np
import pytest
import sympy as sp

import oracle
from oracle import Mesh, Params
from paper_2402_00466_b200 import inputs

RNG = np.random.default_rng(7)


# ---------------------------------------------------------------- quadrature
@pytest.mark.parametrize("ngp", [1, 2, 3])
def test_gauss_rule_exactness(ora, ngp):
    """Gauss-Legendre on [0,1] integrates s^a exactly for a <= 2 ngp - 1 and not beyond (R#18)."""
    x, w = ora.gauss(ngp)
    assert abs(w.sum() - 1.0) < 1e-15
    for a in range(2 * ngp):
        assert abs((w * x**a).sum() - 1.0 / (a + 1)) < 1e-15
    assert abs((w * x ** (2 * ngp)).sum() - 1.0 / (2 * ngp + 1)) > 1e-6


def test_ngp_from_listing2(ora):
    """NGP = 3 for DGstress in {6, 8}, 2 for DGstress == 3, else -1."""
    assert [ora.ngp(n) for n in (3, 6, 8, 5, 1)] == [2, 3, 3, -1, -1]


def test_psi_1_1_paper_value(ora):
    """PSI_1_1 = {1.0}."""
    for s, t in [(0.5, 0.5), (0.1, 0.9)]:
        assert ora.dg_basis(1, s, t).tolist() == [1.0]


# ---------------------------------------------------------------- bases
def test_dg_mass_closed_form(ora):
    """R#5: centred Legendre basis -> M_ref = diag(1, 1/12, 1/12, 1/180, 1/180, 1/144) * |K|.
    The diagonal is the exact integral over the unit square (sympy), independent of quadrature."""
    s, t = sp.symbols("s t")
    S, T = s - sp.Rational(1, 2), t - sp.Rational(1, 2)
    # exact norms of the orthogonal family (closed form)
    exact = [1, sp.Rational(1, 12), sp.Rational(1, 12), sp.Rational(1, 180), sp.Rational(1, 180), sp.Rational(1, 144),
             sp.Rational(1, 2160), sp.Rational(1, 2160)]
    fam = [sp.Integer(1), S, T, S**2 - sp.Rational(1, 12), T**2 - sp.Rational(1, 12), S * T,
           (S**2 - sp.Rational(1, 12)) * T, S * (T**2 - sp.Rational(1, 12))]
    for k, f in enumerate(fam):
        assert sp.integrate(sp.integrate(f * f, (s, 0, 1)), (t, 0, 1)) == exact[k]
        for l in range(k):   # orthogonal family (R#5, R#24)
            assert sp.integrate(sp.integrate(f * fam[l], (s, 0, 1)), (t, 0, 1)) == 0
    for k, f in enumerate(fam):   # the oracle's basis is this family, in this order
        for (sv, tv) in [(0.1, 0.7), (0.9, 0.35)]:
            assert abs(ora.dg_basis(8, sv, tv)[k] - float(f.subs({s: sv, t: tv}))) < 1e-15
    for (hx, hy) in [(1.0, 1.0), (2.0, 3.0)]:
        mesh = Mesh(4, 3, lx=4 * hx, ly=3 * hy)
        M = ora.element_mass(mesh, 2, 1, 6, 3)
        np.testing.assert_allclose(M, np.diag([float(e) for e in exact[:6]]) * hx * hy, rtol=1e-14, atol=1e-15)
        M8 = ora.element_mass(mesh, 1, 2, 8, 3)
        np.testing.assert_allclose(M8, np.diag([float(e) for e in exact]) * hx * hy, rtol=1e-14, atol=1e-15)
        M3 = ora.element_mass(mesh, 0, 0, 3, 2)
        np.testing.assert_allclose(M3, np.diag([1, 1 / 12, 1 / 12]) * hx * hy, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("p", [1, 2])
def test_cg_basis_lagrange_properties(ora, p):
    """Q_p Lagrange on equispaced nodes (R#8): Kronecker at nodes, partition of unity,
    derivatives agree with central finite differences."""
    nodes = np.linspace(0, 1, p + 1)
    for jy in range(p + 1):
        for jx in range(p + 1):
            phi, _, _ = ora.cg_basis(p, nodes[jx], nodes[jy])
            e = np.zeros((p + 1) ** 2); e[jy * (p + 1) + jx] = 1
            np.testing.assert_allclose(phi, e, atol=1e-15)
    for s, t in RNG.uniform(0, 1, (5, 2)):
        phi, ds, dt = ora.cg_basis(p, s, t)
        assert abs(phi.sum() - 1) < 1e-14 and abs(ds.sum()) < 1e-13 and abs(dt.sum()) < 1e-13
        h = 1e-6
        fd_s = (ora.cg_basis(p, s + h, t)[0] - ora.cg_basis(p, s - h, t)[0]) / (2 * h)
        fd_t = (ora.cg_basis(p, s, t + h)[0] - ora.cg_basis(p, s, t - h)[0]) / (2 * h)
        np.testing.assert_allclose(ds, fd_s, atol=1e-8)
        np.testing.assert_allclose(dt, fd_t, atol=1e-8)


def test_box_jacobian(ora):
    """Affine box element: |J| = hx hy, J^{-1} = diag(1/hx, 1/hy); sum |K| = Lx Ly."""
    mesh = Mesh(5, 7, lx=10.0, ly=21.0)
    det, Jinv = ora.jacobian(mesh, 3, 4, 0.3, 0.8)
    assert abs(det - 6.0) < 1e-14
    np.testing.assert_allclose(Jinv, [[0.5, 0], [0, 1 / 3]], atol=1e-15)
    tot = sum(ora.jacobian(mesh, ix, iy, 0.5, 0.5)[0] for ix in range(5) for iy in range(7))
    assert abs(tot - 210.0) < 1e-10


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6)])
def test_lumped_mass_closed_form(ora, p, ns):
    """O7: int phi_j = |K| x {1/4} (Q1) or {1/36, 1/9, 4/9} (Q2 corner/edge/centre);
    assembled masses follow by adjacency; sum = Lx Ly."""
    nx, ny, lx, ly = 4, 3, 8.0, 9.0
    mesh = Mesh(nx, ny, lx=lx, ly=ly, p=p, ns=ns, na=min(ns, 6))
    m = ora.lumped_mass(mesh)
    K = (lx / nx) * (ly / ny)
    w1 = {1: [0.5, 0.5], 2: [1 / 6, 2 / 3, 1 / 6]}[p]  # 1D integrals of the Lagrange basis
    NX, NY = p * nx + 1, p * ny + 1
    ref = np.zeros((NY, NX))
    for iy in range(ny):
        for ix in range(nx):
            for jy in range(p + 1):
                for jx in range(p + 1):
                    ref[p * iy + jy, p * ix + jx] += K * w1[jx] * w1[jy]
    np.testing.assert_allclose(m, ref, rtol=1e-14)
    assert abs(m.sum() - lx * ly) < 1e-12 * lx * ly
    if p == 2:  # the named closed forms
        assert abs(m[2, 2] - 4 * K / 36) < 1e-14 * K and abs(m[1, 1] - 4 * K / 9) < 1e-14 * K
        assert abs(m[1, 2] - 2 * K / 9) < 1e-14 * K


# ---------------------------------------------------------------- strain
def _nodal(mesh, f):
    NY, NX = mesh.node_shape
    hx, hy = mesh.lx / mesh.nx, mesh.ly / mesh.ny
    X, Y = np.meshgrid(np.arange(NX) * hx / mesh.p, np.arange(NY) * hy / mesh.p)
    return f(X, Y)


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_strain_constant_velocity_is_zero(ora, p, ns):
    """north_star pin: zero strain rate for constant velocity."""
    mesh = Mesh(5, 4, lx=50e3, ly=40e3, p=p, ns=ns, na=min(ns, 6))
    vx = np.full(mesh.node_shape, 0.37); vy = np.full(mesh.node_shape, -0.21)
    for E in ora.strain(mesh, vx, vy):
        assert np.abs(E).max() < 1e-13 * 0.37 / 1e4


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_strain_linear_velocity_exact(ora, p, ns):
    """north_star pin: v = v0 + G x gives E11 = G11, E22 = G22, E12 = (G12 + G21)/2 in the
    constant coefficient and 0 elsewhere (G12 != G21 catches a transposed gradient)."""
    mesh = Mesh(6, 5, lx=60e3, ly=50e3, p=p, ns=ns, na=min(ns, 6))
    G = np.array([[3e-6, -7e-6], [5e-6, -2e-6]])
    vx = _nodal(mesh, lambda X, Y: 0.1 + G[0, 0] * X + G[0, 1] * Y)
    vy = _nodal(mesh, lambda X, Y: -0.05 + G[1, 0] * X + G[1, 1] * Y)
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    tol = 1e-12 * 1e-5
    for E, val in ((E11, G[0, 0]), (E22, G[1, 1]), (E12, 0.5 * (G[0, 1] + G[1, 0]))):
        np.testing.assert_allclose(E[:, 0], val, atol=tol)
        assert np.abs(E[:, 1:]).max() < tol


def _lagrange_1d(p):
    """Independent 1D Lagrange basis via a Vandermonde solve (numpy polynomial coefficients)."""
    nodes = np.linspace(0, 1, p + 1)
    V = np.vander(nodes, p + 1, increasing=True)
    C = np.linalg.inv(V)  # column j = coefficients of L_j
    L = lambda s: np.array([np.polynomial.polynomial.polyval(s, C[:, j]) for j in range(p + 1)])
    dL = lambda s: np.array([np.polynomial.polynomial.polyval(s, np.polynomial.polynomial.polyder(C[:, j]))
                             for j in range(p + 1)])
    return L, dL


def _brute_strain(mesh, vx, vy):
    """Brute force: exact L2 projection of sym grad(v_h) with an 8-point numpy Gauss rule
    (exact for these degrees), Vandermonde Lagrange bases and the closed-form diagonal mass."""
    p, ns = mesh.p, mesh.ns
    hx, hy = mesh.lx / mesh.nx, mesh.ly / mesh.ny
    xi, wi = np.polynomial.legendre.leggauss(8)
    q, w = 0.5 * (xi + 1), 0.5 * wi
    L, dL = _lagrange_1d(p)
    fam = [lambda S, T: 1 + 0 * S, lambda S, T: S, lambda S, T: T, lambda S, T: S * S - 1 / 12,
           lambda S, T: T * T - 1 / 12, lambda S, T: S * T, lambda S, T: (S * S - 1 / 12) * T,
           lambda S, T: S * (T * T - 1 / 12)][:ns]
    norm = np.array([1, 1 / 12, 1 / 12, 1 / 180, 1 / 180, 1 / 144, 1 / 2160, 1 / 2160])[:ns]
    out = [np.zeros((mesh.n_elem, ns)) for _ in range(3)]
    for iy in range(mesh.ny):
        for ix in range(mesh.nx):
            e = iy * mesh.nx + ix
            ux = vx[p * iy:p * iy + p + 1, p * ix:p * ix + p + 1]
            uy = vy[p * iy:p * iy + p + 1, p * ix:p * ix + p + 1]
            acc = [np.zeros(ns) for _ in range(3)]
            for a in range(8):
                for b in range(8):
                    s, t = q[a], q[b]
                    Ls, Lt, dLs, dLt = L(s), L(t), dL(s), dL(t)
                    dxs = lambda u: (Lt @ u @ dLs) / hx
                    dys = lambda u: (dLt @ u @ Ls) / hy
                    eps = (dxs(ux), 0.5 * (dys(ux) + dxs(uy)), dys(uy))
                    psi = np.array([f(s - 0.5, t - 0.5) for f in fam])
                    for c in range(3):
                        acc[c] += w[a] * w[b] * psi * eps[c]
            for c in range(3):
                out[c][e] = acc[c] / norm
    return out  # order E11, E12, E22


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_strain_brute_force(ora, p, ns):
    """north_star pin (brute force on tiny meshes): random nodal v on a 3x2 mesh."""
    mesh = Mesh(3, 2, lx=3e3, ly=2.5e3, p=p, ns=ns, na=min(ns, 6))
    vx = RNG.uniform(-0.2, 0.2, mesh.node_shape); vy = RNG.uniform(-0.2, 0.2, mesh.node_shape)
    got = ora.strain(mesh, vx, vy)
    ref = _brute_strain(mesh, vx, vy)
    scale = max(np.abs(r).max() for r in ref)
    for g, r in zip(got, ref):
        np.testing.assert_allclose(g, r, atol=1e-13 * scale)


def test_strain_quadratic_cg2_exact(ora):
    """Quadratic v (CG2) whose strain lies in the DG2 space is reproduced exactly:
    vx = x^2 + x y, vy = y^2  ->  eps11 = 2x + y, eps22 = 2y, eps12 = x/2."""
    mesh = Mesh(4, 3, lx=4.0, ly=3.0)
    vx = _nodal(mesh, lambda X, Y: X * X + X * Y)
    vy = _nodal(mesh, lambda X, Y: Y * Y)
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    for iy in range(3):
        for ix in range(4):
            e = iy * 4 + ix
            xc, yc = ix + 0.5, iy + 0.5
            np.testing.assert_allclose(E11[e], [2 * xc + yc, 2, 1, 0, 0, 0], atol=1e-12)
            np.testing.assert_allclose(E22[e], [2 * yc, 0, 2, 0, 0, 0], atol=1e-12)
            np.testing.assert_allclose(E12[e], [0.5 * xc, 0.5, 0, 0, 0, 0], atol=1e-12)


@pytest.mark.parametrize("ns,exact", [(8, True), (6, False)])
def test_strain_ns8_is_the_gradient_space_of_q2(ora, ns, exact):
    """R#24 (stress "in the gradient of the velocity space"): with n_S = 8 the DG strain of
    ANY CG2 velocity equals its symmetric gradient pointwise (the L2 projection onto a space that
    contains it); with n_S = 6 it does not (the S T^2, S^2 T parts are lost).  The pointwise
    gradient comes from independent Vandermonde Lagrange bases, the DG evaluation from sympy's
    family in R#24's order."""
    mesh = Mesh(3, 2, lx=3e3, ly=2.5e3, p=2, ns=ns, na=6)
    r = np.random.default_rng(11)
    vx = r.uniform(-0.2, 0.2, mesh.node_shape); vy = r.uniform(-0.2, 0.2, mesh.node_shape)
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    hx, hy = mesh.lx / mesh.nx, mesh.ly / mesh.ny
    L, dL = _lagrange_1d(2)
    fam = [lambda S, T: 1 + 0 * S, lambda S, T: S, lambda S, T: T, lambda S, T: S * S - 1 / 12,
           lambda S, T: T * T - 1 / 12, lambda S, T: S * T, lambda S, T: (S * S - 1 / 12) * T,
           lambda S, T: S * (T * T - 1 / 12)][:ns]
    worst = 0.0
    scale = 0.2 / min(hx, hy)
    for iy in range(mesh.ny):
        for ix in range(mesh.nx):
            e = iy * mesh.nx + ix
            ux = vx[2 * iy:2 * iy + 3, 2 * ix:2 * ix + 3]; uy = vy[2 * iy:2 * iy + 3, 2 * ix:2 * ix + 3]
            for (sv, tv) in r.uniform(0, 1, (5, 2)):
                Ls, Lt, dLs, dLt = L(sv), L(tv), dL(sv), dL(tv)
                g = ((Lt @ ux @ dLs) / hx, 0.5 * ((dLt @ ux @ Ls) / hy + (Lt @ uy @ dLs) / hx), (dLt @ uy @ Ls) / hy)
                psi = np.array([f(sv - 0.5, tv - 0.5) for f in fam])
                for Ec, gc in zip((E11, E12, E22), g):
                    worst = max(worst, abs(Ec[e] @ psi - gc) / scale)
    if exact:
        assert worst < 1e-13, worst
    else:
        assert worst > 1e-3, worst


# ---------------------------------------------------------------- stress
def _stress_inputs(mesh, seed=3):
    r = np.random.default_rng(seed)
    N, ns, na = mesh.n_elem, mesh.ns, mesh.na
    E = [r.uniform(-1e-6, 1e-6, (N, ns)) for _ in range(3)]
    H = r.uniform(-0.1, 0.1, (N, na)); H[:, 0] = r.uniform(0.2, 2.0, N)
    A = r.uniform(-0.1, 0.1, (N, na)); A[:, 0] = r.uniform(0.7, 1.05, N)
    S = [r.uniform(-1e4, 1e4, (N, ns)) for _ in range(3)]
    return E, H, A, S


@pytest.mark.parametrize("p,ns,na", [(1, 3, 3), (2, 6, 6), (2, 6, 1), (2, 8, 6)])
def test_stress_zero_thickness_decays_exactly(ora, p, ns, na):
    """SPEC S:317 / Listing 1: H = 0 -> P = 0 -> S <- (1 - 1/alpha) S exactly."""
    mesh = Mesh(3, 3, lx=3e3, ly=3e3, p=p, ns=ns, na=na)
    E, H, A, S = _stress_inputs(mesh)
    prm = Params(alpha=7.0)
    out = ora.stress(mesh, prm, *E, np.zeros_like(H), A, *S)
    fac = 1.0 - 1.0 / 7.0
    for o, s in zip(out, S):
        np.testing.assert_array_equal(o, fac * s)


def test_stress_rigid_ice_spec_example(ora):
    """E = 0, H = A = 1, alpha = 2 -> S11 = S11/2 + (-Pstar/4, 0, ...), S12 = S12/2."""
    mesh = Mesh(2, 2, lx=2.0, ly=2.0, p=1, ns=3, na=3)
    N = 4
    E = [np.zeros((N, 3))] * 3
    H = np.tile([1.0, 0, 0], (N, 1)); A = H.copy()
    S = [RNG.uniform(-1, 1, (N, 3)) for _ in range(3)]
    prm = Params(alpha=2.0, Pstar=27500.0)
    o11, o12, o22 = ora.stress(mesh, prm, *E, H, A, *S)
    add = np.array([-0.25 * 27500.0, 0, 0])
    np.testing.assert_allclose(o11, 0.5 * S[0] + add, rtol=1e-14, atol=1e-10)
    np.testing.assert_allclose(o22, 0.5 * S[2] + add, rtol=1e-14, atol=1e-10)
    np.testing.assert_allclose(o12, 0.5 * S[1], rtol=1e-14, atol=1e-12)


def test_stress_fixed_strain_geometric_contraction(ora):
    """SPEC S:332-336 / Eq. (3): with E, H, A fixed the map is affine with slope (1 - 1/alpha):
    successive increments shrink by exactly that ratio."""
    mesh = Mesh(3, 2, lx=3e3, ly=2e3)
    E, H, A, S = _stress_inputs(mesh)
    prm = Params(alpha=5.0)
    prev = S; incs = []
    for _ in range(6):
        nxt = ora.stress(mesh, prm, *E, H, A, *prev)
        incs.append(np.concatenate([(a - b).ravel() for a, b in zip(nxt, prev)]))
        prev = nxt
    for a, b in zip(incs[1:], incs[:-1]):
        np.testing.assert_allclose(a, 0.8 * b, rtol=1e-9, atol=1e-9 * np.abs(b).max())


def test_stress_component_symmetry(ora):
    """swapping E11 <-> E22 swaps S11 <-> S22 (with S11, S22 inputs swapped) and keeps S12."""
    mesh = Mesh(3, 3, lx=3e3, ly=3e3)
    E, H, A, S = _stress_inputs(mesh)
    prm = Params()
    a11, a12, a22 = ora.stress(mesh, prm, E[0], E[1], E[2], H, A, S[0], S[1], S[2])
    b11, b12, b22 = ora.stress(mesh, prm, E[2], E[1], E[0], H, A, S[2], S[1], S[0])
    np.testing.assert_array_equal(a11, b22)
    np.testing.assert_array_equal(a22, b11)
    np.testing.assert_array_equal(a12, b12)


def test_stress_linear_in_pstar(ora):
    """with S = 0, output is linear in Pstar."""
    mesh = Mesh(3, 3, lx=3e3, ly=3e3)
    E, H, A, _ = _stress_inputs(mesh)
    Z = [np.zeros_like(E[0])] * 3
    o1 = ora.stress(mesh, Params(Pstar=1000.0), *E, H, A, *Z)
    o2 = ora.stress(mesh, Params(Pstar=2000.0), *E, H, A, *Z)
    for a, b in zip(o1, o2):
        np.testing.assert_allclose(b, 2 * a, rtol=1e-14, atol=1e-14 * np.abs(b).max())


def test_stress_yield_ellipse(ora):
    """north_star pin: the VP stress lies on/inside Hibler's ellipse (e = 2):
    ((sI + P/2)/(P/2))^2 + (sII/(P/4))^2 = Draw^2 / (DeltaMin^2 + Draw^2) <= 1,
    -> 1 in the plastic limit.  alpha = 1 makes one update return the projection of
    sigma_vp; element-constant fields make it exact in the constant coefficient.
    Many random strain directions (an exchanged 5/8 <-> 3/8 or a wrong Delta weight fails)."""
    mesh = Mesh(8, 8, lx=8e3, ly=8e3, p=2, ns=6, na=6)
    N = mesh.n_elem
    r = np.random.default_rng(11)
    e11, e12, e22 = (r.normal(0, 1e-6, N) for _ in range(3))
    E = [np.zeros((N, 6)) for _ in range(3)]
    E[0][:, 0], E[1][:, 0], E[2][:, 0] = e11, e12, e22
    h = r.uniform(0.5, 2.0, N); a = r.uniform(0.8, 1.0, N)
    H = np.zeros((N, 6)); H[:, 0] = h
    A = np.zeros((N, 6)); A[:, 0] = a
    Z = [np.zeros((N, 6))] * 3
    for dmin, plastic in ((2e-9, False), (1e-15, True)):
        prm = Params(alpha=1.0, DeltaMin=dmin)
        s11, s12, s22 = (o[:, 0] for o in ora.stress(mesh, prm, *E, H, A, *Z))
        P = 27500.0 * h * np.exp(-20 * (1 - a))
        sI = 0.5 * (s11 + s22)
        sII = np.sqrt((0.5 * (s11 - s22)) ** 2 + s12**2)
        F = ((sI + P / 2) / (P / 2)) ** 2 + (sII / (P / 4)) ** 2
        draw2 = 1.25 * (e11**2 + e22**2) + 1.5 * e11 * e22 + e12**2
        np.testing.assert_allclose(F, draw2 / (dmin**2 + draw2), rtol=1e-12)
        assert (F <= 1 + 1e-12).all()
        if plastic:
            np.testing.assert_allclose(F, 1.0, rtol=1e-12)


def test_stress_pure_shear_plastic_strength(ora):
    """Textbook special case: pure shear in the plastic limit gives sigma12 = sign(e12) P/(2e) = P/4
    and sigma11 = sigma22 = -P/2."""
    mesh = Mesh(1, 1, lx=1.0, ly=1.0, p=1, ns=3, na=1)
    E = [np.zeros((1, 3)), np.array([[3e-7, 0, 0]]), np.zeros((1, 3))]
    H = np.array([[1.0]]); A = np.array([[1.0]])
    s11, s12, s22 = ora.stress(mesh, Params(alpha=1.0, DeltaMin=1e-16), *E, H, A, *[np.zeros((1, 3))] * 3)
    np.testing.assert_allclose([s11[0, 0], s12[0, 0], s22[0, 0]], [-13750.0, 6875.0, -13750.0], rtol=1e-12)


def test_stress_clamps(ora):
    """h = max(0, .), a = min(1, max(0, .)): A > 1 behaves as A = 1, H < 0 as H = 0."""
    mesh = Mesh(1, 1, lx=1.0, ly=1.0, p=1, ns=3, na=1)
    E = [np.array([[1e-7, 0, 0]]), np.zeros((1, 3)), np.zeros((1, 3))]
    Z = [np.zeros((1, 3))] * 3
    prm = Params(alpha=1.0)
    a = ora.stress(mesh, prm, *E, np.array([[1.0]]), np.array([[1.7]]), *Z)
    b = ora.stress(mesh, prm, *E, np.array([[1.0]]), np.array([[1.0]]), *Z)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    c = ora.stress(mesh, prm, *E, np.array([[-0.5]]), np.array([[1.0]]), *Z)
    for x in c:
        assert np.abs(x).max() == 0.0


# ---------------------------------------------------------------- divergence
@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_divergence_constant_stress_interior_zero(ora, p, ns):
    """north_star pin: zero divergence of a constant interior stress."""
    mesh = Mesh(5, 4, lx=5e3, ly=4e3, p=p, ns=ns, na=min(ns, 6))
    N = mesh.n_elem
    S = [np.zeros((N, ns)) for _ in range(3)]
    S[0][:, 0], S[1][:, 0], S[2][:, 0] = 1200.0, -300.0, 700.0
    Fx, Fy = ora.divergence(mesh, *S)
    assert np.abs(Fx[1:-1, 1:-1]).max() < 1e-9 and np.abs(Fy[1:-1, 1:-1]).max() < 1e-9
    assert np.abs(Fx[:, 0]).max() > 1.0  # boundary traction is not zero


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_divergence_linear_stress(ora, p, ns):
    """Linear sigma: F_j / m_j = div sigma exactly at interior nodes (lumped mass, exact quadrature).
    sigma11 = a x, sigma12 = b y, sigma22 = d y  ->  div sigma = (a + b, d)."""
    nx, ny, lx, ly = 5, 4, 5e3, 4e3
    mesh = Mesh(nx, ny, lx=lx, ly=ly, p=p, ns=ns, na=min(ns, 6))
    hx, hy = lx / nx, ly / ny
    a, b, d = 3.0, -2.0, 5.0
    S = [np.zeros((mesh.n_elem, ns)) for _ in range(3)]
    for iy in range(ny):
        for ix in range(nx):
            e = iy * nx + ix
            xc, yc = (ix + 0.5) * hx, (iy + 0.5) * hy
            S[0][e, :2] = [a * xc, a * hx]
            S[1][e, [0, 2]] = [b * yc, b * hy]
            S[2][e, [0, 2]] = [d * yc, d * hy]
    Fx, Fy = ora.divergence(mesh, *S)
    m = ora.lumped_mass(mesh)
    np.testing.assert_allclose((Fx / m)[1:-1, 1:-1], a + b, rtol=1e-10)
    np.testing.assert_allclose((Fy / m)[1:-1, 1:-1], d, rtol=1e-10)


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_divergence_strain_adjointness(ora, p, ns):
    """Identity of the weak forms: sum_j v_j . F_j = -sum_K int sigma : eps(v) = -sum_K |K| sum_k
    ||psi_k||^2 (S11 E11 + 2 S12 E12 + S22 E22)_k (sigma in the DG space, exact quadrature).
    A sign or transposition error in either the strain or the divergence breaks it."""
    mesh = Mesh(4, 3, lx=4e3, ly=3e3, p=p, ns=ns, na=min(ns, 6))
    vx = RNG.uniform(-1, 1, mesh.node_shape); vy = RNG.uniform(-1, 1, mesh.node_shape)
    S = [RNG.uniform(-1, 1, (mesh.n_elem, ns)) for _ in range(3)]
    E11, E12, E22 = ora.strain(mesh, vx, vy)
    Fx, Fy = ora.divergence(mesh, *S)
    lhs = (vx * Fx + vy * Fy).sum()
    norm = np.array([1, 1 / 12, 1 / 12, 1 / 180, 1 / 180, 1 / 144, 1 / 2160, 1 / 2160])[:ns]
    K = 1e6
    rhs = -K * ((S[0] * E11 + 2 * S[1] * E12 + S[2] * E22) * norm).sum()
    assert abs(lhs - rhs) < 1e-12 * max(abs(lhs), 1.0) * 10


def test_divergence_brute_force(ora):
    """Brute force (tiny mesh): F = -int sigma . grad phi with an 8-point numpy rule and
    Vandermonde Lagrange bases, assembled by scatter over elements."""
    p, ns = 2, 6
    mesh = Mesh(3, 2, lx=3e3, ly=2.5e3, p=p, ns=ns, na=min(ns, 6))
    hx, hy = 1e3, 1.25e3
    S = [RNG.uniform(-1, 1, (mesh.n_elem, ns)) for _ in range(3)]
    xi, wi = np.polynomial.legendre.leggauss(8)
    q, w = 0.5 * (xi + 1), 0.5 * wi
    L, dL = _lagrange_1d(p)
    Fx = np.zeros(mesh.node_shape); Fy = np.zeros(mesh.node_shape)
    for iy in range(2):
        for ix in range(3):
            e = iy * 3 + ix
            for a in range(8):
                for b in range(8):
                    s, t = q[a], q[b]
                    Sg, Tg = s - 0.5, t - 0.5
                    psi = np.array([1, Sg, Tg, Sg * Sg - 1 / 12, Tg * Tg - 1 / 12, Sg * Tg])
                    s11, s12, s22 = (x[e] @ psi for x in S)
                    gx = np.outer(L(t), dL(s)) / hx   # [jy, jx]
                    gy = np.outer(dL(t), L(s)) / hy
                    W = w[a] * w[b] * hx * hy
                    Fx[2 * iy:2 * iy + 3, 2 * ix:2 * ix + 3] -= W * (s11 * gx + s12 * gy)
                    Fy[2 * iy:2 * iy + 3, 2 * ix:2 * ix + 3] -= W * (s12 * gx + s22 * gy)
    gx_, gy_ = ora.divergence(mesh, *S)
    np.testing.assert_allclose(gx_, Fx, atol=1e-12 * np.abs(Fx).max())
    np.testing.assert_allclose(gy_, Fy, atol=1e-12 * np.abs(Fy).max())


# ---------------------------------------------------------------- prep
def test_prep_nodal_mean_and_floors(ora):
    """R#17: nodal mean of a continuous (linear) DG field is its exact nodal value;
    A clamped to [0,1]; H floored at 1e-4."""
    nx, ny, lx, ly = 4, 3, 4e3, 3e3
    mesh = Mesh(nx, ny, lx=lx, ly=ly)
    hx, hy = lx / nx, ly / ny
    H = np.zeros((mesh.n_elem, 6)); A = np.zeros((mesh.n_elem, 6))
    for iy in range(ny):
        for ix in range(nx):
            e = iy * nx + ix
            xc, yc = (ix + 0.5) * hx, (iy + 0.5) * hy
            H[e, :3] = [1 + 1e-4 * xc, 1e-4 * hx, 0]           # H = 1 + 1e-4 x
            A[e, :3] = [0.5 + 1e-4 * yc, 0, 1e-4 * hy]         # A = 0.5 + 1e-4 y (exceeds 1 near the top)
    Hn, An = ora.prep(mesh, H, A)
    X = _nodal(mesh, lambda X, Y: X); Y = _nodal(mesh, lambda X, Y: Y)
    np.testing.assert_allclose(Hn, 1 + 1e-4 * X, rtol=1e-14)
    np.testing.assert_allclose(An, np.minimum(0.5 + 1e-4 * Y, 1.0), rtol=1e-14)
    Hn0, _ = ora.prep(mesh, -H, A)
    assert (Hn0 == 1e-4).all()


# ---------------------------------------------------------------- velocity
def _free_drift_fixed_point(prm, Hn, An, vn, o, a):
    """Implicit-Euler free drift (Eq. 2 with sigma = 0), solved per node with scipy:
    rho H (v - v^n)/dt = A Fa |a| a + A Fo |o - v| (o - v) + rho H f (v - o) x k."""
    from scipy.optimize import fsolve
    Fa, Fo = prm.rho_atm * prm.C_atm, prm.rho_ocean * prm.C_ocean
    m = prm.rho_ice * Hn

    def res(v):
        d = o - v
        w = np.hypot(*d)
        cor = m * prm.f_c * np.array([v[1] - o[1], o[0] - v[0]])
        return m * (v - vn) / prm.dt - An * Fa * np.hypot(*a) * a - An * Fo * w * d - cor

    return fsolve(res, vn, xtol=1e-14)


def test_velocity_free_drift_fixed_point(ora):
    """O8 with S = 0: iterating the mEVP velocity update converges to the implicit-Euler
    free-drift solution; boundary nodes are exactly 0 (R#16)."""
    mesh = Mesh(3, 3, lx=3e4, ly=3e4, p=2, ns=6, na=6)
    shp = mesh.node_shape
    r = np.random.default_rng(5)
    Hn = r.uniform(0.5, 2, shp); An = r.uniform(0.5, 1, shp)
    vnx, vny = r.uniform(-0.1, 0.1, shp), r.uniform(-0.1, 0.1, shp)
    ox, oy = r.uniform(-0.05, 0.05, shp), r.uniform(-0.05, 0.05, shp)
    ax, ay = r.uniform(-15, 15, shp), r.uniform(-15, 15, shp)
    prm = Params(beta=10.0)
    Z = np.zeros(shp); one = np.ones(shp)
    vx, vy = vnx.copy(), vny.copy()
    for _ in range(2000):
        vx, vy = ora.velocity(mesh, prm, Z, Z, one, Hn, An, vnx, vny, ox, oy, ax, ay, vx, vy)
    assert (vx[0] == 0).all() and (vy[:, -1] == 0).all()
    for J in range(1, shp[0] - 1):
        for I in range(1, shp[1] - 1):
            ref = _free_drift_fixed_point(prm, Hn[J, I], An[J, I], np.array([vnx[J, I], vny[J, I]]),
                                          np.array([ox[J, I], oy[J, I]]), np.array([ax[J, I], ay[J, I]]))
            np.testing.assert_allclose([vx[J, I], vy[J, I]], ref, rtol=1e-10, atol=1e-13)


def test_velocity_quadratic_drag_closed_form(ora):
    """Special case f = 0, o = 0, 1D wind, v^n = 0: fixed point solves
    c v + A Fo v^2 = A Fa a^2  ->  v = (-c + sqrt(c^2 + 4 A Fo A Fa a^2)) / (2 A Fo)."""
    mesh = Mesh(2, 2, lx=2e4, ly=2e4, p=1, ns=3, na=3)
    shp = mesh.node_shape
    prm = Params(f_c=0.0, beta=5.0)
    Hn = np.full(shp, 1.3); An = np.full(shp, 0.9)
    ax = np.full(shp, 12.0); Z = np.zeros(shp); one = np.ones(shp)
    vx, vy = Z.copy(), Z.copy()
    for _ in range(3000):
        vx, vy = ora.velocity(mesh, prm, Z, Z, one, Hn, An, Z, Z, Z, Z, ax, Z, vx, vy)
    c = prm.rho_ice * 1.3 / prm.dt
    k = 0.9 * prm.rho_ocean * prm.C_ocean
    rhs = 0.9 * prm.rho_atm * prm.C_atm * 144.0
    v = (-c + math.sqrt(c * c + 4 * k * rhs)) / (2 * k)
    assert abs(vx[1, 1] - v) < 1e-12 * v and vy[1, 1] == 0.0


def test_velocity_stress_force_balance(ora):
    """With drag and Coriolis off and v^(p-1) = v^n, one update gives
    v = v^n + F/(m c (1+beta)), i.e. the relaxed momentum step rho H dv/dt = div sigma."""
    mesh = Mesh(2, 2, lx=2e4, ly=2e4, p=2, ns=6, na=6)
    shp = mesh.node_shape
    prm = Params(f_c=0.0, rho_atm=0.0, rho_ocean=0.0, beta=3.0)
    r = np.random.default_rng(9)
    Fx, Fy, mass = r.normal(size=shp), r.normal(size=shp), r.uniform(1, 2, shp)
    Hn = np.full(shp, 2.0); Z = np.zeros(shp)
    vn = r.normal(size=shp) * 0.1
    vx, vy = ora.velocity(mesh, prm, Fx, Fy, mass, Hn, Z + 1, vn, vn, Z, Z, Z, Z, vn.copy(), vn.copy())
    c = 900 * 2.0 / 120.0
    np.testing.assert_allclose(vx[1:-1, 1:-1], (vn + Fx / mass / (c * 4.0))[1:-1, 1:-1], rtol=1e-14)
    np.testing.assert_allclose(vy[1:-1, 1:-1], (vn + Fy / mass / (c * 4.0))[1:-1, 1:-1], rtol=1e-14)


# ---------------------------------------------------------------- advection
def _periodic_velocity(mesh, r):
    v = r.uniform(-0.1, 0.1, mesh.node_shape)
    v[-1, :] = v[0, :]; v[:, -1] = v[:, 0]
    return v


@pytest.mark.parametrize("p,ns,na", [(1, 3, 1), (1, 3, 3), (2, 6, 6), (2, 6, 3)])
def test_advection_periodic_mass_conservation(ora, p, ns, na):
    """north_star pin: sum_K |K| c_0 conserved under periodic boundaries (any v, any c)."""
    mesh = Mesh(5, 4, lx=5e3, ly=4e3, p=p, ns=ns, na=na, bc=1)
    r = np.random.default_rng(13)
    vx, vy = _periodic_velocity(mesh, r), _periodic_velocity(mesh, r)
    A = r.uniform(0, 1, (mesh.n_elem, na)); H = r.uniform(0, 2, (mesh.n_elem, na))
    A2, H2 = ora.advect(mesh, 500.0, vx, vy, A, H)
    assert abs(A2[:, 0].sum() - A[:, 0].sum()) < 1e-13 * A[:, 0].sum()
    assert abs(H2[:, 0].sum() - H[:, 0].sum()) < 1e-13 * H[:, 0].sum()
    assert np.abs(A2 - A).max() > 1e-6  # it did move


def test_advection_dg0_is_first_order_upwind(ora):
    """Textbook reduction: DG0 with uniform velocity (U, V) > 0 on a periodic mesh is
    first-order upwind finite volumes: dc/dt = -U (c_i - c_{i-1})/hx - V (c_j - c_{j-1})/hy."""
    nx, ny, lx, ly = 6, 5, 6e3, 5e3
    mesh = Mesh(nx, ny, lx=lx, ly=ly, p=1, ns=3, na=1, bc=1)
    U, V = 0.07, 0.03
    vx = np.full(mesh.node_shape, U); vy = np.full(mesh.node_shape, V)
    c = np.random.default_rng(2).uniform(0, 1, (ny, nx))
    rhs = ora.advect_rhs(mesh, vx, vy, c.reshape(-1, 1)).reshape(ny, nx)
    ref = -U * (c - np.roll(c, 1, axis=1)) / (lx / nx) - V * (c - np.roll(c, 1, axis=0)) / (ly / ny)
    np.testing.assert_allclose(rhs, ref, rtol=1e-12, atol=1e-18)
    # negative velocity takes the other neighbour
    rhs2 = ora.advect_rhs(mesh, -vx, -vy, c.reshape(-1, 1)).reshape(ny, nx)
    ref2 = U * (np.roll(c, -1, axis=1) - c) / (lx / nx) + V * (np.roll(c, -1, axis=0) - c) / (ly / ny)
    np.testing.assert_allclose(rhs2, ref2, rtol=1e-12, atol=1e-18)


@pytest.mark.parametrize("p,ns,na", [(1, 3, 3), (2, 6, 6)])
def test_advection_constant_preserved_by_rotation(ora, p, ns, na):
    """A constant tracer is a steady state of a divergence-free (rigid rotation) flow at every
    interior element (edge quadrature is exact for these degrees)."""
    nx, ny, lx, ly = 6, 6, 6e3, 6e3
    mesh = Mesh(nx, ny, lx=lx, ly=ly, p=p, ns=ns, na=na)
    om = 1e-5
    vx = _nodal(mesh, lambda X, Y: -om * (Y - 3e3)); vy = _nodal(mesh, lambda X, Y: om * (X - 3e3))
    c = np.zeros((mesh.n_elem, na)); c[:, 0] = 0.8
    rhs = ora.advect_rhs(mesh, vx, vy, c).reshape(ny, nx, na)
    assert np.abs(rhs[1:-1, 1:-1]).max() < 1e-18


@pytest.mark.parametrize("p,ns,na", [(1, 3, 3), (2, 6, 6)])
def test_advection_linear_profile_uniform_flow(ora, p, ns, na):
    """c = c0 + b x advected by uniform U: dc/dt = -U b exactly (c0 coefficient), 0 for the rest,
    at every element whose upwind neighbour exists (interior)."""
    nx, ny, lx, ly = 6, 5, 6e3, 5e3
    mesh = Mesh(nx, ny, lx=lx, ly=ly, p=p, ns=ns, na=na)
    U, b = 0.1, 2e-4
    hx = lx / nx
    vx = np.full(mesh.node_shape, U); vy = np.zeros(mesh.node_shape)
    c = np.zeros((mesh.n_elem, na))
    for iy in range(ny):
        for ix in range(nx):
            c[iy * nx + ix, :2] = [0.3 + b * (ix + 0.5) * hx, b * hx]
    rhs = ora.advect_rhs(mesh, vx, vy, c).reshape(ny, nx, na)
    np.testing.assert_allclose(rhs[:, 1:-1, 0], -U * b, rtol=1e-11)
    assert np.abs(rhs[:, 1:-1, 1:]).max() < 1e-16


@pytest.mark.parametrize("na,order", [(1, 1), (3, 2), (6, 3)])
def test_advection_rk_is_taylor_polynomial(ora, na, order):
    """The operator is linear, so Euler / SSP-RK2 / SSP-RK3 equal the Taylor polynomial of
    exp(dt L) of order 1 / 2 / 3 (pins the RK weights)."""
    p, ns = (1, 3) if na != 6 else (2, 6)
    mesh = Mesh(4, 4, lx=4e3, ly=4e3, p=p, ns=ns, na=na, bc=1)
    r = np.random.default_rng(21)
    vx, vy = _periodic_velocity(mesh, r), _periodic_velocity(mesh, r)
    c = r.uniform(0, 1, (mesh.n_elem, na))
    dt = 800.0
    terms = [c]; acc = c.copy()
    for k in range(1, order + 1):
        terms.append(ora.advect_rhs(mesh, vx, vy, terms[-1]) * dt / k)
        acc = acc + terms[-1]
    A2, _ = ora.advect(mesh, dt, vx, vy, c, c)
    np.testing.assert_allclose(A2, acc, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- composition
def test_subcycle_is_composition_of_steps(ora):
    """O9: one subcycle = strain -> stress -> divergence -> velocity (paper order)."""
    mesh = Mesh(6, 5, lx=6e4, ly=5e4, p=2, ns=6, na=6)
    st = inputs.make_case(6, 5, 2, 6, 6, kind="random", lx=6e4, ly=5e4)
    prm = Params()
    out = ora.subcycles(mesh, prm, 1, st)
    E = ora.strain(mesh, st["vx"], st["vy"])
    S = ora.stress(mesh, prm, *E, st["H"], st["A"], st["S11"], st["S12"], st["S22"])
    F = ora.divergence(mesh, *S)
    Hn, An = ora.prep(mesh, st["H"], st["A"])
    m = ora.lumped_mass(mesh)
    v = ora.velocity(mesh, prm, *F, m, Hn, An, st["vx"], st["vy"], st["ox"], st["oy"], st["ax"], st["ay"],
                     st["vx"], st["vy"])
    for k, ref in zip(("S11", "S12", "S22", "vx", "vy"), (*S, *v)):
        np.testing.assert_array_equal(out[k], ref)


def test_oracle_threads_deterministic(ora):
    """OpenMP only over independent loops: 1 thread and all threads agree bitwise."""
    mesh = Mesh(8, 7, lx=8e4, ly=7e4)
    st = inputs.make_case(8, 7, 2, 6, 6, lx=8e4, ly=7e4)
    prm = Params()
    n0 = ora.threads
    a = ora.outer_step(mesh, prm, 3, st)
    ora.L.ora_set_threads(1)
    try:
        b = ora.outer_step(mesh, prm, 3, st)
    finally:
        ora.L.ora_set_threads(n0)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])


# ---------------------------------------------------------------- general (distorted) quads, R#23
def _dmesh(nx=5, ny=4, lx=5e3, ly=4e3, delta=0.25, p=2, ns=6, na=6, seed=31):
    V = inputs.distorted_vertices(nx, ny, lx, ly, delta, seed)
    return Mesh(nx, ny, lx=lx, ly=ly, p=p, ns=ns, na=na, verts=V), V


def test_distorted_element_area_is_shoelace(ora):
    """The Gauss integral of |J| over a bilinear quad equals its polygon (shoelace) area; the
    total equals the box area (boundary vertices fixed)."""
    mesh, V = _dmesh()
    x, w = ora.gauss(3)
    tot = 0.0
    for iy in range(mesh.ny):
        for ix in range(mesh.nx):
            area = sum(w[a] * w[b] * ora.jacobian(mesh, ix, iy, x[a], x[b])[0] for a in range(3) for b in range(3))
            q = [V[iy, ix], V[iy, ix + 1], V[iy + 1, ix + 1], V[iy + 1, ix]]
            shoe = 0.5 * sum(q[i][0] * q[(i + 1) % 4][1] - q[(i + 1) % 4][0] * q[i][1] for i in range(4))
            assert abs(area - shoe) < 1e-9 * shoe and area > 0
            tot += area
    assert abs(tot - mesh.lx * mesh.ly) < 1e-9 * mesh.lx * mesh.ly


def test_distorted_stress_rigid_constant(ora):
    """SPEC S:318 on distorted elements: the projection of a constant is exact for any element
    mass matrix, so E = 0, H = A = 1, alpha = 2 gives S11 = S11/2 + (-Pstar/4, 0, ...)."""
    mesh, _ = _dmesh(p=1, ns=3, na=3)
    N = mesh.n_elem
    E = [np.zeros((N, 3))] * 3
    H = np.tile([1.0, 0, 0], (N, 1)); A = H.copy()
    S = [RNG.uniform(-1, 1, (N, 3)) for _ in range(3)]
    o11, o12, o22 = ora.stress(mesh, Params(alpha=2.0), *E, H, A, *S)
    add = np.array([-0.25 * 27500.0, 0, 0])
    np.testing.assert_allclose(o11, 0.5 * S[0] + add, rtol=1e-13, atol=1e-9)
    np.testing.assert_allclose(o12, 0.5 * S[1], rtol=1e-13, atol=1e-12)


def _node_xy(mesh, V):
    """Physical positions of the CG nodes: the bilinear map of their reference positions."""
    p = mesh.p
    X = np.zeros(mesh.node_shape); Y = np.zeros(mesh.node_shape)
    for iy in range(mesh.ny):
        for ix in range(mesh.nx):
            q = V[iy:iy + 2, ix:ix + 2]
            for jy in range(p + 1):
                for jx in range(p + 1):
                    s, t = jx / p, jy / p
                    pt = (1 - s) * (1 - t) * q[0, 0] + s * (1 - t) * q[0, 1] + (1 - s) * t * q[1, 0] + s * t * q[1, 1]
                    X[p * iy + jy, p * ix + jx], Y[p * iy + jy, p * ix + jx] = pt
    return X, Y


@pytest.mark.parametrize("p,ns", [(1, 3), (2, 6), (2, 8)])
def test_distorted_strain_linear_velocity(ora, p, ns):
    """A physically linear velocity is reproduced by the (sub)parametric CG space on a bilinear
    mesh, so E = sym(G) in the constant coefficient and 0 elsewhere."""
    mesh, V = _dmesh(p=p, ns=ns, na=min(ns, 6))
    X, Y = _node_xy(mesh, V)
    G = np.array([[3e-6, -7e-6], [5e-6, -2e-6]])
    E11, E12, E22 = ora.strain(mesh, 0.1 + G[0, 0] * X + G[0, 1] * Y, -0.05 + G[1, 0] * X + G[1, 1] * Y)
    tol = 1e-11 * 1e-5
    for E, val in ((E11, G[0, 0]), (E22, G[1, 1]), (E12, 0.5 * (G[0, 1] + G[1, 0]))):
        np.testing.assert_allclose(E[:, 0], val, atol=tol)
        assert np.abs(E[:, 1:]).max() < tol


def test_distorted_stress_scale_invariance(ora):
    """iMJwPSI = M_K^{-1} [w |J| psi] is invariant under a uniform scaling of the element
    (|J| cancels): scaling every vertex by 3 leaves the stress update unchanged."""
    mesh, V = _dmesh()
    E, H, A, S = _stress_inputs(mesh)
    a = ora.stress(mesh, Params(), *E, H, A, *S)
    big = Mesh(mesh.nx, mesh.ny, lx=3 * mesh.lx, ly=3 * mesh.ly, verts=3.0 * V)
    b = ora.stress(big, Params(), *E, H, A, *S)
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y, rtol=1e-12, atol=1e-12 * np.abs(x).max())


# ---------------------------------------------------------------- NEXT-4: bound-preserving limiter (R#25)
_FAM6 = [lambda S, T: 1 + 0 * S, lambda S, T: S, lambda S, T: T, lambda S, T: S * S - 1 / 12,
         lambda S, T: T * T - 1 / 12, lambda S, T: S * T]


def _check_points(ngp=3):
    x, _ = np.polynomial.legendre.leggauss(ngp)
    q = 0.5 * (x + 1)
    pts = [(a, b) for b in q for a in q]
    pts += [(1.0, b) for b in q] + [(0.0, b) for b in q] + [(a, 1.0) for a in q] + [(a, 0.0) for a in q]
    return pts


def _eval6(c, s, t):
    return sum(c[k] * f(s - 0.5, t - 0.5) for k, f in enumerate(_FAM6))


def _phys_mean(c, X, Y):
    """|J|-weighted mean of the DG2 polynomial over a bilinear element (independent 6-point rule)."""
    xi, wi = np.polynomial.legendre.leggauss(6)
    q, w = 0.5 * (xi + 1), 0.5 * wi
    num = den = 0.0
    for a in range(6):
        for b in range(6):
            s, t = q[a], q[b]
            xs = (X[1] - X[0]) * (1 - t) + (X[3] - X[2]) * t; xt = (X[2] - X[0]) * (1 - s) + (X[3] - X[1]) * s
            ys = (Y[1] - Y[0]) * (1 - t) + (Y[3] - Y[2]) * t; yt = (Y[2] - Y[0]) * (1 - s) + (Y[3] - Y[1]) * s
            dj = xs * yt - xt * ys
            num += w[a] * w[b] * dj * _eval6(c, s, t); den += w[a] * w[b] * dj
    return num / den


def test_limiter_closed_form(ora):
    """R#25, Zhang-Shu: c = 0.9 + 0.4 S on a box element peaks at the east edge (S = 1/2) at 1.1, so
    theta = (1 - 0.9) / (1.1 - 0.9) = 1/2 and the slope halves; the mean stays; no upper bound -> unchanged."""
    mesh = Mesh(1, 1, lx=1.0, ly=1.0, p=2, ns=6, na=6)
    c = np.array([[0.9, 0.4, 0.0, 0.0, 0.0, 0.0]])
    np.testing.assert_allclose(ora.limit(mesh, c, 0.0, 1.0), [[0.9, 0.2, 0, 0, 0, 0]], atol=1e-15)
    np.testing.assert_array_equal(ora.limit(mesh, c, 0.0), c)
    # mean below the lower bound cannot be fixed: theta = 0 leaves the mean alone
    c2 = np.array([[-0.1, 0.3, 0.1, 0.0, 0.02, 0.0]])
    np.testing.assert_allclose(ora.limit(mesh, c2, 0.0, 1.0), [[-0.1, 0, 0, 0, 0, 0]], atol=1e-15)


@pytest.mark.parametrize("distorted", [False, True])
def test_limiter_keeps_mean_and_bounds(ora, distorted):
    """Random DG2 data: after limiting, the |J|-weighted element mean is unchanged (independent
    6-point integration of the bilinear map) and the values at every check point (volume and edge
    Gauss points) lie in [0, 1]; elements already inside the bounds are untouched."""
    nx, ny, lx, ly = 7, 5, 7e3, 5e3
    V = inputs.distorted_vertices(nx, ny, lx, ly, 0.28) if distorted else None
    mesh = Mesh(nx, ny, lx=lx, ly=ly, p=2, ns=6, na=6, verts=V)
    r = np.random.default_rng(13)
    c = np.zeros((nx * ny, 6))
    c[:, 0] = r.uniform(0.05, 0.95, nx * ny)
    c[:, 1:] = r.uniform(-0.6, 0.6, (nx * ny, 5))
    c[::3, 1:] *= 1e-3                        # some elements well inside the bounds
    out = ora.limit(mesh, c, 0.0, 1.0)
    pts = _check_points()
    hx, hy = lx / nx, ly / ny
    for e in range(nx * ny):
        ix, iy = e % nx, e // nx
        if V is not None:
            X = [V[iy + b, ix + a, 0] for b in (0, 1) for a in (0, 1)]; Y = [V[iy + b, ix + a, 1] for b in (0, 1) for a in (0, 1)]
        else:
            X = [(ix + a) * hx for b in (0, 1) for a in (0, 1)]; Y = [(iy + b) * hy for b in (0, 1) for a in (0, 1)]
        assert abs(_phys_mean(out[e], X, Y) - _phys_mean(c[e], X, Y)) < 1e-14
        vals = [_eval6(out[e], s, t) for s, t in pts]
        assert min(vals) >= -1e-14 and max(vals) <= 1 + 1e-14
        if min(_eval6(c[e], s, t) for s, t in pts) >= 0 and max(_eval6(c[e], s, t) for s, t in pts) <= 1:
            np.testing.assert_array_equal(out[e], c[e])


def test_limited_advection_bounds_and_mass(ora):
    """A discontinuous concentration (1 inside a disc, 0.5 outside, L2-projected into DG2 and limited)
    in a uniform periodic flow within Zhang-Shu's CFL bound: the unlimited SSP-RK3 step overshoots 1
    at the check points, the limited one stays in [0, 1] and conserves the total mass exactly
    (periodic box, the limiter keeps element means)."""
    nx = ny = 24
    lx = ly = 24e3
    mesh = Mesh(nx, ny, lx=lx, ly=ly, p=2, ns=6, na=6, bc=1)
    xi, wi = np.polynomial.legendre.leggauss(5)
    q, w = 0.5 * (xi + 1), 0.5 * wi
    norm = np.array([1, 1 / 12, 1 / 12, 1 / 180, 1 / 180, 1 / 144])
    A = np.zeros((nx * ny, 6))
    for e in range(nx * ny):
        ix, iy = e % nx, e // nx
        for a in range(5):
            for b in range(5):
                x, y = (ix + q[a]) * 1e3, (iy + q[b]) * 1e3
                f = 1.0 if (x - 12e3) ** 2 + (y - 12e3) ** 2 < (5e3) ** 2 else 0.5
                for k, g in enumerate(_FAM6):
                    A[e, k] += w[a] * w[b] * f * g(q[a] - 0.5, q[b] - 0.5) / norm[k]
    A = ora.limit(mesh, A, 0.0, 1.0)          # bounded initial state (the projection's Gibbs overshoot removed)
    H = A.copy()
    shp = mesh.node_shape
    vx, vy = np.full(shp, 0.3), np.full(shp, 0.2)
    dt = 200.0                                # (|u|/hx + |v|/hy) dt = 0.1 <= 1/6: Zhang-Shu's CFL for DG2
    pts = _check_points()
    ev = lambda C: np.array([[_eval6(C[e], s, t) for s, t in pts] for e in range(nx * ny)])
    Au, _ = ora.advect(mesh, dt, vx, vy, A, H)
    Al, Hl = ora.advect_limited(mesh, dt, vx, vy, A, H, 1)
    assert ev(Au).max() > 1 + 1e-3
    vl = ev(Al)
    assert vl.max() <= 1 + 1e-13 and vl.min() >= -1e-13
    assert abs(Al[:, 0].sum() - A[:, 0].sum()) <= 1e-13 * A[:, 0].sum()
    assert ev(Hl).min() >= -1e-13 and abs(Hl[:, 0].sum() - H[:, 0].sum()) <= 1e-13 * H[:, 0].sum()
