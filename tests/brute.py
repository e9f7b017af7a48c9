"""Independent brute-force evaluation of the discretisation on tiny meshes (test infrastructure).

Used by ``tests/test_oracle_brute.py`` to pin the oracle (``-m "not gpu"``).  It shares nothing with
``oracle/oracle.c`` except the readings it implements, and it is built from other
pieces on purpose, so that a slip in the oracle's own building blocks cannot cancel out:

- quadrature: numpy's Gauss-Legendre nodes (``leggauss``), with a high-order rule (8 points) wherever
  the integrand is a polynomial the rule integrates exactly, and the method's own rule (ngp of
  Listing 2) only where the method defines the result through it (the stress projection of
  Listing 2, the advection volume and edge integrals, R#18);
- bases: CG Lagrange polynomials from a Vandermonde solve; the DG family (R#5, R#24) and its
  gradient from sympy (symbolic differentiation, not hand-written derivatives);
- geometry: the bilinear map written out from the vertex array, gradients through the adjugate
  (|J| J^-T, so every weak form is polynomial), edge normals x length from the straight edge's end
  vertices (no tangent evaluation, no normalisation);
- sphere (R#26): the lon-lat element's metric written from the spherical line element
  ds^2 = R^2 cos^2(lat) dlon^2 + R^2 dlat^2 (|J| = R^2 cos(lat) dlon dlat, adjugate diag(R dlat,
  R cos(lat) dlon)), the frame's metric term tan(lat)/R, edge normals x length from the edge's arc
  lengths; every integral with the method's rule (the integrands are not polynomials);
- operators: global matrices assembled by scatter over elements (strain G, divergence D),
  the nodal mean of the DG->CG prep by scatter-and-count, the velocity update in vector form
  with the Coriolis term as the rotation (v - o) x k.

Only tiny meshes (a few dozen elements): everything is plain Python loops.
"""
from __future__ import annotations

import numpy as np
import sympy as sp

# ------------------------------------------------------------------ bases
_s, _t = sp.symbols("s t")
_S, _T = _s - sp.Rational(1, 2), _t - sp.Rational(1, 2)
_FAM = [sp.Integer(1), _S, _T, _S**2 - sp.Rational(1, 12), _T**2 - sp.Rational(1, 12), _S * _T,
        (_S**2 - sp.Rational(1, 12)) * _T, _S * (_T**2 - sp.Rational(1, 12))]   # R#5 / R#24 order
_PSI = sp.lambdify((_s, _t), _FAM, "numpy")
_DPSI_S = sp.lambdify((_s, _t), [sp.diff(f, _s) for f in _FAM], "numpy")
_DPSI_T = sp.lambdify((_s, _t), [sp.diff(f, _t) for f in _FAM], "numpy")


def psi(n, s, t):
    return np.array([float(v) for v in _PSI(s, t)[:n]])


def dpsi(n, s, t):
    return (np.array([float(v) for v in _DPSI_S(s, t)[:n]]),
            np.array([float(v) for v in _DPSI_T(s, t)[:n]]))


def lagrange(p):
    """1D Lagrange basis on p+1 equispaced nodes of [0, 1] via a Vandermonde inverse: (L(s), dL(s))."""
    nodes = np.linspace(0.0, 1.0, p + 1)
    Cf = np.linalg.inv(np.vander(nodes, p + 1, increasing=True))
    P = np.polynomial.polynomial
    L = lambda s: np.array([P.polyval(s, Cf[:, j]) for j in range(p + 1)])
    dL = lambda s: np.array([P.polyval(s, P.polyder(Cf[:, j])) for j in range(p + 1)])
    return L, dL


def gauss(k):
    x, w = np.polynomial.legendre.leggauss(k)
    return 0.5 * (x + 1.0), 0.5 * w


def ngp_of(ns):
    return {3: 2, 6: 3, 8: 3}[ns]


# ------------------------------------------------------------------ mesh
class BMesh:
    """nx x ny quads; ``verts`` (ny+1, nx+1, 2) or None for the box; radius > 0: lon-lat mesh on the
    sphere (lx, ly angular extents [rad], lat0 the southern edge)."""

    def __init__(self, nx, ny, lx, ly, p, ns, na, bc=0, verts=None, radius=0.0, lat0=0.0):
        self.nx, self.ny, self.lx, self.ly, self.p, self.ns, self.na, self.bc = nx, ny, lx, ly, p, ns, na, bc
        self.radius, self.lat0 = radius, lat0
        self.sphere = radius > 0
        # the quadrature of integrals the method evaluates exactly on plane meshes (8 points: exact for
        # the polynomial integrands) or, on the sphere, with its own rule
        self.kq = ngp_of(ns) if self.sphere else 8
        if verts is None:
            X, Y = np.meshgrid(np.arange(nx + 1) * (lx / nx), np.arange(ny + 1) * (ly / ny))
            verts = np.stack([X, Y], axis=-1)
        self.V = np.asarray(verts, dtype=np.float64)
        self.NX, self.NY = p * nx + 1, p * ny + 1
        self.L, self.dL = lagrange(p)

    @property
    def ne(self):
        return self.nx * self.ny

    @property
    def nn(self):
        return self.NX * self.NY

    def corners(self, ix, iy):
        """q[b][a] = vertex (ix + a, iy + b) relative to vertex (ix, iy)."""
        q = self.V[iy:iy + 2, ix:ix + 2].copy()
        return q - q[0, 0]

    def lat(self, iy, t):
        return self.lat0 + (iy + t) * self.ly / self.ny

    def kt(self, iy, t):
        """metric term tan(lat) / R of the sphere's orthonormal frame (0 on plane meshes)"""
        return np.tan(self.lat(iy, t)) / self.radius if self.sphere else 0.0

    def jac(self, ix, iy, s, t):
        """(|J|, adj) with adj = |J| J^-T, so grad f = adj @ (f_s, f_t) / |J|."""
        if self.sphere:
            R, dl, dp = self.radius, self.lx / self.nx, self.ly / self.ny
            c = np.cos(self.lat(iy, t))
            return R * R * c * dl * dp, np.array([[R * dp, 0.0], [0.0, R * c * dl]])
        q = self.corners(ix, iy)
        xs = (1 - t) * (q[0, 1] - q[0, 0]) + t * (q[1, 1] - q[1, 0])      # d(x, y)/ds
        xt = (1 - s) * (q[1, 0] - q[0, 0]) + s * (q[1, 1] - q[0, 1])      # d(x, y)/dt
        det = xs[0] * xt[1] - xt[0] * xs[1]
        adj = np.array([[xt[1], -xs[1]], [-xt[0], xs[0]]])
        return det, adj

    def node(self, ix, iy, jx, jy):
        """Flat global node index of local node (jx, jy) of element (ix, iy)."""
        return (self.p * iy + jy) * self.NX + self.p * ix + jx

    def cg(self, s, t):
        """phi[jy, jx], dphi/ds, dphi/dt at (s, t)."""
        Ls, Lt, dLs, dLt = self.L(s), self.L(t), self.dL(s), self.dL(t)
        return np.outer(Lt, Ls), np.outer(Lt, dLs), np.outer(dLt, Ls)

    def on_boundary(self, k):
        J, I = divmod(k, self.NX)
        return I == 0 or J == 0 or I == self.NX - 1 or J == self.NY - 1


def elem_mass(m: BMesh, ix, iy, n, k=None):
    k = m.kq if k is None else k
    x, w = gauss(k)
    M = np.zeros((n, n))
    for a in range(k):
        for b in range(k):
            det, _ = m.jac(ix, iy, x[a], x[b])
            f = psi(n, x[a], x[b])
            M += w[a] * w[b] * det * np.outer(f, f)
    return M


# ------------------------------------------------------------------ assembled operators
def strain_matrices(m: BMesh):
    """Global G11, G11y, G12x, G12y, G22 (ne*ns x nn): E11 = G11 vx + G11y vy, E22 = G22 vy,
    E12 = G12x vx + G12y vy -- the |J|-weighted L2 projection of sym grad v_h (R#9) with the sphere's
    metric terms (R#26: -v tan/R in eps11, +u tan/(2R) in eps12; G11y = 0 on plane meshes); 8-point
    rule on plane meshes (exact: |J| eps is a polynomial of degree <= 2 ngp - 1 per variable on
    bilinear elements), the method's rule on the sphere."""
    ns, ne, nn, p = m.ns, m.ne, m.nn, m.p
    G = {k: np.zeros((ne * ns, nn)) for k in ("11", "11y", "12x", "12y", "22")}
    kq = m.kq
    x, w = gauss(kq)
    for iy in range(m.ny):
        for ix in range(m.nx):
            e = iy * m.nx + ix
            Minv = np.linalg.inv(elem_mass(m, ix, iy, ns))
            loc = {k: np.zeros((ns, (p + 1) ** 2)) for k in G}
            for a in range(kq):
                for b in range(kq):
                    s, t = x[a], x[b]
                    det, adj = m.jac(ix, iy, s, t)
                    phi, ds, dt = m.cg(s, t)
                    g = adj @ np.stack([ds.ravel(), dt.ravel()])     # |J| grad phi_j, (2, ncg)
                    f = w[a] * w[b] * psi(ns, s, t)
                    kt = det * m.kt(iy, t) * phi.ravel()              # |J| tan/R phi_j
                    loc["11"] += np.outer(f, g[0])
                    loc["11y"] -= np.outer(f, kt)
                    loc["22"] += np.outer(f, g[1])
                    loc["12x"] += 0.5 * (np.outer(f, g[1]) + np.outer(f, kt))
                    loc["12y"] += 0.5 * np.outer(f, g[0])
            cols = [m.node(ix, iy, jx, jy) for jy in range(p + 1) for jx in range(p + 1)]
            for k in G:
                G[k][e * ns:(e + 1) * ns, cols] += Minv @ loc[k]
    return G


def divergence_matrices(m: BMesh):
    """Global D_x, D_y, K (nn x ne*ns): F^x = -(D_x S11 + D_y S12 + K S12), F^y = -(D_x S12 + D_y S22
    - K S11) with D_x[j, (e,k)] = int_K psi_k d phi_j/dx (R#10) and K[j, (e,k)] = int_K psi_k phi_j
    tan(lat)/R (the sphere's metric term, R#26; 0 on plane meshes): the adjoint of strain_matrices."""
    ns, ne, nn, p = m.ns, m.ne, m.nn, m.p
    Dx = np.zeros((nn, ne * ns)); Dy = np.zeros((nn, ne * ns)); K = np.zeros((nn, ne * ns))
    kq = m.kq
    x, w = gauss(kq)
    for iy in range(m.ny):
        for ix in range(m.nx):
            e = iy * m.nx + ix
            rows = [m.node(ix, iy, jx, jy) for jy in range(p + 1) for jx in range(p + 1)]
            for a in range(kq):
                for b in range(kq):
                    s, t = x[a], x[b]
                    det, adj = m.jac(ix, iy, s, t)
                    phi, ds, dt = m.cg(s, t)
                    g = adj @ np.stack([ds.ravel(), dt.ravel()])
                    f = w[a] * w[b] * psi(ns, s, t)
                    cols = range(e * ns, (e + 1) * ns)
                    Dx[np.ix_(rows, cols)] += np.outer(g[0], f)
                    Dy[np.ix_(rows, cols)] += np.outer(g[1], f)
                    K[np.ix_(rows, cols)] += np.outer(det * m.kt(iy, t) * phi.ravel(), f)
    return Dx, Dy, K


def lumped_mass(m: BMesh):
    """m_j = int phi_j over the mesh (8-point rule, exact for Q_p times a bilinear |J|; the method's
    rule on the sphere)."""
    out = np.zeros(m.nn)
    kq = m.kq
    x, w = gauss(kq)
    for iy in range(m.ny):
        for ix in range(m.nx):
            for a in range(kq):
                for b in range(kq):
                    det, _ = m.jac(ix, iy, x[a], x[b])
                    phi, _, _ = m.cg(x[a], x[b])
                    for jy in range(m.p + 1):
                        for jx in range(m.p + 1):
                            out[m.node(ix, iy, jx, jy)] += w[a] * w[b] * det * phi[jy, jx]
    return out


def prep(m: BMesh, H, A):
    """R#17 by scatter-and-count: every element adds its DG value at each of its nodes."""
    hs = np.zeros(m.nn); as_ = np.zeros(m.nn); cnt = np.zeros(m.nn)
    for iy in range(m.ny):
        for ix in range(m.nx):
            e = iy * m.nx + ix
            for jy in range(m.p + 1):
                for jx in range(m.p + 1):
                    k = m.node(ix, iy, jx, jy)
                    f = psi(m.na, jx / m.p, jy / m.p)
                    hs[k] += H[e] @ f; as_[k] += A[e] @ f; cnt[k] += 1
    return np.maximum(hs / cnt, 1e-4), np.clip(as_ / cnt, 0.0, 1.0)


def stress(m: BMesh, prm, E11, E12, E22, H, A, S11, S12, S22):
    """Listing 2 at the stress rule's points; projection iMJwPSI with that rule."""
    ns, na, ngp = m.ns, m.na, ngp_of(m.ns)
    x, w = gauss(ngp)
    out = [S.copy() for S in (S11, S12, S22)]
    ai = 1.0 / prm.alpha
    for iy in range(m.ny):
        for ix in range(m.nx):
            e = iy * m.nx + ix
            Minv = np.linalg.inv(elem_mass(m, ix, iy, ns))
            acc = np.zeros((3, ns))
            for a in range(ngp):
                for b in range(ngp):
                    s, t = x[a], x[b]
                    det, _ = m.jac(ix, iy, s, t)
                    fS, fA = psi(ns, s, t), psi(na, s, t)
                    h = max(0.0, H[e] @ fA)
                    c = min(1.0, max(0.0, A[e] @ fA))
                    P = prm.Pstar * h * np.exp(-prm.C_conc * (1.0 - c))
                    e11, e12, e22 = E11[e] @ fS, E12[e] @ fS, E22[e] @ fS
                    d2 = 1.25 * (e11 * e11 + e22 * e22) + 1.5 * e11 * e22 + e12 * e12
                    D = np.sqrt(prm.DeltaMin ** 2 + d2)
                    Pr = P * np.sqrt(d2) / D if prm.replacement_pressure else P
                    g = (P / D * (0.625 * e11 + 0.375 * e22) - 0.5 * Pr, P / D * 0.25 * e12,
                         P / D * (0.625 * e22 + 0.375 * e11) - 0.5 * Pr)
                    for c_ in range(3):
                        acc[c_] += w[a] * w[b] * det * fS * ai * g[c_]
            for c_ in range(3):
                out[c_][e] = (1.0 - ai) * out[c_][e] + Minv @ acc[c_]
    return out


def velocity(m: BMesh, prm, Fx, Fy, mass, Hn, An, vn, o, a, v):
    """O8 (R#11) in vector form, Jacobi: every term uses v^(p-1) = v.  Arrays are (nn, 2)."""
    mm = prm.rho_ice * Hn
    c = mm / prm.dt
    Fa, Fo = prm.rho_atm * prm.C_atm, prm.rho_ocean * prm.C_ocean
    d = o - v
    wv = np.linalg.norm(d, axis=1)
    amag = np.linalg.norm(a, axis=1)
    rel = v - o
    cross = np.stack([rel[:, 1], -rel[:, 0]], axis=1)               # (v - o) x k
    F = np.stack([Fx, Fy], axis=1)
    rhs = (c[:, None] * (prm.beta * v + vn) + An[:, None] * (Fa * amag[:, None] * a + Fo * wv[:, None] * o)
           + (mm * prm.f_c)[:, None] * cross + F / mass[:, None])
    out = rhs / (c * (1 + prm.beta) + An * Fo * wv)[:, None]
    for k in range(m.nn):
        if m.on_boundary(k):
            out[k] = 0.0
    return out


def subcycles(m: BMesh, prm, nsub, st):
    """n subcycles by assembled global operators: E = G v, S <- stress, F = -D S, v <- velocity."""
    G = strain_matrices(m)
    Dx, Dy, K = divergence_matrices(m)
    mass = lumped_mass(m)
    Hn, An = prep(m, st["H"], st["A"])
    ns = m.ns
    v = np.stack([st["vx"].ravel(), st["vy"].ravel()], axis=1)
    vn = v.copy()
    o = np.stack([st["ox"].ravel(), st["oy"].ravel()], axis=1)
    a = np.stack([st["ax"].ravel(), st["ay"].ravel()], axis=1)
    S = [st[k].copy() for k in ("S11", "S12", "S22")]
    for _ in range(nsub):
        E11 = (G["11"] @ v[:, 0] + G["11y"] @ v[:, 1]).reshape(-1, ns)
        E22 = (G["22"] @ v[:, 1]).reshape(-1, ns)
        E12 = (G["12x"] @ v[:, 0] + G["12y"] @ v[:, 1]).reshape(-1, ns)
        S = stress(m, prm, E11, E12, E22, st["H"], st["A"], *S)
        s11, s12, s22 = (x.ravel() for x in S)
        Fx = -(Dx @ s11 + Dy @ s12 + K @ s12)
        Fy = -(Dx @ s12 + Dy @ s22 - K @ s11)
        v = velocity(m, prm, Fx, Fy, mass, Hn, An, vn, o, a, v)
    shp = (m.NY, m.NX)
    return dict(vx=v[:, 0].reshape(shp), vy=v[:, 1].reshape(shp), S11=S[0], S12=S[1], S22=S[2])


# ------------------------------------------------------------------ advection
def _edge(m: BMesh, ix, iy, edge):
    """(points on the edge as functions of r, neighbour's matching points, N = outward normal x length).
    edge 0 east, 1 west, 2 north, 3 south.  The edge is straight (bilinear map), so N is its end-vertex
    difference rotated a quarter turn outwards.  On the sphere the edges are a meridian arc (length
    R dlat, normal +-east) and a parallel arc (R cos(lat) dlon, normal +-north)."""
    if m.sphere:
        R, dl, dp = m.radius, m.lx / m.nx, m.ly / m.ny
        return [((lambda r: (1.0, r)), (lambda r: (0.0, r)), np.array([R * dp, 0.0]), (ix + 1, iy)),
                ((lambda r: (0.0, r)), (lambda r: (1.0, r)), np.array([-R * dp, 0.0]), (ix - 1, iy)),
                ((lambda r: (r, 1.0)), (lambda r: (r, 0.0)), np.array([0.0, R * np.cos(m.lat(iy, 1.0)) * dl]), (ix, iy + 1)),
                ((lambda r: (r, 0.0)), (lambda r: (r, 1.0)), np.array([0.0, -R * np.cos(m.lat(iy, 0.0)) * dl]), (ix, iy - 1))][edge]
    q = m.corners(ix, iy)
    if edge == 0:
        d = q[1, 1] - q[0, 1]; N = np.array([d[1], -d[0]])
        return (lambda r: (1.0, r)), (lambda r: (0.0, r)), N, (ix + 1, iy)
    if edge == 1:
        d = q[1, 0] - q[0, 0]; N = np.array([-d[1], d[0]])
        return (lambda r: (0.0, r)), (lambda r: (1.0, r)), N, (ix - 1, iy)
    if edge == 2:
        d = q[1, 1] - q[1, 0]; N = np.array([-d[1], d[0]])
        return (lambda r: (r, 1.0)), (lambda r: (r, 0.0)), N, (ix, iy + 1)
    d = q[0, 1] - q[0, 0]; N = np.array([d[1], -d[0]])
    return (lambda r: (r, 0.0)), (lambda r: (r, 1.0)), N, (ix, iy - 1)


def advect_rhs(m: BMesh, vx, vy, c):
    """M_K dc/dt = int_K c v.grad psi - sum_e int_e c_hat (v.n) psi (Eq. 1, R#18), upwind c_hat, with the
    stress rule's ngp points in the volume and on each edge (the method's quadrature)."""
    na, ngp = m.na, ngp_of(m.ns)
    x, w = gauss(ngp)
    vxf, vyf = vx.ravel(), vy.ravel()
    out = np.zeros((m.ne, na))

    def vel(ix, iy, s, t):
        phi, _, _ = m.cg(s, t)
        idx = [m.node(ix, iy, jx, jy) for jy in range(m.p + 1) for jx in range(m.p + 1)]
        f = phi.ravel()
        return np.array([f @ vxf[idx], f @ vyf[idx]])

    for iy in range(m.ny):
        for ix in range(m.nx):
            e = iy * m.nx + ix
            b = np.zeros(na)
            for a in range(ngp):
                for bb in range(ngp):
                    s, t = x[a], x[bb]
                    _, adj = m.jac(ix, iy, s, t)
                    ds, dt = dpsi(na, s, t)
                    g = adj @ np.stack([ds, dt])                     # |J| grad psi_k
                    b += w[a] * w[bb] * (c[e] @ psi(na, s, t)) * (vel(ix, iy, s, t) @ g)
            for edge in range(4):
                own, nb, N, (jx_, jy_) = _edge(m, ix, iy, edge)
                if not (0 <= jx_ < m.nx and 0 <= jy_ < m.ny):
                    if m.bc == 0:
                        continue
                    jx_, jy_ = jx_ % m.nx, jy_ % m.ny
                en = jy_ * m.nx + jx_
                for qq in range(ngp):
                    s, t = own(x[qq])
                    vN = vel(ix, iy, s, t) @ N
                    ch = c[e] @ psi(na, s, t) if vN > 0 else c[en] @ psi(na, *nb(x[qq]))
                    b -= w[qq] * ch * vN * psi(na, s, t)
            out[e] = np.linalg.solve(elem_mass(m, ix, iy, na), b)
    return out
