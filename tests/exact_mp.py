"""Exact (40-digit mpmath) evaluation of S after ONE mEVP subcycle at single elements of an axis-aligned
CG2 box mesh, following the oracle's definitions written out independently: O4 strain = L2 projection
of sym grad v_h with the 3x3 Gauss rule, Listing 2 at the Gauss points, projection with the
diagonal box mass (R#5, R#24).  The float64 test inputs are taken as exact.  Test infrastructure: used
by tests/test_oracle_exact.py (pins the oracle's accuracy) and scripts/exact_stress.py."""
import mpmath as mp
import numpy as np

mp.mp.dps = 40
XI = mp.sqrt(mp.mpf(3) / 5)
GX = [(1 - XI) / 2, mp.mpf(1) / 2, (1 + XI) / 2]
GW = [mp.mpf(5) / 18, mp.mpf(8) / 18, mp.mpf(5) / 18]
NORM = [mp.mpf(1), mp.mpf(1) / 12, mp.mpf(1) / 12, mp.mpf(1) / 180, mp.mpf(1) / 180, mp.mpf(1) / 144,
        mp.mpf(1) / 2160, mp.mpf(1) / 2160]


def psi(s, t):
    S, T = s - mp.mpf(1) / 2, t - mp.mpf(1) / 2
    return [mp.mpf(1), S, T, S * S - mp.mpf(1) / 12, T * T - mp.mpf(1) / 12, S * T,
            (S * S - mp.mpf(1) / 12) * T, S * (T * T - mp.mpf(1) / 12)]


def lag(s):
    return [2 * (s - mp.mpf(1) / 2) * (s - 1), -4 * s * (s - 1), 2 * s * (s - mp.mpf(1) / 2)], \
           [4 * s - 3, -8 * s + 4, 4 * s - 1]


def exact_S(st, nx, lx, ly, ny, ns, na, e, prm):
    ix, iy = e % nx, e // nx
    hx, hy = mp.mpf(lx) / nx, mp.mpf(ly) / ny
    ux = [[mp.mpf(float(st["vx"][2 * iy + jy, 2 * ix + jx])) for jx in range(3)] for jy in range(3)]
    uy = [[mp.mpf(float(st["vy"][2 * iy + jy, 2 * ix + jx])) for jx in range(3)] for jy in range(3)]
    G = [(GX[gx], GX[gy], GW[gx] * GW[gy]) for gy in range(3) for gx in range(3)]
    eps = []
    for (s, t, w) in G:
        Ls, dLs = lag(s); Lt, dLt = lag(t)
        d = lambda u, a, b: sum(u[jy][jx] * a[jx] * b[jy] for jy in range(3) for jx in range(3))
        vxx, vxy = d(ux, dLs, Lt) / hx, d(ux, Ls, dLt) / hy
        vyx, vyy = d(uy, dLs, Lt) / hx, d(uy, Ls, dLt) / hy
        eps.append((vxx, (vxy + vyx) / 2, vyy))
    R = [[psi(s, t)[k] * w / NORM[k] for (s, t, w) in G] for k in range(ns)]
    E = [[sum(R[k][g] * eps[g][c] for g in range(9)) for k in range(ns)] for c in range(3)]
    ainv = 1 / mp.mpf(prm.alpha)
    fac = 1 - ainv
    out = [[fac * mp.mpf(float(st[n][e, k])) for k in range(ns)] for n in ("S11", "S12", "S22")]
    for g, (s, t, w) in enumerate(G):
        ps = psi(s, t)
        e11, e12, e22 = (sum(E[c][k] * ps[k] for k in range(ns)) for c in range(3))
        h = max(sum(mp.mpf(float(st["H"][e, k])) * ps[k] for k in range(na)), 0)
        a = min(max(sum(mp.mpf(float(st["A"][e, k])) * ps[k] for k in range(na)), 0), 1)
        P = mp.mpf(prm.Pstar) * h * mp.exp(-mp.mpf(prm.C_conc) * (1 - a))
        D = mp.sqrt(mp.mpf(prm.DeltaMin) ** 2 + mp.mpf(5) / 4 * (e11 ** 2 + e22 ** 2) + mp.mpf(3) / 2 * e11 * e22 + e12 ** 2)
        r = (ainv * (P / D * (mp.mpf(5) / 8 * e11 + mp.mpf(3) / 8 * e22) - P / 2),
             ainv * (P / D * e12 / 4),
             ainv * (P / D * (mp.mpf(5) / 8 * e22 + mp.mpf(3) / 8 * e11) - P / 2))
        for c in range(3):
            for k in range(ns):
                out[c][k] += R[k][g] * r[c]
    return np.array([[float(x) for x in row] for row in out])
