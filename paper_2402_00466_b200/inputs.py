"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no quadrature, basis
evaluation, projection or rheology): it evaluates closed-form analytic fields
at node coordinates and fills DG coefficient rows with centred finite
differences of those fields.  It imports only numpy.  DESIGN.md §5 states the
recipe; it is a proposal because the paper cites the VP cyclone benchmark
 but gives no formulas.

All arrays are float64 in the C-ABI layouts:
  DG field : (N_e, n) row-major, element e = iy*nx + ix
  CG field : (p*ny+1, p*nx+1) row-major
A *window* (ix0, iy0, wx, wy) of a global mesh can be generated on its own, with
global coordinates, so large configs can be cut into oracle-sized pieces and
row strips can be generated per rank.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SEED_BASE = 240200466
KM_PER_DAY = 1000.0 / 86400.0


@dataclass(frozen=True)
class Config:
    name: str
    nx: int
    ny: int
    p: int
    ns: int
    na: int
    nsub: int
    lx: float = 512e3
    ly: float = 512e3
    kind: str = "warm"
    advect: bool = False
    alpha: float = 1500.0   # = beta; R#13: raised with resolution (mEVP needs alpha*beta >> gamma ~ 1/dx^2)


# BASELINE.json configs (C5 is per GPU: Ly = P * 512 km)
CONFIGS = {
    "C1": Config("C1", 16, 16, 1, 3, 3, 10, kind="random"),
    "C2": Config("C2", 256, 256, 2, 6, 6, 100),
    "C3": Config("C3", 2048, 2048, 2, 6, 6, 100, advect=True, alpha=25000.0),
    "C4": Config("C4", 4096, 4096, 2, 6, 6, 100, advect=True, alpha=25000.0),
    "C5": Config("C5", 8192, 8192, 2, 6, 6, 100, advect=True, alpha=100000.0),   # R#13: 25000 is unstable at 62.5 m
}


def default_params() -> dict:
    """Physical constants (R#12/R#13); all configurable."""
    return dict(rho_ice=900.0, rho_atm=1.3, rho_ocean=1026.0, C_atm=1.2e-3, C_ocean=5.5e-3,
                f_c=1.46e-4, Pstar=27500.0, DeltaMin=2e-9, C_conc=20.0, alpha=1500.0,
                beta=1500.0, dt=120.0, replacement_pressure=0)


def _node_xy(nx, ny, p, lx, ly, window):
    ix0, iy0, wx, wy = window
    hx, hy = lx / nx, ly / ny
    I = np.arange(p * ix0, p * (ix0 + wx) + 1, dtype=np.float64)
    J = np.arange(p * iy0, p * (iy0 + wy) + 1, dtype=np.float64)
    X, Y = np.meshgrid(I * (hx / p), J * (hy / p))
    return X, Y


def _elem_xy(nx, ny, lx, ly, window):
    ix0, iy0, wx, wy = window
    hx, hy = lx / nx, ly / ny
    xc = (np.arange(ix0, ix0 + wx) + 0.5) * hx
    yc = (np.arange(iy0, iy0 + wy) + 0.5) * hy
    X, Y = np.meshgrid(xc, yc)
    return X.ravel(), Y.ravel(), hx, hy


def dg_rows(f, nx, ny, lx, ly, n, window):
    """Coefficient rows from centred differences of an analytic f(x, y):
    c0 = f(centre); c1, c2 = first differences across the element; c3, c4 =
    second differences; c5 = mixed difference.  Truncated to n columns."""
    X, Y, hx, hy = _elem_xy(nx, ny, lx, ly, window)
    a, b = 0.5 * hx, 0.5 * hy
    f00 = f(X, Y)
    fe, fw, fn, fs = f(X + a, Y), f(X - a, Y), f(X, Y + b), f(X, Y - b)
    cols = [f00, fe - fw, fn - fs, 2.0 * (fe + fw - 2.0 * f00), 2.0 * (fn + fs - 2.0 * f00),
            f(X + a, Y + b) - f(X + a, Y - b) - f(X - a, Y + b) + f(X - a, Y - b)]
    return np.ascontiguousarray(np.stack(cols[:n], axis=1))


def warm_velocity(x, y, lx, ly, U0=0.1):
    """v0 = U0 (sin(pi x/Lx) sin(2 pi y/Ly), -sin(2 pi x/Lx) sin(pi y/Ly)); zero on the box boundary."""
    vx = U0 * np.sin(np.pi * x / lx) * np.sin(2 * np.pi * y / ly)
    vy = -U0 * np.sin(2 * np.pi * x / lx) * np.sin(np.pi * y / ly)
    return vx, vy


def ice_height(lx, ly):
    return lambda x, y: 0.3 + 0.005 * (np.sin(6e-5 * x) + np.sin(3e-5 * y))


def ice_conc(lx, ly):
    return lambda x, y: 0.95 + 0.05 * np.cos(2 * np.pi * x / lx) * np.cos(2 * np.pi * y / ly)


def cyclone_forcing(x, y, lx, ly, t=0.0):
    """Ocean o = 0.01 (2y/Ly-1, 1-2x/Lx); wind a = -(W e/r0) exp(-r/r0) R_theta (x - c(t)),
    c(t) = (Lx/2, Ly/2) + 51.2 km/day * t * (1, 1), W = 15 m/s, r0 = 100 km, theta = 72 deg."""
    ox = 0.01 * (2.0 * y / ly - 1.0)
    oy = 0.01 * (1.0 - 2.0 * x / lx)
    cx = 0.5 * lx + 51.2 * KM_PER_DAY * t
    cy = 0.5 * ly + 51.2 * KM_PER_DAY * t
    dx, dy = x - cx, y - cy
    r = np.sqrt(dx * dx + dy * dy)
    W, r0, th = 15.0, 100e3, math.radians(72.0)
    s = -(W * math.e / r0) * np.exp(-r / r0)
    ax = s * (math.cos(th) * dx + math.sin(th) * dy)
    ay = s * (-math.sin(th) * dx + math.cos(th) * dy)
    return ox, oy, ax, ay


def make_case(nx, ny, p, ns, na, kind="warm", seed=SEED_BASE, lx=512e3, ly=512e3, t=0.0,
              window=None) -> dict:
    """Generate one state + forcing.  kind: 'warm' (warm box + cyclone), 'random'
    (seeded uniform fields, tiny meshes), 'rest' (v=0 start).  ``window`` =
    (ix0, iy0, wx, wy) in elements selects a sub-box with global coordinates."""
    if window is None:
        window = (0, 0, nx, ny)
    ix0, iy0, wx, wy = window
    X, Y = _node_xy(nx, ny, p, lx, ly, window)
    ox, oy, ax, ay = cyclone_forcing(X, Y, lx, ly, t)
    N = wx * wy
    if kind in ("warm", "rest"):
        vx, vy = warm_velocity(X, Y, lx, ly)
        if kind == "rest":
            vx, vy = np.zeros_like(vx), np.zeros_like(vy)
        H = dg_rows(ice_height(lx, ly), nx, ny, lx, ly, na, window)
        A = dg_rows(ice_conc(lx, ly), nx, ny, lx, ly, na, window)
        S = [np.zeros((N, ns)) for _ in range(3)]
    elif kind == "random":
        rng = np.random.default_rng(seed)
        shp = X.shape
        vx = rng.uniform(-0.2, 0.2, shp)
        vy = rng.uniform(-0.2, 0.2, shp)
        for v in (vx, vy):  # zero on the global box boundary
            gI = np.arange(p * ix0, p * (ix0 + wx) + 1)
            gJ = np.arange(p * iy0, p * (iy0 + wy) + 1)
            v[:, (gI == 0) | (gI == p * nx)] = 0.0
            v[(gJ == 0) | (gJ == p * ny), :] = 0.0
        S = [rng.uniform(-1e4, 1e4, (N, ns)) for _ in range(3)]
        H = rng.uniform(-0.2, 0.2, (N, na)); H[:, 0] = rng.uniform(0.0, 2.0, N)
        A = rng.uniform(-0.2, 0.2, (N, na)); A[:, 0] = rng.uniform(0.5, 1.1, N)
        ox = rng.uniform(-0.05, 0.05, shp); oy = rng.uniform(-0.05, 0.05, shp)
        ax = rng.uniform(-20, 20, shp); ay = rng.uniform(-20, 20, shp)
    else:
        raise ValueError(kind)
    c = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    return dict(vx=c(vx), vy=c(vy), S11=c(S[0]), S12=c(S[1]), S22=c(S[2]), A=c(A), H=c(H),
                ox=c(ox), oy=c(oy), ax=c(ax), ay=c(ay))


def distorted_vertices(nx, ny, lx, ly, delta=0.25, seed=SEED_BASE + 7) -> np.ndarray:
    """(ny+1, nx+1, 2) vertices of a box mesh whose interior vertices are moved by a seeded uniform
    offset of up to delta * (hx, hy) / 2 per axis (distortion < 0.3 keeps every
    quad convex, so all Jacobians stay positive).  Boundary vertices stay on the box."""
    rng = np.random.default_rng(seed)
    hx, hy = lx / nx, ly / ny
    X, Y = np.meshgrid(np.arange(nx + 1) * hx, np.arange(ny + 1) * hy)
    dx = rng.uniform(-0.5, 0.5, X.shape) * delta * hx
    dy = rng.uniform(-0.5, 0.5, Y.shape) * delta * hy
    dx[:, [0, -1]] = 0.0; dy[[0, -1], :] = 0.0
    dx[[0, -1], :] = 0.0; dy[:, [0, -1]] = 0.0
    return np.ascontiguousarray(np.stack([X + dx, Y + dy], axis=-1))


def make_config_case(cfg: Config, window=None, t=0.0, seed=None) -> dict:
    idx = list(CONFIGS).index(cfg.name) if cfg.name in CONFIGS else 0
    return make_case(cfg.nx, cfg.ny, cfg.p, cfg.ns, cfg.na, kind=cfg.kind,
                     seed=SEED_BASE + idx if seed is None else seed,
                     lx=cfg.lx, ly=cfg.ly, t=t, window=window)
