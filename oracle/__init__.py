"""ORACLE — test infrastructure only.

ctypes wrapper around ``oracle/liboracle.so`` (plain FP64 C, see oracle.c).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2402_00466_b200`` never imports it and shares no code
with it.

Two builds exist so tests can measure the oracle's own rounding floor
("self-consistency floor"): ``plain`` (-ffp-contract=off, no
FMA) and ``fma`` (-mfma -ffp-contract=fast).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_VARIANTS = {
    "plain": ("liboracle.so", ["-O2", "-fno-fast-math", "-ffp-contract=off"]),
    "fma": ("liboracle_fma.so", ["-O2", "-fno-fast-math", "-mfma", "-ffp-contract=fast"]),
}
_LIBS: dict[str, C.CDLL] = {}


def build(variant: str = "plain", force: bool = False) -> str:
    """Compile the oracle shared library with gcc (OpenMP, FP64, -O2)."""
    name, flags = _VARIANTS[variant]
    out = os.path.join(_HERE, name)
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        cmd = ["gcc", "-std=c11", "-shared", "-fPIC", "-fopenmp", *flags, "-o", out, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return out


class OraMesh(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("lx", C.c_double), ("ly", C.c_double),
        ("p", C.c_int), ("ns", C.c_int), ("na", C.c_int), ("bc", C.c_int),
        ("verts", C.POINTER(C.c_double)), ("radius", C.c_double), ("lat0", C.c_double),
    ]


class OraParams(C.Structure):
    _fields_ = [
        ("rho_ice", C.c_double), ("rho_atm", C.c_double), ("rho_ocean", C.c_double),
        ("C_atm", C.c_double), ("C_ocean", C.c_double), ("f_c", C.c_double),
        ("Pstar", C.c_double), ("DeltaMin", C.c_double), ("C_conc", C.c_double),
        ("alpha", C.c_double), ("beta", C.c_double), ("dt", C.c_double),
        ("replacement_pressure", C.c_int),
    ]


_P = C.POINTER(C.c_double)


def lib(variant: str = "plain") -> C.CDLL:
    if variant not in _LIBS:
        L = C.CDLL(build(variant))
        L.ora_ngp.restype = C.c_int
        L.ora_gauss.restype = C.c_int
        L.ora_element_jacobian.restype = C.c_double
        L.ora_num_threads.restype = C.c_int
        _LIBS[variant] = L
    return _LIBS[variant]


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_P)


@dataclass
class Mesh:
    nx: int
    ny: int
    lx: float = 512e3
    ly: float = 512e3
    p: int = 2
    ns: int = 6
    na: int = 6
    bc: int = 0
    verts: np.ndarray | None = None   # (ny+1, nx+1, 2) vertex coordinates; None = box
    radius: float = 0.0               # > 0: lon-lat mesh on the sphere (R#26); lx, ly in radians
    lat0: float = 0.0                 # southern edge latitude [rad] (sphere)

    def c(self) -> OraMesh:
        vp = None
        if self.verts is not None:
            self._vkeep = np.ascontiguousarray(self.verts, dtype=np.float64)
            vp = self._vkeep.ctypes.data_as(_P)
        return OraMesh(self.nx, self.ny, self.lx, self.ly, self.p, self.ns, self.na, self.bc, vp,
                       float(self.radius), float(self.lat0))

    @property
    def n_elem(self) -> int:
        return self.nx * self.ny

    @property
    def node_shape(self) -> tuple[int, int]:
        return (self.p * self.ny + 1, self.p * self.nx + 1)


@dataclass
class Params:
    rho_ice: float = 900.0
    rho_atm: float = 1.3
    rho_ocean: float = 1026.0
    C_atm: float = 1.2e-3
    C_ocean: float = 5.5e-3
    f_c: float = 1.46e-4
    Pstar: float = 27500.0
    DeltaMin: float = 2e-9
    C_conc: float = 20.0
    alpha: float = 1500.0
    beta: float = 1500.0
    dt: float = 120.0
    replacement_pressure: int = 0

    def c(self) -> OraParams:
        return OraParams(self.rho_ice, self.rho_atm, self.rho_ocean, self.C_atm, self.C_ocean,
                         self.f_c, self.Pstar, self.DeltaMin, self.C_conc, self.alpha, self.beta,
                         self.dt, self.replacement_pressure)


def _check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with code {rc}")


class Oracle:
    """Thin callable facade; every method copies inputs it mutates."""

    def __init__(self, variant: str = "plain", threads: int | None = None):
        self.L = lib(variant)
        if threads:
            self.L.ora_set_threads(int(threads))

    @property
    def threads(self) -> int:
        return int(self.L.ora_num_threads())

    # --- building blocks -------------------------------------------------
    def ngp(self, ns: int) -> int:
        return int(self.L.ora_ngp(ns))

    def gauss(self, ngp: int):
        x = np.zeros(3); w = np.zeros(3)
        _check(self.L.ora_gauss(ngp, _ptr(x), _ptr(w)), "gauss")
        return x[:ngp].copy(), w[:ngp].copy()

    def dg_basis(self, n: int, s: float, t: float) -> np.ndarray:
        out = np.zeros(8)
        self.L.ora_dg_basis(n, C.c_double(s), C.c_double(t), _ptr(out))
        return out[:n].copy()

    def cg_basis(self, p: int, s: float, t: float):
        phi = np.zeros(9); ds = np.zeros(9); dt = np.zeros(9)
        self.L.ora_cg_basis(p, C.c_double(s), C.c_double(t), _ptr(phi), _ptr(ds), _ptr(dt))
        n = (p + 1) ** 2
        return phi[:n].copy(), ds[:n].copy(), dt[:n].copy()

    def jacobian(self, mesh: Mesh, ix: int, iy: int, s: float, t: float):
        Jinv = np.zeros(4)
        m = mesh.c()
        det = self.L.ora_element_jacobian(C.byref(m), ix, iy, C.c_double(s), C.c_double(t), _ptr(Jinv))
        return det, Jinv.reshape(2, 2)

    def element_mass(self, mesh: Mesh, ix: int, iy: int, n: int, ngp: int) -> np.ndarray:
        M = np.zeros(n * n)
        m = mesh.c()
        _check(self.L.ora_element_mass(C.byref(m), ix, iy, n, ngp, _ptr(M)), "element_mass")
        return M.reshape(n, n)

    # --- hot-path steps --------------------------------------------------
    def strain(self, mesh: Mesh, vx, vy):
        N, ns = mesh.n_elem, mesh.ns
        E = [np.zeros(N * ns) for _ in range(3)]
        m = mesh.c()
        _check(self.L.ora_strain(C.byref(m), _ptr(_f(vx)), _ptr(_f(vy)), *[_ptr(e) for e in E]), "strain")
        return tuple(e.reshape(N, ns) for e in E)

    def stress(self, mesh: Mesh, prm: Params, E11, E12, E22, H, A, S11, S12, S22):
        S = [_f(x).copy() for x in (S11, S12, S22)]
        m, pr = mesh.c(), prm.c()
        _check(self.L.ora_stress(C.byref(m), C.byref(pr), _ptr(_f(E11)), _ptr(_f(E12)), _ptr(_f(E22)),
                                 _ptr(_f(H)), _ptr(_f(A)), *[_ptr(s) for s in S]), "stress")
        return tuple(s.reshape(mesh.n_elem, mesh.ns) for s in S)

    def divergence(self, mesh: Mesh, S11, S12, S22):
        shp = mesh.node_shape
        Fx = np.zeros(shp); Fy = np.zeros(shp)
        m = mesh.c()
        _check(self.L.ora_divergence(C.byref(m), _ptr(_f(S11)), _ptr(_f(S12)), _ptr(_f(S22)),
                                     _ptr(Fx), _ptr(Fy)), "divergence")
        return Fx, Fy

    def lumped_mass(self, mesh: Mesh):
        out = np.zeros(mesh.node_shape)
        m = mesh.c()
        _check(self.L.ora_lumped_mass(C.byref(m), _ptr(out)), "lumped_mass")
        return out

    def prep(self, mesh: Mesh, H, A):
        Hn = np.zeros(mesh.node_shape); An = np.zeros(mesh.node_shape)
        m = mesh.c()
        _check(self.L.ora_prep(C.byref(m), _ptr(_f(H)), _ptr(_f(A)), _ptr(Hn), _ptr(An)), "prep")
        return Hn, An

    def velocity(self, mesh: Mesh, prm: Params, Fx, Fy, mass, Hn, An, vnx, vny, ox, oy, ax, ay, vx, vy):
        vx = _f(vx).copy(); vy = _f(vy).copy()
        m, pr = mesh.c(), prm.c()
        _check(self.L.ora_velocity(C.byref(m), C.byref(pr), *[_ptr(_f(a)) for a in
                                   (Fx, Fy, mass, Hn, An, vnx, vny, ox, oy, ax, ay)],
                                   _ptr(vx), _ptr(vy)), "velocity")
        return vx, vy

    def subcycles(self, mesh: Mesh, prm: Params, nsub: int, st: dict, vn=None) -> dict:
        """n mEVP subcycles; ``st`` holds vx, vy, S11, S12, S22, A, H, ox, oy, ax, ay.
        v^n defaults to the incoming v (BEGIN_STEP semantics)."""
        out = {k: _f(v).copy() for k, v in st.items()}
        vnx = _f(st["vx"]).copy() if vn is None else _f(vn[0])
        vny = _f(st["vy"]).copy() if vn is None else _f(vn[1])
        m, pr = mesh.c(), prm.c()
        _check(self.L.ora_subcycles(C.byref(m), C.byref(pr), int(nsub), _ptr(out["H"]), _ptr(out["A"]),
                                    _ptr(out["ox"]), _ptr(out["oy"]), _ptr(out["ax"]), _ptr(out["ay"]),
                                    _ptr(vnx), _ptr(vny), _ptr(out["vx"]), _ptr(out["vy"]),
                                    _ptr(out["S11"]), _ptr(out["S12"]), _ptr(out["S22"])), "subcycles")
        return out

    def advect_rhs(self, mesh: Mesh, vx, vy, c):
        out = np.zeros((mesh.n_elem, mesh.na))
        m = mesh.c()
        _check(self.L.ora_advect_rhs(C.byref(m), _ptr(_f(vx)), _ptr(_f(vy)), _ptr(_f(c)), _ptr(out)),
               "advect_rhs")
        return out

    def advect(self, mesh: Mesh, dt: float, vx, vy, A, H):
        A = _f(A).copy(); H = _f(H).copy()
        m = mesh.c()
        _check(self.L.ora_advect(C.byref(m), C.c_double(dt), _ptr(_f(vx)), _ptr(_f(vy)), _ptr(A), _ptr(H)),
               "advect")
        return A, H

    def limit(self, mesh: Mesh, c, lo: float, hi: float = float("inf")):
        c = _f(c).copy()
        m = mesh.c()
        _check(self.L.ora_limit(C.byref(m), C.c_double(lo), C.c_double(hi), _ptr(c)), "limit")
        return c

    def advect_limited(self, mesh: Mesh, dt: float, vx, vy, A, H, limiter: int = 1):
        A = _f(A).copy(); H = _f(H).copy()
        m = mesh.c()
        _check(self.L.ora_advect_limited(C.byref(m), C.c_double(dt), _ptr(_f(vx)), _ptr(_f(vy)), _ptr(A), _ptr(H),
                                         int(limiter)), "advect_limited")
        return A, H

    def outer_step(self, mesh: Mesh, prm: Params, nsub: int, st: dict, do_advect: bool = True) -> dict:
        out = {k: _f(v).copy() for k, v in st.items()}
        m, pr = mesh.c(), prm.c()
        _check(self.L.ora_outer_step(C.byref(m), C.byref(pr), int(nsub), int(bool(do_advect)),
                                     _ptr(out["ox"]), _ptr(out["oy"]), _ptr(out["ax"]), _ptr(out["ay"]),
                                     _ptr(out["vx"]), _ptr(out["vy"]), _ptr(out["S11"]), _ptr(out["S12"]),
                                     _ptr(out["S22"]), _ptr(out["A"]), _ptr(out["H"])), "outer_step")
        return out


def _f(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
