"""Shared helpers for the GPU-vs-oracle parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import oracle
from paper_2402_00466_b200 import inputs

GROUPS = {"S": ("S11", "S12", "S22"), "v": ("vx", "vy"), "A": ("A",), "H": ("H",)}


def group_err(got: dict, ref: dict, keys) -> float:
    """Group-normalised relative max-norm error:
    max_{c in G, i} |X_gpu - X_ora| / max_{c in G, i} |X_ora|."""
    num = max(float(np.abs(np.asarray(got[k]) - np.asarray(ref[k])).max()) for k in keys)
    den = max(float(np.abs(np.asarray(ref[k])).max()) for k in keys)
    return num / den if den > 0 else num


def parity(got: dict, ref: dict, init: dict | None = None, groups=("S", "v")) -> dict:
    """Errors of the fields and (if ``init`` is given) of the increments X - X0."""
    out = {}
    for g in groups:
        keys = GROUPS[g]
        out[g] = group_err(got, ref, keys)
        if init is not None:
            gi = {k: np.asarray(got[k]) - np.asarray(init[k]) for k in keys}
            ri = {k: np.asarray(ref[k]) - np.asarray(init[k]) for k in keys}
            if max(float(np.abs(v).max()) for v in ri.values()) > 0:
                out["d" + g] = group_err(gi, ri, keys)
    return out


def ora_mesh(nx, ny, p, ns, na, lx=512e3, ly=512e3, bc=0) -> oracle.Mesh:
    return oracle.Mesh(nx, ny, lx=lx, ly=ly, p=p, ns=ns, na=na, bc=bc)


def ora_params(pp) -> oracle.Params:
    from dataclasses import asdict
    return oracle.Params(**asdict(pp))


def case(nx, ny, p=2, ns=6, na=6, kind="warm", lx=512e3, ly=512e3, seed=inputs.SEED_BASE, window=None):
    return inputs.make_case(nx, ny, p, ns, na, kind=kind, lx=lx, ly=ly, seed=seed, window=window)
