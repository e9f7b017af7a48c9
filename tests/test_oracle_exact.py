"""Pin: the oracle's stress after one subcycle against a 40-digit evaluation of the same
definitions (tests/exact_mp.py: O4 strain, Listing 2, box projection; R#5, R#24).

This pins two things the other pins cannot: (1) every term of the strain -> stress -> projection
chain (a dropped term, a wrong coefficient or index shows up at >= 1e-6), and (2) the oracle's
rounding: the VP law amplifies strain rounding by P/Delta, so the oracle must be
within the north_star one-subcycle bar (1e-12, group-normalised like tests/parity.py) of the exact
value, or it could not referee the GPU at that bar."""
import numpy as np
import pytest

import oracle
from tests.exact_mp import exact_S
from tests.parity import case


class _P:
    alpha, Pstar, C_conc, DeltaMin = 1500.0, 27500.0, 20.0, 2e-9


@pytest.mark.parametrize("nxe,nye,ns,lx,ly,kind,nsample", [
    (37, 29, 8, 512e3, 512e3, "warm", 0),      # every element
    (37, 29, 6, 512e3, 512e3, "warm", 0),
    (70, 75, 8, 140e3, 150e3, "warm", 300),
    (70, 75, 6, 140e3, 150e3, "warm", 300),
    (20, 17, 8, 20e3, 17e3, "random", 0),      # S^0 != 0: the (1 - 1/alpha) S term
])
@pytest.mark.parametrize("variant", ["plain", "fma"])
def test_oracle_stress_within_bar_of_exact(nxe, nye, ns, lx, ly, kind, nsample, variant):
    st = case(nxe, nye, 2, ns, 6, kind, lx, ly)
    m = oracle.Mesh(nxe, nye, lx, ly, 2, ns, 6)
    R = oracle.Oracle(variant).subcycles(m, oracle.Params(), 1, st)
    got = np.stack([R["S11"], R["S12"], R["S22"]], 1)
    scale = np.abs(got).max()
    els = np.arange(nxe * nye)
    if nsample:   # random elements + the worst-conditioned ones (where the two oracle builds differ most)
        other = oracle.Oracle("fma" if variant == "plain" else "plain").subcycles(m, oracle.Params(), 1, st)
        d = np.abs(got - np.stack([other["S11"], other["S12"], other["S22"]], 1)).max(axis=(1, 2))
        els = np.unique(np.r_[np.random.default_rng(5).choice(els, nsample, replace=False), np.argsort(-d)[:30]])
    err = max(np.abs(got[e] - exact_S(st, nxe, lx, ly, nye, ns, 6, int(e), _P)).max() for e in els) / scale
    assert err <= 1e-12, err
