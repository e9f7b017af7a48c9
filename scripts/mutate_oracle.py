"""Mutation check of the oracle's pins (VERDICT r01 "Next round" item 1).

Each mutant is one plausible bug written into a scratch copy of ``oracle/oracle.c``; the oracle's
``-m "not gpu"`` pin files are then run against the mutated build.  A mutant is *killed* when at least
one pin fails.  Every mutant must be killed; a survivor names a part of the oracle that nothing other
than the oracle itself checks.

    python scripts/mutate_oracle.py [--only NAME ...] [--log profiles/mutation_r02.log]

Runs on CPU in the container (gcc + pytest-xdist), about 20 s per mutant.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN_FILES = ["tests/test_oracle_pins.py", "tests/test_oracle_exact.py", "tests/test_oracle_brute.py"]

# (name, what the bug is, exact text in oracle.c, replacement)
MUTANTS = [
    # --- the four VERDICT r01 survivors
    ("prep_single_element", "DG->CG prep takes the first adjacent element instead of the mean (R#17)",
     "hs += hv; as += av; ++cnt;", "if (cnt == 0) { hs = hv; as = av; cnt = 1; }"),
    ("velocity_gauss_seidel", "vy's Coriolis term uses the new vx (Gauss-Seidel instead of Jacobi, R#11)",
     "+ mm * prm->f_c * (ox[n] - vxo) + Fy[n] / mass[n];", "+ mm * prm->f_c * (ox[n] - nx_ / den) + Fy[n] / mass[n];"),
    ("lumped_mass_element00_J", "lumped mass evaluates |J| of element (0,0) for every element",
     "double detJ = ora_element_jacobian(m, (int)ix, (int)iy, s, t, NULL);",
     "double detJ = ora_element_jacobian(m, 0, 0, s, t, NULL);"),
    ("advect_box_edge_length", "advection edge flux uses the box edge length on distorted meshes",
     "b[k] -= wq * len * chat * vn * psi[k];",
     "b[k] -= wq * (col == 1 ? m->ly / m->ny : m->lx / m->nx) * chat * vn * psi[k];"),
    # --- round-1 mutation list
    ("stress_swap_5_8_3_8", "g11 with 3/8 e11 + 5/8 e22 (Listing 1 coefficients exchanged)",
     "((5.0 / 8.0) * e11[g] + (3.0 / 8.0) * e22[g])", "((3.0 / 8.0) * e11[g] + (5.0 / 8.0) * e22[g])"),
    ("stress_e12_factor", "g12 = P/Delta e12 / 2 instead of / 4",
     "(PDelta * (1.0 / 4.0) * e12[g])", "(PDelta * (1.0 / 2.0) * e12[g])"),
    ("stress_delta_weight", "Delta with 1.25 e11 e22 instead of 1.5",
     "+ 1.50 * e11[g] * e22[g]", "+ 1.25 * e11[g] * e22[g]"),
    ("divergence_transposed", "F^y with sigma22 d/dx + sigma12 d/dy (transposed operand)",
     "ly[j] -= w * detJ * (s12 * gxj + s22 * gyj - s11 * phi[j] * kt);",
     "ly[j] -= w * detJ * (s22 * gxj + s12 * gyj - s11 * phi[j] * kt);"),
    ("coriolis_sign", "Coriolis term with the wrong sign in x",
     "+ mm * prm->f_c * (vyo - oy[n])", "+ mm * prm->f_c * (oy[n] - vyo)"),
    ("rk3_weights", "SSP-RK3 second stage 1/2, 1/2 instead of 3/4, 1/4",
     "c2[i] = 0.75 * c0[i] + 0.25 * (c1[i] + dt * L[i]);", "c2[i] = 0.5 * c0[i] + 0.5 * (c1[i] + dt * L[i]);"),
    ("rk2_weights", "SSP-RK2 final stage 1/4, 3/4 instead of 1/2, 1/2",
     "c[i] = 0.5 * c0[i] + 0.5 * (c1[i] + dt * L[i]);", "c[i] = 0.25 * c0[i] + 0.75 * (c1[i] + dt * L[i]);"),
    ("upwind_side", "downwind trace instead of upwind",
     "double chat = vn > 0 ?", "double chat = vn < 0 ?"),
    ("basis_offset", "psi_3 = S^2 - 1/6 (non-orthogonal offset)",
     "all[3] = S * S - 1.0 / 12.0;", "all[3] = S * S - 1.0 / 6.0;"),
    ("pressure_exponent", "P = P* h exp(-C a) instead of exp(-C (1 - a))",
     "exp(-prm->C_conc * (1.0 - aG[g]))", "exp(-prm->C_conc * aG[g])"),
    ("drag_without_A", "ocean drag in the denominator without the concentration factor",
     "double den = c * (1.0 + beta) + An[n] * Fo * w;", "double den = c * (1.0 + beta) + Fo * w;"),
    ("h_floor", "nodal H floored at 1e-3 instead of 1e-4",
     "fmax(h, 1e-4)", "fmax(h, 1e-3)"),
    ("grad_Jinv_transposed", "physical gradient with J^-1 instead of J^-T",
     "*gx = Jinv[0] * gs + Jinv[2] * gt;\n    *gy = Jinv[1] * gs + Jinv[3] * gt;",
     "*gx = Jinv[0] * gs + Jinv[1] * gt;\n    *gy = Jinv[2] * gs + Jinv[3] * gt;"),
    # --- more
    ("element_mass_element00_J", "DG mass matrix with |J| of element (0,0)",
     "double detJ = ora_element_jacobian(m, ix, iy, s, t, NULL);\n            double psi[MAXN];\n            ora_dg_basis(n, s, t, psi);",
     "double detJ = ora_element_jacobian(m, 0, 0, s, t, NULL);\n            double psi[MAXN];\n            ora_dg_basis(n, s, t, psi);"),
    ("divergence_drops_sw", "divergence gather skips the south-west element of each node (F^x)",
     "fx += rx[e * ncg + j];", "if (ix == I / p - 1 && iy == J / p - 1) continue; fx += rx[e * ncg + j];"),
    ("west_normal_sign", "west edge keeps the east-facing normal",
     "if (edge == 1 || edge == 3) { nrm[0] = -nrm[0]; nrm[1] = -nrm[1]; }",
     "if (edge == 3) { nrm[0] = -nrm[0]; nrm[1] = -nrm[1]; }"),
    ("neighbour_trace_flipped", "east neighbour's trace read at t = 1 - r",
     "if (edge == 0) { s = 1.0; t = r; sn = 0.0; tn = r; col = 1; }",
     "if (edge == 0) { s = 1.0; t = r; sn = 0.0; tn = 1.0 - r; col = 1; }"),
    ("limiter_drops_mean", "limiter scales c without restoring the mean",
     "ce[0] += (1.0 - theta) * cbar;", "ce[0] += 0.0 * cbar;"),
    ("strain_e12_no_half", "eps12 = dvx/dy + dvy/dx (engineering shear)",
     "eps12 = 0.5 * (dvxdy + dvydx + kt * vgx)", "eps12 = (dvxdy + dvydx + kt * vgx)"),
    ("stress_relaxation_factor", "S <- (1 - 1/alpha^2) S + ...",
     "double fac = 1.0 - alphaInv;", "double fac = 1.0 - alphaInv * alphaInv;"),
    ("jinv_cofactor_sign", "J^-1 off-diagonal with the wrong sign",
     "Jinv[1] = -xt / det;", "Jinv[1] = xt / det;"),
    ("velocity_beta_on_vn", "beta multiplies v^n instead of v^(p-1)",
     "c * (beta * vxo + vnx[n])", "c * (beta * vnx[n] + vxo)"),
    ("lumped_mass_phi0", "lumped mass integrates phi_0 for every local node",
     "acc += w * detJ * phi[j];", "acc += w * detJ * phi[0];"),
    ("prep_no_A_clamp", "nodal A not clamped to 1",
     "An[node_index(m, I, J)] = fmin(fmax(a, 0.0), 1.0);", "An[node_index(m, I, J)] = fmax(a, 0.0);"),
    ("stress_no_h_clamp", "Gauss-point h not clamped at 0",
     "hG[g] = fmax(hv, 0.0);", "hG[g] = hv;"),
    ("replacement_pressure_power", "replacement pressure P Delta_raw^2 / Delta",
     "Prep = P[g] * sqrt(draw2) / DELTA;", "Prep = P[g] * draw2 / DELTA;"),
    ("air_drag_linear", "air drag F_a a instead of F_a |a| a",
     "An[n] * (Fa * amag * ax[n] + Fo * w * ox[n])", "An[n] * (Fa * ax[n] + Fo * w * ox[n])"),
    ("advect_volume_sign", "advection volume term with the wrong sign",
     "b[k] += w * detJ * cv * (ux * gxk + uy * gyk);", "b[k] -= w * detJ * cv * (ux * gxk + uy * gyk);"),
    # --- sphere (R#26)
    ("sph_strain_metric_sign", "sphere: eps11 metric term with the wrong sign",
     "double eps11 = dvxdx - kt * vgy", "double eps11 = dvxdx + kt * vgy"),
    ("sph_strain_metric_dropped", "sphere: eps12 without its metric term",
     "eps12 = 0.5 * (dvxdy + dvydx + kt * vgx)", "eps12 = 0.5 * (dvxdy + dvydx)"),
    ("sph_divergence_metric_dropped", "sphere: F^x without the metric term",
     "lx[j] -= w * detJ * (s11 * gxj + s12 * gyj + s12 * phi[j] * kt);", "lx[j] -= w * detJ * (s11 * gxj + s12 * gyj);"),
    ("sph_jacobian_no_cos", "sphere: |J| without cos(lat)",
     "return R * R * c * dlon * dlat;", "return R * R * dlon * dlat;"),
    ("sph_parallel_edge_no_cos", "sphere: parallel-arc edge length without cos(lat)",
     "if (col == 0) { T[0] = R * cos(sph_lat(m, iy, t)) * dlon; T[1] = 0.0; }",
     "if (col == 0) { T[0] = R * dlon; T[1] = 0.0; }"),
    ("sph_metric_at_centre", "sphere: metric evaluated at the element-centre latitude",
     "return tan(sph_lat(m, iy, t)) / m->radius;", "return tan(sph_lat(m, iy, 0.5)) / m->radius;"),
    ("sph_dlon_dlat_swapped", "sphere: J^-1 with dlat in the longitude entry",
     "Jinv[0] = 1.0 / (R * c * dlon); Jinv[1] = 0.0;", "Jinv[0] = 1.0 / (R * c * dlat); Jinv[1] = 0.0;"),
    ("strain_vy_typo", "strain reads vx where vy is meant",
     "double ux = vx[n] - cx, uy = vy[n] - cy;", "double ux = vx[n] - cx, uy = vx[n] - cy;"),
]


def run_one(name, old, new, jobs):
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    cnt = src.count(old)
    if cnt != 1:
        return "BAD-PATTERN", f"pattern found {cnt} times", 0.0
    with tempfile.TemporaryDirectory(prefix=f"mut_{name}_") as tmp:
        shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(tmp, "oracle"),
                        ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        shutil.copytree(os.path.join(ROOT, "tests"), os.path.join(tmp, "tests"),
                        ignore=shutil.ignore_patterns("__pycache__"))
        os.makedirs(os.path.join(tmp, "paper_2402_00466_b200"))
        for f in ("__init__.py", "inputs.py"):
            shutil.copy(os.path.join(ROOT, "paper_2402_00466_b200", f), os.path.join(tmp, "paper_2402_00466_b200", f))
        with open(os.path.join(tmp, "oracle", "oracle.c"), "w") as fh:
            fh.write(src.replace(old, new))
        t0 = time.time()
        build = subprocess.run([sys.executable, "-c", "import oracle; oracle.build('plain'); oracle.build('fma')"],
                               cwd=tmp, capture_output=True, text=True)
        if build.returncode != 0:
            return "BUILD-FAILED", build.stderr[-300:], time.time() - t0
        r = subprocess.run([sys.executable, "-m", "pytest", *PIN_FILES, "-q", "-x", "-p", "no:cacheprovider",
                            "-n", str(jobs), "-m", "not gpu"], cwd=tmp, capture_output=True, text=True)
        dt = time.time() - t0
        failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED ")]
        if r.returncode == 0:
            return "SURVIVED", "all pins passed", dt
        if failed:   # rc 1, or 2 when xdist interrupts the session after the first failure (-x)
            return "killed", failed[0], dt
        return "ERROR", r.stdout[-300:] + r.stderr[-300:], dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--jobs", type=int, default=min(8, os.cpu_count() or 1))
    ap.add_argument("--log")
    a = ap.parse_args()
    lines = []
    survivors = 0
    for name, what, old, new in MUTANTS:
        if a.only and name not in a.only:
            continue
        status, detail, dt = run_one(name, old, new, a.jobs)
        survivors += status != "killed"
        ln = f"{status:12s} {name:28s} {dt:6.1f}s  {what}  ->  {detail}"
        print(ln, flush=True)
        lines.append(ln)
    summary = f"{len(lines) - survivors}/{len(lines)} mutants killed by the oracle pins ({', '.join(PIN_FILES)})"
    print(summary)
    if a.log:
        with open(a.log, "w") as fh:
            fh.write("# python scripts/mutate_oracle.py  (status, mutant, time, bug -> first failing pin)\n")
            fh.write("\n".join(lines) + "\n" + summary + "\n")
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()
