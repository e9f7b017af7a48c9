/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).  Never linked, loaded or
 * called by the product path (paper_2402_00466_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline and --impl reference)
 * may use it.
 *
 * Plain FP64 C, written step by step from PAPER.md and the DESIGN.md
 * readings R#1..R#22.  Every element operation is done the slow, literal way:
 *   - Gauss points and weights from the textbook rule, per element;
 *   - the bilinear element map and its Jacobian evaluated at every point
 *     (constant on the box, computed anyway);
 *   - physical gradients through J^{-1};
 *   - the element mass matrix assembled by quadrature and solved by Gaussian
 *     elimination with partial pivoting (no closed-form inverse);
 *   - the divergence assembled per node from element contributions.
 * No blocking, fusion, folding of constants or reordering beyond what the
 * equations say.  OpenMP parallelises only independent element / node loops,
 * so results are deterministic and thread-count independent.
 *
 * parity unpinned: none of the functions below; each is pinned by a
 * `-m "not gpu"` test in tests/test_oracle_*.py.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXN 8      /* max DG dofs      */
#define MAXCG 9     /* max CG dofs      */
#define MAXG 9      /* max Gauss points */

int ora_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ora_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Listing 2: NGP = (DGstress==8||DGstress==6) ? 3 : (DGstress==3 ? 2 : -1). */
int ora_ngp(int ns) {
    if (ns == 8 || ns == 6) return 3;
    if (ns == 3) return 2;
    return -1;
}

/* Gauss-Legendre rule on [0,1] (textbook nodes on [-1,1] mapped by (1+xi)/2,
 * weights halved).  Points ascending.  R#18 (same ngp everywhere). */
int ora_gauss(int ngp, double* x, double* w) {
    if (ngp == 1) {
        x[0] = 0.5; w[0] = 1.0;
    } else if (ngp == 2) {
        double xi = 1.0 / sqrt(3.0);
        x[0] = 0.5 * (1.0 - xi); x[1] = 0.5 * (1.0 + xi);
        w[0] = 0.5; w[1] = 0.5;
    } else if (ngp == 3) {
        double xi = sqrt(3.0 / 5.0);
        x[0] = 0.5 * (1.0 - xi); x[1] = 0.5; x[2] = 0.5 * (1.0 + xi);
        w[0] = 0.5 * 5.0 / 9.0; w[1] = 0.5 * 8.0 / 9.0; w[2] = 0.5 * 5.0 / 9.0;
    } else {
        return -1;
    }
    return 0;
}

/* DG basis, R#5: centred Legendre on the reference square, S = s-1/2, T = t-1/2:
 * {1, S, T, S^2-1/12, T^2-1/12, S*T}, first n of them.  PSI_1_1 = {1.0}.
 * n = 8 (R#24): + (S^2-1/12) T, S (T^2-1/12) -- the full gradient space of Q2. */
void ora_dg_basis(int n, double s, double t, double* psi) {
    double S = s - 0.5, T = t - 0.5;
    double all[8];
    all[0] = 1.0;
    all[1] = S;
    all[2] = T;
    all[3] = S * S - 1.0 / 12.0;
    all[4] = T * T - 1.0 / 12.0;
    all[5] = S * T;
    all[6] = (S * S - 1.0 / 12.0) * T;
    all[7] = S * (T * T - 1.0 / 12.0);
    for (int k = 0; k < n; ++k) psi[k] = all[k];
}

/* Reference-coordinate gradient of the DG basis above. */
static void ora_dg_basis_grad(int n, double s, double t, double* dpsids, double* dpsidt) {
    double S = s - 0.5, T = t - 0.5;
    double ds[8] = {0.0, 1.0, 0.0, 2.0 * S, 0.0, T, 2.0 * S * T, T * T - 1.0 / 12.0};
    double dt[8] = {0.0, 0.0, 1.0, 0.0, 2.0 * T, S, S * S - 1.0 / 12.0, 2.0 * S * T};
    for (int k = 0; k < n; ++k) { dpsids[k] = ds[k]; dpsidt[k] = dt[k]; }
}

/* 1D Lagrange polynomials on equispaced nodes {0,1} (p=1) or {0,1/2,1} (p=2), R#8. */
static void lagrange1d(int p, double s, double* L, double* dL) {
    if (p == 1) {
        L[0] = 1.0 - s;  dL[0] = -1.0;
        L[1] = s;        dL[1] = 1.0;
    } else {
        L[0] = 2.0 * (s - 0.5) * (s - 1.0);   dL[0] = 4.0 * s - 3.0;
        L[1] = -4.0 * s * (s - 1.0);          dL[1] = -8.0 * s + 4.0;
        L[2] = 2.0 * s * (s - 0.5);           dL[2] = 4.0 * s - 1.0;
    }
}

/* CG basis Q_p (tensor Lagrange), local node j = jy*(p+1)+jx (R#8). */
void ora_cg_basis(int p, double s, double t, double* phi, double* dphids, double* dphidt) {
    double Ls[3], dLs[3], Lt[3], dLt[3];
    lagrange1d(p, s, Ls, dLs);
    lagrange1d(p, t, Lt, dLt);
    for (int jy = 0; jy <= p; ++jy)
        for (int jx = 0; jx <= p; ++jx) {
            int j = jy * (p + 1) + jx;
            if (phi) phi[j] = Ls[jx] * Lt[jy];
            if (dphids) dphids[j] = dLs[jx] * Lt[jy];
            if (dphidt) dphidt[j] = Ls[jx] * dLt[jy];
        }
}

/* Bilinear (Q1) element map from the four vertices: the box x_{a,b} = (a*hx, b*hy), or the
 * mesh's vertex array for general quads (R#23). */
/* The element's four vertices relative to its first one (x_{a,b} - x_{0,0}).  Only derivatives of
 * the bilinear map are ever used, and sum_k grad N_k = 0, so this is exact in real arithmetic; it
 * keeps J exact in floating point too (differences of nearby vertices are exact), where absolute
 * coordinates (~1e5 m on ~1e2 m elements) would cost ~1e-13 relative in J - amplified past the
 * north_star bar by the near-cancellation of volume and edge terms in the advection (R#23). */
static void element_vertices(const ora_mesh* m, int ix, int iy, double X[4], double Y[4]) {
    double hx = m->lx / m->nx, hy = m->ly / m->ny;
    for (int k = 0; k < 4; ++k) {
        int kx = k & 1, ky = k >> 1;
        if (m->verts) {
            long v = (long)(iy + ky) * (m->nx + 1) + (ix + kx);
            long v0 = (long)iy * (m->nx + 1) + ix;
            X[k] = m->verts[2 * v] - m->verts[2 * v0];
            Y[k] = m->verts[2 * v + 1] - m->verts[2 * v0 + 1];
        } else {
            X[k] = kx * hx;
            Y[k] = ky * hy;
        }
    }
}

/* Spherical lat-lon mesh (R#26): element (ix, iy) covers longitudes ix dlon + s dlon and
 * latitudes lat0 + (iy + t) dlat.  In the local orthonormal east-north frame the map's Jacobian is
 * diag(R cos(lat) dlon, R dlat); physical vector components are (east, north). */
static int is_sphere(const ora_mesh* m) { return m->radius > 0.0 && !m->verts; }
static double sph_lat(const ora_mesh* m, int iy, double t) { return m->lat0 + (iy + t) * (m->ly / m->ny); }

/* The metric (Christoffel) coefficient tan(lat) / R of the orthonormal frame on the sphere at (iy, t);
 * 0 on plane meshes.  It enters the strain rate of a vector field,
 *   eps11 = (1/(R cos lat)) du/dlon - v tan(lat)/R,  eps22 = (1/R) dv/dlat,
 *   eps12 = 1/2 [(1/(R cos lat)) dv/dlon + (1/R) du/dlat + u tan(lat)/R],
 * and, as its adjoint, the weak stress divergence (R#26). */
static double metric_tan(const ora_mesh* m, int iy, double t) {
    if (!is_sphere(m)) return 0.0;
    return tan(sph_lat(m, iy, t)) / m->radius;
}

/* |J| of the bilinear map at (s,t); fills J^{-1} row-major ([ds/dx ds/dy; dt/dx dt/dy]).
 * On the sphere: |J| = R^2 cos(lat) dlon dlat, J^{-1} = diag(1 / (R cos(lat) dlon), 1 / (R dlat)). */
double ora_element_jacobian(const ora_mesh* m, int ix, int iy, double s, double t, double Jinv[4]) {
    if (is_sphere(m)) {
        double dlon = m->lx / m->nx, dlat = m->ly / m->ny, R = m->radius, c = cos(sph_lat(m, iy, t));
        (void)ix; (void)s;
        if (Jinv) {
            Jinv[0] = 1.0 / (R * c * dlon); Jinv[1] = 0.0;
            Jinv[2] = 0.0;                  Jinv[3] = 1.0 / (R * dlat);
        }
        return R * R * c * dlon * dlat;
    }
    double X[4], Y[4];
    element_vertices(m, ix, iy, X, Y);
    double phi[4], ds[4], dt[4];
    ora_cg_basis(1, s, t, phi, ds, dt);
    double xs = 0, xt = 0, ys = 0, yt = 0;
    for (int k = 0; k < 4; ++k) {
        xs += ds[k] * X[k]; xt += dt[k] * X[k];
        ys += ds[k] * Y[k]; yt += dt[k] * Y[k];
    }
    double det = xs * yt - xt * ys;
    if (Jinv) {
        Jinv[0] = yt / det;  Jinv[1] = -xt / det;
        Jinv[2] = -ys / det; Jinv[3] = xs / det;
    }
    return det;
}

/* Tangent vector of the element map along s (col 0) or t (col 1); on the sphere in the local
 * east-north frame: (R cos(lat) dlon, 0) and (0, R dlat). */
static void element_tangent(const ora_mesh* m, int ix, int iy, double s, double t, int col, double* T) {
    if (is_sphere(m)) {
        double dlon = m->lx / m->nx, dlat = m->ly / m->ny, R = m->radius;
        (void)ix; (void)s;
        if (col == 0) { T[0] = R * cos(sph_lat(m, iy, t)) * dlon; T[1] = 0.0; }
        else { T[0] = 0.0; T[1] = R * dlat; }
        return;
    }
    double X[4], Y[4];
    element_vertices(m, ix, iy, X, Y);
    double phi[4], ds[4], dt[4];
    ora_cg_basis(1, s, t, phi, ds, dt);
    double a = 0, b = 0;
    for (int k = 0; k < 4; ++k) {
        double d = col == 0 ? ds[k] : dt[k];
        a += d * X[k];
        b += d * Y[k];
    }
    T[0] = a; T[1] = b;
}

/* Physical gradient = J^{-T} * reference gradient. */
static void phys_grad(const double Jinv[4], double gs, double gt, double* gx, double* gy) {
    *gx = Jinv[0] * gs + Jinv[2] * gt;
    *gy = Jinv[1] * gs + Jinv[3] * gt;
}

/* Element mass matrix M_K = sum_g w_g |J_g| psi(g) psi(g)^T (R#5, O3). */
int ora_element_mass(const ora_mesh* m, int ix, int iy, int n, int ngp, double* M) {
    double xg[3], wg[3];
    if (ora_gauss(ngp, xg, wg)) return -1;
    for (int a = 0; a < n * n; ++a) M[a] = 0.0;
    for (int gy = 0; gy < ngp; ++gy)
        for (int gx = 0; gx < ngp; ++gx) {
            double s = xg[gx], t = xg[gy], w = wg[gx] * wg[gy];
            double detJ = ora_element_jacobian(m, ix, iy, s, t, NULL);
            double psi[MAXN];
            ora_dg_basis(n, s, t, psi);
            for (int a = 0; a < n; ++a)
                for (int b = 0; b < n; ++b) M[a * n + b] += w * detJ * psi[a] * psi[b];
        }
    return 0;
}

/* Dense solve A x = b (in place, x -> b) by Gaussian elimination with partial pivoting. */
int ora_solve(int n, double* A, double* b) {
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (fabs(A[r * n + c]) > fabs(A[piv * n + c])) piv = r;
        if (A[piv * n + c] == 0.0) return -1;
        if (piv != c) {
            for (int k = 0; k < n; ++k) {
                double tmp = A[c * n + k]; A[c * n + k] = A[piv * n + k]; A[piv * n + k] = tmp;
            }
            double tb = b[c]; b[c] = b[piv]; b[piv] = tb;
        }
        for (int r = c + 1; r < n; ++r) {
            double f = A[r * n + c] / A[c * n + c];
            for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
            b[r] -= f * b[c];
        }
    }
    for (int r = n - 1; r >= 0; --r) {
        double acc = b[r];
        for (int k = r + 1; k < n; ++k) acc -= A[r * n + k] * b[k];
        b[r] = acc / A[r * n + r];
    }
    return 0;
}

/* Solve M_K x = b with a fresh copy of M_K. */
static int solve_mass(int n, const double* M, double* b) {
    double Mc[MAXN * MAXN];
    memcpy(Mc, M, sizeof(double) * n * n);
    return ora_solve(n, Mc, b);
}

static int check_mesh(const ora_mesh* m) {
    if (!m || m->nx < 1 || m->ny < 1 || !(m->lx > 0) || !(m->ly > 0)) return -1;
    if (m->radius < 0.0 || (m->radius > 0.0 && (m->verts || fabs(m->lat0) >= 1.5707963267948966 ||
                                                fabs(m->lat0 + m->ly) >= 1.5707963267948966)))
        return -1;
    if (m->p == 1 && m->ns != 3) return -2;
    if (m->p == 2 && m->ns != 6 && m->ns != 8) return -2;
    if (m->p != 1 && m->p != 2) return -2;
    if (m->na != 1 && m->na != 3 && m->na != 6) return -2;
    if (m->p == 1 && m->na == 6) return -2;
    return 0;
}

static long node_index(const ora_mesh* m, long I, long J) { return J * (long)(m->p * m->nx + 1) + I; }

/* Global node id of local CG node j of element (ix, iy) (R#8). */
static long elem_node(const ora_mesh* m, int ix, int iy, int j) {
    int p = m->p, jx = j % (p + 1), jy = j / (p + 1);
    return node_index(m, (long)p * ix + jx, (long)p * iy + jy);
}

/* O4 strain (Table 1 "strain"; R#9): E_c = M_K^{-1} sum_g w_g |J_g| psi(g) eps_c(g),
 * eps11 = d vx/dx, eps22 = d vy/dy, eps12 = (d vx/dy + d vy/dx)/2 from the CG field; on the sphere
 * (R#26) with the metric terms -vy tan(lat)/R in eps11 and +vx tan(lat)/(2R) in eps12. */
int ora_strain(const ora_mesh* m, const double* vx, const double* vy,
               double* E11, double* E12, double* E22) {
    int rc = check_mesh(m); if (rc) return rc;
    int ns = m->ns, ngp = ora_ngp(ns), ncg = (m->p + 1) * (m->p + 1);
    double xg[3], wg[3];
    ora_gauss(ngp, xg, wg);
    long N = (long)m->nx * m->ny;
    int err = 0;
#pragma omp parallel for schedule(static) reduction(| : err)
    for (long e = 0; e < N; ++e) {
        int ix = (int)(e % m->nx), iy = (int)(e / m->nx);
        double M[MAXN * MAXN];
        ora_element_mass(m, ix, iy, ns, ngp, M);
        double b11[MAXN] = {0}, b12[MAXN] = {0}, b22[MAXN] = {0};
        /* grad v_h = sum_j (v_j - c) grad phi_j for any constant c, because the CG basis is a
         * partition of unity (sum_j grad phi_j = 0).  With c = the element's mean nodal velocity the
         * sum no longer cancels large equal parts: on smooth fields the plain sum loses ~|v|/|dv| ulps,
         * which the VP law then amplifies by P/Delta past the parity bar (R#20). */
        double cx = 0.0, cy = 0.0;
        for (int j = 0; j < ncg; ++j) { long n = elem_node(m, ix, iy, j); cx += vx[n]; cy += vy[n]; }
        cx /= ncg; cy /= ncg;
        for (int gy = 0; gy < ngp; ++gy)
            for (int gx = 0; gx < ngp; ++gx) {
                double s = xg[gx], t = xg[gy], w = wg[gx] * wg[gy];
                double Jinv[4];
                double detJ = ora_element_jacobian(m, ix, iy, s, t, Jinv);
                double phi[MAXCG], dps[MAXCG], dpt[MAXCG];
                ora_cg_basis(m->p, s, t, phi, dps, dpt);
                double dvxdx = 0, dvxdy = 0, dvydx = 0, dvydy = 0, ugx = 0, ugy = 0;
                for (int j = 0; j < ncg; ++j) {
                    double gxj, gyj;
                    phys_grad(Jinv, dps[j], dpt[j], &gxj, &gyj);
                    long n = elem_node(m, ix, iy, j);
                    double ux = vx[n] - cx, uy = vy[n] - cy;
                    dvxdx += ux * gxj; dvxdy += ux * gyj;
                    dvydx += uy * gxj; dvydy += uy * gyj;
                    ugx += phi[j] * ux; ugy += phi[j] * uy;
                }
                /* sphere (R#26): the metric terms of the orthonormal frame, with v at the point */
                double kt = metric_tan(m, iy, t);
                double vgx = cx + ugx, vgy = cy + ugy;
                double eps11 = dvxdx - kt * vgy, eps22 = dvydy, eps12 = 0.5 * (dvxdy + dvydx + kt * vgx);
                double psi[MAXN];
                ora_dg_basis(ns, s, t, psi);
                for (int k = 0; k < ns; ++k) {
                    b11[k] += w * detJ * psi[k] * eps11;
                    b12[k] += w * detJ * psi[k] * eps12;
                    b22[k] += w * detJ * psi[k] * eps22;
                }
            }
        err |= solve_mass(ns, M, b11) | solve_mass(ns, M, b12) | solve_mass(ns, M, b22);
        for (int k = 0; k < ns; ++k) {
            E11[e * ns + k] = b11[k]; E12[e * ns + k] = b12[k]; E22[e * ns + k] = b22[k];
        }
    }
    return err ? -3 : 0;
}

/* O5 stress update: Listing 2, literally.
 *   h = max(0, H_i PSI<na,NGP>), a = min(1, max(0, A_i PSI<na,NGP>))
 *   P = Pstar * h * exp(-C (1-a)), C = 20
 *   e_c = E_c,i PSI<ns,NGP>
 *   DELTA = sqrt(DeltaMin^2 + 1.25 (e11^2+e22^2) + 1.5 e11 e22 + e12^2)
 *   S_c,i = (1 - 1/alpha) S_c,i + iMJwPSI_i (alphaInv (...))^T
 * iMJwPSI_i = M_K^{-1} [w_g |J_g| psi(g)] built column by column with the dense solve. */
int ora_stress(const ora_mesh* m, const ora_params* prm,
               const double* E11, const double* E12, const double* E22,
               const double* H, const double* A,
               double* S11, double* S12, double* S22) {
    int rc = check_mesh(m); if (rc) return rc;
    int ns = m->ns, na = m->na, ngp = ora_ngp(ns), ng = ngp * ngp;
    double xg[3], wg[3];
    ora_gauss(ngp, xg, wg);
    long N = (long)m->nx * m->ny;
    int err = 0;
#pragma omp parallel for schedule(static) reduction(| : err)
    for (long e = 0; e < N; ++e) {
        int ix = (int)(e % m->nx), iy = (int)(e / m->nx);
        double M[MAXN * MAXN];
        ora_element_mass(m, ix, iy, ns, ngp, M);
        double iMJwPSI[MAXN][MAXG];
        double hG[MAXG], aG[MAXG], P[MAXG], e11[MAXG], e12[MAXG], e22[MAXG];
        for (int gy = 0; gy < ngp; ++gy)
            for (int gx = 0; gx < ngp; ++gx) {
                int g = gy * ngp + gx;
                double s = xg[gx], t = xg[gy], w = wg[gx] * wg[gy];
                double detJ = ora_element_jacobian(m, ix, iy, s, t, NULL);
                double psiS[MAXN], psiA[MAXN];
                ora_dg_basis(ns, s, t, psiS);
                ora_dg_basis(na, s, t, psiA);
                double col[MAXN];
                for (int k = 0; k < ns; ++k) col[k] = w * detJ * psiS[k];
                err |= solve_mass(ns, M, col);
                for (int k = 0; k < ns; ++k) iMJwPSI[k][g] = col[k];
                double hv = 0, av = 0;
                for (int k = 0; k < na; ++k) { hv += H[e * na + k] * psiA[k]; av += A[e * na + k] * psiA[k]; }
                hG[g] = fmax(hv, 0.0);
                aG[g] = fmin(fmax(av, 0.0), 1.0);
                P[g] = prm->Pstar * hG[g] * exp(-prm->C_conc * (1.0 - aG[g]));
                double a11 = 0, a12 = 0, a22 = 0;
                for (int k = 0; k < ns; ++k) {
                    a11 += E11[e * ns + k] * psiS[k];
                    a12 += E12[e * ns + k] * psiS[k];
                    a22 += E22[e * ns + k] * psiS[k];
                }
                e11[g] = a11; e12[g] = a12; e22[g] = a22;
            }
        double alphaInv = 1.0 / prm->alpha;
        double fac = 1.0 - alphaInv;
        double r11[MAXG], r12[MAXG], r22[MAXG];
        for (int g = 0; g < ng; ++g) {
            double draw2 = 1.25 * (e11[g] * e11[g] + e22[g] * e22[g]) + 1.50 * e11[g] * e22[g] + e12[g] * e12[g];
            double DELTA = sqrt(prm->DeltaMin * prm->DeltaMin + draw2);
            double PDelta = P[g] / DELTA;
            double Prep = P[g];
            if (prm->replacement_pressure) Prep = P[g] * sqrt(draw2) / DELTA; /* R#4 variant */
            r11[g] = alphaInv * (PDelta * ((5.0 / 8.0) * e11[g] + (3.0 / 8.0) * e22[g]) - 0.5 * Prep);
            r12[g] = alphaInv * (PDelta * (1.0 / 4.0) * e12[g]);
            r22[g] = alphaInv * (PDelta * ((5.0 / 8.0) * e22[g] + (3.0 / 8.0) * e11[g]) - 0.5 * Prep);
        }
        for (int k = 0; k < ns; ++k) {
            double p11 = 0, p12 = 0, p22 = 0;
            for (int g = 0; g < ng; ++g) {
                p11 += iMJwPSI[k][g] * r11[g];
                p12 += iMJwPSI[k][g] * r12[g];
                p22 += iMJwPSI[k][g] * r22[g];
            }
            S11[e * ns + k] = fac * S11[e * ns + k] + p11;
            S12[e * ns + k] = fac * S12[e * ns + k] + p12;
            S22[e * ns + k] = fac * S22[e * ns + k] + p22;
        }
    }
    return err ? -3 : 0;
}

/* O6 divergence (Table 1 "divergence"; R#10): weak form
 *   F^x_j = - sum_{K ∋ j} sum_g w_g |J_g| [sigma11 dphi_j/dx + sigma12 dphi_j/dy]
 *   F^y_j = - sum_{K ∋ j} sum_g w_g |J_g| [sigma12 dphi_j/dx + sigma22 dphi_j/dy]
 * sigma_c(g) = sum_k S_c,k psi_k(g).  Element contributions first, then a
 * per-node gather over the adjacent elements.  On the sphere (R#26) the adjoint of the strain's
 * metric terms: + sigma12 phi_j tan(lat)/R in F^x, - sigma11 phi_j tan(lat)/R in F^y. */
int ora_divergence(const ora_mesh* m, const double* S11, const double* S12, const double* S22,
                   double* Fx, double* Fy) {
    int rc = check_mesh(m); if (rc) return rc;
    int ns = m->ns, p = m->p, ngp = ora_ngp(ns), ncg = (p + 1) * (p + 1);
    double xg[3], wg[3];
    ora_gauss(ngp, xg, wg);
    long N = (long)m->nx * m->ny;
    double* rx = (double*)malloc(sizeof(double) * N * ncg);
    double* ry = (double*)malloc(sizeof(double) * N * ncg);
    if (!rx || !ry) { free(rx); free(ry); return -4; }
#pragma omp parallel for schedule(static)
    for (long e = 0; e < N; ++e) {
        int ix = (int)(e % m->nx), iy = (int)(e / m->nx);
        double lx[MAXCG] = {0}, ly[MAXCG] = {0};
        for (int gy = 0; gy < ngp; ++gy)
            for (int gx = 0; gx < ngp; ++gx) {
                double s = xg[gx], t = xg[gy], w = wg[gx] * wg[gy];
                double Jinv[4];
                double detJ = ora_element_jacobian(m, ix, iy, s, t, Jinv);
                double psi[MAXN];
                ora_dg_basis(ns, s, t, psi);
                double s11 = 0, s12 = 0, s22 = 0;
                for (int k = 0; k < ns; ++k) {
                    s11 += S11[e * ns + k] * psi[k];
                    s12 += S12[e * ns + k] * psi[k];
                    s22 += S22[e * ns + k] * psi[k];
                }
                double phi[MAXCG], dps[MAXCG], dpt[MAXCG];
                ora_cg_basis(p, s, t, phi, dps, dpt);
                double kt = metric_tan(m, iy, t);   /* sphere: the adjoint of the strain's metric terms */
                for (int j = 0; j < ncg; ++j) {
                    double gxj, gyj;
                    phys_grad(Jinv, dps[j], dpt[j], &gxj, &gyj);
                    lx[j] -= w * detJ * (s11 * gxj + s12 * gyj + s12 * phi[j] * kt);
                    ly[j] -= w * detJ * (s12 * gxj + s22 * gyj - s11 * phi[j] * kt);
                }
            }
        for (int j = 0; j < ncg; ++j) { rx[e * ncg + j] = lx[j]; ry[e * ncg + j] = ly[j]; }
    }
    long NX = (long)p * m->nx + 1, NY = (long)p * m->ny + 1;
#pragma omp parallel for schedule(static)
    for (long J = 0; J < NY; ++J)
        for (long I = 0; I < NX; ++I) {
            double fx = 0, fy = 0;
            for (long iy = J / p - 1; iy <= J / p; ++iy)
                for (long ix = I / p - 1; ix <= I / p; ++ix) {
                    if (ix < 0 || iy < 0 || ix >= m->nx || iy >= m->ny) continue;
                    long jx = I - p * ix, jy = J - p * iy;
                    if (jx < 0 || jx > p || jy < 0 || jy > p) continue;
                    long e = iy * m->nx + ix;
                    int j = (int)(jy * (p + 1) + jx);
                    fx += rx[e * ncg + j];
                    fy += ry[e * ncg + j];
                }
            Fx[node_index(m, I, J)] = fx;
            Fy[node_index(m, I, J)] = fy;
        }
    free(rx); free(ry);
    return 0;
}

/* O7 lumped mass: m_j = sum_{K ∋ j} sum_g w_g |J_g| phi_j(g). */
int ora_lumped_mass(const ora_mesh* m, double* mass) {
    int rc = check_mesh(m); if (rc) return rc;
    int p = m->p, ngp = ora_ngp(m->ns), ncg = (p + 1) * (p + 1);
    double xg[3], wg[3];
    ora_gauss(ngp, xg, wg);
    long NX = (long)p * m->nx + 1, NY = (long)p * m->ny + 1;
#pragma omp parallel for schedule(static)
    for (long J = 0; J < NY; ++J)
        for (long I = 0; I < NX; ++I) {
            double acc = 0;
            for (long iy = J / p - 1; iy <= J / p; ++iy)
                for (long ix = I / p - 1; ix <= I / p; ++ix) {
                    if (ix < 0 || iy < 0 || ix >= m->nx || iy >= m->ny) continue;
                    long jx = I - p * ix, jy = J - p * iy;
                    if (jx < 0 || jx > p || jy < 0 || jy > p) continue;
                    int j = (int)(jy * (p + 1) + jx);
                    for (int gy = 0; gy < ngp; ++gy)
                        for (int gx = 0; gx < ngp; ++gx) {
                            double s = xg[gx], t = xg[gy], w = wg[gx] * wg[gy];
                            double detJ = ora_element_jacobian(m, (int)ix, (int)iy, s, t, NULL);
                            double phi[MAXCG];
                            ora_cg_basis(p, s, t, phi, NULL, NULL);
                            acc += w * detJ * phi[j];
                        }
                }
            mass[node_index(m, I, J)] = acc;
        }
    (void)ncg;
    return 0;
}

/* O10 DG -> CG (R#17): nodal mean over the adjacent elements of the DG
 * polynomial evaluated at the node, A clamped to [0,1], H floored at 1e-4. */
int ora_prep(const ora_mesh* m, const double* H, const double* A, double* Hn, double* An) {
    int rc = check_mesh(m); if (rc) return rc;
    int p = m->p, na = m->na;
    long NX = (long)p * m->nx + 1, NY = (long)p * m->ny + 1;
#pragma omp parallel for schedule(static)
    for (long J = 0; J < NY; ++J)
        for (long I = 0; I < NX; ++I) {
            double hs = 0, as = 0; int cnt = 0;
            for (long iy = J / p - 1; iy <= J / p; ++iy)
                for (long ix = I / p - 1; ix <= I / p; ++ix) {
                    if (ix < 0 || iy < 0 || ix >= m->nx || iy >= m->ny) continue;
                    long jx = I - p * ix, jy = J - p * iy;
                    if (jx < 0 || jx > p || jy < 0 || jy > p) continue;
                    long e = iy * m->nx + ix;
                    double psi[MAXN];
                    ora_dg_basis(na, (double)jx / p, (double)jy / p, psi);
                    double hv = 0, av = 0;
                    for (int k = 0; k < na; ++k) { hv += H[e * na + k] * psi[k]; av += A[e * na + k] * psi[k]; }
                    hs += hv; as += av; ++cnt;
                }
            double h = hs / cnt, a = as / cnt;
            Hn[node_index(m, I, J)] = fmax(h, 1e-4);
            An[node_index(m, I, J)] = fmin(fmax(a, 0.0), 1.0);
        }
    return 0;
}

static int on_boundary(const ora_mesh* m, long I, long J) {
    return I == 0 || J == 0 || I == (long)m->p * m->nx || J == (long)m->p * m->ny;
}

/* O8 velocity update (Eq. 2 P:107-111 with mEVP beta-relaxation; R#11, R#14, R#16).
 * Jacobi in (x, y): every right-hand side uses v^(p-1).  Boundary nodes -> 0. */
int ora_velocity(const ora_mesh* m, const ora_params* prm,
                 const double* Fx, const double* Fy, const double* mass,
                 const double* Hn, const double* An,
                 const double* vnx, const double* vny,
                 const double* ox, const double* oy, const double* ax, const double* ay,
                 double* vx, double* vy) {
    int rc = check_mesh(m); if (rc) return rc;
    if (m->bc != 0) return -2;
    long NX = (long)m->p * m->nx + 1, NY = (long)m->p * m->ny + 1;
    double Fa = prm->rho_atm * prm->C_atm, Fo = prm->rho_ocean * prm->C_ocean;
    double beta = prm->beta;
#pragma omp parallel for schedule(static)
    for (long J = 0; J < NY; ++J)
        for (long I = 0; I < NX; ++I) {
            long n = node_index(m, I, J);
            if (on_boundary(m, I, J)) { vx[n] = 0.0; vy[n] = 0.0; continue; }
            double vxo = vx[n], vyo = vy[n];
            double mm = prm->rho_ice * Hn[n];
            double c = mm / prm->dt;
            double w = sqrt((ox[n] - vxo) * (ox[n] - vxo) + (oy[n] - vyo) * (oy[n] - vyo));
            double amag = sqrt(ax[n] * ax[n] + ay[n] * ay[n]);
            double den = c * (1.0 + beta) + An[n] * Fo * w;
            double nx_ = c * (beta * vxo + vnx[n]) + An[n] * (Fa * amag * ax[n] + Fo * w * ox[n])
                         + mm * prm->f_c * (vyo - oy[n]) + Fx[n] / mass[n];
            double ny_ = c * (beta * vyo + vny[n]) + An[n] * (Fa * amag * ay[n] + Fo * w * oy[n])
                         + mm * prm->f_c * (ox[n] - vxo) + Fy[n] / mass[n];
            vx[n] = nx_ / den;
            vy[n] = ny_ / den;
        }
    return 0;
}

/* One outer step's n mEVP subcycles (Table 1 rows strain..velocity):
 * strain -> stress -> divergence -> velocity, n times, with v^n, H, A fixed. */
int ora_subcycles(const ora_mesh* m, const ora_params* prm, int nsub,
                  const double* H, const double* A,
                  const double* ox, const double* oy, const double* ax, const double* ay,
                  const double* vnx, const double* vny,
                  double* vx, double* vy, double* S11, double* S12, double* S22) {
    int rc = check_mesh(m); if (rc) return rc;
    long N = (long)m->nx * m->ny;
    long NN = ((long)m->p * m->nx + 1) * ((long)m->p * m->ny + 1);
    int ns = m->ns;
    double* E11 = (double*)malloc(sizeof(double) * N * ns);
    double* E12 = (double*)malloc(sizeof(double) * N * ns);
    double* E22 = (double*)malloc(sizeof(double) * N * ns);
    double* Fx = (double*)malloc(sizeof(double) * NN);
    double* Fy = (double*)malloc(sizeof(double) * NN);
    double* mass = (double*)malloc(sizeof(double) * NN);
    double* Hn = (double*)malloc(sizeof(double) * NN);
    double* An = (double*)malloc(sizeof(double) * NN);
    if (!E11 || !E12 || !E22 || !Fx || !Fy || !mass || !Hn || !An) { rc = -4; goto done; }
    if ((rc = ora_lumped_mass(m, mass))) goto done;
    if ((rc = ora_prep(m, H, A, Hn, An))) goto done;
    for (int it = 0; it < nsub; ++it) {
        if ((rc = ora_strain(m, vx, vy, E11, E12, E22))) goto done;
        if ((rc = ora_stress(m, prm, E11, E12, E22, H, A, S11, S12, S22))) goto done;
        if ((rc = ora_divergence(m, S11, S12, S22, Fx, Fy))) goto done;
        if ((rc = ora_velocity(m, prm, Fx, Fy, mass, Hn, An, vnx, vny, ox, oy, ax, ay, vx, vy))) goto done;
    }
done:
    free(E11); free(E12); free(E22); free(Fx); free(Fy); free(mass); free(Hn); free(An);
    return rc;
}

/* CG velocity at reference point (s,t) of element (ix,iy). */
static void cg_velocity(const ora_mesh* m, int ix, int iy, double s, double t,
                        const double* vx, const double* vy, double* ux, double* uy) {
    int ncg = (m->p + 1) * (m->p + 1);
    double phi[MAXCG];
    ora_cg_basis(m->p, s, t, phi, NULL, NULL);
    double a = 0, b = 0;
    for (int j = 0; j < ncg; ++j) {
        long n = elem_node(m, ix, iy, j);
        a += phi[j] * vx[n]; b += phi[j] * vy[n];
    }
    *ux = a; *uy = b;
}

static double dg_eval(int na, const double* c, double s, double t) {
    double psi[MAXN];
    ora_dg_basis(na, s, t, psi);
    double v = 0;
    for (int k = 0; k < na; ++k) v += c[k] * psi[k];
    return v;
}

/* O11 advection right-hand side (Eq. 1; R#18):
 *   M_K dc/dt = int_K c (v . grad psi) - sum_edges int_e c_hat (v . n) psi,
 * c_hat = trace from the side the flow leaves (v.n > 0 w.r.t. K's outward
 * normal -> K itself, else the neighbour).  Closed box: boundary edges carry
 * no flux.  Periodic: neighbours wrap. */
int ora_advect_rhs(const ora_mesh* m, const double* vx, const double* vy,
                   const double* c, double* rhs) {
    int rc = check_mesh(m); if (rc) return rc;
    int na = m->na, ngp = ora_ngp(m->ns);
    double xg[3], wg[3];
    ora_gauss(ngp, xg, wg);
    long N = (long)m->nx * m->ny;
    int err = 0;
#pragma omp parallel for schedule(static) reduction(| : err)
    for (long e = 0; e < N; ++e) {
        int ix = (int)(e % m->nx), iy = (int)(e / m->nx);
        double b[MAXN] = {0};
        /* volume term */
        for (int gy = 0; gy < ngp; ++gy)
            for (int gx = 0; gx < ngp; ++gx) {
                double s = xg[gx], t = xg[gy], w = wg[gx] * wg[gy];
                double Jinv[4];
                double detJ = ora_element_jacobian(m, ix, iy, s, t, Jinv);
                double ux, uy;
                cg_velocity(m, ix, iy, s, t, vx, vy, &ux, &uy);
                double cv = dg_eval(na, c + e * na, s, t);
                double dps[MAXN], dpt[MAXN];
                ora_dg_basis_grad(na, s, t, dps, dpt);
                for (int k = 0; k < na; ++k) {
                    double gxk, gyk;
                    phys_grad(Jinv, dps[k], dpt[k], &gxk, &gyk);
                    b[k] += w * detJ * cv * (ux * gxk + uy * gyk);
                }
            }
        /* edge terms: 0 east (s=1), 1 west (s=0), 2 north (t=1), 3 south (t=0) */
        for (int edge = 0; edge < 4; ++edge) {
            int nbx = ix, nby = iy;
            if (edge == 0) nbx = ix + 1;
            if (edge == 1) nbx = ix - 1;
            if (edge == 2) nby = iy + 1;
            if (edge == 3) nby = iy - 1;
            if (nbx < 0 || nbx >= m->nx || nby < 0 || nby >= m->ny) {
                if (m->bc == 0) continue; /* closed box: no boundary flux (R#16) */
                nbx = (nbx + m->nx) % m->nx;
                nby = (nby + m->ny) % m->ny;
            }
            long en = (long)nby * m->nx + nbx;
            for (int q = 0; q < ngp; ++q) {
                double r = xg[q], wq = wg[q];
                double s, t, sn, tn;
                int col;
                if (edge == 0) { s = 1.0; t = r; sn = 0.0; tn = r; col = 1; }
                else if (edge == 1) { s = 0.0; t = r; sn = 1.0; tn = r; col = 1; }
                else if (edge == 2) { s = r; t = 1.0; sn = r; tn = 0.0; col = 0; }
                else { s = r; t = 0.0; sn = r; tn = 1.0; col = 0; }
                double T[2];
                element_tangent(m, ix, iy, s, t, col, T);
                double len = sqrt(T[0] * T[0] + T[1] * T[1]);
                double nrm[2];
                if (col == 1) { nrm[0] = T[1] / len; nrm[1] = -T[0] / len; }  /* east outward */
                else { nrm[0] = -T[1] / len; nrm[1] = T[0] / len; }           /* north outward */
                if (edge == 1 || edge == 3) { nrm[0] = -nrm[0]; nrm[1] = -nrm[1]; }
                double ux, uy;
                cg_velocity(m, ix, iy, s, t, vx, vy, &ux, &uy);
                double vn = ux * nrm[0] + uy * nrm[1];
                double chat = vn > 0 ? dg_eval(na, c + e * na, s, t) : dg_eval(na, c + en * na, sn, tn);
                double psi[MAXN];
                ora_dg_basis(na, s, t, psi);
                for (int k = 0; k < na; ++k) b[k] -= wq * len * chat * vn * psi[k];
            }
        }
        double M[MAXN * MAXN];
        ora_element_mass(m, ix, iy, na, ngp, M);
        err |= solve_mass(na, M, b);
        for (int k = 0; k < na; ++k) rhs[e * na + k] = b[k];
    }
    return err ? -3 : 0;
}

/* Explicit RK of the advection ("higher order explicit Runge-Kutta"; R#18):
 * na=1 forward Euler, na=3 SSP-RK2 (Heun), na=6 SSP-RK3 (Shu-Osher). */
int ora_limit(const ora_mesh* m, double lo, double hi, double* c);

/* SSP-RK stages; with limiter != 0 the bound-preserving limiter (R#25) acts on every stage value. */
static int advect_one(const ora_mesh* m, double dt, const double* vx, const double* vy, double* c,
                      int limiter, double lo, double hi) {
    long n = (long)m->nx * m->ny * m->na;
    double* c0 = (double*)malloc(sizeof(double) * n);
    double* c1 = (double*)malloc(sizeof(double) * n);
    double* L = (double*)malloc(sizeof(double) * n);
    int rc = 0;
    if (!c0 || !c1 || !L) { rc = -4; goto done; }
    memcpy(c0, c, sizeof(double) * n);
    if ((rc = ora_advect_rhs(m, vx, vy, c0, L))) goto done;
    for (long i = 0; i < n; ++i) c1[i] = c0[i] + dt * L[i];
    if (limiter) ora_limit(m, lo, hi, c1);
    if (m->na == 1) {
        memcpy(c, c1, sizeof(double) * n);
    } else if (m->na == 3) {
        if ((rc = ora_advect_rhs(m, vx, vy, c1, L))) goto done;
        for (long i = 0; i < n; ++i) c[i] = 0.5 * c0[i] + 0.5 * (c1[i] + dt * L[i]);
        if (limiter) ora_limit(m, lo, hi, c);
    } else {
        if ((rc = ora_advect_rhs(m, vx, vy, c1, L))) goto done;
        double* c2 = c; /* reuse output as stage 2 */
        for (long i = 0; i < n; ++i) c2[i] = 0.75 * c0[i] + 0.25 * (c1[i] + dt * L[i]);
        if (limiter) ora_limit(m, lo, hi, c2);
        if ((rc = ora_advect_rhs(m, vx, vy, c2, L))) goto done;
        for (long i = 0; i < n; ++i) c[i] = (1.0 / 3.0) * c0[i] + (2.0 / 3.0) * (c2[i] + dt * L[i]);
        if (limiter) ora_limit(m, lo, hi, c);
    }
done:
    free(c0); free(c1); free(L);
    return rc;
}

int ora_advect(const ora_mesh* m, double dt, const double* vx, const double* vy,
               double* A, double* H) {
    int rc = check_mesh(m); if (rc) return rc;
    if ((rc = advect_one(m, dt, vx, vy, A, 0, 0.0, 0.0))) return rc;
    return advect_one(m, dt, vx, vy, H, 0, 0.0, 0.0);
}

/* NEXT-4 (R#25): bound-preserving scaling limiter of Zhang & Shu (maximum-principle-satisfying DG),
 * per element: with the physical mean cbar = int c |J| / int |J| (Gauss rule of the advection) and
 * the extremes cmin, cmax of c over the points where the scheme evaluates it - the ngp x ngp volume
 * Gauss points and the ngp Gauss points of each of the 4 edges -
 *   theta = min(1, (cbar - lo) / (cbar - cmin) if cmin < lo, (hi - cbar) / (cmax - cbar) if cmax > hi),
 * clamped to [0, 1], and c <- cbar + theta (c - cbar): the mean (mass) is kept, the values at the
 * check points land in [lo, hi] (hi = +inf for no upper bound). */
int ora_limit(const ora_mesh* m, double lo, double hi, double* c) {
    int rc = check_mesh(m); if (rc) return rc;
    int na = m->na, ngp = ora_ngp(m->ns), ng = ngp * ngp;
    if (na == 1) return 0;                       /* DG0: c is its own mean */
    double xg[3], wg[3];
    ora_gauss(ngp, xg, wg);
    long N = (long)m->nx * m->ny;
#pragma omp parallel for schedule(static)
    for (long e = 0; e < N; ++e) {
        int ix = (int)(e % m->nx), iy = (int)(e / m->nx);
        double* ce = c + e * na;
        double psi[MAXN], mass = 0.0, integ = 0.0;
        double cmin = INFINITY, cmax = -INFINITY;
        for (int gy = 0; gy < ngp; ++gy)
            for (int gx = 0; gx < ngp; ++gx) {
                double s = xg[gx], t = xg[gy], w = wg[gx] * wg[gy];
                double detJ = ora_element_jacobian(m, ix, iy, s, t, NULL);
                ora_dg_basis(na, s, t, psi);
                double v = 0.0;
                for (int k = 0; k < na; ++k) v += ce[k] * psi[k];
                integ += w * detJ * v;
                mass += w * detJ;
                cmin = fmin(cmin, v); cmax = fmax(cmax, v);
            }
        for (int edge = 0; edge < 4; ++edge)
            for (int q = 0; q < ngp; ++q) {
                double s = edge == 0 ? 1.0 : (edge == 1 ? 0.0 : xg[q]);
                double t = edge == 2 ? 1.0 : (edge == 3 ? 0.0 : xg[q]);
                ora_dg_basis(na, s, t, psi);
                double v = 0.0;
                for (int k = 0; k < na; ++k) v += ce[k] * psi[k];
                cmin = fmin(cmin, v); cmax = fmax(cmax, v);
            }
        double cbar = integ / mass, theta = 1.0;
        if (cmin < lo) theta = fmin(theta, (cbar - lo) / (cbar - cmin));
        if (cmax > hi) theta = fmin(theta, (hi - cbar) / (cmax - cbar));
        theta = fmax(0.0, fmin(1.0, theta));
        if (theta < 1.0) {
            /* c <- cbar + theta (c - cbar): psi_0 = 1, so the constant goes into coefficient 0 */
            for (int k = 0; k < na; ++k) ce[k] *= theta;
            ce[0] += (1.0 - theta) * cbar;
        }
    }
    (void)ng;
    return 0;
}

int ora_advect_limited(const ora_mesh* m, double dt, const double* vx, const double* vy,
                       double* A, double* H, int limiter) {
    int rc = check_mesh(m); if (rc) return rc;
    if ((rc = advect_one(m, dt, vx, vy, A, limiter, 0.0, 1.0))) return rc;       /* A in [0, 1] */
    return advect_one(m, dt, vx, vy, H, limiter, 0.0, INFINITY);                  /* H >= 0      */
}

/* One outer step in paper order (R#15): advect A, H with the current v,
 * snapshot v^n, then n mEVP subcycles. */
int ora_outer_step(const ora_mesh* m, const ora_params* prm, int nsub, int do_advect,
                   const double* ox, const double* oy, const double* ax, const double* ay,
                   double* vx, double* vy, double* S11, double* S12, double* S22,
                   double* A, double* H) {
    int rc = check_mesh(m); if (rc) return rc;
    if (do_advect && (rc = ora_advect(m, prm->dt, vx, vy, A, H))) return rc;
    long NN = ((long)m->p * m->nx + 1) * ((long)m->p * m->ny + 1);
    double* vnx = (double*)malloc(sizeof(double) * NN);
    double* vny = (double*)malloc(sizeof(double) * NN);
    if (!vnx || !vny) { free(vnx); free(vny); return -4; }
    memcpy(vnx, vx, sizeof(double) * NN);
    memcpy(vny, vy, sizeof(double) * NN);
    rc = ora_subcycles(m, prm, nsub, H, A, ox, oy, ax, ay, vnx, vny, vx, vy, S11, S12, S22);
    free(vnx); free(vny);
    return rc;
}
