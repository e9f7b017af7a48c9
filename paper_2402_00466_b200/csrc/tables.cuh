// K0 — element-matrix precompute (DESIGN.md §6 K0).
//
// Builds, on the device, every reference-element table the kernels use for
// one space (p, n_S) = (1, 3), (2, 6) or (2, 8), in FP64, and the kernels then read them from
// __constant__ memory (uniform across a warp -> constant-bank operands, the
// placement P:220 and P:254 recommend).  On the affine box every element map
// is x = x0 + diag(hx, hy) (s, t), so the per-element M_i^{-1} of Listing 1
// ("pre-assembled and stored for each element") collapses to one
// reference table R = M_ref^{-1} PSI W (|J| cancels) plus the scale
// factors 1/hx, 1/hy passed per launch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nxk {

struct RefTab {
    int ngp, ng, ncg;
    double gx[3], gw[3];        // 1D Gauss-Legendre on [0,1]
    double w[9];                // tensor weights, g = gy*ngp + gx
    double psi[8][9];           // DG basis psi_k(g) (hierarchical: PSI<n> = first n rows)
    double dpsis[8][9];         // d psi_k / ds at g
    double dpsit[8][9];         // d psi_k / dt at g
    double phi[9][9];           // CG basis phi_j(g)
    double dphis[9][9];         // d phi_j / ds at g
    double dphit[9][9];         // d phi_j / dt at g
    double mref[8];             // reference DG mass (diagonal: orthogonal basis)
    double R[8][9];             // iMJwPSI of the reference element: psi_k(g) w_g / mref_k
    double Ks[9][9];            // strain composite [g][j] = sum_k psi_k(g) sum_g' R[k][g'] dphis[j][g']
    double Kt[9][9];
    double Ds[9][8];            // divergence composite [j][k] = sum_g w_g dphis[j][g] psi_k(g)
    double Dt[9][8];
    double psinode[8][9];       // psi_k at CG node j (DG -> CG nodal evaluation)
    double L1[3][3];            // 1D Lagrange L_j(gx_q)
    double psiedge[4][8][3];    // psi_k on edge e at point q: e = 0 east (s=1), 1 west (s=0), 2 north (t=1), 3 south (t=0)
    double w1int[3];            // 1D integral of L_j over [0,1]
    double invm[3][3];          // 1 / (lumped node-mass factor) for in-element node position (q, jy)
};

__constant__ RefTab c_tab[3];   // [tab_index(p, n_S)]: (1,3) (2,6) (2,8)

__host__ __device__ constexpr int tab_index(int p, int ns) { return ns == 8 ? 2 : p - 1; }

// Lagrange basis on equispaced nodes x_m = m/p, product form.
__device__ inline void lagrange_eval(int p, double s, double* L, double* dL) {
    for (int j = 0; j <= p; ++j) {
        double xj = (double)j / p, val = 1.0, der = 0.0;
        for (int m = 0; m <= p; ++m) {
            if (m == j) continue;
            double xm = (double)m / p;
            double term = 1.0 / (xj - xm);
            // derivative by the product rule, accumulated alongside
            der = der * (s - xm) * term + val * term;
            val = val * (s - xm) * term;
        }
        L[j] = val; dL[j] = der;
    }
}

// Centred Legendre family on [0,1]: l0 = 1, l1 = S, l2 = S^2 - 1/12 (S = s - 1/2);
// 2D index k -> (a, b): (0,0) (1,0) (0,1) (2,0) (0,2) (1,1), and for n_S = 8 (R#24) (2,1) (1,2).
__device__ inline void legendre1(double s, double* l, double* dl) {
    double S = s - 0.5;
    l[0] = 1.0; l[1] = S; l[2] = S * S - 1.0 / 12.0;
    dl[0] = 0.0; dl[1] = 1.0; dl[2] = 2.0 * S;
}
__device__ inline void dg_basis(double s, double t, double* psi, double* ds, double* dt) {
    const int A[8] = {0, 1, 0, 2, 0, 1, 2, 1}, B[8] = {0, 0, 1, 0, 2, 1, 1, 2};
    double ls[3], dls[3], lt[3], dlt[3];
    legendre1(s, ls, dls);
    legendre1(t, lt, dlt);
    for (int k = 0; k < 8; ++k) {
        psi[k] = ls[A[k]] * lt[B[k]];
        if (ds) ds[k] = dls[A[k]] * lt[B[k]];
        if (dt) dt[k] = ls[A[k]] * dlt[B[k]];
    }
}

// One thread builds the whole table for degree p (it is tiny: ~800 doubles).
__global__ void k_build_tables(RefTab* out, int p, int ns) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    RefTab T;
    memset(&T, 0, sizeof(T));
    const int ngp = p + 1, ng = ngp * ngp, ncg = (p + 1) * (p + 1);
    T.ngp = ngp; T.ng = ng; T.ncg = ncg;
    // Gauss-Legendre (textbook abscissae +-1/sqrt3; 0, +-sqrt(3/5)) mapped to [0,1]
    if (ngp == 2) {
        double xi = rsqrt(3.0);
        T.gx[0] = 0.5 - 0.5 * xi; T.gx[1] = 0.5 + 0.5 * xi;
        T.gw[0] = 0.5; T.gw[1] = 0.5;
    } else {
        double xi = sqrt(0.6);
        T.gx[0] = 0.5 - 0.5 * xi; T.gx[1] = 0.5; T.gx[2] = 0.5 + 0.5 * xi;
        T.gw[0] = 5.0 / 18.0; T.gw[1] = 8.0 / 18.0; T.gw[2] = 5.0 / 18.0;
    }
    double L[3][3], dL[3][3];  // [q][j]
    for (int q = 0; q < ngp; ++q) lagrange_eval(p, T.gx[q], L[q], dL[q]);
    for (int j = 0; j <= p; ++j)
        for (int q = 0; q < ngp; ++q) T.L1[j][q] = L[q][j];
    for (int gy = 0; gy < ngp; ++gy)
        for (int gx = 0; gx < ngp; ++gx) {
            int g = gy * ngp + gx;
            T.w[g] = T.gw[gx] * T.gw[gy];
            double ps[8], ds[8], dt[8];
            dg_basis(T.gx[gx], T.gx[gy], ps, ds, dt);
            for (int k = 0; k < 8; ++k) { T.psi[k][g] = ps[k]; T.dpsis[k][g] = ds[k]; T.dpsit[k][g] = dt[k]; }
            for (int jy = 0; jy <= p; ++jy)
                for (int jx = 0; jx <= p; ++jx) {
                    int j = jy * (p + 1) + jx;
                    T.phi[j][g] = L[gx][jx] * L[gy][jy];
                    T.dphis[j][g] = dL[gx][jx] * L[gy][jy];
                    T.dphit[j][g] = L[gx][jx] * dL[gy][jy];
                }
        }
    for (int k = 0; k < 8; ++k) {
        double m = 0.0;
        for (int g = 0; g < ng; ++g) m += T.w[g] * T.psi[k][g] * T.psi[k][g];
        T.mref[k] = m;
        for (int g = 0; g < ng; ++g) T.R[k][g] = T.psi[k][g] * T.w[g] / m;
    }
    // strain composite: e(g) = sum_k psi_k(g) E_k, E_k = sum_g' R[k][g'] eps(g'), eps = dphi . v
    for (int g = 0; g < ng; ++g)
        for (int j = 0; j < ncg; ++j) {
            double as = 0.0, at = 0.0;
            for (int k = 0; k < ns; ++k) {
                double rs = 0.0, rt = 0.0;
                for (int h = 0; h < ng; ++h) { rs += T.R[k][h] * T.dphis[j][h]; rt += T.R[k][h] * T.dphit[j][h]; }
                as += T.psi[k][g] * rs; at += T.psi[k][g] * rt;
            }
            T.Ks[g][j] = as; T.Kt[g][j] = at;
        }
    for (int j = 0; j < ncg; ++j)
        for (int k = 0; k < ns; ++k) {
            double as = 0.0, at = 0.0;
            for (int g = 0; g < ng; ++g) { as += T.w[g] * T.dphis[j][g] * T.psi[k][g]; at += T.w[g] * T.dphit[j][g] * T.psi[k][g]; }
            T.Ds[j][k] = as; T.Dt[j][k] = at;
        }
    for (int jy = 0; jy <= p; ++jy)
        for (int jx = 0; jx <= p; ++jx) {
            double ps[8];
            dg_basis((double)jx / p, (double)jy / p, ps, nullptr, nullptr);
            for (int k = 0; k < 8; ++k) T.psinode[k][jy * (p + 1) + jx] = ps[k];
        }
    for (int q = 0; q < ngp; ++q) {
        double r = T.gx[q], ps[8];
        dg_basis(1.0, r, ps, nullptr, nullptr); for (int k = 0; k < 8; ++k) T.psiedge[0][k][q] = ps[k];
        dg_basis(0.0, r, ps, nullptr, nullptr); for (int k = 0; k < 8; ++k) T.psiedge[1][k][q] = ps[k];
        dg_basis(r, 1.0, ps, nullptr, nullptr); for (int k = 0; k < 8; ++k) T.psiedge[2][k][q] = ps[k];
        dg_basis(r, 0.0, ps, nullptr, nullptr); for (int k = 0; k < 8; ++k) T.psiedge[3][k][q] = ps[k];
    }
    for (int j = 0; j <= p; ++j) {
        double a = 0.0;
        for (int q = 0; q < ngp; ++q) a += T.gw[q] * L[q][j];
        T.w1int[j] = a;
    }
    // node-mass factor: a vertex column collects w1int[0] + w1int[p] from the two adjacent elements
    for (int q = 0; q < p; ++q)
        for (int jy = 0; jy < p; ++jy) {
            double fx = (q == 0) ? T.w1int[0] + T.w1int[p] : T.w1int[q];
            double fy = (jy == 0) ? T.w1int[0] + T.w1int[p] : T.w1int[jy];
            T.invm[q][jy] = 1.0 / (fx * fy);
        }
    *out = T;
}

}  // namespace nxk
