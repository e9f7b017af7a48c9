// NEXT-1: the Listing 2 stress update on general quadrilaterals, with
// the per-element inverse map iMJwPSI_i = M_i^{-1} [w_g |J_g| psi(g)] either pre-assembled and
// stored for each element (Listing 1 caption) or recomputed on the fly from the element's
// four vertices ("fewer reads are required if we compute the matrices on-the-fly").
// This is the paper's Table 2 experiment on B200.  Geometry: bilinear map of the four
// vertices (DESIGN R#23); M_i by the stress Gauss rule, factorised by Cholesky.
#pragma once
#include "kernels.cuh"

namespace nxk {

struct GenArgs {
    const double* verts;   // (ny+1) x (nx+1) x 2
    double* maps;          // NS*NG planes: maps[(k*NG + g) * eplane + e]
    const double* E; double* S; const double* H; const double* A;
    int64_t eplane, epitch;
    int nx, ny;
    double ainv, fac, dmin2, Pstar, C_conc;
    int repl;
};

// Bilinear map x(s,t) of the element's four vertices: |J| = d0 + d1 s + d2 t exactly (the s t terms
// of x_s y_t - x_t y_s cancel), so |J| at the Gauss points and the element mass matrix need only the
// three coefficients.  Returns c0 = |J|(1/2, 1/2), d1, d2.
template <int P>
__device__ __forceinline__ void gen_geom(const GenArgs& a, int ix, int iy, double& c0, double& d1, double& d2) {
    const double* v00 = a.verts + 2 * ((int64_t)iy * (a.nx + 1) + ix);
    const double* v01 = v00 + 2 * (a.nx + 1);
    const double ax = v00[2] - v00[0], ay = v00[3] - v00[1];          // X10 - X00
    const double bx = v01[0] - v00[0], by = v01[1] - v00[1];          // X01 - X00
    const double cx = (v01[2] - v01[0]) - ax, cy = (v01[3] - v01[1]) - ay;   // X11 - X01 - X10 + X00
    const double d0 = ax * by - bx * ay;
    d1 = ax * cy - cx * ay;
    d2 = cx * by - bx * cy;
    c0 = d0 + 0.5 * (d1 + d2);
}
template <int P>
__device__ __forceinline__ void gen_wdet(double c0, double d1, double d2, double (&wdet)[Deg<P>::NG]) {
    const RefTab& T = c_tab[P - 1];
    constexpr int NGP = Deg<P>::NGP;
#pragma unroll
    for (int gy = 0; gy < NGP; ++gy)
#pragma unroll
        for (int gx = 0; gx < NGP; ++gx)
            wdet[gy * NGP + gx] = T.w[gy * NGP + gx] * fma(d1, T.gx[gx] - 0.5, fma(d2, T.gx[gy] - 0.5, c0));
}

// Cholesky factor (packed lower triangle, diagonal stored as its reciprocal) of
// M = sum_g w_g |J_g| psi psi^T in closed form:
// M = c0 D + d1 M_S + d2 M_T, D = diag(1, 1/12, 1/12, 1/180, 1/180, 1/144), M_S couples
// (0,1) 1/12, (1,3) 1/180, (2,5) 1/144 and M_T (0,2) 1/12, (2,4) 1/180, (1,5) 1/144 (exact
// moments of the centred Legendre family; the Gauss rule integrates them exactly).
template <int NS>
__device__ __forceinline__ void gen_mass_chol_n(double c0, double d1, double d2, double (&L)[NS * (NS + 1) / 2]) {
    const double D[6] = {1.0, 1.0 / 12.0, 1.0 / 12.0, 1.0 / 180.0, 1.0 / 180.0, 1.0 / 144.0};
    auto Mij = [&](int i, int j) -> double {   // lower triangle, indices are compile-time after unrolling
        if (i == j) return c0 * D[i];
        if (i == 1 && j == 0) return d1 * (1.0 / 12.0);
        if (i == 2 && j == 0) return d2 * (1.0 / 12.0);
        if (NS == 6 && i == 3 && j == 1) return d1 * (1.0 / 180.0);
        if (NS == 6 && i == 5 && j == 2) return d1 * (1.0 / 144.0);
        if (NS == 6 && i == 4 && j == 2) return d2 * (1.0 / 180.0);
        if (NS == 6 && i == 5 && j == 1) return d2 * (1.0 / 144.0);
        return 0.0;
    };
    // rectangular constant-trip loops with compile-time guards: fully unrolled, L stays in registers
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        double d = Mij(j, j);
#pragma unroll
        for (int k = 0; k < NS; ++k)
            if (k < j) d -= L[j * (j + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
        const double id = rsqrt_nr(d);          // the diagonal is kept as 1 / L_jj
        L[j * (j + 1) / 2 + j] = id;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            if (i <= j) continue;
            double v = Mij(i, j);
#pragma unroll
            for (int k = 0; k < NS; ++k)
                if (k < j) v -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
            L[i * (i + 1) / 2 + j] = v * id;
        }
    }
}
template <int P>
__device__ __forceinline__ void gen_mass_chol(double c0, double d1, double d2, double (&L)[Deg<P>::NS * (Deg<P>::NS + 1) / 2]) {
    gen_mass_chol_n<Deg<P>::NS>(c0, d1, d2, L);
}

template <int NS>
__device__ __forceinline__ void chol_solve(const double (&L)[NS * (NS + 1) / 2], double (&b)[NS]) {
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        double v = b[i];
#pragma unroll
        for (int k = 0; k < NS; ++k)
            if (k < i) v -= L[i * (i + 1) / 2 + k] * b[k];
        b[i] = v * L[i * (i + 1) / 2 + i];
    }
#pragma unroll
    for (int ii = 0; ii < NS; ++ii) {
        const int i = NS - 1 - ii;
        double v = b[i];
#pragma unroll
        for (int k = 0; k < NS; ++k)
            if (k > i) v -= L[k * (k + 1) / 2 + i] * b[k];
        b[i] = v * L[i * (i + 1) / 2 + i];
    }
}

// pre-assembly of iMJwPSI for every element (once per mesh)
template <int P>
__global__ void k_gen_maps(GenArgs a) {
    constexpr int NS = Deg<P>::NS, NG = Deg<P>::NG;
    const RefTab& T = c_tab[P - 1];
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, iy = blockIdx.y;
    if (ix >= a.nx || iy >= a.ny) return;
    double c0, d1, d2, det[NG], L[NS * (NS + 1) / 2];
    gen_geom<P>(a, ix, iy, c0, d1, d2);
    gen_wdet<P>(c0, d1, d2, det);
    gen_mass_chol<P>(c0, d1, d2, L);
    const int64_t e = (int64_t)iy * a.epitch + ix;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        double col[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) col[k] = det[g] * T.psi[k][g];
        chol_solve<NS>(L, col);
#pragma unroll
        for (int k = 0; k < NS; ++k) a.maps[(k * NG + g) * a.eplane + e] = col[k];
    }
}

// Listing 2 on general quads; ONFLY selects the on-the-fly map
template <int P, int NA, bool ONFLY>
__global__ void __launch_bounds__(128) k_stress_general(GenArgs a) {
    constexpr int NS = Deg<P>::NS, NG = Deg<P>::NG;
    const RefTab& T = c_tab[P - 1];
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, iy = blockIdx.y;
    if (ix >= a.nx || iy >= a.ny) return;
    const int64_t e = (int64_t)iy * a.epitch + ix;
    double r11[NG], r12[NG], r22[NG];
    if constexpr (P == 2 && NA == 6) {
        // structured Gauss-point values (separable P2 evaluation, as in k_subcycle_tma)
        double c[6], ev11[9], ev12[9], ev22[9], hg[9], ag[9];
#pragma unroll
        for (int k = 0; k < 6; ++k) c[k] = a.E[(0 * NS + k) * a.eplane + e];
        eval_gp<true, true>(c, ev11);
#pragma unroll
        for (int k = 0; k < 6; ++k) c[k] = a.E[(1 * NS + k) * a.eplane + e];
        eval_gp<true, true>(c, ev12);
#pragma unroll
        for (int k = 0; k < 6; ++k) c[k] = a.E[(2 * NS + k) * a.eplane + e];
        eval_gp<true, true>(c, ev22);
#pragma unroll
        for (int k = 0; k < 6; ++k) c[k] = a.H[k * a.eplane + e];
        eval_gp<true, true>(c, hg);
#pragma unroll
        for (int k = 0; k < 6; ++k) c[k] = a.A[k * a.eplane + e];
        eval_gp<true, true>(c, ag);
        const double hA = 0.5 * a.ainv;
#pragma unroll
        for (int g = 0; g < 9; ++g) {
            const double hv = fmax(hg[g], 0.0), av = fmin(fmax(ag[g], 0.0), 1.0);
            const double ph = a.Pstar * hv * exp(-a.C_conc * (1.0 - av)) * hA;   // alpha^{-1} P / 2
            const double x = ev11[g], y = ev22[g], z = ev12[g];
            const double draw2 = fma(z, z, fma(1.5 * x, y, 1.25 * fma(x, x, y * y)));
            const double rD = rsqrt_nr(draw2 + a.dmin2);
            const double pr = ph * rD;
            const double sub = a.repl ? pr * (draw2 > 0.0 ? draw2 * rsqrt_nr(draw2) : 0.0) : ph;
            r11[g] = fma(pr, fma(1.25, x, 0.75 * y), -sub);
            r22[g] = fma(pr, fma(1.25, y, 0.75 * x), -sub);
            r12[g] = 0.5 * pr * z;
        }
    } else {
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        double hv = 0, av = 0, e11 = 0, e12 = 0, e22 = 0;
#pragma unroll
        for (int k = 0; k < NA; ++k) { hv = fma(a.H[k * a.eplane + e], T.psi[k][g], hv); av = fma(a.A[k * a.eplane + e], T.psi[k][g], av); }
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            e11 = fma(a.E[(0 * NS + k) * a.eplane + e], T.psi[k][g], e11);
            e12 = fma(a.E[(1 * NS + k) * a.eplane + e], T.psi[k][g], e12);
            e22 = fma(a.E[(2 * NS + k) * a.eplane + e], T.psi[k][g], e22);
        }
        hv = fmax(hv, 0.0); av = fmin(fmax(av, 0.0), 1.0);
        const double Pp = a.Pstar * hv * exp(-a.C_conc * (1.0 - av));
        const double draw2 = 1.25 * (e11 * e11 + e22 * e22) + 1.5 * e11 * e22 + e12 * e12;
        const double DELTA = sqrt(a.dmin2 + draw2);
        const double PD = Pp / DELTA;
        const double Pr = a.repl ? Pp * sqrt(draw2) / DELTA : Pp;
        r11[g] = a.ainv * (PD * (0.625 * e11 + 0.375 * e22) - 0.5 * Pr);
        r12[g] = a.ainv * (PD * 0.25 * e12);
        r22[g] = a.ainv * (PD * (0.625 * e22 + 0.375 * e11) - 0.5 * Pr);
    }
    }
    double x11[NS], x12[NS], x22[NS];
    if (ONFLY) {
        double c0, d1, d2, det[NG], L[NS * (NS + 1) / 2];
        gen_geom<P>(a, ix, iy, c0, d1, d2);
        gen_wdet<P>(c0, d1, d2, det);
        gen_mass_chol<P>(c0, d1, d2, L);
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            double b11 = 0, b12 = 0, b22 = 0;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const double wp = det[g] * T.psi[k][g];
                b11 = fma(wp, r11[g], b11); b12 = fma(wp, r12[g], b12); b22 = fma(wp, r22[g], b22);
            }
            x11[k] = b11; x12[k] = b12; x22[k] = b22;
        }
        chol_solve<NS>(L, x11); chol_solve<NS>(L, x12); chol_solve<NS>(L, x22);
    } else {
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            double p11 = 0, p12 = 0, p22 = 0;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const double m = a.maps[(k * NG + g) * a.eplane + e];
                p11 = fma(m, r11[g], p11); p12 = fma(m, r12[g], p12); p22 = fma(m, r22[g], p22);
            }
            x11[k] = p11; x12[k] = p12; x22[k] = p22;
        }
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        double* s = a.S + e;
        s[(0 * NS + k) * a.eplane] = fma(a.fac, s[(0 * NS + k) * a.eplane], x11[k]);
        s[(1 * NS + k) * a.eplane] = fma(a.fac, s[(1 * NS + k) * a.eplane], x12[k]);
        s[(2 * NS + k) * a.eplane] = fma(a.fac, s[(2 * NS + k) * a.eplane], x22[k]);
    }
}

}  // namespace nxk
