// NEXT-1 for the whole outer step: the unfused step kernels on general (distorted)
// quadrilaterals with the bilinear map of each element's four vertices (DESIGN R#23).
//   w |J| grad(phi) = w adj(J)^T grad_ref(phi): |J| cancels in every weak form, so strain,
//   divergence and the advection volume term need no division; the element mass matrix is the
//   closed form c0 D + d1 M_S + d2 M_T of general_quads.cuh (Cholesky, reciprocal diagonal).
//   Edge normals x |edge| come from the edge's two end vertices, identical on both sides.
// Kernels: lumped node masses (once per mesh), strain, divergence (element contributions, then a
// fixed-order node gather), velocity (uses the lumped masses), advection stage.
#pragma once
#include "general_quads.cuh"

namespace nxk {

struct GeomJ { double xs, xt, ys, yt; };   // columns of J at a point

struct ElemGeom {
    double X00, Y00, ax, ay, bx, by, cx, cy;
    __device__ __forceinline__ GeomJ at(double s, double t) const {
        return GeomJ{fma(t, cx, ax), fma(s, cx, bx), fma(t, cy, ay), fma(s, cy, by)};
    }
};
__device__ __forceinline__ ElemGeom elem_geom(const double* verts, int nx, int ix, int iy) {
    const double* v00 = verts + 2 * ((int64_t)iy * (nx + 1) + ix);
    const double* v01 = v00 + 2 * (nx + 1);
    ElemGeom g;
    g.X00 = v00[0]; g.Y00 = v00[1];
    g.ax = v00[2] - v00[0]; g.ay = v00[3] - v00[1];
    g.bx = v01[0] - v00[0]; g.by = v01[1] - v00[1];
    g.cx = (v01[2] - v01[0]) - g.ax; g.cy = (v01[3] - v01[1]) - g.ay;
    return g;
}

struct GenStepArgs {
    const double* verts;
    const double* vx_in; const double* vy_in; double* vx_out; double* vy_out;
    double* S; double* E; double* Fx; double* Fy; double* contrib;   // contrib: 2*NCG planes
    double* mlump;
    double* imlump;                         // -1 / m (0 where m <= 0): the fused subcycle's F / m factor
    const double* H; const double* A;
    const double* c1; const double* rx0; const double* ry0; const double* cafo; const double* ox; const double* oy;
    int64_t eplane, epitch, npitch;
    int nx, ny;
    double beta, b1, kc;
};

// lumped mass m_j = sum_{K ∋ j} sum_g w_g |J_g| phi_j(g)  (per node, fixed order SW, SE, NW, NE)
template <int P>
__global__ void k_gen_lumped(GenStepArgs a) {
    const RefTab& T = c_tab[P - 1];
    constexpr int NGP = P + 1;
    const int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y;
    if (I > P * a.nx || J > P * a.ny) return;
    double m = 0.0;
#pragma unroll
    for (int dy = 1; dy >= 0; --dy)
#pragma unroll
        for (int dx = 1; dx >= 0; --dx) {
            const int ex = I / P - dx, ey = J / P - dy, jx = I - P * ex, jy = J - P * ey;
            if (ex < 0 || ex >= a.nx || ey < 0 || ey >= a.ny || jx < 0 || jx > P || jy < 0 || jy > P) continue;
            double c0, d1, d2;
            GenArgs ga{}; ga.verts = a.verts; ga.nx = a.nx;
            gen_geom<P>(ga, ex, ey, c0, d1, d2);
            const int j = jy * (P + 1) + jx;
#pragma unroll
            for (int gy = 0; gy < NGP; ++gy)
#pragma unroll
                for (int gx = 0; gx < NGP; ++gx) {
                    const int g = gy * NGP + gx;
                    m = fma(T.w[g] * fma(d1, T.gx[gx] - 0.5, fma(d2, T.gx[gy] - 0.5, c0)), T.phi[j][g], m);
                }
        }
    a.mlump[(int64_t)J * a.npitch + I] = m;
    if (a.imlump) a.imlump[(int64_t)J * a.npitch + I] = m > 0.0 ? -rcp_nr(m) : 0.0;   // the fused kernel's factor
}

// strain: E_c = M_K^{-1} sum_g w_g |J_g| psi(g) eps_c(g), with w |J| eps from adj(J) (R#9)
template <int P>
__global__ void k_strain_gen(GenStepArgs a) {
    constexpr int NS = Deg<P>::NS, NGP = P + 1, NCG = (P + 1) * (P + 1);
    const RefTab& T = c_tab[P - 1];
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, iy = blockIdx.y;
    if (ix >= a.nx || iy >= a.ny) return;
    double ux[NCG], uy[NCG];
    const int64_t nref = (int64_t)(P * iy + P / 2) * a.npitch + P * ix + P / 2;
    const double rx = a.vx_in[nref], ry = a.vy_in[nref];   // reference node: cancellation-free differences
#pragma unroll
    for (int jy = 0; jy <= P; ++jy)
#pragma unroll
        for (int jx = 0; jx <= P; ++jx) {
            const int64_t n = (int64_t)(P * iy + jy) * a.npitch + P * ix + jx;
            ux[jy * (P + 1) + jx] = a.vx_in[n] - rx; uy[jy * (P + 1) + jx] = a.vy_in[n] - ry;
        }
    const ElemGeom G = elem_geom(a.verts, a.nx, ix, iy);
    double b11[NS], b12[NS], b22[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) { b11[k] = 0.0; b12[k] = 0.0; b22[k] = 0.0; }
#pragma unroll
    for (int gy = 0; gy < NGP; ++gy)
#pragma unroll
        for (int gx = 0; gx < NGP; ++gx) {
            const int g = gy * NGP + gx;
            const GeomJ Jg = G.at(T.gx[gx], T.gx[gy]);
            double us = 0, ut = 0, vs = 0, vt = 0;
#pragma unroll
            for (int j = 0; j < NCG; ++j) {
                us = fma(T.dphis[j][g], ux[j], us); ut = fma(T.dphit[j][g], ux[j], ut);
                vs = fma(T.dphis[j][g], uy[j], vs); vt = fma(T.dphit[j][g], uy[j], vt);
            }
            // w |J| (d/dx, d/dy) = w (yt d/ds - ys d/dt, -xt d/ds + xs d/dt)
            const double w = T.w[g];
            const double e11 = w * (Jg.yt * us - Jg.ys * ut);
            const double e22 = w * (Jg.xs * vt - Jg.xt * vs);
            const double e12 = 0.5 * w * ((Jg.xs * ut - Jg.xt * us) + (Jg.yt * vs - Jg.ys * vt));
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                b11[k] = fma(T.psi[k][g], e11, b11[k]);
                b12[k] = fma(T.psi[k][g], e12, b12[k]);
                b22[k] = fma(T.psi[k][g], e22, b22[k]);
            }
        }
    double c0, d1, d2, L[NS * (NS + 1) / 2];
    GenArgs ga{}; ga.verts = a.verts; ga.nx = a.nx;
    gen_geom<P>(ga, ix, iy, c0, d1, d2);
    gen_mass_chol<P>(c0, d1, d2, L);
    chol_solve<NS>(L, b11); chol_solve<NS>(L, b12); chol_solve<NS>(L, b22);
    const int64_t e = (int64_t)iy * a.epitch + ix;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        a.E[(0 * NS + k) * a.eplane + e] = b11[k];
        a.E[(1 * NS + k) * a.eplane + e] = b12[k];
        a.E[(2 * NS + k) * a.eplane + e] = b22[k];
    }
}

// divergence, element part: r_j = -sum_g w |J| (sigma . grad phi_j) for the NCG local nodes
template <int P>
__global__ void k_div_contrib_gen(GenStepArgs a) {
    constexpr int NS = Deg<P>::NS, NGP = P + 1, NCG = (P + 1) * (P + 1);
    const RefTab& T = c_tab[P - 1];
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, iy = blockIdx.y;
    if (ix >= a.nx || iy >= a.ny) return;
    const int64_t e = (int64_t)iy * a.epitch + ix;
    double s11[NS], s12[NS], s22[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        s11[k] = a.S[(0 * NS + k) * a.eplane + e]; s12[k] = a.S[(1 * NS + k) * a.eplane + e];
        s22[k] = a.S[(2 * NS + k) * a.eplane + e];
    }
    const ElemGeom G = elem_geom(a.verts, a.nx, ix, iy);
    double rx[NCG], ry[NCG];
#pragma unroll
    for (int j = 0; j < NCG; ++j) { rx[j] = 0.0; ry[j] = 0.0; }
#pragma unroll
    for (int gy = 0; gy < NGP; ++gy)
#pragma unroll
        for (int gx = 0; gx < NGP; ++gx) {
            const int g = gy * NGP + gx;
            const GeomJ Jg = G.at(T.gx[gx], T.gx[gy]);
            double a11 = 0, a12 = 0, a22 = 0;
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                a11 = fma(s11[k], T.psi[k][g], a11); a12 = fma(s12[k], T.psi[k][g], a12); a22 = fma(s22[k], T.psi[k][g], a22);
            }
            const double w = T.w[g];
#pragma unroll
            for (int j = 0; j < NCG; ++j) {
                const double gxj = Jg.yt * T.dphis[j][g] - Jg.ys * T.dphit[j][g];   // |J| dphi/dx
                const double gyj = Jg.xs * T.dphit[j][g] - Jg.xt * T.dphis[j][g];   // |J| dphi/dy
                rx[j] -= w * (a11 * gxj + a12 * gyj);
                ry[j] -= w * (a12 * gxj + a22 * gyj);
            }
        }
#pragma unroll
    for (int j = 0; j < NCG; ++j) {
        a.contrib[j * a.eplane + e] = rx[j];
        a.contrib[(NCG + j) * a.eplane + e] = ry[j];
    }
}
// divergence, node gather in the fixed order SW, SE, NW, NE
template <int P>
__global__ void k_div_gather_gen(GenStepArgs a) {
    constexpr int NCG = (P + 1) * (P + 1);
    const int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y;
    if (I > P * a.nx || J > P * a.ny) return;
    double fx = 0.0, fy = 0.0;
#pragma unroll
    for (int dy = 1; dy >= 0; --dy)
#pragma unroll
        for (int dx = 1; dx >= 0; --dx) {
            const int ex = I / P - dx, ey = J / P - dy, jx = I - P * ex, jy = J - P * ey;
            if (ex < 0 || ex >= a.nx || ey < 0 || ey >= a.ny || jx < 0 || jx > P || jy < 0 || jy > P) continue;
            const int64_t e = (int64_t)ey * a.epitch + ex;
            const int j = jy * (P + 1) + jx;
            fx += a.contrib[j * a.eplane + e];
            fy += a.contrib[(NCG + j) * a.eplane + e];
        }
    const int64_t n = (int64_t)J * a.npitch + I;
    a.Fx[n] = fx; a.Fy[n] = fy;
}

// velocity (R#11) with the per-node lumped mass of the general mesh
template <int P>
__global__ void k_velocity_gen(GenStepArgs a) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y;
    if (I > P * a.nx || J > P * a.ny) return;
    const int64_t n = (int64_t)J * a.npitch + I;
    if (I == 0 || I == P * a.nx || J == 0 || J == P * a.ny) { a.vx_out[n] = 0.0; a.vy_out[n] = 0.0; return; }
    const double mass = a.mlump[n];
    const double vxo = a.vx_in[n], vyo = a.vy_in[n];
    const double c1 = a.c1[n], cf = a.cafo[n], oxv = a.ox[n], oyv = a.oy[n];
    const double w = sqrt((oxv - vxo) * (oxv - vxo) + (oyv - vyo) * (oyv - vyo));
    const double den = c1 * a.b1 + cf * w;
    const double nx_ = c1 * a.beta * vxo + a.rx0[n] + cf * w * oxv + c1 * a.kc * vyo + a.Fx[n] / mass;
    const double ny_ = c1 * a.beta * vyo + a.ry0[n] + cf * w * oyv - c1 * a.kc * vxo + a.Fy[n] / mass;
    a.vx_out[n] = nx_ / den;
    a.vy_out[n] = ny_ / den;
}

// ---------------------------------------------------------------- advection on general quads
template <int P, int NA>
__device__ __forceinline__ void gen_edge_flux(int dir, const Cf<NA>& lo, const Cf<NA>& hi, const double* vxn,
                                              const double* vyn, double ex, double ey, bool open, double* FA, double* FH) {
    // (ex, ey) = edge vector from its first to its second end vertex (lo's east or north edge);
    // normal x |edge| for the +x-ish (vertical edge) / +y-ish (horizontal edge) direction
    const RefTab& T = c_tab[P - 1];
    const double nxl = dir == 0 ? ey : -ey, nyl = dir == 0 ? -ex : ex;
    const int elo = dir == 0 ? 0 : 2, ehi = dir == 0 ? 1 : 3;
#pragma unroll
    for (int q = 0; q < P + 1; ++q) {
        double ux = 0.0, uy = 0.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) { ux = fma(T.L1[j][q], vxn[j], ux); uy = fma(T.L1[j][q], vyn[j], uy); }
        const double vn = fma(ux, nxl, uy * nyl);   // (v . n) |edge|
        double lA = 0.0, lH = 0.0, hA = 0.0, hH = 0.0;
#pragma unroll
        for (int k = 0; k < NA; ++k) {
            lA = fma(lo.A[k], T.psiedge[elo][k][q], lA); lH = fma(lo.H[k], T.psiedge[elo][k][q], lH);
            hA = fma(hi.A[k], T.psiedge[ehi][k][q], hA); hH = fma(hi.H[k], T.psiedge[ehi][k][q], hH);
        }
        const bool from_lo = vn > 0.0;
        const double vo = open ? vn : 0.0;
        FA[q] = (from_lo ? lA : hA) * vo;
        FH[q] = (from_lo ? lH : hH) * vo;
    }
}

struct GenAdvArgs {
    AdvArgs b;
    const double* verts;
    int ny;
};

template <int P, int NA>
__global__ void __launch_bounds__(32 * ADV_ROWS, 3) k_advect_gen(GenAdvArgs ga) {
    constexpr int NGP = P + 1;
    const RefTab& T = c_tab[P - 1];
    const AdvArgs& a = ga.b;
    __shared__ double sFA[ADV_ROWS][32][NGP], sFH[ADV_ROWS][32][NGP];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int ix = blockIdx.x * 32 + tx;
    const int lr = a.erow_begin + blockIdx.y * ADV_ROWS + ty;
    const bool valid = ix < a.nx && lr < a.erow_end;
    const int ixc = valid ? ix : 0, lrc = valid ? lr : a.erow_begin;
    const int64_t e = (int64_t)lrc * a.epitch + ixc;
    Cf<NA> me; load_coef<P, NA>(a, e, me);
    double ux[P + 1][P + 1], uy[P + 1][P + 1];
#pragma unroll
    for (int jy = 0; jy <= P; ++jy)
#pragma unroll
        for (int jx = 0; jx <= P; ++jx) {
            const int64_t n = (int64_t)(P * lrc + jy) * a.npitch + P * ixc + jx;
            ux[jy][jx] = a.vx[n]; uy[jy][jx] = a.vy[n];
        }
    const double* v00 = ga.verts + 2 * ((int64_t)lrc * (a.nx + 1) + ixc);
    const double* v01 = v00 + 2 * (a.nx + 1);
    auto nb_index = [&](int ex, int ey, bool& open) -> int64_t {
        open = true;
        if (ex < 0 || ex >= a.nx) { open = false; return e; }
        if (ey < a.erow_begin || ey >= a.erow_end) { open = false; return e; }
        return (int64_t)ey * a.epitch + ex;
    };
    double FeA[NGP], FeH[NGP], FnA[NGP], FnH[NGP], FwA[NGP], FwH[NGP], FsA[NGP], FsH[NGP];
    double vxn[P + 1], vyn[P + 1];
    {   // east edge: vertices (ix+1, iy) -> (ix+1, iy+1)
        bool open; const int64_t en = nb_index(ixc + 1, lrc, open);
        Cf<NA> nb; load_coef<P, NA>(a, en, nb);
#pragma unroll
        for (int j = 0; j <= P; ++j) { vxn[j] = ux[j][P]; vyn[j] = uy[j][P]; }
        gen_edge_flux<P, NA>(0, me, nb, vxn, vyn, v01[2] - v00[2], v01[3] - v00[3], open, FeA, FeH);
    }
    {   // north edge: vertices (ix, iy+1) -> (ix+1, iy+1)
        bool open; const int64_t en = nb_index(ixc, lrc + 1, open);
        Cf<NA> nb; load_coef<P, NA>(a, en, nb);
#pragma unroll
        for (int j = 0; j <= P; ++j) { vxn[j] = ux[P][j]; vyn[j] = uy[P][j]; }
        gen_edge_flux<P, NA>(1, me, nb, vxn, vyn, v01[2] - v01[0], v01[3] - v01[1], open, FnA, FnH);
    }
#pragma unroll
    for (int q = 0; q < NGP; ++q) {
        FwA[q] = __shfl_up_sync(0xffffffffu, FeA[q], 1);
        FwH[q] = __shfl_up_sync(0xffffffffu, FeH[q], 1);
    }
    if (tx == 0) {   // west edge = the west neighbour's east edge: (ix, iy) -> (ix, iy+1)
        bool open; const int64_t wn = nb_index(ixc - 1, lrc, open);
        Cf<NA> nb; load_coef<P, NA>(a, wn, nb);
#pragma unroll
        for (int j = 0; j <= P; ++j) { vxn[j] = ux[j][0]; vyn[j] = uy[j][0]; }
        gen_edge_flux<P, NA>(0, nb, me, vxn, vyn, v01[0] - v00[0], v01[1] - v00[1], open, FwA, FwH);
    }
#pragma unroll
    for (int q = 0; q < NGP; ++q) { sFA[ty][tx][q] = FnA[q]; sFH[ty][tx][q] = FnH[q]; }
    __syncthreads();
    if (ty > 0) {
#pragma unroll
        for (int q = 0; q < NGP; ++q) { FsA[q] = sFA[ty - 1][tx][q]; FsH[q] = sFH[ty - 1][tx][q]; }
    } else {   // south edge = the south neighbour's north edge: (ix, iy) -> (ix+1, iy)
        bool open; const int64_t sn = nb_index(ixc, lrc - 1, open);
        Cf<NA> nb; load_coef<P, NA>(a, sn, nb);
#pragma unroll
        for (int j = 0; j <= P; ++j) { vxn[j] = ux[0][j]; vyn[j] = uy[0][j]; }
        gen_edge_flux<P, NA>(1, nb, me, vxn, vyn, v00[2] - v00[0], v00[3] - v00[1], open, FsA, FsH);
    }
    if (!valid) return;
    const ElemGeom G = elem_geom(ga.verts, a.nx, ixc, lrc);
    double LA[NA], LH[NA];
#pragma unroll
    for (int k = 0; k < NA; ++k) { LA[k] = 0.0; LH[k] = 0.0; }
#pragma unroll
    for (int gy = 0; gy < NGP; ++gy)
#pragma unroll
        for (int gx = 0; gx < NGP; ++gx) {
            const int g = gy * NGP + gx;
            const GeomJ Jg = G.at(T.gx[gx], T.gx[gy]);
            double vxg = 0.0, vyg = 0.0, cA = 0.0, cH = 0.0;
#pragma unroll
            for (int jy = 0; jy <= P; ++jy)
#pragma unroll
                for (int jx = 0; jx <= P; ++jx) {
                    const int j = jy * (P + 1) + jx;
                    vxg = fma(T.phi[j][g], ux[jy][jx], vxg);
                    vyg = fma(T.phi[j][g], uy[jy][jx], vyg);
                }
#pragma unroll
            for (int k = 0; k < NA; ++k) { cA = fma(me.A[k], T.psi[k][g], cA); cH = fma(me.H[k], T.psi[k][g], cH); }
            // w |J| v . grad psi_k = w [vx (yt psi_s - ys psi_t) + vy (xs psi_t - xt psi_s)]
            const double ps = T.w[g] * (vxg * Jg.yt - vyg * Jg.xt), pt = T.w[g] * (vyg * Jg.xs - vxg * Jg.ys);
#pragma unroll
            for (int k = 1; k < NA; ++k) {
                const double gk = ps * T.dpsis[k][g] + pt * T.dpsit[k][g];
                LA[k] = fma(cA, gk, LA[k]);
                LH[k] = fma(cH, gk, LH[k]);
            }
        }
#pragma unroll
    for (int q = 0; q < NGP; ++q) {
        const double w = T.gw[q];
#pragma unroll
        for (int k = 0; k < NA; ++k) {
            LA[k] -= w * (FeA[q] * T.psiedge[0][k][q] - FwA[q] * T.psiedge[1][k][q] + FnA[q] * T.psiedge[2][k][q] - FsA[q] * T.psiedge[3][k][q]);
            LH[k] -= w * (FeH[q] * T.psiedge[0][k][q] - FwH[q] * T.psiedge[1][k][q] + FnH[q] * T.psiedge[2][k][q] - FsH[q] * T.psiedge[3][k][q]);
        }
    }
    // M_K^{-1}: closed-form element mass of the first NA basis functions
    double c0, d1, d2;
    {
        GenArgs gga{}; gga.verts = ga.verts; gga.nx = a.nx;
        gen_geom<P>(gga, ix, lr, c0, d1, d2);
    }
    if (NA == 1) {
        LA[0] *= 1.0 / c0; LH[0] *= 1.0 / c0;
    } else {
        double L[NA * (NA + 1) / 2];
        gen_mass_chol_n<NA>(c0, d1, d2, L);
        chol_solve<NA>(L, LA); chol_solve<NA>(L, LH);
    }
    const int64_t eo = (int64_t)lr * a.epitch + ix;
#pragma unroll
    for (int k = 0; k < NA; ++k) {
        const double outA = a.a1 * (me.A[k] + a.dt * LA[k]);
        const double outH = a.a1 * (me.H[k] + a.dt * LH[k]);
        a.Aout[k * a.eplane + eo] = (a.a0 != 0.0) ? a.a0 * a.A0[k * a.eplane + eo] + outA : outA;
        a.Hout[k * a.eplane + eo] = (a.a0 != 0.0) ? a.a0 * a.H0[k * a.eplane + eo] + outH : outH;
    }
}

}  // namespace nxk
