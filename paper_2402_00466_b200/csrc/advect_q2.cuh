// K4 for CG2 velocity and DG2 tracers (n_A = 6, the configs' pair): the advection stage of
// kernels.cuh (k_advect) with the reference tables folded into the code:
//   Q2 values at the Gauss points / on edges   row pass (V0+V2, V0-V2, V1) -> 0.3 s + 0.4 V1 +- a d
//   DG2 traces on an edge                       A + T B + c_q q(T) with A, B from 3 coefficients
//   volume term  int c v.grad psi_k             1D moments sum w G, sum w S G, sum w T G of c vx, c vy
//   edge term    int c_hat (v.n) psi_k          moments sum w F, sum w T F, sum w q(T) F
// Same block layout and flux sharing as k_advect: each element evaluates its east and north
// edges; the west edge comes from lane-1 by shuffle, the south edge from the row below
// through shared memory; block-border elements evaluate those edges with the same function,
// so both sides of every edge use bitwise-identical fluxes.
#pragma once
#include "kernels.cuh"
#include "subcycle_tma.cuh"   // eval_gp: DG2 values at the 3 x 3 Gauss points

namespace nxk {

constexpr double kAdvA = 0.38729833462074170;   // sqrt(3/5)/2

__device__ __forceinline__ void q2_interp3(double n0, double n1, double n2, double out[3]) {
    const double s = n0 + n2, d = n0 - n2, m = fma(0.3, s, 0.4 * n1);
    out[0] = fma(kAdvA, d, m); out[1] = n1; out[2] = fma(-kAdvA, d, m);
}
// trace at s = 1 (east side, sg = +1) or s = 0 (sg = -1), at the 3 edge Gauss points in t
__device__ __forceinline__ void trace_s(const double c[6], double sg, double out[3]) {
    const double A = fma(sg * 0.5, c[1], fma(c[3], 1.0 / 6.0, c[0])), B = fma(sg * 0.5, c[5], c[2]);
    const double P = fma(c[4], 1.0 / 15.0, A);
    out[0] = fma(-kAdvA, B, P); out[1] = fma(c[4], -1.0 / 12.0, A); out[2] = fma(kAdvA, B, P);
}
// trace at t = 1 (north, sg = +1) or t = 0 (sg = -1), at the 3 edge Gauss points in s
__device__ __forceinline__ void trace_t(const double c[6], double sg, double out[3]) {
    const double A = fma(sg * 0.5, c[2], fma(c[4], 1.0 / 6.0, c[0])), B = fma(sg * 0.5, c[5], c[1]);
    const double P = fma(c[3], 1.0 / 15.0, A);
    out[0] = fma(-kAdvA, B, P); out[1] = fma(c[3], -1.0 / 12.0, A); out[2] = fma(kAdvA, B, P);
}
// upwind flux values on one edge for both tracers: vn = normal velocity (positive from lo to hi)
__device__ __forceinline__ void q2_edge(bool vert, const Cf<6>& lo, const Cf<6>& hi, const double vn[3], bool open,
                                        double FA[3], double FH[3]) {
    double la[3], lh[3], ha[3], hh[3];
    if (vert) { trace_s(lo.A, 1.0, la); trace_s(lo.H, 1.0, lh); trace_s(hi.A, -1.0, ha); trace_s(hi.H, -1.0, hh); }
    else { trace_t(lo.A, 1.0, la); trace_t(lo.H, 1.0, lh); trace_t(hi.A, -1.0, ha); trace_t(hi.H, -1.0, hh); }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const bool up = vn[q] > 0.0;
        const double v = open ? vn[q] : 0.0;
        FA[q] = (up ? la[q] : ha[q]) * v;
        FH[q] = (up ? lh[q] : hh[q]) * v;
    }
}
// edge moments: m0 = sum w F, m1 = sum w T F, m2 = sum w (T^2 - 1/12) F
__device__ __forceinline__ void edge_mom(const double F[3], double& m0, double& m1, double& m2) {
    const double s = F[0] + F[2];
    m0 = fma(5.0, s, 8.0 * F[1]) * (1.0 / 18.0);
    m1 = (F[2] - F[0]) * (5.0 * kAdvA / 18.0);
    m2 = fma(-2.0, F[1], s) * (1.0 / 54.0);
}
// volume moments of G[gy][gx]: M00 = sum w G, M10 = sum w S G, M01 = sum w T G
__device__ __forceinline__ void vol_mom(const double G[3][3], double& M00, double& M10, double& M01) {
    double X0[3], X1[3];
#pragma unroll
    for (int gy = 0; gy < 3; ++gy) {
        X0[gy] = fma(5.0, G[gy][0] + G[gy][2], 8.0 * G[gy][1]) * (1.0 / 18.0);
        X1[gy] = (G[gy][2] - G[gy][0]) * (5.0 * kAdvA / 18.0);
    }
    M00 = fma(5.0, X0[0] + X0[2], 8.0 * X0[1]) * (1.0 / 18.0);
    M10 = fma(5.0, X1[0] + X1[2], 8.0 * X1[1]) * (1.0 / 18.0);
    M01 = (X0[2] - X0[0]) * (5.0 * kAdvA / 18.0);
}
__device__ __forceinline__ void gp_vals(const double c[6], double e[3][3]) {
    const double c0 = fma(c[4], 1.0 / 15.0, c[0]), c1 = fma(c[4], -1.0 / 12.0, c[0]);
    const double t2 = kAdvA * c[2], t5 = kAdvA * c[5];
    const double Av[3] = {c0 - t2, c1, c0 + t2}, Bv[3] = {c[1] - t5, c[1], c[1] + t5};
#pragma unroll
    for (int gy = 0; gy < 3; ++gy) {
        const double Pq = fma(c[3], 1.0 / 15.0, Av[gy]);
        e[gy][0] = fma(-kAdvA, Bv[gy], Pq);
        e[gy][2] = fma(kAdvA, Bv[gy], Pq);
        e[gy][1] = fma(c[3], -1.0 / 12.0, Av[gy]);
    }
}

// SPH (NEXT-4, R#26): lon-lat sphere rows - the volume integrand carries |J| / (R^2 dlon dlat) = cos(lat)
// with the gradient's 1/(R cos dlon), 1/(R dlat) (a.ihx, a.ihy), the parallel-arc edges their cos(lat)
// (the same node-row value on both sides of an edge, so fluxes still cancel bitwise), and the update
// applies the row's block inverse of the cos-weighted DG mass (row table of nxsdg.cu).
template <bool SPH = false>
__global__ void __launch_bounds__(32 * ADV_ROWS, 3) k_advect_q2(AdvArgs a) {
    __shared__ double sFA[ADV_ROWS][32][3], sFH[ADV_ROWS][32][3];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int ix = blockIdx.x * 32 + tx;
    const int lr = a.erow_begin + blockIdx.y * ADV_ROWS + ty;
    const bool valid = ix < a.nx && lr < a.erow_end;
    const int ixc = valid ? ix : 0, lrc = valid ? lr : a.erow_begin;
    const int64_t e = (int64_t)lrc * a.epitch + ixc;
    Cf<6> me; load_coef<2, 6>(a, e, me);
    // RK combine input c0 (stages 2, 3): loaded up front so its latency overlaps the compute
    double c0A[6], c0H[6];
    if (a.a0 != 0.0) {
#pragma unroll
        for (int k = 0; k < 6; ++k) { c0A[k] = a.A0[k * a.eplane + e]; c0H[k] = a.H0[k * a.eplane + e]; }
    }
    double ux[3][3], uy[3][3];
#pragma unroll
    for (int jy = 0; jy < 3; ++jy)
#pragma unroll
        for (int jx = 0; jx < 3; ++jx) {
            const int64_t n = (int64_t)(2 * lrc + jy) * a.npitch + 2 * ixc + jx;
            ux[jy][jx] = a.vx[n]; uy[jy][jx] = a.vy[n];
        }
    auto nb_index = [&](int ex, int ey, bool& open) -> int64_t {
        open = true;
        if (ex < 0 || ex >= a.nx) { if (!a.periodic) { open = false; return e; } ex = (ex + a.nx) % a.nx; }
        if (ey < a.erow_begin && !a.has_south) { if (!a.periodic) { open = false; return e; } ey = a.erow_end - 1; }
        if (ey >= a.erow_end && !a.has_north) { if (!a.periodic) { open = false; return e; } ey = a.erow_begin; }
        return (int64_t)ey * a.epitch + ex;
    };
    double FeA[3], FeH[3], FnA[3], FnH[3], FwA[3], FwH[3], FsA[3], FsH[3];
    {
        bool open; const int64_t en = nb_index(ixc + 1, lrc, open);
        Cf<6> nb; load_coef<2, 6>(a, en, nb);
        double vn[3]; q2_interp3(ux[0][2], ux[1][2], ux[2][2], vn);
        q2_edge(true, me, nb, vn, open, FeA, FeH);
    }
    {
        bool open; const int64_t en = nb_index(ixc, lrc + 1, open);
        Cf<6> nb; load_coef<2, 6>(a, en, nb);
        double vn[3]; q2_interp3(uy[2][0], uy[2][1], uy[2][2], vn);
        q2_edge(false, me, nb, vn, open, FnA, FnH);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        FwA[q] = __shfl_up_sync(0xffffffffu, FeA[q], 1);
        FwH[q] = __shfl_up_sync(0xffffffffu, FeH[q], 1);
    }
    if (tx == 0) {
        bool open; const int64_t wn = nb_index(ixc - 1, lrc, open);
        Cf<6> nb; load_coef<2, 6>(a, wn, nb);
        double vn[3]; q2_interp3(ux[0][0], ux[1][0], ux[2][0], vn);
        q2_edge(true, nb, me, vn, open, FwA, FwH);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) { sFA[ty][tx][q] = FnA[q]; sFH[ty][tx][q] = FnH[q]; }
    __syncthreads();
    if (ty > 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q) { FsA[q] = sFA[ty - 1][tx][q]; FsH[q] = sFH[ty - 1][tx][q]; }
    } else {
        bool open; const int64_t sn = nb_index(ixc, lrc - 1, open);
        Cf<6> nb; load_coef<2, 6>(a, sn, nb);
        double vn[3]; q2_interp3(uy[0][0], uy[0][1], uy[0][2], vn);
        q2_edge(false, nb, me, vn, open, FsA, FsH);
    }
    if (!valid) return;
    // ---- volume term: velocity and tracers at the Gauss points (separable), then moments
    double gvx[3][3], gvy[3][3];
    {
        double X[3][3], Y[3][3];
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) { q2_interp3(ux[jy][0], ux[jy][1], ux[jy][2], X[jy]); q2_interp3(uy[jy][0], uy[jy][1], uy[jy][2], Y[jy]); }
#pragma unroll
        for (int g = 0; g < 3; ++g) {
            double o[3];
            q2_interp3(X[0][g], X[1][g], X[2][g], o); gvx[0][g] = o[0]; gvx[1][g] = o[1]; gvx[2][g] = o[2];
            q2_interp3(Y[0][g], Y[1][g], Y[2][g], o); gvy[0][g] = o[0]; gvy[1][g] = o[1]; gvy[2][g] = o[2];
        }
    }
    const double mr[6] = {1.0, 12.0, 12.0, 180.0, 180.0, 144.0};   // 1 / reference mass
    const int64_t eo = (int64_t)lr * a.epitch + ix;
    const double* __restrict__ srow = SPH ? a.sph_rows + (int64_t)lr * kSphRow : nullptr;
    // volume factors (folded into the integrand on the sphere) and north / south edge factors
    const double vsx = SPH ? 1.0 : a.ihx, vsy = SPH ? 1.0 : a.ihy;
    const double eny = SPH ? a.ihy * __ldg(srow + SPH_COS_N) : a.ihy, esy = SPH ? a.ihy * __ldg(srow + SPH_COS_S) : a.ihy;
#pragma unroll
    for (int tr = 0; tr < 2; ++tr) {
        const double* c = tr == 0 ? me.A : me.H;
        const double* Fe = tr == 0 ? FeA : FeH; const double* Fw = tr == 0 ? FwA : FwH;
        const double* Fn = tr == 0 ? FnA : FnH; const double* Fs = tr == 0 ? FsA : FsH;
        double cg[3][3], Gx[3][3], Gy[3][3];
        gp_vals(c, cg);
#pragma unroll
        for (int gy = 0; gy < 3; ++gy) {
            const double fx = SPH ? a.ihx : 1.0, fy = SPH ? a.ihy * __ldg(srow + SPH_COS + gy) : 1.0;
#pragma unroll
            for (int g = 0; g < 3; ++g) {
                Gx[gy][g] = SPH ? cg[gy][g] * gvx[gy][g] * fx : cg[gy][g] * gvx[gy][g];
                Gy[gy][g] = SPH ? cg[gy][g] * gvy[gy][g] * fy : cg[gy][g] * gvy[gy][g];
            }
        }
        double x00, x10, x01, y00, y10, y01;
        vol_mom(Gx, x00, x10, x01);
        vol_mom(Gy, y00, y10, y01);
        double L[6];
        L[0] = 0.0;
        L[1] = vsx * x00;
        L[2] = vsy * y00;
        L[3] = 2.0 * vsx * x10;
        L[4] = 2.0 * vsy * y01;
        L[5] = fma(vsx, x01, vsy * y10);
        double m0, m1, m2;
        edge_mom(Fe, m0, m1, m2);   // east, outward +x
        L[0] -= a.ihx * m0; L[1] -= a.ihx * 0.5 * m0; L[2] -= a.ihx * m1; L[3] -= a.ihx * m0 * (1.0 / 6.0);
        L[4] -= a.ihx * m2; L[5] -= a.ihx * 0.5 * m1;
        edge_mom(Fw, m0, m1, m2);   // west, outward -x
        L[0] += a.ihx * m0; L[1] -= a.ihx * 0.5 * m0; L[2] += a.ihx * m1; L[3] += a.ihx * m0 * (1.0 / 6.0);
        L[4] += a.ihx * m2; L[5] -= a.ihx * 0.5 * m1;
        edge_mom(Fn, m0, m1, m2);   // north, outward +y
        L[0] -= eny * m0; L[1] -= eny * m1; L[2] -= eny * 0.5 * m0; L[3] -= eny * m2;
        L[4] -= eny * m0 * (1.0 / 6.0); L[5] -= eny * 0.5 * m1;
        edge_mom(Fs, m0, m1, m2);   // south, outward -y
        L[0] += esy * m0; L[1] += esy * m1; L[2] -= esy * 0.5 * m0; L[3] += esy * m2;
        L[4] += esy * m0 * (1.0 / 6.0); L[5] -= esy * 0.5 * m1;
        double* out = tr == 0 ? a.Aout : a.Hout;
        const double* c0 = tr == 0 ? c0A : c0H;
        double nc[6], Ld[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) Ld[k] = L[k] * mr[k];
        if constexpr (SPH) {   // the row's cos-weighted mass: block inverse (modes {0,2,4}, {1,5}, {3})
            double p[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) p[k] = Ld[k];
            sph_apply_q(srow, p, Ld);
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const double v = a.a1 * fma(a.dt, Ld[k], c[k]);
            nc[k] = (a.a0 != 0.0) ? fma(a.a0, c0[k], v) : v;
        }
        if (a.limit) {   // R#25 fused: extremes over the 9 volume and 12 edge Gauss points, scale about the mean
            double gv[9], ev[4][3];
            eval_gp<true, true>(nc, gv);
            trace_s(nc, 1.0, ev[0]); trace_s(nc, -1.0, ev[1]); trace_t(nc, 1.0, ev[2]); trace_t(nc, -1.0, ev[3]);
            double cmin = gv[0], cmax = gv[0];
#pragma unroll
            for (int g = 1; g < 9; ++g) { cmin = fmin(cmin, gv[g]); cmax = fmax(cmax, gv[g]); }
#pragma unroll
            for (int ed = 0; ed < 4; ++ed)
#pragma unroll
                for (int q = 0; q < 3; ++q) { cmin = fmin(cmin, ev[ed][q]); cmax = fmax(cmax, ev[ed][q]); }
            const double cbar = nc[0], lo = 0.0, hi = tr == 0 ? 1.0 : INFINITY;
            double theta = 1.0;
            if (cmin < lo) theta = fmin(theta, (cbar - lo) / (cbar - cmin));
            if (cmax > hi) theta = fmin(theta, (hi - cbar) / (cmax - cbar));
            theta = fmax(0.0, fmin(1.0, theta));
            if (theta < 1.0) {
                nc[0] = fma(1.0 - theta, cbar, theta * nc[0]);
#pragma unroll
                for (int k = 1; k < 6; ++k) nc[k] *= theta;
            }
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) out[k * a.eplane + eo] = nc[k];
    }
}

}  // namespace nxk
