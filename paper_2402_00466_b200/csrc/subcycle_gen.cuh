// NEXT-1 fused: the whole mEVP subcycle (strain -> Listing 2 -> divergence gather -> velocity) on a
// GENERAL quad mesh (bilinear map of each element's four vertices, DESIGN R#23) in one pass, with
// the geometry recomputed on the fly from the vertices - nothing per element is stored.
//
// Same warp mapping, TMA job pipeline and node gather as k_subcycle_tma (CG2/DG2, n_S = 6); each job
// additionally stages the element row's two vertex rows and the two owned rows of lumped node masses.
// Per element:
//   geometry   a = X10-X00, b = X01-X00, c = X11-X01-X10+X00:  J(s,t) = [a + c t | b + c s],
//              |J| = c0 + d1 S + d2 T (centred, exactly linear), M_K = c0 D + d1 M_S + d2 M_T
//              (closed form, Cholesky with reciprocal diagonal: general_quads.cuh)
//   strain     the reference derivatives d/ds v, d/dt v at the Gauss points are exact in the n_S = 8
//              space (R#24), so their coefficients come from the same node differences as the box
//              kernel; w |J| eps = w adj(J)^T grad_ref v; E_c = M_K^{-1} sum_g w psi (|J| eps_c)(g)
//   stress     Listing 2 at the Gauss points with P_g from the outer-step prep; then
//              S <- (1 - 1/alpha) S + M_K^{-1} sum_g w |J_g| psi r(g)
//   divergence r_j = sum_g w sigma(g) . adj(J_g)^T grad_ref phi_j(g), evaluated separably with the
//              1D Lagrange values / derivatives at the Gauss abscissae; F / m with the lumped mass
#pragma once
#include "subcycle_tma.cuh"
#include "general_quads.cuh"

namespace nxk {

struct K2GenMaps {
    CUtensorMap S, Pg, vx, vy, C, X, M;    // box-kernel maps + vertices + lumped masses
};

struct __align__(128) K2GenStage {
    K2Stage<double, 6> b;
    alignas(128) double X[2][K2_VCOLS];    // vertex rows lr, lr+1: 33 vertices x (x, y)
    alignas(128) double M[2][K2_CCOLS];    // -1 / lumped mass of node rows 2 lr, 2 lr + 1 (owned columns)
};
__host__ __device__ constexpr uint32_t k2g_tx_bytes() {
    return k2_tx_bytes<double, 6>() + 2 * K2_VCOLS * 8 + 2 * K2_CCOLS * 8;
}
// LC ("late constants", NXSDG_OPT_CONST_STAGING = 1 for this kernel): the stage has no node-constant
// box; once the stress update has consumed S and P_g, lane 0 TMA-loads the job's six node constants
// into that region (7.5 KB >= 5952 B) on a second mbarrier, and the velocity update waits for it.
// 13.1 KB stages instead of 19 KB: 4 CTAs (8 warps) per SM fit instead of 3.
struct __align__(128) K2GenStageLC {
    K2StageNC<double, 6> b;
    alignas(128) double X[2][K2_VCOLS];
    alignas(128) double M[2][K2_CCOLS];
};
__host__ __device__ constexpr uint32_t k2g_const_bytes() { return 6 * 2 * K2_CCOLS * 8; }
template <bool LC> struct K2GenStageSel { using T = K2GenStage; };
template <> struct K2GenStageSel<true> { using T = K2GenStageLC; };

// Raw Gauss sums of the six P2 moments: the plain moment sum_g w psi_k G_g is tau_k q_k (tau_k = M_ref,k x
// the box projection's scale of proj_coeffs, with the 1D sums 5 G(-a) + 8 G(0) + 5 G(a) taken as
// G(-a) + 1.6 G(0) + G(a)), so the scales fold into the mass solve below.
__device__ __forceinline__ void proj_raw(const double G[9], double (&q)[6]) {
    double X0[3], X1[3], X2[3];
#pragma unroll
    for (int gy = 0; gy < 3; ++gy) {
        const double s = G[gy * 3] + G[gy * 3 + 2], d = G[gy * 3 + 2] - G[gy * 3], m = G[gy * 3 + 1];
        X0[gy] = fma(1.6, m, s);
        X1[gy] = d;
        X2[gy] = fma(-2.0, m, s);
    }
    const double s0 = X0[0] + X0[2];
    q[0] = fma(1.6, X0[1], s0);
    q[1] = fma(1.6, X1[1], X1[0] + X1[2]);
    q[2] = X0[2] - X0[0];
    q[3] = fma(1.6, X2[1], X2[0] + X2[2]);
    q[4] = fma(-2.0, X0[1], s0);
    q[5] = X1[2] - X1[0];
}
constexpr double kTau0 = 25.0 / 324.0, kTau1 = 5.0 * (1.0 / 12.0) * (kC / 18.0), kTau2 = kTau1;
constexpr double kTau3 = 5.0 * (1.0 / 180.0) * (10.0 / 54.0), kTau4 = kTau3, kTau5 = (1.0 / 144.0) * (kC * kC);

// Sparse LDL^T of M_K = c0 D + d1 M_S + d2 M_T (general_quads.cuh): its off-diagonal pattern is (1,0), (2,0),
// (3,1), (5,1), (4,2), (5,2); eliminated in the order 3, 4, 0, 1, 2, 5 it fills only (2,1), so a solve
// costs 7 + 7 FMAs and 6 products instead of the dense Cholesky's 2 x 15 FMAs and 12 products, and the
// factor needs 4 reciprocals (1/c0 serves the pivots c0/180, c0/180, c0).  The moment scales tau are
// folded in: with y_i = tau_i yh_i the forward pass runs on the raw sums q (g_ij = l_ij tau_j / tau_i) and
// the pivots become rho_i = tau_i / p_i.  Same matrix as the oracle's M_i, another elimination order.
struct MassLDL6 {
    double l13, l10, l24, l20, l21, l51, l52;    // unit lower factor (backward substitution)
    double g13, g10, g24, g20, g21, g51, g52;    // forward coefficients on the raw sums
    double rho[6];
};
__device__ __forceinline__ void mass_ldl6(double c0, double d1, double d2, MassLDL6& F) {
    const double ic = rcp_nr(c0);
    F.l13 = d1 * ic; F.l24 = d2 * ic;                       // pivots 3, 4: c0 / 180; m31 = d1 / 180, m42 = d2 / 180
    F.l10 = F.l13 * (1.0 / 12.0); F.l20 = F.l24 * (1.0 / 12.0);   // pivot 0: c0; m10 = d1 / 12, m20 = d2 / 12
    const double m21 = -(d1 * F.l20) * (1.0 / 12.0);       // fill: -m10 m20 / c0
    const double p1 = fma(-d1 * (1.0 / 80.0), F.l13, c0 * (1.0 / 12.0));   // c0/12 - m31^2/p3 - m10^2/p0
    const double ip1 = rcp_nr(p1);
    F.l21 = m21 * ip1;
    const double m51 = d2 * (1.0 / 144.0);
    F.l51 = m51 * ip1;
    const double p2 = fma(-F.l21, m21, fma(-d2 * (1.0 / 80.0), F.l24, c0 * (1.0 / 12.0)));
    const double ip2 = rcp_nr(p2);
    const double m52 = fma(-F.l21, m51, d1 * (1.0 / 144.0));
    F.l52 = m52 * ip2;
    const double p5 = fma(-F.l52, m52, fma(-F.l51, m51, c0 * (1.0 / 144.0)));
    const double ip5 = rcp_nr(p5);
    F.g13 = F.l13 * (kTau3 / kTau1); F.g10 = F.l10 * (kTau0 / kTau1);
    F.g24 = F.l24 * (kTau4 / kTau2); F.g20 = F.l20 * (kTau0 / kTau2);
    F.g21 = F.l21 * (kTau1 / kTau2); F.g51 = F.l51 * (kTau1 / kTau5); F.g52 = F.l52 * (kTau2 / kTau5);
    F.rho[0] = kTau0 * ic; F.rho[3] = (180.0 * kTau3) * ic; F.rho[4] = (180.0 * kTau4) * ic;
    F.rho[1] = kTau1 * ip1; F.rho[2] = kTau2 * ip2; F.rho[5] = kTau5 * ip5;
}
// x = M_K^{-1} (sc tau (.) q)
__device__ __forceinline__ void ldl6_solve(const MassLDL6& F, const double (&q)[6], double sc, double (&x)[6]) {
    const double y1 = fma(-F.g10, q[0], fma(-F.g13, q[3], q[1]));
    const double y2 = fma(-F.g21, y1, fma(-F.g20, q[0], fma(-F.g24, q[4], q[2])));
    const double y5 = fma(-F.g52, y2, fma(-F.g51, y1, q[5]));
    const double x5 = (sc * F.rho[5]) * y5;
    const double x2 = fma(-F.l52, x5, (sc * F.rho[2]) * y2);
    const double x1 = fma(-F.l51, x5, fma(-F.l21, x2, (sc * F.rho[1]) * y1));
    x[0] = fma(-F.l20, x2, fma(-F.l10, x1, (sc * F.rho[0]) * q[0]));
    x[4] = fma(-F.l24, x2, (sc * F.rho[4]) * q[4]);
    x[3] = fma(-F.l13, x1, (sc * F.rho[3]) * q[3]);
    x[1] = x1; x[2] = x2; x[5] = x5;
}

__device__ __forceinline__ const double* gen_const_box(const K2GenStage& t) { return &t.b.C[0][0][0]; }
__device__ __forceinline__ const double* gen_const_box(const K2GenStageLC& t) { return &t.b.S[0][0]; }

template <bool REPL, int STAGES, bool LC = false>
__global__ void __launch_bounds__(32 * K2_WARPS, 2) k_subcycle_gen(const __grid_constant__ K2GenMaps maps, SubArgs a) {
    using Stage = typename K2GenStageSel<LC>::T;
    using NC6 = K2StageNC<double, 6>;
    static_assert(!LC || offsetof(NC6, vx) >= 6 * 2 * K2_CCOLS * 8, "the constants fit before vx");
    extern __shared__ __align__(1024) unsigned char k2_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    Stage* stg = reinterpret_cast<Stage*>(k2_smem) + wib * STAGES;
    uint64_t* bar = reinterpret_cast<uint64_t*>(k2_smem + K2_WARPS * STAGES * sizeof(Stage)) + wib * STAGES;
    const int twarps = gridDim.x * K2_WARPS;
    const int gw = blockIdx.x * K2_WARPS + wib;
    const int nunits = units_total(a);
    if (gw >= nunits) return;
    const uint64_t pol_st = l2_policy(a.l2_hints & 2 ? 1 : 0);   // stores: evict_first by default
    // LC: one more mbarrier per stage for the late constants, after the job descriptors
    uint64_t* barC = reinterpret_cast<uint64_t*>(reinterpret_cast<int4*>(bar + K2_WARPS * STAGES - wib * STAGES) +
                                                 K2_WARPS * STAGES) + wib * STAGES;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&bar[s], 1);
            if constexpr (LC) mbar_init(&barC[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    struct Cur { int u, lr, lr1, ix0; bool ring, first, ok; };
    auto start_unit = [&](int u, Cur& c) {
        for (;;) {                        // skip empty sub-units (ragged last chunk)
            c.ok = u < nunits;
            if (!c.ok) return;
            int strip, lr0, lr1;
            unit_rows(a, u, strip, lr0, lr1);
            if (lr0 < lr1) {
                c.u = u; c.lr1 = lr1; c.ix0 = strip * 31;
                c.ring = lr0 > 0; c.lr = c.ring ? lr0 - 1 : lr0; c.first = true;
                return;
            }
            u = a.work_counter ? twarps + atomicAdd(a.work_counter, 1) : u + twarps;
        }
    };
    auto advance = [&](Cur& c) {
        ++c.lr; c.ring = false; c.first = false;
        if (c.lr >= c.lr1) {
            const int nu = a.work_counter ? twarps + atomicAdd(a.work_counter, 1) : c.u + twarps;
            start_unit(nu, c);
        }
    };
    int4* jobs = reinterpret_cast<int4*>(bar + K2_WARPS * STAGES - wib * STAGES) + wib * STAGES;
    auto record = [&](const Cur& c, int st) {
        jobs[st] = make_int4(c.ok ? c.u : -1, c.lr, c.lr1, (c.ring ? 1 : 0) | (c.first ? 2 : 0));
    };
    auto issue = [&](const Cur& c, int s) {
        Stage* t = stg + s;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[s], k2g_tx_bytes() - (LC ? k2g_const_bytes() : 0u));
        const int xs = (c.ix0 - 1) & ~1;
        tma3(&t->b.S[0][0], &maps.S, &bar[s], xs, c.lr, 0);
        tma3(&t->b.Pg[0][0], &maps.Pg, &bar[s], xs, c.lr, 0);
        tma2(&t->b.vx[0][0], &maps.vx, &bar[s], 2 * (c.ix0 - 1), 2 * c.lr);
        tma2(&t->b.vy[0][0], &maps.vy, &bar[s], 2 * (c.ix0 - 1), 2 * c.lr);
        if constexpr (!LC) tma3(&t->b.C[0][0][0], &maps.C, &bar[s], 2 * c.ix0, 2 * c.lr, 0);
        tma2(&t->X[0][0], &maps.X, &bar[s], 2 * (c.ix0 - 1), c.lr);
        tma2(&t->M[0][0], &maps.M, &bar[s], 2 * c.ix0, 2 * c.lr);
    };

    const double fac = a.fac, hA = 0.5 * a.ainv;
    const int64_t npitch = a.npitch, eplane = a.eplane;
    Cur pre;
    if (lane == 0) {
        start_unit(gw, pre);
        record(pre, 0);
        issue(pre, 0);
#pragma unroll
        for (int k = 1; k < STAGES - 1; ++k) {
            advance(pre);
            record(pre, k);
            if (pre.ok) issue(pre, k);
        }
    }
    __syncwarp();
    uint32_t phase = 0, phaseC = 0;
    int s = 0;
    double carx[2] = {0.0, 0.0}, cary[2] = {0.0, 0.0};
    for (;;) {
        const int sp = (s + STAGES - 1) % STAGES;
        if (lane == 0) {
            if (pre.ok) advance(pre);
            record(pre, sp);
            if (pre.ok) issue(pre, sp);
        }
        Cur cur;
        {
            const int4 jd = jobs[s];
            cur.ok = jd.x >= 0;
            if (!cur.ok) break;
            cur.u = jd.x; cur.lr = jd.y; cur.lr1 = jd.z; cur.ring = jd.w & 1; cur.first = (jd.w & 2) != 0;
            cur.ix0 = (cur.u % a.nstrips) * 31;
        }
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
        const Stage& t = stg[s];
        const int ix = cur.ix0 - 1 + lane, lr = cur.lr;
        const int eo = (cur.ix0 - 1) - ((cur.ix0 - 1) & ~1);
        const bool evalid = ix >= 0 && ix < a.nx;
        if (cur.first) { carx[0] = carx[1] = cary[0] = cary[1] = 0.0; }

        // ---- geometry of this element (zero-filled boxes outside the mesh: use a unit square there)
        double ax_, ay_, bx_, by_, cx_, cy_;
        {
            const double x00 = t.X[0][2 * lane], y00 = t.X[0][2 * lane + 1];
            const double x10 = t.X[0][2 * lane + 2], y10 = t.X[0][2 * lane + 3];
            const double x01 = t.X[1][2 * lane], y01 = t.X[1][2 * lane + 1];
            const double x11 = t.X[1][2 * lane + 2], y11 = t.X[1][2 * lane + 3];
            ax_ = x10 - x00; ay_ = y10 - y00; bx_ = x01 - x00; by_ = y01 - y00;
            cx_ = (x11 - x01) - ax_; cy_ = (y11 - y01) - ay_;
            if (!evalid) { ax_ = 1.0; ay_ = 0.0; bx_ = 0.0; by_ = 1.0; cx_ = 0.0; cy_ = 0.0; }
        }
        const double d0 = ax_ * by_ - bx_ * ay_, d1 = ax_ * cy_ - cx_ * ay_, d2 = cx_ * by_ - bx_ * cy_;
        const double c0 = d0 + 0.5 * (d1 + d2);
        MassLDL6 F;
        mass_ldl6(c0, d1, d2, F);
        // J columns at the Gauss point (gx, gy): x_s = ax + cx t, x_t = bx + cx s, y_s = ay + cy t, y_t = by + cy s
        auto jac = [&](int gx, int gy, double& xs, double& xt, double& ys, double& yt) {
            const double sg = 0.5 + (gx - 1) * kA, tg = 0.5 + (gy - 1) * kA;
            xs = fma(cx_, tg, ax_); xt = fma(cx_, sg, bx_); ys = fma(cy_, tg, ay_); yt = fma(cy_, sg, by_);
        };

        // ---- node values (local box columns 2*lane .. 2*lane+2)
        double Vx[3][3], Vy[3][3];
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
            const double2 a2 = *reinterpret_cast<const double2*>(&t.b.vx[jy][2 * lane]);
            const double2 b2 = *reinterpret_cast<const double2*>(&t.b.vy[jy][2 * lane]);
            Vx[jy][0] = a2.x; Vx[jy][1] = a2.y; Vx[jy][2] = t.b.vx[jy][2 * lane + 2];
            Vy[jy][0] = b2.x; Vy[jy][1] = b2.y; Vy[jy][2] = t.b.vy[jy][2 * lane + 2];
        }
        // ---- strain: pointwise reference derivatives at the Gauss points, w |J| eps, projection
        double e11[9], e12[9], e22[9];
        {
            double Dsx[9], Dtx[9], Dsy[9], Dty[9];
            {
                double E8[8];
                strain_s(Vx, E8); eval_gp<false, true>(E8, Dsx);
                strain_t(Vx, E8); eval_gp<true, false>(E8, Dtx);
                strain_s(Vy, E8); eval_gp<false, true>(E8, Dsy);
                strain_t(Vy, E8); eval_gp<true, false>(E8, Dty);
            }
#pragma unroll
            for (int gy = 0; gy < 3; ++gy)
#pragma unroll
                for (int gx = 0; gx < 3; ++gx) {
                    const int g = gy * 3 + gx;
                    double xs, xt, ys, yt;
                    jac(gx, gy, xs, xt, ys, yt);
                    const double x = fma(yt, Dsx[g], -ys * Dtx[g]);                           // |J| d vx / dx
                    const double y = fma(xs, Dty[g], -xt * Dsy[g]);                           // |J| d vy / dy
                    e11[g] = x + y;                                                           // |J| u (trace)
                    e22[g] = x - y;                                                           // |J| w, x 1/2 below
                    e12[g] = fma(xs, Dtx[g], -xt * Dsx[g]) + fma(yt, Dsy[g], -ys * Dty[g]);     // x 1/2 below
                }
            double E11[6], E12[6], E22[6], q[6];
            proj_raw(e11, q); ldl6_solve(F, q, 1.0, E11);
            proj_raw(e12, q); ldl6_solve(F, q, 0.5, E12);
            proj_raw(e22, q); ldl6_solve(F, q, 0.5, E22);
            eval_gp<true, true>(E11, e11); eval_gp<true, true>(E12, e12); eval_gp<true, true>(E22, e22);
        }
        // ---- VP stress at the Gauss points (Listing 2), alpha^{-1} folded in as in the box kernel,
        // on the projected trace u = eps11 + eps22 (e11), half difference w = (eps11 - eps22) / 2 (e22) and
        // eps12 (e12): Delta^2 = u^2 + w^2 + eps12^2 and g11, g22 = a +- b with a = p u - P/2, b = p w / 2
        // (the box kernel's form), so S11 and S22 come from the projections of a and b.
        // |J_g| = c0 + d1 S_g + d2 T_g, separably; it multiplies p / Delta and the pressure term
        const double Jx[3] = {fma(d1, -kA, c0), c0, fma(d1, kA, c0)};
#pragma unroll
        for (int g = 0; g < 9; ++g) {
            const double u = e11[g], w = e22[g], z = e12[g];
            const double draw2 = fma(u, u, fma(w, w, z * z));
            const double rD = rsqrt_nr(draw2 + a.dmin2);
            const double ph = t.b.Pg[g][eo + lane] * hA;
            const double jd = g / 3 == 1 ? Jx[g % 3] : fma(d2, (g / 3 - 1) * kA, Jx[g % 3]);   // |J_g|
            const double pr = ph * rD, prj = jd * pr;
            const double subj = REPL ? prj * (draw2 > 0.0 ? draw2 * rsqrt_nr(draw2) : 0.0) : jd * ph;
            e11[g] = fma(prj, u, -subj);      // |J| a
            e22[g] = prj * w;                 // |J| 2 b
            e12[g] = prj * z;
        }
        double S11[6], S12[6], S22[6];
        {
            double q[6], Sa[6], Sb[6];
            proj_raw(e11, q); ldl6_solve(F, q, 1.0, Sa);
            proj_raw(e22, q); ldl6_solve(F, q, 0.5, Sb);
            proj_raw(e12, q); ldl6_solve(F, q, 0.5, S12);
#pragma unroll
            for (int k = 0; k < 6; ++k) { S11[k] = Sa[k] + Sb[k]; S22[k] = Sa[k] - Sb[k]; }
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            S11[k] = fma(fac, t.b.S[k][eo + lane], S11[k]);
            S12[k] = fma(fac, t.b.S[6 + k][eo + lane], S12[k]);
            S22[k] = fma(fac, t.b.S[12 + k][eo + lane], S22[k]);
        }
        // LC: S and P_g of this stage are consumed; load the node constants into their place
        if constexpr (LC) {
            if (!cur.ring) {
                asm volatile("" ::: "memory");   // every lane's reads of the stage are issued before the barrier
                __syncwarp();
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&barC[s], k2g_const_bytes());
                    tma3(const_cast<double*>(&t.b.S[0][0]), &maps.C, &barC[s], 2 * cur.ix0, 2 * lr, 0);
                }
            }
        }
        if (!cur.ring && evalid && lane >= 1) {
            const int64_t e = (int64_t)lr * a.epitch + ix;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                st_hint(a.S_out + k * eplane + e, S11[k], pol_st);
                st_hint(a.S_out + (6 + k) * eplane + e, S12[k], pol_st);
                st_hint(a.S_out + (12 + k) * eplane + e, S22[k], pol_st);
            }
        }
        // ---- divergence: r_j = sum_g w sigma . adj(J)^T grad_ref phi_j, separable in (gx, gy)
        double rX[3][3], rY[3][3];
        {
            double s11[9], s12[9], s22[9];
            eval_gp<true, true>(S11, s11); eval_gp<true, true>(S12, s12); eval_gp<true, true>(S22, s22);
            double AX[9], BX[9], AY[9], BY[9];
#pragma unroll
            for (int gy = 0; gy < 3; ++gy)
#pragma unroll
                for (int gx = 0; gx < 3; ++gx) {
                    const int g = gy * 3 + gx;
                    double xs, xt, ys, yt;
                    jac(gx, gy, xs, xt, ys, yt);
                    AX[g] = fma(s11[g], yt, -s12[g] * xt);     // coefficient of d phi / ds (weights below)
                    BX[g] = fma(s12[g], xs, -s11[g] * ys);     // coefficient of d phi / dt
                    AY[g] = fma(s12[g], yt, -s22[g] * xt);
                    BY[g] = fma(s22[g], xs, -s12[g] * ys);
                }
            // r(jx, jy) = sum_gy [ (sum_gx w L'_jx AX) w L_jy + (sum_gx w L_jx BX) w L'_jy ] (and Y): 1D
            // contractions over gx for each gy, then over gy
            double uAX[3][3], uBX[3][3], uAY[3][3], uBY[3][3];   // [gy][jx]
#pragma unroll
            for (int gy = 0; gy < 3; ++gy) {
                lag_der3(AX[gy * 3], AX[gy * 3 + 1], AX[gy * 3 + 2], uAX[gy]);
                lag_val3(BX[gy * 3], BX[gy * 3 + 1], BX[gy * 3 + 2], uBX[gy]);
                lag_der3(AY[gy * 3], AY[gy * 3 + 1], AY[gy * 3 + 2], uAY[gy]);
                lag_val3(BY[gy * 3], BY[gy * 3 + 1], BY[gy * 3 + 2], uBY[gy]);
            }
#pragma unroll
            for (int jx = 0; jx < 3; ++jx) {
                double vA[3], dB[3], vAy[3], dBy[3];
                lag_val3(uAX[0][jx], uAX[1][jx], uAX[2][jx], vA);
                lag_der3(uBX[0][jx], uBX[1][jx], uBX[2][jx], dB);
                lag_val3(uAY[0][jx], uAY[1][jx], uAY[2][jx], vAy);
                lag_der3(uBY[0][jx], uBY[1][jx], uBY[2][jx], dBy);
#pragma unroll
                for (int jy = 0; jy < 3; ++jy) {
                    rX[jx][jy] = evalid ? vA[jy] + dB[jy] : 0.0;
                    rY[jx][jy] = evalid ? vAy[jy] + dBy[jy] : 0.0;
                }
            }
        }
        // ---- per-node gather (row below, W, E) + velocity update with the lumped mass (R#11)
        const bool nvalid = lane >= 1 && ix >= 0 && ix <= a.nx && !cur.ring;
        double sumx[2][2], sumy[2][2];
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
            const double wx = __shfl_up_sync(0xffffffffu, rX[2][jy], 1);
            const double wy = __shfl_up_sync(0xffffffffu, rY[2][jy], 1);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                double sx = rX[q][jy], sy = rY[q][jy];
                if (q == 0) { sx = wx + sx; sy = wy + sy; }
                if (jy == 2) { carx[q] = sx; cary[q] = sy; continue; }
                if (jy == 0) { sx = carx[q] + sx; sy = cary[q] + sy; }
                sumx[jy][q] = sx; sumy[jy][q] = sy;
            }
        }
        if constexpr (LC) {
            if (!cur.ring) {
                mbar_wait(&barC[s], (phaseC >> s) & 1u);
                phaseC ^= 1u << s;
            }
        }
        const double (*CC)[2][K2_CCOLS] = reinterpret_cast<const double (*)[2][K2_CCOLS]>(gen_const_box(t));
        if (nvalid) {
            const bool brow0 = lr == a.erow_begin && a.bottom_boundary;
#pragma unroll
            for (int jy = 0; jy < 2; ++jy) {
                double nvx[2], nvy[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int I = 2 * ix + q;
                    const int cc = 2 * lane - 2 + q;
                    const double im = t.M[jy][cc];                            // F = -r / m (-1 / m staged)
                    const double fx = sumx[jy][q] * im, fy = sumy[jy][q] * im;
                    const double vxo = Vx[jy][q], vyo = Vy[jy][q];
                    const double c1 = CC[0][jy][cc], r0x = CC[1][jy][cc], r0y = CC[2][jy][cc];
                    const double cf = CC[3][jy][cc], oxv = CC[4][jy][cc], oyv = CC[5][jy][cc];
                    const double dx = oxv - vxo, dy = oyv - vyo;
                    const double w2 = fma(dx, dx, dy * dy);
                    const double w = w2 > 0.0 ? w2 * rsqrt_nr(w2) : 0.0;
                    const double cw = cf * w;
                    const double rden = rcp_nr(fma(c1, a.b1, cw));
                    const double cb = c1 * a.beta, ck = c1 * a.kc;
                    const double ux = (fma(cb, vxo, r0x) + fma(cw, oxv, fma(ck, vyo, fx))) * rden;
                    const double uy = (fma(cb, vyo, r0y) + fma(cw, oyv, fma(-ck, vxo, fy))) * rden;
                    const bool bnd = (I == 0) || (I == 2 * a.nx) || (jy == 0 && brow0);
                    nvx[q] = bnd ? 0.0 : ux;
                    nvy[q] = bnd ? 0.0 : uy;
                }
                const int64_t n = (int64_t)(2 * lr + jy) * npitch + 2 * ix;
                if (ix < a.nx) {
                    st_hint2(a.vx_out + n, nvx[0], nvx[1], pol_st);
                    st_hint2(a.vy_out + n, nvy[0], nvy[1], pol_st);
                } else {
                    a.vx_out[n] = 0.0;
                    a.vy_out[n] = 0.0;
                }
            }
        }
        if (a.top_boundary && lr == a.erow_end - 1 && nvalid) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int I = 2 * ix + q;
                if (I > 2 * a.nx) continue;
                a.vx_out[(int64_t)(2 * a.erow_end) * npitch + I] = 0.0;
                a.vy_out[(int64_t)(2 * a.erow_end) * npitch + I] = 0.0;
            }
        }
        __syncwarp();
        s = (s + 1) % STAGES;
    }
}

}  // namespace nxk
