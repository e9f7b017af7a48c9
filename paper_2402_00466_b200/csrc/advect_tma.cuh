// K4, persistent TMA-staged form of the structured CG2/DG2 advection stage (Eq. (1),
// P:102-106, upwind DG).  The arithmetic is k_advect_q2's, call for call (same traces, fluxes,
// moments and update; the compiler may contract a few products differently, ~1e-15); what changes is how the data
// reaches the registers, the part that kept k_advect_q2 at ~60 % of HBM (16 % warps active, every
// element loading its east and north neighbours' coefficients again through L1/L2):
//
//   - a warp owns a strip of 31 element columns (+ lane 0 = the ring column ix0 - 1, whose east flux
//     is lane 1's west flux) and marches up a chunk of element rows;
//   - every row of the chunk, plus one ring row below and one above, is loaded ONCE by TMA into a
//     ring of shared-memory slots: the A and H coefficients of 34 columns (the strip + both neighbours)
//     and the two node rows of v the row adds (2k+1, 2k+2; the row below supplies node row 2k);
//   - a row is processed when the row above has landed: east neighbours come from the slot, west
//     fluxes by shuffle, south / north fluxes from the slots of the rows below / above (each interior
//     horizontal edge is evaluated by the two rows sharing it with the same function on the same
//     inputs: bitwise-identical fluxes, mass conserved to the rounding of the sums);
//   - the RK combine input c0 (stages 2, 3) is prefetched into registers before the wait.
// Closed box (boundary edges carry no flux; out-of-range rows / columns arrive zero-filled by TMA and are
// masked by `open`); periodic meshes, the limiter and the sphere use k_advect_q2.
#pragma once
#include "advect_q2.cuh"
#include "prep_q2.cuh"

namespace nxk {

// 2 warps per CTA, 4 CTAs (8 warps) per SM at 232 registers.  Measured alternatives (round 2,
// profiles/ab_adv_prep_r02.log): 3 warps x 3 CTAs at 222 registers ran the three stages in 6.05 ms per outer
// step against 4.51 ms; 10 warps x 1 CTA at 200 registers does not launch (register granularity).
constexpr int ADV_TMA_WARPS = 2;
#ifndef ADV_TMA_MINB
#define ADV_TMA_MINB 3
#endif
constexpr int ADV_COLS = 34;                   // FP64 box: 16-B aligned start (ix0 - 1) & ~1, covers ix0 + 31

struct __align__(128) AdvSlot {
    alignas(128) double A[6][ADV_COLS];        // 1632 B
    alignas(128) double H[6][ADV_COLS];
    alignas(128) double vx[2][K2_VCOLS];       // node rows 2k+1, 2k+2; 1056 B
    alignas(128) double vy[2][K2_VCOLS];
};
constexpr uint32_t kAdvTx = 2u * 6u * ADV_COLS * 8u + 2u * 2u * K2_VCOLS * 8u;

// the RK combine input c0 = (A^n, H^n) of one job (stages 2, 3): one buffer per warp, TMA-loaded while the
// previous job computes (a plain register prefetch left one DFMA with a quarter of the stage's stall samples)
struct __align__(128) AdvC0 {
    alignas(128) double A[6][ADV_COLS];
    alignas(128) double H[6][ADV_COLS];
};
constexpr uint32_t kAdvC0Tx = 2u * 6u * ADV_COLS * 8u;

struct AdvMaps {
    CUtensorMap A, H;     // 3D {nx, erows_local, 6}, box {34, 1, 6}: the stage input planes
    CUtensorMap vx, vy;   // 2D node grid, box {66, 2}
    CUtensorMap A0, H0;   // the RK combine input planes (same geometry as A, H)
};
// dynamic shared memory of k_advect_tma: slots [warps][STAGES] | c0 buffers [warps] | slot barriers
// [warps][STAGES] | c0 barriers [warps] (padded to 16 B) | job descriptors [warps][STAGES]
__host__ __device__ constexpr size_t adv_bar_off(int st) {
    return (size_t)ADV_TMA_WARPS * st * sizeof(AdvSlot) + (size_t)ADV_TMA_WARPS * sizeof(AdvC0);
}
__host__ __device__ constexpr size_t adv_desc_off(int st) {
    return adv_bar_off(st) + (((size_t)ADV_TMA_WARPS * (st + 1) * 8 + 15) / 16) * 16;
}
__host__ __device__ constexpr size_t adv_smem_bytes(int st) { return adv_desc_off(st) + (size_t)ADV_TMA_WARPS * st * 16; }

struct AdvTmaArgs {
    AdvArgs a;
    int nstrips, ty, nchunks;
    int dbg;                                   // debug: lane 0 prints its positions (NXSDG_DEBUG_ADV_TMA)
};

// STAGES = 3 ("late" ring): row k + 2 goes into the slot of row k - 1 as soon as job k has read what it
// needs of row k - 1 (its top v node row, and the south flux for a unit's first job), so a job still
// waits only for a row issued one job earlier; 3 slots per warp fit 5 CTAs (10 warps) per SM at <= 204
// registers where 4 slots fit 4 (8 warps)
// Raw moments (session 3).  k_advect_q2 forms the edge moments m0 = sum w F, m1 = sum w T F, m2 = sum w q(T) F
// and the volume moments, scales them, accumulates L_k with the 1 / h factors and then applies dt mr_k a1.  Here
// the moments stay raw (1D Gauss sums with the weights (5, 8, 5) taken as (1, 1.6, 1)) and every scale -
// 5/18, 5a/18, 1/54, 1/6, 1/2, 1/h, dt, mr_k, a1 - is folded on the host into 18 coefficients per stage
// (AdvArgs::kc, adv_coeffs in nxsdg.cu), so a tracer's update costs ~70 FP64 operations instead of ~150
// (the stage is bound by FP64 dependency latency).  Same quantities, another rounding order (~1e-16).
__device__ __forceinline__ void edge_raw(const double F[3], double& r0, double& r1, double& r2) {
    const double s = F[0] + F[2];
    r0 = fma(1.6, F[1], s);      // m0 = 5/18 r0
    r1 = F[2] - F[0];            // m1 = 5a/18 r1
    r2 = fma(-2.0, F[1], s);     // m2 = r2 / 54
}
// raw volume moments of G[gy][gx]: M00 = (5/18)^2 R00, M10 = (5/18)(5a/18) R10, M01 = (5/18)(5a/18) R01
__device__ __forceinline__ void vol_raw(const double G[3][3], double& R00, double& R10, double& R01) {
    double x0[3], x1[3];
#pragma unroll
    for (int gy = 0; gy < 3; ++gy) {
        x0[gy] = fma(1.6, G[gy][1], G[gy][0] + G[gy][2]);
        x1[gy] = G[gy][2] - G[gy][0];
    }
    R00 = fma(1.6, x0[1], x0[0] + x0[2]);
    R10 = fma(1.6, x1[1], x1[0] + x1[2]);
    R01 = x0[2] - x0[0];
}

template <int STAGES>
__global__ void __launch_bounds__(32 * ADV_TMA_WARPS, STAGES == 3 ? 5 : ADV_TMA_MINB)
k_advect_tma(const __grid_constant__ AdvMaps maps, AdvTmaArgs ta) {
    static_assert(STAGES >= 3, "rows k-1, k, k+1 in use");
    constexpr bool LATE = STAGES == 3;
    constexpr int P = LATE ? 0 : STAGES - 3;       // positions in flight beyond the three a job uses
    const AdvArgs& a = ta.a;
    extern __shared__ __align__(1024) unsigned char adv_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    AdvSlot* slot = reinterpret_cast<AdvSlot*>(adv_smem) + wib * STAGES;
    AdvC0* c0buf = reinterpret_cast<AdvC0*>(adv_smem + ADV_TMA_WARPS * STAGES * sizeof(AdvSlot)) + wib;
    uint64_t* bar = reinterpret_cast<uint64_t*>(adv_smem + adv_bar_off(STAGES)) + wib * STAGES;
    uint64_t* bar0 = reinterpret_cast<uint64_t*>(adv_smem + adv_bar_off(STAGES)) + ADV_TMA_WARPS * STAGES + wib;
    int4* desc = reinterpret_cast<int4*>(adv_smem + adv_desc_off(STAGES)) + wib * STAGES;
    const int twarps = gridDim.x * ADV_TMA_WARPS, gw = blockIdx.x * ADV_TMA_WARPS + wib;
    const int nunits = ta.nstrips * ta.nchunks;
    if (gw >= nunits) return;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        mbar_init(bar0, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    // load cursor (lane 0): the warp's units gw, gw + twarps, ...; each unit contributes the rows
    // lr0 - 1 .. lr1 (ring below, the chunk, ring above); desc = (unit, row, job?, 0)
    struct Cur { int u, k, lr0, lr1; bool ok; };
    auto unit_start = [&](int u, Cur& c) {
        c.ok = u < nunits;
        if (!c.ok) return;
        const int chunk = u / ta.nstrips;
        c.u = u;
        c.lr0 = a.erow_begin + chunk * ta.ty;
        c.lr1 = min(c.lr0 + ta.ty, a.erow_end);
        c.k = c.lr0 - 1;
    };
    auto step = [&](Cur& c) {
        if (++c.k > c.lr1) unit_start(c.u + twarps, c);
    };
    auto issue = [&](const Cur& c, int s) {
        desc[s] = make_int4(c.ok ? c.u : -1, c.k, (c.ok && c.k >= c.lr0 && c.k < c.lr1) ? 1 : 0, 0);
        if (!c.ok) return;
        AdvSlot* t = slot + s;
        const int ix0 = (c.u % ta.nstrips) * 31;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[s], kAdvTx);
        const int xs = (ix0 - 1) & ~1;
        tma3(&t->A[0][0], &maps.A, &bar[s], xs, c.k, 0);
        tma3(&t->H[0][0], &maps.H, &bar[s], xs, c.k, 0);
        tma2(&t->vx[0][0], &maps.vx, &bar[s], 2 * (ix0 - 1), 2 * c.k + 1);
        tma2(&t->vy[0][0], &maps.vy, &bar[s], 2 * (ix0 - 1), 2 * c.k + 1);
    };
    Cur cur;
    if (lane == 0) {
        unit_start(gw, cur);
        for (int q = 0; q <= (LATE ? 1 : P); ++q) {       // positions 0 .. P (LATE: 0, 1)
            issue(cur, q);
            if (cur.ok) step(cur);
        }
    }
    __syncwarp();
    uint32_t phase = 0;
    auto wait_slot = [&](int s) {
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
    };
    // c0 of a job (row r of unit u) into the warp's buffer; c0_inflight: issued and not yet consumed
    uint32_t ph0 = 0;
    bool c0_inflight = false;
    auto issue_c0 = [&](int u, int r) {   // lane 0; every lane's reads of the buffer are done (__syncwarp)
        const int xs = (((u % ta.nstrips) * 31) - 1) & ~1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar0, kAdvC0Tx);
        tma3(&c0buf->A[0][0], &maps.A0, bar0, xs, r, 0);
        tma3(&c0buf->H[0][0], &maps.H0, bar0, xs, r, 0);
    };
    const bool rk = a.a0 != 0.0;
    const int4 d0 = desc[0];
    if (d0.x < 0) return;
    wait_slot(0);
    // the north flux of a job is the south flux of the unit's next job (same edge, same function, same
    // inputs): carried in registers instead of evaluated twice; the unit's first job evaluates its own
    int prev_unit = -1;
    double cNA[3] = {0.0, 0.0, 0.0}, cNH[3] = {0.0, 0.0, 0.0};   // raw moments (r0, r1, r2) of the north edge
    for (int i = 0;; ++i) {
        const int sL = (i + STAGES - 1) % STAGES, sM = i % STAGES, sU = (i + 1) % STAGES;
        const int4 dM = desc[sM];
        if (dM.x < 0) break;
        if (!LATE && lane == 0) {              // position i + 1 + P into the slot of position i - 2 (done)
            issue(cur, (i + 1 + P) % STAGES);
            if (cur.ok) step(cur);
        }
        // LATE: position i + 2 into the slot of position i - 1 once nothing reads it any more (a ring
        // position reads nothing of it; a job after its south flux, below)
        auto issue_late = [&]() {
            if constexpr (LATE) {
                __syncwarp();
                if (lane == 0) {
                    issue(cur, sL);
                    if (cur.ok) step(cur);
                }
            }
        };
        if (!dM.z) issue_late();
        const int4 dU = desc[sU];              // issued at iteration i - P or in the prologue
        if (ta.dbg && lane == 0)
            printf("adv_tma blk %d w %d i %d M(u%d k%d j%d) U(u%d k%d j%d) rows [%d,%d) erows %d\n", blockIdx.x, wib, i,
                   dM.x, dM.y, dM.z, dU.x, dU.y, dU.z, a.erow_begin, a.erow_end, a.erows_local);
        // the RK combine input c0 (stages 2, 3): prefetched by TMA during the previous job of the unit, or (a
        // unit's first job) issued now - it is waited for only at the update, at the end of the job
        if (dM.z && rk && !c0_inflight) {
            if (lane == 0) issue_c0(dM.x, dM.y);
            c0_inflight = true;
        }
        if (dU.x >= 0) wait_slot(sU);          // position i+1 belongs to the same unit when i is a job
        if (dM.z) {                            // a job: element row r = dM.y of strip dM.x % nstrips
            const int r = dM.y;
            const int ix0 = (dM.x % ta.nstrips) * 31, ix = ix0 - 1 + lane;
            const int eo = (ix0 - 1) - ((ix0 - 1) & ~1);
            const bool valid = lane >= 1 && ix < a.nx;
            const AdvSlot& L = slot[sL];
            const AdvSlot& M = slot[sM];
            const AdvSlot& U = slot[sU];
            Cf<6> me, nb;
#pragma unroll
            for (int k = 0; k < 6; ++k) { me.A[k] = M.A[k][eo + lane]; me.H[k] = M.H[k][eo + lane]; }
            double ux[3][3], uy[3][3];   // node rows 2r (row below's slot), 2r+1, 2r+2
#pragma unroll
            for (int jx = 0; jx < 3; ++jx) {
                ux[0][jx] = L.vx[1][2 * lane + jx]; uy[0][jx] = L.vy[1][2 * lane + jx];
                ux[1][jx] = M.vx[0][2 * lane + jx]; uy[1][jx] = M.vy[0][2 * lane + jx];
                ux[2][jx] = M.vx[1][2 * lane + jx]; uy[2][jx] = M.vy[1][2 * lane + jx];
            }
            double FeA[3], FeH[3], FnA[3], FnH[3], FsA[3], FsH[3];
            {   // east edge (closed box: no flux through x = Lx)
#pragma unroll
                for (int k = 0; k < 6; ++k) { nb.A[k] = M.A[k][eo + lane + 1]; nb.H[k] = M.H[k][eo + lane + 1]; }
                double vn[3]; q2_interp3(ux[0][2], ux[1][2], ux[2][2], vn);
                q2_edge(true, me, nb, vn, ix >= 0 && ix + 1 < a.nx, FeA, FeH);
            }
            {   // north edge: the row above (ghost / next row, or none at the global top)
#pragma unroll
                for (int k = 0; k < 6; ++k) { nb.A[k] = U.A[k][eo + lane]; nb.H[k] = U.H[k][eo + lane]; }
                double vn[3]; q2_interp3(uy[2][0], uy[2][1], uy[2][2], vn);
                q2_edge(false, me, nb, vn, r + 1 < a.erow_end || a.has_north, FnA, FnH);
            }
            // raw edge moments (east, north here; west by shuffle of the east ones, south carried or evaluated)
            double rE[2][3], rN[2][3], rW[2][3], rS[2][3];
            edge_raw(FeA, rE[0][0], rE[0][1], rE[0][2]); edge_raw(FeH, rE[1][0], rE[1][1], rE[1][2]);
            edge_raw(FnA, rN[0][0], rN[0][1], rN[0][2]); edge_raw(FnH, rN[1][0], rN[1][1], rN[1][2]);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                rW[0][q] = __shfl_up_sync(0xffffffffu, rE[0][q], 1);
                rW[1][q] = __shfl_up_sync(0xffffffffu, rE[1][q], 1);
            }
            if (prev_unit == dM.x) {   // the previous job was the row below in this unit: its north moments
#pragma unroll
                for (int q = 0; q < 3; ++q) { rS[0][q] = cNA[q]; rS[1][q] = cNH[q]; }
            } else {   // south edge: the row below (ring row of the unit)
#pragma unroll
                for (int k = 0; k < 6; ++k) { nb.A[k] = L.A[k][eo + lane]; nb.H[k] = L.H[k][eo + lane]; }
                double vn[3]; q2_interp3(uy[0][0], uy[0][1], uy[0][2], vn);
                q2_edge(false, nb, me, vn, r > a.erow_begin || a.has_south, FsA, FsH);
                edge_raw(FsA, rS[0][0], rS[0][1], rS[0][2]); edge_raw(FsH, rS[1][0], rS[1][1], rS[1][2]);
            }
#pragma unroll
            for (int q = 0; q < 3; ++q) { cNA[q] = rN[0][q]; cNH[q] = rN[1][q]; }
            prev_unit = dM.x;
            issue_late();                      // row k - 1 (slot sL) is consumed
            // ---- volume term and update: k_advect_q2's code
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
            const int64_t eo_g = (int64_t)r * a.epitch + ix;
            double ncv[2][6];
#pragma unroll
            for (int tr = 0; tr < 2; ++tr) {
                const double* c = tr == 0 ? me.A : me.H;
                double cg[3][3], Gx[3][3], Gy[3][3];
                gp_vals(c, cg);
#pragma unroll
                for (int gy = 0; gy < 3; ++gy)
#pragma unroll
                    for (int g = 0; g < 3; ++g) { Gx[gy][g] = cg[gy][g] * gvx[gy][g]; Gy[gy][g] = cg[gy][g] * gvy[gy][g]; }
                double X00, X10, X01, Y00, Y10, Y01;
                vol_raw(Gx, X00, X10, X01);
                vol_raw(Gy, Y00, Y10, Y01);
                const double* e = rE[tr]; const double* w = rW[tr]; const double* n = rN[tr]; const double* so = rS[tr];
                const double d0x = w[0] - e[0], s0x = e[0] + w[0], d1x = w[1] - e[1], s1x = e[1] + w[1], d2x = w[2] - e[2];
                const double d0y = so[0] - n[0], s0y = n[0] + so[0], d1y = so[1] - n[1], s1y = n[1] + so[1], d2y = so[2] - n[2];
                // dt a1 mr_k L_k (k_advect_q2's L_k, every scale in a.kc)
                double Lk[6];
                Lk[0] = fma(a.kc[0], d0x, a.kc[1] * d0y);
                Lk[1] = fma(a.kc[2], X00, fma(a.kc[3], s0x, a.kc[4] * d1y));
                Lk[2] = fma(a.kc[5], Y00, fma(a.kc[6], d1x, a.kc[7] * s0y));
                Lk[3] = fma(a.kc[8], X10, fma(a.kc[9], d0x, a.kc[10] * d2y));
                Lk[4] = fma(a.kc[11], Y01, fma(a.kc[12], d2x, a.kc[13] * d0y));
                Lk[5] = fma(a.kc[14], X01, fma(a.kc[15], Y10, fma(a.kc[16], s1x, a.kc[17] * s1y)));
                if (tr == 0 && rk) {           // the job's c0 has landed in the buffer
                    mbar_wait(bar0, ph0);
                    ph0 ^= 1u;
                }
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    const double v = fma(a.a1, c[k], Lk[k]);
                    ncv[tr][k] = rk ? fma(a.a0, tr == 0 ? c0buf->A[k][eo + lane] : c0buf->H[k][eo + lane], v) : v;
                }
            }
            if (rk) {                          // every lane has read c0: the next job of this unit prefetches its own
                __syncwarp();
                c0_inflight = dU.x == dM.x && dU.z;
                if (lane == 0 && c0_inflight) issue_c0(dU.x, dU.y);
            }
            if (valid) {
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    a.Aout[k * a.eplane + eo_g] = ncv[0][k];
                    a.Hout[k * a.eplane + eo_g] = ncv[1][k];
                }
                if (a.Pg != nullptr) {   // last stage, single rank: the outer-step prep's P at the Gauss
                    double P[9];         // points of the new A, H (R#17 / Listing 2), bitwise = k_prep_elems_q2
                    pg_q2(ncv[1], ncv[0], a.Pstar, a.C_conc, P);
#pragma unroll
                    for (int g = 0; g < 9; ++g) a.Pg[g * a.eplane + eo_g] = P[g];
                }
            }
        }
        __syncwarp();   // every lane is done with slot sL before iteration i + 1 refills it
    }
}

}  // namespace nxk
