// Outer-step prep (row a1; Listing 2, R#17) for the configs' CG2 / DG2 pair (n_A = 6),
// structured: the table-driven k_prep_nodes<2, 6> / k_prep_elems<2, 6> of kernels.cuh looked the DG
// basis up in __constant__ with a per-thread node index (divergent constant-cache accesses, 4 gathers of
// 12 coefficients per node); here the DG2 values at the Q2 node positions (S, T in {-1/2, 0, 1/2}) are
// folded into the code, one thread updates the 2 x 2 nodes an element owns from the 4 elements around
// them, and the per-node arithmetic is k_prep_nodes' own (same sums in the same order: bitwise equal).
// The P at the Gauss points (pg_q2) is shared with the last advection stage, which produces it for
// the new A, H while they are still in registers.
#pragma once
#include "advect_q2.cuh"
#include "prep_node.cuh"

namespace nxk {

// P = P* h exp(-C (1 - a)) at the 9 Gauss points, h = max(0, H), a = clamp(A, 0, 1) (Listing 2)
__device__ __forceinline__ void pg_q2(const double h[6], const double c[6], double Pstar, double C, double P[9]) {
    double hg[3][3], ag[3][3];
    gp_vals(h, hg);
    gp_vals(c, ag);
#pragma unroll
    for (int gy = 0; gy < 3; ++gy)
#pragma unroll
        for (int gx = 0; gx < 3; ++gx) {
            const double hv = fmax(hg[gy][gx], 0.0), av = fmin(fmax(ag[gy][gx], 0.0), 1.0);
            P[gy * 3 + gx] = Pstar * hv * exp(-C * (1.0 - av));
        }
}

__global__ void k_prep_elems_q2(PrepArgs a) {
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, lr = blockIdx.y;
    if (ix >= a.nx || lr >= a.erows_local) return;
    const int64_t e = (int64_t)lr * a.epitch + ix;
    double h[6], c[6], P[9];
#pragma unroll
    for (int k = 0; k < 6; ++k) { h[k] = a.H[k * a.eplane + e]; c[k] = a.A[k * a.eplane + e]; }
    pg_q2(h, c, a.Pstar, a.C_conc, P);
#pragma unroll
    for (int g = 0; g < 9; ++g) a.Pg[g * a.eplane + e] = P[g];
}

__device__ __forceinline__ void prep_node_out(const PrepArgs& a, int jr, int I, double hs, double as, int cnt) {
    const int64_t n = (int64_t)jr * a.npitch + I;
    const PrepNodeOut o = prep_node_calc(a, hs, as, cnt, a.ax[n], a.ay[n], a.vx[n], a.vy[n], a.ox[n], a.oy[n]);
    a.c1[n] = o.c1; a.rx0[n] = o.rx0; a.ry0[n] = o.ry0; a.cafo[n] = o.cafo;
}

// thread (ix, pr): nodes (2 ix + q, 2 pr + jy), q, jy in {0, 1}, from elements (ix - 1 | ix, pr - 1 | pr)
__global__ void k_prep_nodes_q2(PrepArgs a) {
    const int ix = blockIdx.x * blockDim.x + threadIdx.x;
    const int pr = blockIdx.y * blockDim.y + threadIdx.y + (a.node_row_begin >> 1);
    if (ix > a.nx || 2 * pr >= a.node_row_end) return;
    // the 4 elements around the nodes [dy][dx]: dy = 0 the row below (pr - 1), dx = 0 the west one (ix - 1)
    double hE[2][2][6], aE[2][2][6];
    bool ok[2][2];
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
            const int ex = ix - 1 + dx, ey = pr - 1 + dy;
            ok[dy][dx] = ex >= 0 && ex < a.nx && ey >= 0 && ey < a.elem_rows_with_nodes;
            const int64_t e = (int64_t)(ok[dy][dx] ? ey : 0) * a.epitch + (ok[dy][dx] ? ex : 0);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                hE[dy][dx][k] = ok[dy][dx] ? a.H[k * a.eplane + e] : 0.0;
                aE[dy][dx][k] = ok[dy][dx] ? a.A[k * a.eplane + e] : 0.0;
            }
        }
#pragma unroll
    for (int jy = 0; jy < 2; ++jy) {
        const int jr = 2 * pr + jy;
        if (jr < a.node_row_begin || jr >= a.node_row_end) continue;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (2 * ix + q > 2 * a.nx) continue;
            double hs = 0.0, as = 0.0;
            int cnt = 0;
            // k_prep_nodes' order: SW, SE, NW, NE (the node's local position in each)
            if (jy == 0 && q == 0) {
                if (ok[0][0]) { hs += dg2_node<2, 2>(hE[0][0]); as += dg2_node<2, 2>(aE[0][0]); ++cnt; }
                if (ok[0][1]) { hs += dg2_node<0, 2>(hE[0][1]); as += dg2_node<0, 2>(aE[0][1]); ++cnt; }
                if (ok[1][0]) { hs += dg2_node<2, 0>(hE[1][0]); as += dg2_node<2, 0>(aE[1][0]); ++cnt; }
                if (ok[1][1]) { hs += dg2_node<0, 0>(hE[1][1]); as += dg2_node<0, 0>(aE[1][1]); ++cnt; }
            } else if (jy == 0) {
                if (ok[0][1]) { hs += dg2_node<1, 2>(hE[0][1]); as += dg2_node<1, 2>(aE[0][1]); ++cnt; }
                if (ok[1][1]) { hs += dg2_node<1, 0>(hE[1][1]); as += dg2_node<1, 0>(aE[1][1]); ++cnt; }
            } else if (q == 0) {
                if (ok[1][0]) { hs += dg2_node<2, 1>(hE[1][0]); as += dg2_node<2, 1>(aE[1][0]); ++cnt; }
                if (ok[1][1]) { hs += dg2_node<0, 1>(hE[1][1]); as += dg2_node<0, 1>(aE[1][1]); ++cnt; }
            } else {
                if (ok[1][1]) { hs += dg2_node<1, 1>(hE[1][1]); as += dg2_node<1, 1>(aE[1][1]); ++cnt; }
            }
            prep_node_out(a, jr, 2 * ix + q, hs, as, cnt);
        }
    }
}

// Row-marching form of k_prep_nodes_q2 (same sums, same order: bitwise equal): a warp owns a strip of 31
// element columns plus a ring lane (lane 0 = the column west of the strip, which only supplies its values)
// and marches up a chunk of element rows; each element's 12 coefficients are read once, its DG values at
// its 9 local nodes are formed once, the west neighbour's arrive by shuffle and the row below's top-node
// values are carried in registers (the chunk's first row evaluates its row below itself).  Per row every
// load the row needs - the element's coefficients and the 2 x 2 nodes' six inputs as 16-B pairs - is
// issued in one batch before any of it is used: one memory latency per row (ncu showed the first form,
// with separate coefficient, west-element and node-input phases, long-scoreboard bound at 42 % occupancy).
struct PrepNodeVals { double h[9], a[9]; };   // [jy * 3 + jx]
struct PrepCoef { double h[6], a[6]; };

__device__ __forceinline__ void prep_coef(const PrepArgs& a, int ex, int ey, bool ok, PrepCoef& c) {
    const int64_t e = (int64_t)(ok ? ey : 0) * a.epitch + (ok ? ex : 0);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        c.h[k] = ok ? __ldg(a.H + k * a.eplane + e) : 0.0;
        c.a[k] = ok ? __ldg(a.A + k * a.eplane + e) : 0.0;
    }
}
__device__ __forceinline__ void prep_vals(const PrepCoef& c, PrepNodeVals& v) {
    v.h[0] = dg2_node<0, 0>(c.h); v.h[1] = dg2_node<1, 0>(c.h); v.h[2] = dg2_node<2, 0>(c.h);
    v.h[3] = dg2_node<0, 1>(c.h); v.h[4] = dg2_node<1, 1>(c.h); v.h[5] = dg2_node<2, 1>(c.h);
    v.h[6] = dg2_node<0, 2>(c.h); v.h[7] = dg2_node<1, 2>(c.h); v.h[8] = dg2_node<2, 2>(c.h);
    v.a[0] = dg2_node<0, 0>(c.a); v.a[1] = dg2_node<1, 0>(c.a); v.a[2] = dg2_node<2, 0>(c.a);
    v.a[3] = dg2_node<0, 1>(c.a); v.a[4] = dg2_node<1, 1>(c.a); v.a[5] = dg2_node<2, 1>(c.a);
    v.a[6] = dg2_node<0, 2>(c.a); v.a[7] = dg2_node<1, 2>(c.a); v.a[8] = dg2_node<2, 2>(c.a);
}
// the six inputs of a lane's node pair (2 ix, 2 ix + 1) on one node row (the pair is 16-B aligned: npitch is
// even; at ix = nx the second node is row padding, loaded but never used)
struct PrepNodeIn { double2 ax, ay, vx, vy, ox, oy; };
__device__ __forceinline__ void prep_in(const PrepArgs& a, int64_t n, bool ok, PrepNodeIn& p) {
    const double2 z = make_double2(0.0, 0.0);
    p.ax = ok ? __ldg(reinterpret_cast<const double2*>(a.ax + n)) : z;
    p.ay = ok ? __ldg(reinterpret_cast<const double2*>(a.ay + n)) : z;
    p.vx = ok ? __ldg(reinterpret_cast<const double2*>(a.vx + n)) : z;
    p.vy = ok ? __ldg(reinterpret_cast<const double2*>(a.vy + n)) : z;
    p.ox = ok ? __ldg(reinterpret_cast<const double2*>(a.ox + n)) : z;
    p.oy = ok ? __ldg(reinterpret_cast<const double2*>(a.oy + n)) : z;
}

__host__ __device__ constexpr int prep_march_strips(int nx) { return (nx + 1 + 30) / 31; }

__global__ void __launch_bounds__(128) k_prep_nodes_march(PrepArgs a, int chunk) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nstrips = prep_march_strips(a.nx);       // element columns 0 .. nx (column nx: node column 2 nx)
    const int pr_lo = a.node_row_begin >> 1, pr_hi = (a.node_row_end + 1) >> 1;   // element rows with owned nodes
    const int nchunks = (pr_hi - pr_lo + chunk - 1) / chunk;
    if (warp >= nstrips * nchunks) return;
    const int strip = warp % nstrips, ch = warp / nstrips;
    const int ix = strip * 31 - 1 + lane;              // lane 0: the ring column west of the strip
    const int pr0 = pr_lo + ch * chunk, pr1 = min(pr0 + chunk, pr_hi);
    const bool colok = lane >= 1 && ix <= a.nx;
    auto okE = [&](int ex, int ey) { return ex >= 0 && ex < a.nx && ey >= 0 && ey < a.elem_rows_with_nodes; };
    // row below the chunk (pr0 - 1): own values, the west ones by shuffle
    PrepNodeVals below, belowW;
    bool okB = okE(ix, pr0 - 1), okBW;
    {
        PrepCoef cb;
        prep_coef(a, ix, pr0 - 1, okB, cb);
        prep_vals(cb, below);
#pragma unroll
        for (int j = 0; j < 9; ++j) { belowW.h[j] = __shfl_up_sync(0xffffffffu, below.h[j], 1); belowW.a[j] = __shfl_up_sync(0xffffffffu, below.a[j], 1); }
        okBW = __shfl_up_sync(0xffffffffu, okB, 1);
    }
    for (int pr = pr0; pr < pr1; ++pr) {
        const bool okM = okE(ix, pr);
        PrepCoef cM;
        prep_coef(a, ix, pr, okM, cM);
        PrepNodeIn in[2];
        bool rowok[2];
#pragma unroll
        for (int jy = 0; jy < 2; ++jy) {
            const int jr = 2 * pr + jy;
            rowok[jy] = colok && jr >= a.node_row_begin && jr < a.node_row_end;
            prep_in(a, (int64_t)jr * a.npitch + 2 * ix, rowok[jy], in[jy]);
        }
        PrepNodeVals me, W;
        prep_vals(cM, me);
#pragma unroll
        for (int j = 0; j < 9; ++j) { W.h[j] = __shfl_up_sync(0xffffffffu, me.h[j], 1); W.a[j] = __shfl_up_sync(0xffffffffu, me.a[j], 1); }
        const bool okW = __shfl_up_sync(0xffffffffu, okM, 1);
#pragma unroll
        for (int jy = 0; jy < 2; ++jy) {
            if (!rowok[jy]) continue;
            const int jr = 2 * pr + jy;
            PrepNodeOut o[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                double hs = 0.0, as = 0.0;
                int cnt = 0;
                // k_prep_nodes' order SW, SE, NW, NE with the node's position in each element
                if (jy == 0 && q == 0) {
                    if (okBW) { hs += belowW.h[8]; as += belowW.a[8]; ++cnt; }
                    if (okB) { hs += below.h[6]; as += below.a[6]; ++cnt; }
                    if (okW) { hs += W.h[2]; as += W.a[2]; ++cnt; }
                    if (okM) { hs += me.h[0]; as += me.a[0]; ++cnt; }
                } else if (jy == 0) {
                    if (okB) { hs += below.h[7]; as += below.a[7]; ++cnt; }
                    if (okM) { hs += me.h[1]; as += me.a[1]; ++cnt; }
                } else if (q == 0) {
                    if (okW) { hs += W.h[5]; as += W.a[5]; ++cnt; }
                    if (okM) { hs += me.h[3]; as += me.a[3]; ++cnt; }
                } else {
                    if (okM) { hs += me.h[4]; as += me.a[4]; ++cnt; }
                }
                const PrepNodeIn& p = in[jy];
                o[q] = q == 0 ? prep_node_calc(a, hs, as, cnt, p.ax.x, p.ay.x, p.vx.x, p.vy.x, p.ox.x, p.oy.x)
                              : prep_node_calc(a, hs, as, cnt, p.ax.y, p.ay.y, p.vx.y, p.vy.y, p.ox.y, p.oy.y);
            }
            const int64_t n = (int64_t)jr * a.npitch + 2 * ix;
            if (ix < a.nx) {
                *reinterpret_cast<double2*>(a.c1 + n) = make_double2(o[0].c1, o[1].c1);
                *reinterpret_cast<double2*>(a.rx0 + n) = make_double2(o[0].rx0, o[1].rx0);
                *reinterpret_cast<double2*>(a.ry0 + n) = make_double2(o[0].ry0, o[1].ry0);
                *reinterpret_cast<double2*>(a.cafo + n) = make_double2(o[0].cafo, o[1].cafo);
            } else {                                    // ix = nx: node column 2 nx only
                a.c1[n] = o[0].c1; a.rx0[n] = o[0].rx0; a.ry0[n] = o[0].ry0; a.cafo[n] = o[0].cafo;
            }
        }
        below = me; belowW = W; okB = okM; okBW = okW;
    }
}

}  // namespace nxk
