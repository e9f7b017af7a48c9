// Hot-path kernels for sm_100a, FP64.  DESIGN.md §6 has the byte and
// instruction budgets; the citations name the PAPER.md passage each step follows.
//
// Device layout:
//   element fields  : SoA planes, plane k at base + k*eplane, element (lr, ix) at lr*nx + ix,
//                     lr = local element row (ghost rows included)
//   node fields     : row-pitched grid, node (jr, I) at jr*npitch + I, jr = local node row
//   S buffer        : 3*NS planes: S11[0..NS), S12[0..NS), S22[0..NS)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tables.cuh"

namespace nxk {

template <int P, int NS_ = (P == 1) ? 3 : 6> struct Deg {
    static constexpr int NS = NS_;                // DG stress dofs (R#6; 8 = R#24)
    static constexpr int TAB = tab_index(P, NS_);  // c_tab slot
    static constexpr int NGP = P + 1;             // Listing 2
    static constexpr int NG = NGP * NGP;
    static constexpr int NCG = (P + 1) * (P + 1);
};

// --------------------------------------------------------------------------
// Outer-step constants (K0p): nodal H, A (R#17) folded into the per-node
// velocity constants of O8, and P at the element Gauss points.
// --------------------------------------------------------------------------
struct PrepArgs {
    const double* H; const double* A;          // NA planes each
    const double* vx; const double* vy;        // v^n (current v)
    const double* ox; const double* oy; const double* ax; const double* ay;
    double* c1; double* rx0; double* ry0; double* cafo;
    double* Pg;                                // NG planes
    int64_t eplane, npitch, epitch;            // plane stride, node row pitch, element row pitch
    int nx, erows_local;                       // stored element rows (incl. ghosts)
    int node_row_begin, node_row_end;          // owned local node rows [begin, end)
    int elem_rows_with_nodes;                  // element rows that touch stored nodes (excl. upper ghost)
    double rho_ice, Fa, Fo, f_c, dt, Pstar, C_conc;
    double rdt;                                // 1 / dt
};

template <int P, int NA>
__global__ void k_prep_nodes(PrepArgs a) {
    const RefTab& T = c_tab[P - 1];
    int I = blockIdx.x * blockDim.x + threadIdx.x;
    int jr = a.node_row_begin + blockIdx.y;
    if (I > P * a.nx || jr >= a.node_row_end) return;
    double hs = 0.0, as = 0.0;
    int cnt = 0;
    // adjacent elements in fixed order SW, SE, NW, NE
#pragma unroll
    for (int dy = 1; dy >= 0; --dy)
#pragma unroll
        for (int dx = 1; dx >= 0; --dx) {
            int ex = I / P - dx, ey = jr / P - dy;
            int jx = I - P * ex, jy = jr - P * ey;
            if (ex < 0 || ex >= a.nx || ey < 0 || ey >= a.elem_rows_with_nodes) continue;
            if (jx < 0 || jx > P || jy < 0 || jy > P) continue;
            int j = jy * (P + 1) + jx;
            int64_t e = (int64_t)ey * a.epitch + ex;
            double hv = 0.0, av = 0.0;
#pragma unroll
            for (int k = 0; k < NA; ++k) {
                hv += a.H[k * a.eplane + e] * T.psinode[k][j];
                av += a.A[k * a.eplane + e] * T.psinode[k][j];
            }
            hs += hv; as += av; ++cnt;
        }
    double Hn = fmax(hs / cnt, 1e-4);
    double An = fmin(fmax(as / cnt, 0.0), 1.0);
    int64_t n = (int64_t)jr * a.npitch + I;
    double m = a.rho_ice * Hn;
    double c1 = m / a.dt;
    double axv = a.ax[n], ayv = a.ay[n];
    double amag = sqrt(axv * axv + ayv * ayv);
    double drag = An * a.Fa * amag;
    a.c1[n] = c1;
    a.rx0[n] = c1 * a.vx[n] + drag * axv - m * a.f_c * a.oy[n];
    a.ry0[n] = c1 * a.vy[n] + drag * ayv + m * a.f_c * a.ox[n];
    a.cafo[n] = An * a.Fo;
}

template <int P, int NA>
__global__ void k_prep_elems(PrepArgs a) {
    constexpr int NG = Deg<P>::NG;
    const RefTab& T = c_tab[P - 1];
    int ix = blockIdx.x * blockDim.x + threadIdx.x;
    int lr = blockIdx.y;
    if (ix >= a.nx || lr >= a.erows_local) return;
    int64_t e = (int64_t)lr * a.epitch + ix;
    double h[NA], c[NA];
#pragma unroll
    for (int k = 0; k < NA; ++k) { h[k] = a.H[k * a.eplane + e]; c[k] = a.A[k * a.eplane + e]; }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        double hv = 0.0, av = 0.0;
#pragma unroll
        for (int k = 0; k < NA; ++k) { hv += h[k] * T.psi[k][g]; av += c[k] * T.psi[k][g]; }
        hv = fmax(hv, 0.0);
        av = fmin(fmax(av, 0.0), 1.0);
        a.Pg[g * a.eplane + e] = a.Pstar * hv * exp(-a.C_conc * (1.0 - av));
    }
}

// --------------------------------------------------------------------------
// Fused subcycle kernel: strain + stress + divergence gather + velocity, one
// pass over HBM per subcycle (DESIGN.md §6 "K_sub").
//
// Mapping: one warp = a strip of 32 element columns (lane 0 is the ring
// element ix0-1, recomputed; lanes 1..31 own their elements) marching up a
// chunk of element rows, preceded by one ring row.  A lane owns the node
// columns P*ix .. P*ix+P-1 of its element.  Node values and divergence
// contributions move between lanes by warp shuffles; node-row sums carry
// in registers from one element row to the next.  No shared memory, no
// atomics: every node sum has the fixed order (row below, then W, E), so the
// result is deterministic and independent of the strip/chunk/rank partition.
// --------------------------------------------------------------------------
struct SubArgs {
    const double* __restrict__ S_in; double* __restrict__ S_out;
    const double* __restrict__ Pg;
    const double* __restrict__ vx_in; const double* __restrict__ vy_in;
    double* __restrict__ vx_out; double* __restrict__ vy_out;
    const double* __restrict__ c1; const double* __restrict__ rx0; const double* __restrict__ ry0;
    const double* __restrict__ cafo; const double* __restrict__ ox; const double* __restrict__ oy;
    int64_t eplane, npitch, epitch;
    int nx, nstrips, ty;
    int erow_begin, erow_end;       // owned local element rows
    int bottom_boundary;            // local element row erow_begin touches global node row 0
    int top_boundary;               // node row P*erow_end is the global top row
    double ihx, ihy, fac, ainv, dmin2, beta, b1, kc;
    int repl;
    int* work_counter;              // TMA kernel: dynamic unit counter (zeroed before the launch), or null
    int chunk0, chunk_step, nsel;   // chunk selection: chunks chunk0 + i*chunk_step, i < nsel
    // P2P transport, fused peer stores (TMA kernel): the rows a neighbour needs are stored straight
    // into its buffers (peer memory) as they are computed; null pointers = off
    double* peer_vx_up; double* peer_vy_up; double* peer_S_up;   // upper neighbour's new-state buffers
    double* peer_vx_dn; double* peer_vy_dn;                      // lower neighbour's
    int up_node_row0;               // local node rows >= this go up (to the neighbour's rows 0 ..)
    int up_elem_row;                // local element row whose S goes up (to the neighbour's row 0)
    int dn_node_row, dn_dst_row;    // local node row that goes down, and its row at the neighbour
    int64_t peer_up_eplane;         // the upper neighbour's element plane stride
    int ntail, qtail;               // persistent kernels: the last ntail selected chunks are split into
                                    // qtail sub-units each (0 / 1 = off)
    int l2_hints;                   // box TMA kernel: L2 eviction-policy bits (subcycle_tma.cuh)
    int vcarry;                     // box TMA kernel: shared v node row carried in registers (subcycle_tma.cuh)
    // NEXT-4 sphere (R#26; box TMA kernel instantiated with SPH): per local element row geometry table
    // (kSphRow doubles, nxsdg.cu sphere_tables); ihx = 1 / (R dlon), ihy = 1 / (R dlat) then
    const double* __restrict__ sph_rows;
    // the first fused subcycle of an outer step forming the node constants itself (box TMA kernel
    // instantiated with PREP, single rank): the prep's inputs / outputs and constants
    PrepArgs pa;
    // two subcycles per launch (box TMA kernel instantiated with PAIR): pass A's outputs S^{p+1}, v^{p+1}
    double* Sx; double* vxx; double* vyx;
};
// sphere row table layout (doubles per local element row)
constexpr int kSphRow = 32;
enum { SPH_COS = 0, SPH_SINR = 3, SPH_QA = 6, SPH_QB = 15, SPH_QC = 19, SPH_IMU = 20, SPH_COS_S = 26, SPH_COS_N = 27 };

// Unit u of a persistent kernel's work list -> strip and element rows [lr0, lr1) (lr0 >= lr1: empty).
// Whole chunks come first, strip-fastest; the last a.ntail selected chunks follow as a.qtail
// sub-units each, so the final units handed out are short and the warps finish together
// (tail split).  Every partition gives bitwise the same result (ring recomputation,
// fixed-order node sums).
__device__ __forceinline__ int units_total(const SubArgs& a) {
    return a.nstrips * (a.nsel + a.ntail * (a.qtail - 1));
}
__device__ __forceinline__ void unit_rows(const SubArgs& a, int u, int& strip, int& lr0, int& lr1) {
    const int nbulk = a.nstrips * (a.nsel - a.ntail);
    int i, sub = 0, q = 1;
    if (u < nbulk) {
        strip = u % a.nstrips; i = u / a.nstrips;
    } else {
        const int v = u - nbulk, k = v / a.nstrips;
        strip = v % a.nstrips; i = a.nsel - a.ntail + k / a.qtail; sub = k % a.qtail; q = a.qtail;
    }
    const int c0 = a.erow_begin + (a.chunk0 + i * a.chunk_step) * a.ty, c1 = min(c0 + a.ty, a.erow_end);
    const int per = (a.ty + q - 1) / q;
    lr0 = c0 + sub * per; lr1 = min(lr0 + per, c1);
}

template <int P, int NS_ = Deg<P>::NS>
__global__ void __launch_bounds__(128) k_subcycle(SubArgs a) {
    using D = Deg<P, NS_>;
    constexpr int NS = D::NS, NG = D::NG, NCG = D::NCG;
    const RefTab& T = c_tab[D::TAB];
    const int lane = threadIdx.x & 31;
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int strip = gwarp % a.nstrips, ci = gwarp / a.nstrips;
    if (ci >= a.nsel) return;                    // whole warp exits together
    const int lr0 = a.erow_begin + (a.chunk0 + ci * a.chunk_step) * a.ty;
    if (lr0 >= a.erow_end) return;
    const int lr1 = min(lr0 + a.ty, a.erow_end);
    const int ix = strip * 31 - 1 + lane;
    const bool evalid = ix >= 0 && ix < a.nx;
    const int I0 = P * ix;                        // first node column of this lane
    const bool nvalid = lane >= 1 && ix >= 0 && ix <= a.nx;   // lane owns node columns
    const int64_t npitch = a.npitch, eplane = a.eplane;

    // rolling node window: rows 0..P of the current element row, own columns q < P,
    // and the extra column I0 + P (lane+1's first column) per row
    double vx[P + 1][P], vy[P + 1][P], vxe[P + 1], vye[P + 1];
    double carx[P], cary[P];

    auto load_row = [&](int jr, double* rx, double* ry, double& ex, double& ey) {
        const double* px = a.vx_in + (int64_t)jr * npitch;
        const double* py = a.vy_in + (int64_t)jr * npitch;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            int I = I0 + q;
            bool ok = ix >= 0 && I <= P * a.nx;
            rx[q] = ok ? __ldg(px + I) : 0.0;
            ry[q] = ok ? __ldg(py + I) : 0.0;
        }
        double sx = __shfl_down_sync(0xffffffffu, rx[0], 1);
        double sy = __shfl_down_sync(0xffffffffu, ry[0], 1);
        if (lane == 31) {
            int I = I0 + P;
            bool ok = I <= P * a.nx;
            sx = ok ? __ldg(px + I) : 0.0;
            sy = ok ? __ldg(py + I) : 0.0;
        }
        ex = sx; ey = sy;
    };

    int lr = lr0 > 0 ? lr0 - 1 : lr0;   // ring row below the chunk when it exists
    bool ring = lr < lr0;
    load_row(P * lr, vx[0], vy[0], vxe[0], vye[0]);
#pragma unroll
    for (int q = 0; q < P; ++q) { carx[q] = 0.0; cary[q] = 0.0; }

    for (; lr < lr1; ++lr) {
#pragma unroll
        for (int r = 1; r <= P; ++r) load_row(P * lr + r, vx[r], vy[r], vxe[r], vye[r]);
        const int64_t e = (int64_t)lr * a.epitch + ix;
        double s11[NS], s12[NS], s22[NS], pg[NG];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            s11[k] = evalid ? __ldg(a.S_in + (0 * NS + k) * eplane + e) : 0.0;
            s12[k] = evalid ? __ldg(a.S_in + (1 * NS + k) * eplane + e) : 0.0;
            s22[k] = evalid ? __ldg(a.S_in + (2 * NS + k) * eplane + e) : 0.0;
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) pg[g] = evalid ? __ldg(a.Pg + g * eplane + e) : 0.0;

        // ---- strain at the Gauss points (Table 1 "strain"; composite K = Pi_DG dphi)
        //      + stress update per Gauss point (Listing 2) accumulated into S
#pragma unroll
        for (int k = 0; k < NS; ++k) { s11[k] *= a.fac; s12[k] *= a.fac; s22[k] *= a.fac; }
        // velocities relative to one node of the element: the strain rows sum to zero, so this
        // is exact in real arithmetic and removes the cancellation of sum_j K_j v_j (the VP law
        // amplifies strain roundoff by P/Delta near rigid ice)
        double dvx[NCG], dvy[NCG];
        {
            const double rx_ = vx[P / 2][P / 2 < P ? P / 2 : 0], ry_ = vy[P / 2][P / 2 < P ? P / 2 : 0];
#pragma unroll
            for (int jy = 0; jy <= P; ++jy)
#pragma unroll
                for (int jx = 0; jx <= P; ++jx) {
                    const double ux = (jx < P) ? vx[jy][jx < P ? jx : 0] : vxe[jy];
                    const double uy = (jx < P) ? vy[jy][jx < P ? jx : 0] : vye[jy];
                    dvx[jy * (P + 1) + jx] = ux - rx_;
                    dvy[jy * (P + 1) + jx] = uy - ry_;
                }
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            double dxs = 0.0, dxt = 0.0, dys = 0.0, dyt = 0.0;
#pragma unroll
            for (int jy = 0; jy <= P; ++jy)
#pragma unroll
                for (int jx = 0; jx <= P; ++jx) {
                    const int j = jy * (P + 1) + jx;
                    const double ux = dvx[j], uy = dvy[j];
                    dxs = fma(T.Ks[g][j], ux, dxs);
                    dxt = fma(T.Kt[g][j], ux, dxt);
                    dys = fma(T.Ks[g][j], uy, dys);
                    dyt = fma(T.Kt[g][j], uy, dyt);
                }
            const double e11 = a.ihx * dxs;
            const double e22 = a.ihy * dyt;
            const double e12 = 0.5 * (a.ihy * dxt + a.ihx * dys);
            const double draw2 = 1.25 * (e11 * e11 + e22 * e22) + 1.5 * e11 * e22 + e12 * e12;
            const double rD = rsqrt(a.dmin2 + draw2);           // 1 / DELTA
            const double Pa = pg[g] * a.ainv;                   // alpha^{-1} P
            const double PD = Pa * rD;                          // alpha^{-1} P / DELTA
            const double Ph = a.repl ? 0.5 * PD * sqrt(draw2) : 0.5 * Pa;
            const double g11 = PD * (0.625 * e11 + 0.375 * e22) - Ph;
            const double g12 = PD * (0.25 * e12);
            const double g22 = PD * (0.625 * e22 + 0.375 * e11) - Ph;
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                s11[k] = fma(T.R[k][g], g11, s11[k]);
                s12[k] = fma(T.R[k][g], g12, s12[k]);
                s22[k] = fma(T.R[k][g], g22, s22[k]);
            }
        }
        if (!ring && evalid && lane >= 1) {
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                a.S_out[(0 * NS + k) * eplane + e] = s11[k];
                a.S_out[(1 * NS + k) * eplane + e] = s12[k];
                a.S_out[(2 * NS + k) * eplane + e] = s22[k];
            }
        }

        // ---- divergence contributions of this element to its NCG nodes,
        //      sum_k D[j][k] S_k; the minus sign and 1/lumped-mass are applied at the node
        double rx[NCG], ry[NCG];
#pragma unroll
        for (int j = 0; j < NCG; ++j) {
            double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                ax = fma(T.Ds[j][k], s11[k], ax);
                bx = fma(T.Dt[j][k], s12[k], bx);
                ay = fma(T.Ds[j][k], s12[k], ay);
                by = fma(T.Dt[j][k], s22[k], by);
            }
            rx[j] = evalid ? a.ihx * ax + a.ihy * bx : 0.0;
            ry[j] = evalid ? a.ihx * ay + a.ihy * by : 0.0;
        }

        // ---- per-node gather (fixed order: row below, W element, E element) + velocity update
#pragma unroll
        for (int jy = 0; jy <= P; ++jy) {
            const double wx = __shfl_up_sync(0xffffffffu, rx[jy * (P + 1) + P], 1);
            const double wy = __shfl_up_sync(0xffffffffu, ry[jy * (P + 1) + P], 1);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                double sx = rx[jy * (P + 1) + q], sy = ry[jy * (P + 1) + q];
                if (q == 0) { sx = wx + sx; sy = wy + sy; }
                if (jy == P) { carx[q] = sx; cary[q] = sy; continue; }
                if (jy == 0) { sx = carx[q] + sx; sy = cary[q] + sy; }
                if (ring || !nvalid) continue;
                const int I = I0 + q;
                if (I > P * a.nx) continue;
                const int jr = P * lr + jy;
                const int64_t n = (int64_t)jr * npitch + I;
                const bool bnd = (I == 0) || (I == P * a.nx) || (jy == 0 && lr == a.erow_begin && a.bottom_boundary);
                double nvx = 0.0, nvy = 0.0;
                if (!bnd) {
                    const double im = T.invm[q][jy < P ? jy : 0];
                    const double fx = -sx * im, fy = -sy * im;   // F / lumped mass
                    const double vxo = vx[jy][q], vyo = vy[jy][q];
                    const double c1 = __ldg(a.c1 + n), cf = __ldg(a.cafo + n);
                    const double oxv = __ldg(a.ox + n), oyv = __ldg(a.oy + n);
                    const double dx = oxv - vxo, dy = oyv - vyo;
                    const double w = sqrt(dx * dx + dy * dy);
                    const double cw = cf * w;
                    const double rden = 1.0 / fma(c1, a.b1, cw);
                    const double cb = c1 * a.beta, ck = c1 * a.kc;
                    nvx = (cb * vxo + __ldg(a.rx0 + n) + cw * oxv + ck * vyo + fx) * rden;
                    nvy = (cb * vyo + __ldg(a.ry0 + n) + cw * oyv - ck * vxo + fy) * rden;
                }
                a.vx_out[n] = nvx;
                a.vy_out[n] = nvy;
            }
        }
        // roll the node window
#pragma unroll
        for (int q = 0; q < P; ++q) { vx[0][q] = vx[P][q]; vy[0][q] = vy[P][q]; }
        vxe[0] = vxe[P]; vye[0] = vye[P];
        ring = false;
    }
    // global top boundary row (Dirichlet)
    if (a.top_boundary && lr1 == a.erow_end && nvalid) {
        const int jr = P * lr1;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const int I = I0 + q;
            if (I > P * a.nx) continue;
            a.vx_out[(int64_t)jr * npitch + I] = 0.0;
            a.vy_out[(int64_t)jr * npitch + I] = 0.0;
        }
    }
}

// --------------------------------------------------------------------------
// Unfused debug steps (NXSDG_UNFUSED / nxsdg_run_step): the four Table 1
// steps as separate kernels, written literally (E materialised, Listing 2 with
// P recomputed from H, A, F materialised).  Parity of each step alone.
// --------------------------------------------------------------------------
struct StepArgs {
    const double* vx_in; const double* vy_in; double* vx_out; double* vy_out;
    double* S;  double* E;  double* Fx; double* Fy;  const double* H; const double* A;
    const double* c1; const double* rx0; const double* ry0; const double* cafo;
    const double* ox; const double* oy;
    int64_t eplane, npitch, epitch;
    int nx, erow_begin, erow_end, elem_rows_with_nodes;
    int node_row_begin, node_row_end;
    int node_row_global0;          // global index of local node row 0
    int node_rows_global;          // P*ny + 1
    double ihx, ihy, area, fac, ainv, dmin2, beta, b1, kc, Pstar, C_conc;
    int repl;
};

// Table 1 "strain": E_c = R . eps_c(g), eps from the CG gradient at the Gauss points.
template <int P, int NS_ = Deg<P>::NS>
__global__ void k_strain(StepArgs a) {
    using D = Deg<P, NS_>;
    constexpr int NS = D::NS, NG = D::NG;
    const RefTab& T = c_tab[D::TAB];
    int ix = blockIdx.x * blockDim.x + threadIdx.x;
    int lr = a.erow_begin + blockIdx.y;
    if (ix >= a.nx || lr >= a.erow_end) return;
    double ux[P + 1][P + 1], uy[P + 1][P + 1];
    const int64_t nref = (int64_t)(P * lr + P / 2) * a.npitch + P * ix + P / 2;
    const double rx_ = a.vx_in[nref], ry_ = a.vy_in[nref];   // reference node (see k_subcycle)
    for (int jy = 0; jy <= P; ++jy)
        for (int jx = 0; jx <= P; ++jx) {
            int64_t n = (int64_t)(P * lr + jy) * a.npitch + P * ix + jx;
            ux[jy][jx] = a.vx_in[n] - rx_; uy[jy][jx] = a.vy_in[n] - ry_;
        }
    double E11[NS] = {}, E12[NS] = {}, E22[NS] = {};
    for (int g = 0; g < NG; ++g) {
        double dxs = 0, dxt = 0, dys = 0, dyt = 0;
        for (int jy = 0; jy <= P; ++jy)
            for (int jx = 0; jx <= P; ++jx) {
                int j = jy * (P + 1) + jx;
                dxs += T.dphis[j][g] * ux[jy][jx]; dxt += T.dphit[j][g] * ux[jy][jx];
                dys += T.dphis[j][g] * uy[jy][jx]; dyt += T.dphit[j][g] * uy[jy][jx];
            }
        double e11 = a.ihx * dxs, e22 = a.ihy * dyt, e12 = 0.5 * (a.ihy * dxt + a.ihx * dys);
        for (int k = 0; k < NS; ++k) {
            E11[k] += T.R[k][g] * e11; E12[k] += T.R[k][g] * e12; E22[k] += T.R[k][g] * e22;
        }
    }
    int64_t e = (int64_t)lr * a.epitch + ix;
    for (int k = 0; k < NS; ++k) {
        a.E[(0 * NS + k) * a.eplane + e] = E11[k];
        a.E[(1 * NS + k) * a.eplane + e] = E12[k];
        a.E[(2 * NS + k) * a.eplane + e] = E22[k];
    }
}

// Listing 2 literally, with the stored E and P from H, A.
template <int P, int NA, int NS_ = Deg<P>::NS>
__global__ void k_stress(StepArgs a) {
    using D = Deg<P, NS_>;
    constexpr int NS = D::NS, NG = D::NG;
    const RefTab& T = c_tab[D::TAB];
    int ix = blockIdx.x * blockDim.x + threadIdx.x;
    int lr = a.erow_begin + blockIdx.y;
    if (ix >= a.nx || lr >= a.erow_end) return;
    int64_t e = (int64_t)lr * a.epitch + ix;
    double r11[NG], r12[NG], r22[NG];
    for (int g = 0; g < NG; ++g) {
        double hv = 0, av = 0, e11 = 0, e12 = 0, e22 = 0;
        for (int k = 0; k < NA; ++k) { hv += a.H[k * a.eplane + e] * T.psi[k][g]; av += a.A[k * a.eplane + e] * T.psi[k][g]; }
        for (int k = 0; k < NS; ++k) {
            e11 += a.E[(0 * NS + k) * a.eplane + e] * T.psi[k][g];
            e12 += a.E[(1 * NS + k) * a.eplane + e] * T.psi[k][g];
            e22 += a.E[(2 * NS + k) * a.eplane + e] * T.psi[k][g];
        }
        hv = fmax(hv, 0.0); av = fmin(fmax(av, 0.0), 1.0);
        double Pp = a.Pstar * hv * exp(-a.C_conc * (1.0 - av));
        double draw2 = 1.25 * (e11 * e11 + e22 * e22) + 1.5 * e11 * e22 + e12 * e12;
        double DELTA = sqrt(a.dmin2 + draw2);
        double PD = Pp / DELTA;
        double Pr = a.repl ? Pp * sqrt(draw2) / DELTA : Pp;
        r11[g] = a.ainv * (PD * (0.625 * e11 + 0.375 * e22) - 0.5 * Pr);
        r12[g] = a.ainv * (PD * 0.25 * e12);
        r22[g] = a.ainv * (PD * (0.625 * e22 + 0.375 * e11) - 0.5 * Pr);
    }
    for (int k = 0; k < NS; ++k) {
        double p11 = 0, p12 = 0, p22 = 0;
        for (int g = 0; g < NG; ++g) { p11 += T.R[k][g] * r11[g]; p12 += T.R[k][g] * r12[g]; p22 += T.R[k][g] * r22[g]; }
        double* s = a.S + e;
        s[(0 * NS + k) * a.eplane] = a.fac * s[(0 * NS + k) * a.eplane] + p11;
        s[(1 * NS + k) * a.eplane] = a.fac * s[(1 * NS + k) * a.eplane] + p12;
        s[(2 * NS + k) * a.eplane] = a.fac * s[(2 * NS + k) * a.eplane] + p22;
    }
}

// Table 1 "divergence": F_j = -|K| sum_{K ∋ j} (ihx Ds[j].S11 + ihy Dt[j].S12, ...), per-node gather.
template <int P, int NS_ = Deg<P>::NS>
__global__ void k_divergence(StepArgs a) {
    constexpr int NS = NS_;
    const RefTab& T = c_tab[Deg<P, NS_>::TAB];
    int I = blockIdx.x * blockDim.x + threadIdx.x;
    int jr = a.node_row_begin + blockIdx.y;
    if (I > P * a.nx || jr >= a.node_row_end) return;
    double fx = 0.0, fy = 0.0;
    for (int dy = 1; dy >= 0; --dy)
        for (int dx = 1; dx >= 0; --dx) {
            int ex = I / P - dx, ey = jr / P - dy;
            int jx = I - P * ex, jy = jr - P * ey;
            if (ex < 0 || ex >= a.nx || ey < 0 || ey >= a.elem_rows_with_nodes) continue;
            if (jx < 0 || jx > P || jy < 0 || jy > P) continue;
            int j = jy * (P + 1) + jx;
            int64_t e = (int64_t)ey * a.epitch + ex;
            double ax = 0, bx = 0, ay = 0, by = 0;
            for (int k = 0; k < NS; ++k) {
                double s11 = a.S[(0 * NS + k) * a.eplane + e], s12 = a.S[(1 * NS + k) * a.eplane + e];
                double s22 = a.S[(2 * NS + k) * a.eplane + e];
                ax += T.Ds[j][k] * s11; bx += T.Dt[j][k] * s12;
                ay += T.Ds[j][k] * s12; by += T.Dt[j][k] * s22;
            }
            fx += a.ihx * ax + a.ihy * bx;
            fy += a.ihx * ay + a.ihy * by;
        }
    int64_t n = (int64_t)jr * a.npitch + I;
    a.Fx[n] = -a.area * fx;
    a.Fy[n] = -a.area * fy;
}

// Table 1 "velocity", O8 with the stored F.
template <int P>
__global__ void k_velocity(StepArgs a) {
    const RefTab& T = c_tab[P - 1];
    int I = blockIdx.x * blockDim.x + threadIdx.x;
    int jr = a.node_row_begin + blockIdx.y;
    if (I > P * a.nx || jr >= a.node_row_end) return;
    int64_t n = (int64_t)jr * a.npitch + I;
    int Jg = a.node_row_global0 + jr;
    if (I == 0 || I == P * a.nx || Jg == 0 || Jg == a.node_rows_global - 1) {
        a.vx_out[n] = 0.0; a.vy_out[n] = 0.0; return;
    }
    double mass = a.area / T.invm[I % P][Jg % P];
    double vxo = a.vx_in[n], vyo = a.vy_in[n];
    double c1 = a.c1[n], cf = a.cafo[n], oxv = a.ox[n], oyv = a.oy[n];
    double w = sqrt((oxv - vxo) * (oxv - vxo) + (oyv - vyo) * (oyv - vyo));
    double den = c1 * a.b1 + cf * w;
    double nx_ = c1 * a.beta * vxo + a.rx0[n] + cf * w * oxv + c1 * a.kc * vyo + a.Fx[n] / mass;
    double ny_ = c1 * a.beta * vyo + a.ry0[n] + cf * w * oyv - c1 * a.kc * vxo + a.Fy[n] / mass;
    a.vx_out[n] = nx_ / den;
    a.vy_out[n] = ny_ / den;
}

// --------------------------------------------------------------------------
// K4 — DG upwind advection stage of A and H (Eq. 1) with the
// RK combine out = a0 c0 + a1 (cin + dt L(cin)).  Block = 32 x 8 elements.
// Each element computes the flux values on its east and north edges once;
// the west edge comes from lane-1 by warp shuffle, the south edge from the
// row below through shared memory; block-border elements evaluate those edges
// with the same function, so both sides see bitwise-identical fluxes and the
// scheme conserves mass exactly up to the final sums.
// --------------------------------------------------------------------------
struct AdvArgs {
    const double* Ain; const double* Hin;     // NA planes
    const double* A0; const double* H0;
    double* Aout; double* Hout;
    const double* vx; const double* vy;
    int64_t eplane, npitch, epitch;
    int nx, erow_begin, erow_end;             // owned local rows
    int has_south, has_north;                 // ghost rows exist below/above (multi-rank)
    int periodic, erows_local;
    double ihx, ihy, dt, a0, a1;
    int limit;                                // k_advect_q2: fused R#25 limiter on the stage output
    const double* sph_rows;                   // k_advect_q2<true>: sphere row tables (R#26), ihx = 1/(R dlon)
    double* Pg; double Pstar, C_conc;         // k_advect_tma, last stage: also write P at the Gauss points
    double kc[18];                            // k_advect_tma: the stage's folded moment coefficients (adv_coeffs)
};

template <int NA> struct Cf { double A[NA], H[NA]; };

template <int P, int NA>
__device__ inline void load_coef(const AdvArgs& a, int64_t e, Cf<NA>& c) {
#pragma unroll
    for (int k = 0; k < NA; ++k) { c.A[k] = a.Ain[k * a.eplane + e]; c.H[k] = a.Hin[k * a.eplane + e]; }
}

// Upwind flux values F_q = c_hat (v.n) on one edge; dir 0 = vertical edge (normal +x), 1 = horizontal (+y).
// lo = element on the negative side, hi = element on the positive side, vn_nodes = normal
// velocity at the P+1 CG nodes on the edge.  valid_lo/hi select zero flux at a closed boundary.
template <int P, int NA>
__device__ inline void edge_flux(int dir, const Cf<NA>& lo, const Cf<NA>& hi, const double* vn_nodes,
                                 bool open, double* FA, double* FH) {
    const RefTab& T = c_tab[P - 1];
    const int elo = dir == 0 ? 0 : 2, ehi = dir == 0 ? 1 : 3;   // lo sees the edge as east/north, hi as west/south
#pragma unroll
    for (int q = 0; q < P + 1; ++q) {
        double vn = 0.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) vn = fma(T.L1[j][q], vn_nodes[j], vn);
        // both traces, then a branch-free upwind select (lanes disagree on the flow direction)
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

constexpr int ADV_ROWS = 4;   // block = 32 x ADV_ROWS elements

template <int P, int NA>
__global__ void __launch_bounds__(32 * ADV_ROWS, 3) k_advect(AdvArgs a) {
    constexpr int NGP = P + 1, NG = NGP * NGP;
    const RefTab& T = c_tab[P - 1];
    __shared__ double sFA[ADV_ROWS][32][NGP], sFH[ADV_ROWS][32][NGP];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int ix = blockIdx.x * 32 + tx;
    const int lr = a.erow_begin + blockIdx.y * ADV_ROWS + ty;
    const bool valid = ix < a.nx && lr < a.erow_end;
    const int ixc = valid ? ix : 0, lrc = valid ? lr : a.erow_begin;
    const int64_t e = (int64_t)lrc * a.epitch + ixc;
    Cf<NA> me; load_coef<P, NA>(a, e, me);
    // node velocities of this element
    double ux[P + 1][P + 1], uy[P + 1][P + 1];
#pragma unroll
    for (int jy = 0; jy <= P; ++jy)
#pragma unroll
        for (int jx = 0; jx <= P; ++jx) {
            int64_t n = (int64_t)(P * lrc + jy) * a.npitch + P * ixc + jx;
            ux[jy][jx] = a.vx[n]; uy[jy][jx] = a.vy[n];
        }
    // neighbours
    auto nb_index = [&](int ex, int ey, bool& open) -> int64_t {
        open = true;
        if (ex < 0 || ex >= a.nx) { if (!a.periodic) { open = false; return e; } ex = (ex + a.nx) % a.nx; }
        if (ey < a.erow_begin && !a.has_south) { if (!a.periodic) { open = false; return e; } ey = a.erow_end - 1; }
        if (ey >= a.erow_end && !a.has_north) { if (!a.periodic) { open = false; return e; } ey = a.erow_begin; }
        return (int64_t)ey * a.epitch + ex;
    };
    // east edge (this element = lo)
    double FeA[NGP], FeH[NGP], FnA[NGP], FnH[NGP], FwA[NGP], FwH[NGP], FsA[NGP], FsH[NGP];
    {
        bool open; int64_t en = nb_index(ixc + 1, lrc, open);
        Cf<NA> nb; load_coef<P, NA>(a, en, nb);
        double vn[P + 1];
#pragma unroll
        for (int j = 0; j <= P; ++j) vn[j] = ux[j][P];
        edge_flux<P, NA>(0, me, nb, vn, open, FeA, FeH);
    }
    {
        bool open; int64_t en = nb_index(ixc, lrc + 1, open);
        Cf<NA> nb; load_coef<P, NA>(a, en, nb);
        double vn[P + 1];
#pragma unroll
        for (int j = 0; j <= P; ++j) vn[j] = uy[P][j];
        edge_flux<P, NA>(1, me, nb, vn, open, FnA, FnH);
    }
    // west edge: lane-1's east edge
#pragma unroll
    for (int q = 0; q < NGP; ++q) {
        FwA[q] = __shfl_up_sync(0xffffffffu, FeA[q], 1);
        FwH[q] = __shfl_up_sync(0xffffffffu, FeH[q], 1);
    }
    if (tx == 0) {
        bool open; int64_t wn = nb_index(ixc - 1, lrc, open);
        Cf<NA> nb; load_coef<P, NA>(a, wn, nb);
        double vn[P + 1];
#pragma unroll
        for (int j = 0; j <= P; ++j) vn[j] = ux[j][0];
        edge_flux<P, NA>(0, nb, me, vn, open, FwA, FwH);
    }
    // south edge: the row below's north edge
#pragma unroll
    for (int q = 0; q < NGP; ++q) { sFA[ty][tx][q] = FnA[q]; sFH[ty][tx][q] = FnH[q]; }
    __syncthreads();
    if (ty > 0) {
#pragma unroll
        for (int q = 0; q < NGP; ++q) { FsA[q] = sFA[ty - 1][tx][q]; FsH[q] = sFH[ty - 1][tx][q]; }
    } else {
        bool open; int64_t sn = nb_index(ixc, lrc - 1, open);
        Cf<NA> nb; load_coef<P, NA>(a, sn, nb);
        double vn[P + 1];
#pragma unroll
        for (int j = 0; j <= P; ++j) vn[j] = uy[0][j];
        edge_flux<P, NA>(1, nb, me, vn, open, FsA, FsH);
    }
    if (!valid) return;
    // volume term: int c v . grad psi_k
    double LA[NA], LH[NA];
#pragma unroll
    for (int k = 0; k < NA; ++k) { LA[k] = 0.0; LH[k] = 0.0; }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
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
        const double wx = T.w[g] * vxg * a.ihx, wy = T.w[g] * vyg * a.ihy;
#pragma unroll
        for (int k = 1; k < NA; ++k) {
            const double gk = wx * T.dpsis[k][g] + wy * T.dpsit[k][g];
            LA[k] = fma(cA, gk, LA[k]);
            LH[k] = fma(cH, gk, LH[k]);
        }
    }
    // edges: -(1/|K|) int_e c_hat (v.n) psi ; |e|/|K| = 1/hx (vertical), 1/hy (horizontal)
#pragma unroll
    for (int q = 0; q < NGP; ++q) {
        const double wqx = T.gw[q] * a.ihx, wqy = T.gw[q] * a.ihy;
#pragma unroll
        for (int k = 0; k < NA; ++k) {
            LA[k] -= wqx * (FeA[q] * T.psiedge[0][k][q] - FwA[q] * T.psiedge[1][k][q])
                   + wqy * (FnA[q] * T.psiedge[2][k][q] - FsA[q] * T.psiedge[3][k][q]);
            LH[k] -= wqx * (FeH[q] * T.psiedge[0][k][q] - FwH[q] * T.psiedge[1][k][q])
                   + wqy * (FnH[q] * T.psiedge[2][k][q] - FsH[q] * T.psiedge[3][k][q]);
        }
    }
    const int64_t eo = (int64_t)lr * a.epitch + ix;
#pragma unroll
    for (int k = 0; k < NA; ++k) {
        const double la = LA[k] / T.mref[k], lh = LH[k] / T.mref[k];
        const double outA = a.a1 * (me.A[k] + a.dt * la);
        const double outH = a.a1 * (me.H[k] + a.dt * lh);
        a.Aout[k * a.eplane + eo] = (a.a0 != 0.0) ? a.a0 * a.A0[k * a.eplane + eo] + outA : outA;
        a.Hout[k * a.eplane + eo] = (a.a0 != 0.0) ? a.a0 * a.H0[k * a.eplane + eo] + outH : outH;
    }
}

// --------------------------------------------------------------------------
// Synthetic VP-benchmark forcing at time t (DESIGN.md §5 recipe; NEXT-2 moving cyclone), on the
// owned node rows: o = 0.01 (2y/Ly - 1, 1 - 2x/Lx); a = -(W e / r0) exp(-r/r0) R_theta (x - c(t)),
// c(t) = (Lx/2, Ly/2) + 51.2 km/day t (1, 1), W = 15 m/s, r0 = 100 km, theta = 72 deg.
// --------------------------------------------------------------------------
// --------------------------------------------------------------------------
// NEXT-4 (R#25): Zhang-Shu bound-preserving scaling limiter, applied to an advection stage's output
// (owned rows): theta from the extremes over the volume and edge Gauss points (the points where the
// scheme evaluates the tracer), c <- cbar + theta (c - cbar) about the |J|-weighted element mean
// cbar = c0 + (d1 c1 + d2 c2) / (12 C0)  (|J| = C0 + d1 S + d2 T; d1 = d2 = 0 on the box).
// A in [0, 1], H >= 0.
// --------------------------------------------------------------------------
struct LimArgs {
    double* A; double* H; const double* verts;   // verts: general quads (single rank), else null
    int64_t eplane, epitch;
    int nx, erow_begin, erow_end;
};
template <int P, int NA>
__global__ void k_limit(LimArgs a) {
    const RefTab& T = c_tab[P - 1];
    constexpr int NGP = P + 1, NG = NGP * NGP;
    const int ix = blockIdx.x * blockDim.x + threadIdx.x, lr = a.erow_begin + blockIdx.y;
    if (ix >= a.nx || lr >= a.erow_end) return;
    const int64_t e = (int64_t)lr * a.epitch + ix;
    double d1 = 0.0, d2 = 0.0, C0 = 1.0;
    if (a.verts) {
        const double* v00 = a.verts + 2 * ((int64_t)lr * (a.nx + 1) + ix);
        const double* v01 = v00 + 2 * (a.nx + 1);
        const double ax = v00[2] - v00[0], ay = v00[3] - v00[1], bx = v01[0] - v00[0], by = v01[1] - v00[1];
        const double cx = (v01[2] - v01[0]) - ax, cy = (v01[3] - v01[1]) - ay;
        const double d0 = ax * by - bx * ay;
        d1 = ax * cy - cx * ay; d2 = cx * by - bx * cy;
        C0 = d0 + 0.5 * (d1 + d2);
    }
#pragma unroll
    for (int f = 0; f < 2; ++f) {
        double* base = f == 0 ? a.A : a.H;
        const double lo = 0.0, hi = f == 0 ? 1.0 : INFINITY;
        double c[NA];
#pragma unroll
        for (int k = 0; k < NA; ++k) c[k] = base[k * a.eplane + e];
        double cmin = INFINITY, cmax = -INFINITY;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < NA; ++k) v = fma(c[k], T.psi[k][g], v);
            cmin = fmin(cmin, v); cmax = fmax(cmax, v);
        }
#pragma unroll
        for (int ed = 0; ed < 4; ++ed)
#pragma unroll
            for (int q = 0; q < NGP; ++q) {
                double v = 0.0;
#pragma unroll
                for (int k = 0; k < NA; ++k) v = fma(c[k], T.psiedge[ed][k][q], v);
                cmin = fmin(cmin, v); cmax = fmax(cmax, v);
            }
        const double cbar = c[0] + (d1 * c[1] + d2 * c[2]) / (12.0 * C0);
        double theta = 1.0;
        if (cmin < lo) theta = fmin(theta, (cbar - lo) / (cbar - cmin));
        if (cmax > hi) theta = fmin(theta, (hi - cbar) / (cmax - cbar));
        theta = fmax(0.0, fmin(1.0, theta));
        if (theta < 1.0) {
#pragma unroll
            for (int k = 0; k < NA; ++k) base[k * a.eplane + e] = (k == 0 ? fma(1.0 - theta, cbar, theta * c[0]) : theta * c[k]);
        }
    }
}

struct ForcingArgs {
    double* ox; double* oy; double* ax; double* ay;
    int64_t npitch;
    int ncols, row_begin, row_end, global_row0;   // owned local node rows; global index of local row 0
    double dxn, dyn, lx, ly, t;                    // node spacing hx/p, hy/p; global extents
};

__global__ void k_cyclone_forcing(ForcingArgs a) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int jr = a.row_begin + blockIdx.y;
    if (I >= a.ncols || jr >= a.row_end) return;
    const double x = I * a.dxn, y = (a.global_row0 + jr) * a.dyn;
    const int64_t n = (int64_t)jr * a.npitch + I;
    a.ox[n] = 0.01 * (2.0 * y / a.ly - 1.0);
    a.oy[n] = 0.01 * (1.0 - 2.0 * x / a.lx);
    const double shift = 51.2 * (1000.0 / 86400.0) * a.t;
    const double dx = x - (0.5 * a.lx + shift), dy = y - (0.5 * a.ly + shift);
    const double r = sqrt(dx * dx + dy * dy);
    const double W = 15.0, r0 = 100e3, th = 72.0 * 3.14159265358979323846 / 180.0;
    const double sc = -(W * 2.71828182845904523536 / r0) * exp(-r / r0);
    const double ct = cos(th), st = sin(th);
    a.ax[n] = sc * (ct * dx + st * dy);
    a.ay[n] = sc * (-st * dx + ct * dy);
}

// --------------------------------------------------------------------------
// ABI layout conversion: AoS rows (n per element) <-> SoA planes.
// --------------------------------------------------------------------------
// NEXT-3 mixed precision: FP64 <-> FP32 copies of the stress / P_g planes at call boundaries
__global__ void k_cvt_d2f(const double* __restrict__ src, float* __restrict__ dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (float)src[i];
}
__global__ void k_cvt_f2d(const float* __restrict__ src, double* __restrict__ dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (double)src[i];
}

// compact ABI element e = row*nx + col  <->  device (row + row_off)*epitch + col
__global__ void k_aos_to_soa(const double* src, double* dst, int64_t nelem, int n, int64_t eplane, int64_t row_off,
                             int nx, int64_t epitch) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nelem * n) return;
    int64_t e = i / n; int k = (int)(i % n);
    dst[k * eplane + (e / nx + row_off) * epitch + e % nx] = src[i];
}
__global__ void k_soa_to_aos(const double* src, double* dst, int64_t nelem, int n, int64_t eplane, int64_t row_off,
                             int nx, int64_t epitch) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nelem * n) return;
    int64_t e = i / n; int k = (int)(i % n);
    dst[i] = src[k * eplane + (e / nx + row_off) * epitch + e % nx];
}

}  // namespace nxk
