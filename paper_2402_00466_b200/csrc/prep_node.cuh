// The per-node arithmetic of the outer-step prep (row a1, R#11, R#17) for the CG2 / DG2 pair, shared
// by every kernel that forms the node constants: the row-marching prep (prep_q2.cuh) and the first fused
// subcycle of an outer step (subcycle_tma.cuh, PREP): the same functions on the same sums in the same
// order, so all of them give bitwise the same constants.
#pragma once
#include "kernels.cuh"

namespace nxk {

// DG2 value at local node (jx, jy) (s, t = jx/2, jy/2): sum_k c_k psi_k, the k order of k_prep_nodes
template <int JX, int JY>
__device__ __forceinline__ double dg2_node(const double* c) {
    constexpr double S = 0.5 * JX - 0.5, T = 0.5 * JY - 0.5;
    constexpr double psi[6] = {1.0, S, T, S * S - 1.0 / 12.0, T * T - 1.0 / 12.0, S * T};
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k)   // explicit FMAs (the same rounding in every kernel), zero terms skipped
        if (psi[k] != 0.0) v = fma(c[k], psi[k], v);
    return v;
}

// the per-node arithmetic of the prep (k_prep_nodes' formulas), shared by both CG2/DG2 prep kernels
struct PrepNodeOut { double c1, rx0, ry0, cafo; };
__device__ __forceinline__ PrepNodeOut prep_node_calc(const PrepArgs& a, double hs, double as, int cnt, double axv,
                                                      double ayv, double vxv, double vyv, double oxv, double oyv) {
    // a node touches 1, 2 or 4 elements of the structured mesh: the mean's division is an exact power-of-2
    // scaling (no FP64 division sequence); 1/dt comes from the host
    const double rc = cnt == 4 ? 0.25 : (cnt == 2 ? 0.5 : (cnt == 1 ? 1.0 : 1.0 / cnt));
    const double Hn = cnt ? fmax(hs * rc, 1e-4) : 1e-4;
    const double An = cnt ? fmin(fmax(as * rc, 0.0), 1.0) : 0.0;
    const double m = a.rho_ice * Hn;
    const double c1 = m * a.rdt;
    const double amag = sqrt(fma(axv, axv, ayv * ayv));
    const double drag = An * a.Fa * amag;
    const double mf = m * a.f_c;
    PrepNodeOut o;                                   // explicit FMAs: the same rounding in every prep kernel
    o.c1 = c1;
    o.rx0 = fma(c1, vxv, fma(drag, axv, -mf * oyv));
    o.ry0 = fma(c1, vyv, fma(drag, ayv, mf * oxv));
    o.cafo = An * a.Fo;
    return o;
}
}  // namespace nxk
