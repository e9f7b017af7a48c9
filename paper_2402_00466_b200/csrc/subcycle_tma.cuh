// K_sub for CG2/DG2 (the bench path): fused strain + stress + divergence gather + velocity,
// TMA-staged and written with the tensor-product structure of the Q2/P2 reference element.
//
// Same mapping as k_subcycle<P> (kernels.cuh): a warp owns a strip of 31 element columns
// (+ lane 0 = ring column ix0-1, recomputed) and marches up a chunk of element rows
// (+ one ring row below).  Differences:
//  * data staging: for every element row ("job") lane 0 issues five TMA loads
//    (cp.async.bulk.tensor) into a per-warp shared-memory stage, double-buffered and
//    tracked by an mbarrier: S (3 n_S planes x 34 elements), P_g (9 x 34), vx / vy (3 node
//    rows x 66 columns) and the six node constants (2 rows x 62 columns).  The next job's
//    loads are in flight while the current one computes; OOB boxes are zero-filled, which
//    also covers the ragged right edge and the ring at ix0-1 = -1.  Warps are persistent and
//    walk a static round-robin list of (strip, chunk) units, prefetching across units.
//  * arithmetic: every reference table is folded into the code.  On the affine Q2/P2
//    element:
//      strain coefficients  E(d/ds v)_(a,b) = sum DX[a][jx] BY[b][jy] v   -> first and second
//                           node differences (exact cancellation-free form), 20 flops each
//      Gauss-point values   e(S,T) = A(T) + S B(T) + E3 q(S)              -> 22 flops / field
//      projection R         1D moments over gx then gy                    -> ~40 flops / field
//      divergence D         Z(jy) = sum_b S_(a,b) BY[b][jy], r = Z DX      -> ~30 flops / part
//    with DX = [[-1,0,1],[1/3,-2/3,1/3],0], BY = [[1/6,2/3,1/6],[-1/12,0,1/12],[1/90,-1/45,1/90]],
//    Gauss S in {-a, 0, a}, a = sqrt(3/5)/2, weights (5, 8, 5)/18, q(+-a) = 1/15, q(0) = -1/12.
//    tests/test_gpu_parity.py checks this kernel against the oracle and against the
//    table-driven k_subcycle<2> (whose tables come from the K0 kernel).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstddef>
#include <cstdio>
#include "prep_node.cuh"

namespace nxk {

constexpr int K2_WARPS = 2;          // warps per CTA (independent work lists)
constexpr int K2_MAX_STAGES = 4;     // pipeline depth is a template parameter (2..4)
constexpr int K2_VCOLS = 66;         // node columns per v box: 2*32 + 2
constexpr int K2_CCOLS = 62;         // owned node columns per const box: 2*31
// Element columns per S / P_g box.  The TMA start column must be 16-B aligned: for FP64 storage
// the box starts at (ix0-1) & ~1 and is 34 wide, for FP32 storage (NEXT-3 mixed precision) at
// (ix0-1) & ~3 and 36 wide; lanes read at the offset (ix0-1) - start.
template <typename SF> struct K2Cols { static constexpr int E = sizeof(SF) == 8 ? 34 : 36, ALIGN = 16 / sizeof(SF); };
__host__ __device__ constexpr int round128(int b) { return (b + 127) / 128 * 128; }

// One job's shared-memory stage; every TMA destination starts on a 128-B boundary.
// CL = false: the six node constants are a fifth TMA box of the stage.  CL = true: they are not
// staged; each lane loads its own 24 doubles straight into registers (coalesced 16-B loads issued
// before the job's stage is waited for, consumed by the velocity update at its end), which takes
// 35 % off the stage and lets 4 CTAs (8 warps) share an SM instead of 2.
template <typename SF, int NS = 6>
struct __align__(128) K2StageNC {
    static constexpr int EC = K2Cols<SF>::E;
    alignas(128) SF S[3 * NS][EC];             // planes S11[0..NS), S12[0..NS), S22[0..NS)
    alignas(128) SF Pg[9][EC];
    alignas(128) double vx[3][K2_VCOLS];       // 1584 B
    alignas(128) double vy[3][K2_VCOLS];
};
template <typename SF, int NS = 6>
struct __align__(128) K2Stage : K2StageNC<SF, NS> {
    alignas(128) double C[6][2][K2_CCOLS];     // 5952 B  c1, rx0, ry0, cafo, ox, oy
};
static_assert(sizeof(K2Stage<double>) == 16896, "stage layout");
static_assert(sizeof(K2Stage<double, 8>) == 18432, "stage layout (n_S = 8)");
static_assert(sizeof(K2StageNC<double>) == 10880, "stage layout (constants in registers)");
template <typename SF, int NS, bool CL> struct K2StageSel { using T = K2Stage<SF, NS>; };
template <typename SF, int NS> struct K2StageSel<SF, NS, true> { using T = K2StageNC<SF, NS>; };
template <typename SF, int NS = 6, bool CL = false>
__host__ __device__ constexpr uint32_t k2_tx_bytes() {
    return (3 * NS + 9) * K2Cols<SF>::E * sizeof(SF) + 2 * 3 * K2_VCOLS * 8 + (CL ? 0 : 6 * 2 * K2_CCOLS * 8);
}
__device__ __forceinline__ double2 ldg_stream2(const double* p) {   // read once: keep it out of L1
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

struct K2Maps {
    CUtensorMap S, Pg, vx, vy, C;    // 5 x 128 B, 64-B aligned
    CUtensorMap vx2, vy2;            // 2-row v boxes: the new node rows of a unit's continuing job
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    for (uint32_t it = 0;; ++it) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
        if (ok) return;
        if (it > (1u << 26)) {   // never hang the GPU on a lost transaction
            printf("nxsdg: TMA mbarrier timeout block %d thread %d parity %u\n", blockIdx.x, threadIdx.x, parity);
            __trap();
        }
    }
}
// L2 eviction policies (createpolicy) for the cache-hinted TMA loads / global accesses below
__device__ __forceinline__ uint64_t l2_policy(int kind) {   // 0 evict_normal, 1 evict_first, 2 evict_last
    uint64_t p;
    if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma3h(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
        ::"r"(su32(dst)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(z), "r"(su32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma2h(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(su32(dst)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(su32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ double2 ldg_stream2h(const double* p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint2(double* p, double x, double y, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(x), "d"(y), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(su32(dst)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(z), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(su32(dst)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(su32(bar)) : "memory");
}

// Branch-free FP64 reciprocal / reciprocal square root: the MUFU seed (~20 bits) plus one
// third-order correction (error ~ seed^3 ~ 2^-60, i.e. <= 1 ulp after rounding).  Valid for
// positive normal arguments, which is all this kernel feeds them (Delta^2 >= DeltaMin^2 > 0,
// c1 (1 + beta) + cAFo w > 0); no slow-path branches, unlike the IEEE-exact library calls.
__device__ __forceinline__ double rsqrt_nr(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-(x * r), r, 1.0);          // 1 - x r^2
    return fma(r * e, fma(0.375, e, 0.5), r);        // r (1 + e/2 + 3 e^2/8)
}
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);                // 1 - x r
    return fma(r, fma(e, e, e), r);                  // r (1 + e + e^2)
}

// ---------------------------------------------------------------- element math (Q2/P2)
constexpr double kA = 0.38729833462074170;       // sqrt(3/5)/2: Gauss S, T in {-kA, 0, kA}
constexpr double kQ = 1.0 / 15.0;                // S^2 - 1/12 at S = +-kA
constexpr double kQ0 = -1.0 / 12.0;              // ... at S = 0
constexpr double kC = 10.0 * kA / 3.0;           // 12 * (5/18) * kA: first-moment scale

// The stress part is templated on the arithmetic type T (double; float for NEXT-3's F32 stress
// update).  Node differences are formed in FP64 and then converted.
__device__ __forceinline__ float rsqrt_t(float x) { return rsqrtf(x); }
__device__ __forceinline__ double rsqrt_t(double x) { return rsqrt_nr(x); }

// strain coefficients of d/ds v (k = 0..NS-1; k = 3 and 6 identically zero: no l2(S) part).
// The n_S = 8 space (R#24) adds E_7 = <d/ds v, l1(S) l2(T)> / (1/2160) = 8 (second difference of s1).
template <typename T, int NS>
__device__ __forceinline__ void strain_s(const double V[3][3], T (&E)[NS]) {
    T s0[3], s1[3];
#pragma unroll
    for (int jy = 0; jy < 3; ++jy) {
        const T d01 = (T)(V[jy][1] - V[jy][0]), d12 = (T)(V[jy][2] - V[jy][1]);
        s0[jy] = d01 + d12; s1[jy] = d12 - d01;
    }
    E[0] = (s0[0] + s0[2] + T(4) * s0[1]) * T(1.0 / 6.0);
    E[1] = (s1[0] + s1[2] + T(4) * s1[1]) * T(2.0 / 3.0);
    E[2] = s0[2] - s0[0];
    E[3] = T(0);
    E[4] = T(2) * (s0[0] + s0[2]) - T(4) * s0[1];
    E[5] = T(4) * (s1[2] - s1[0]);
    if constexpr (NS == 8) {
        E[6] = T(0);
        E[7] = T(8) * (s1[0] + s1[2] - T(2) * s1[1]);
    }
}
// strain coefficients of d/dt v (k = 4 and 7 identically zero; n_S = 8 adds E_6)
template <typename T, int NS>
__device__ __forceinline__ void strain_t(const double V[3][3], T (&E)[NS]) {
    T t0[3], t1[3];
#pragma unroll
    for (int jx = 0; jx < 3; ++jx) {
        const T d01 = (T)(V[1][jx] - V[0][jx]), d12 = (T)(V[2][jx] - V[1][jx]);
        t0[jx] = d01 + d12; t1[jx] = d12 - d01;
    }
    E[0] = (t0[0] + t0[2] + T(4) * t0[1]) * T(1.0 / 6.0);
    E[1] = t0[2] - t0[0];
    E[2] = (t1[0] + t1[2] + T(4) * t1[1]) * T(2.0 / 3.0);
    E[3] = T(2) * (t0[0] + t0[2]) - T(4) * t0[1];
    E[4] = T(0);
    E[5] = T(4) * (t1[2] - t1[0]);
    if constexpr (NS == 8) {
        E[6] = T(8) * (t1[0] + t1[2] - T(2) * t1[1]);
        E[7] = T(0);
    }
}
// E = a Es + b Et over the coefficients, skipping the structural zeros of the d/ds strain (k = 3,
// and 6 for n_S = 8) and of the d/dt strain (k = 4, and 7)
template <typename T, int NS>
__device__ __forceinline__ void combine(const T (&Es)[NS], const T (&Et)[NS], T ca, T cb, T (&E)[NS]) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const bool zs = k == 3 || (NS == 8 && k == 6), zt = k == 4 || (NS == 8 && k == 7);
        E[k] = zs ? cb * Et[k] : (zt ? ca * Es[k] : fma(ca, Es[k], cb * Et[k]));
    }
}
// values at the 9 Gauss points (g = gy*3 + gx) of sum_k E_k psi_k; HAS3/HAS4 drop known zeros.
// e(S, T) = A(T) + S B(T) + q(S) Q(T): A = E0 + E2 T + E4 q(T), B = E1 + E5 T (+ E7 q(T)),
// Q = E3 (+ E6 T) -- the bracketed terms are the n_S = 8 functions (R#24).
template <bool HAS3, bool HAS4, typename T, int NS>
__device__ __forceinline__ void eval_gp(const T (&E)[NS], T e[9]) {
    const T a = T(kA), q = T(kQ), q0 = T(kQ0);
    const T c0 = HAS4 ? fma(E[4], q, E[0]) : E[0];
    const T c1 = HAS4 ? fma(E[4], q0, E[0]) : E[0];
    const T t2 = a * E[2], t5 = a * E[5];
    const T Av[3] = {c0 - t2, c1, c0 + t2};
    T Bv[3] = {E[1] - t5, E[1], E[1] + t5};
    T Qv[3] = {E[3], E[3], E[3]};
    if constexpr (NS == 8) {
        const T b7 = fma(E[7], q, E[1]);                    // E1 + E7 q(T) at T = +-a
        Bv[0] = b7 - t5; Bv[1] = fma(E[7], q0, E[1]); Bv[2] = b7 + t5;
        const T t6 = a * E[6];
        Qv[0] = E[3] - t6; Qv[2] = E[3] + t6;
    }
    constexpr bool HASQ = HAS3 || NS == 8;
#pragma unroll
    for (int gy = 0; gy < 3; ++gy) {
        const T Pq = HASQ ? fma(Qv[gy], q, Av[gy]) : Av[gy];
        e[gy * 3 + 0] = fma(-a, Bv[gy], Pq);
        e[gy * 3 + 2] = fma(a, Bv[gy], Pq);
        e[gy * 3 + 1] = HASQ ? fma(Qv[gy], q0, Av[gy]) : Av[gy];
    }
}
// S_k <- fac S_k + sc * (R G)_k  (R = M_ref^{-1} psi_k(g) w_g) by 1D moments;
// n_S = 8: p6 = 2160 sum w q(S) T G, p7 = 2160 sum w S q(T) G, both (100 a / 9) x second moments
template <typename T, int NS>
__device__ __forceinline__ void proj_coeffs(const T G[9], double sc, T (&p)[NS]) {
    T X0[3], X1[3], X2[3];
#pragma unroll
    for (int gy = 0; gy < 3; ++gy) {
        const T s = G[gy * 3] + G[gy * 3 + 2], d = G[gy * 3 + 2] - G[gy * 3], m = G[gy * 3 + 1];
        X0[gy] = fma(T(5), s, T(8) * m);
        X1[gy] = d;
        X2[gy] = fma(T(-2), m, s);
    }
    p[0] = fma(T(5), X0[0] + X0[2], T(8) * X0[1]) * T(sc / 324.0);
    p[1] = fma(T(5), X1[0] + X1[2], T(8) * X1[1]) * T(sc * kC / 18.0);
    p[2] = (X0[2] - X0[0]) * T(sc * kC / 18.0);
    p[3] = fma(T(5), X2[0] + X2[2], T(8) * X2[1]) * T(sc * 10.0 / 54.0);
    p[4] = fma(T(-2), X0[1], X0[0] + X0[2]) * T(sc * 10.0 / 54.0);
    p[5] = (X1[2] - X1[0]) * T(sc * kC * kC);
    if constexpr (NS == 8) {
        p[6] = (X2[2] - X2[0]) * T(sc * 100.0 * kA / 9.0);
        p[7] = fma(T(-2), X1[1], X1[0] + X1[2]) * T(sc * 100.0 * kA / 9.0);
    }
}
template <typename T, int NS>
__device__ __forceinline__ void project(const T G[9], double sc, T fac, T (&S)[NS]) {
    T p[NS];
    proj_coeffs(G, sc, p);
#pragma unroll
    for (int k = 0; k < NS; ++k) S[k] = fma(fac, S[k], p[k]);
}
// The pair (g11, g22) = (a + b, a - b) projected together: S11 <- fac S11 + R a + R b,
// S22 <- fac S22 + R a - R b, with b's factor 1/2 in its scale (sb = 0.5)
template <typename T, int NS>
__device__ __forceinline__ void project_pair(const T Ga[9], const T Gb[9], T fac, T (&S11)[NS], T (&S22)[NS]) {
    T pa[NS], pb[NS];
    proj_coeffs(Ga, 1.0, pa);
    proj_coeffs(Gb, 0.5, pb);
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        S11[k] = fma(fac, S11[k], pa[k] + pb[k]);
        S22[k] = fma(fac, S22[k], pa[k] - pb[k]);
    }
}
// r[jx][jy] += f(jx) f(jy) sum_k Ds[j][k] S_k * h  (d/ds part, uses k = 0,1,2,4,5 and 7), where
// f(0) = f(2) = 1, f(1) = 1/2 is the lumped-mass ratio of the node type (corner 1/9, edge 2/9,
// centre 4/9 of |K|: 1/m = -9 f(jx) f(jy) with h = -9/hx), folded into the constants
template <int NS>
__device__ __forceinline__ void div_s(const double (&S)[NS], double h, double r[3][3]) {
    const double u = fma(S[4], h * (1.0 / 90.0), S[0] * (h / 6.0)), v = S[2] * (h / 12.0);
    const double Z0[3] = {u - v, fma(S[0], h * (1.0 / 3.0), -S[4] * (h / 90.0)), u + v};
    double p = S[1] * (h / 6.0), m = S[1] * (h * 1.0 / 3.0);
    if constexpr (NS == 8) { p = fma(S[7], h * (1.0 / 90.0), p); m = fma(S[7], -h * (1.0 / 90.0), m); }
    const double w = S[5] * (h / 12.0);
    const double Z1[3] = {p - w, m, p + w};
#pragma unroll
    for (int jy = 0; jy < 3; ++jy) {
        const double t = Z1[jy] * (1.0 / 3.0);
        r[0][jy] += t - Z0[jy];
        r[1][jy] += Z1[jy] * (-1.0 / 3.0);
        r[2][jy] += t + Z0[jy];
    }
}
// r[jx][jy] += f(jx) f(jy) sum_k Dt[j][k] S_k * h  (d/dt part, uses k = 0,1,2,3,5 and 6)
template <int NS>
__device__ __forceinline__ void div_t(const double (&S)[NS], double h, double r[3][3]) {
    const double u = fma(S[3], h * (1.0 / 90.0), S[0] * (h / 6.0)), v = S[1] * (h / 12.0);
    const double W0[3] = {u - v, fma(S[0], h * (1.0 / 3.0), -S[3] * (h / 90.0)), u + v};
    double p = S[2] * (h / 6.0), m = S[2] * (h * 1.0 / 3.0);
    if constexpr (NS == 8) { p = fma(S[6], h * (1.0 / 90.0), p); m = fma(S[6], -h * (1.0 / 90.0), m); }
    const double w = S[5] * (h / 12.0);
    const double W1[3] = {p - w, m, p + w};
#pragma unroll
    for (int jx = 0; jx < 3; ++jx) {
        const double t = W1[jx] * (1.0 / 3.0);
        r[jx][0] += t - W0[jx];
        r[jx][1] += W1[jx] * (-1.0 / 3.0);
        r[jx][2] += t + W0[jx];
    }
}

// ---------------------------------------------------------------- sphere (NEXT-4, R#26)
// On a lon-lat element the metric varies with latitude only, i.e. with t: in the orthonormal east-north
// frame |J| = R^2 cos(lat) dlon dlat, J^-1 = diag(1 / (R cos(lat) dlon), 1 / (R dlat)), and the frame's
// metric term tan(lat)/R enters the strain (eps11 -= v tan/R, eps12 += u tan/(2R)) and, as its adjoint,
// the divergence.  So the fused kernel evaluates the strain pointwise at the 3 x 3 Gauss points (gy =
// latitude row), projects |J| eps / (R^2 dlon dlat) = cos(lat) eps with the box moments and the row's
// cos-weighted DG mass, whose inverse is block-diagonal in the S-degree of the centred Legendre modes
// ({0, 2, 4}, {1, 5}, {3}: the per-row blocks Q = M_row^{-1} M_ref of the row table), and contracts the
// divergence with the 1D Lagrange values / derivatives at the Gauss abscissae.  Row tables: nxsdg.cu.
__device__ __forceinline__ void q2_gauss3(double n0, double n1, double n2, double out[3]) {
    const double s = n0 + n2, d = n0 - n2, m = fma(0.3, s, 0.4 * n1);
    out[0] = fma(kA, d, m); out[1] = n1; out[2] = fma(-kA, d, m);
}
// the Q2 field V[jy][jx] at the 9 Gauss points (g = gy*3 + gx)
__device__ __forceinline__ void q2_at_gauss(const double V[3][3], double out[9]) {
    double X[3][3];
#pragma unroll
    for (int jy = 0; jy < 3; ++jy) q2_gauss3(V[jy][0], V[jy][1], V[jy][2], X[jy]);
#pragma unroll
    for (int gx = 0; gx < 3; ++gx) {
        double o[3];
        q2_gauss3(X[0][gx], X[1][gx], X[2][gx], o);
        out[gx] = o[0]; out[3 + gx] = o[1]; out[6 + gx] = o[2];
    }
}
// exact pointwise d/ds, d/dt of a Q2 field at the Gauss points: the derivative lies in the n_S = 8
// space (R#24), whose strain coefficients are exact
__device__ __forceinline__ void q2_ds_at_gauss(const double V[3][3], double out[9]) {
    double E[8];
    strain_s<double, 8>(V, E);
    eval_gp<true, true>(E, out);
}
__device__ __forceinline__ void q2_dt_at_gauss(const double V[3][3], double out[9]) {
    double E[8];
    strain_t<double, 8>(V, E);
    eval_gp<true, true>(E, out);
}
// E = Q p with the row's blocks (p: the box moments M_ref^{-1} sum_g w_g psi(g) G(g))
__device__ __forceinline__ void sph_apply_q(const double* __restrict__ row, const double (&p)[6], double (&E)[6]) {
    const double* QA = row + SPH_QA;
    const double* QB = row + SPH_QB;
    E[0] = fma(__ldg(QA + 0), p[0], fma(__ldg(QA + 1), p[2], __ldg(QA + 2) * p[4]));
    E[2] = fma(__ldg(QA + 3), p[0], fma(__ldg(QA + 4), p[2], __ldg(QA + 5) * p[4]));
    E[4] = fma(__ldg(QA + 6), p[0], fma(__ldg(QA + 7), p[2], __ldg(QA + 8) * p[4]));
    E[1] = fma(__ldg(QB + 0), p[1], __ldg(QB + 1) * p[5]);
    E[5] = fma(__ldg(QB + 2), p[1], __ldg(QB + 3) * p[5]);
    E[3] = __ldg(row + SPH_QC) * p[3];
}
// DG strain of v on a sphere row, evaluated at the Gauss points as the trace u = e11 + e22, the half
// difference w = (e11 - e22)/2 and e12 (the box kernel's variables); ihx = 1 / (R dlon), ihy = 1 / (R dlat)
__device__ __forceinline__ void sph_strain(const double Vx[3][3], const double Vy[3][3], const double* __restrict__ row,
                                           double ihx, double ihy, double eu[9], double ew[9], double e12[9]) {
    double dsx[9], dtx[9], dsy[9], dty[9], vxg[9], vyg[9];
    q2_ds_at_gauss(Vx, dsx); q2_dt_at_gauss(Vx, dtx);
    q2_ds_at_gauss(Vy, dsy); q2_dt_at_gauss(Vy, dty);
    q2_at_gauss(Vx, vxg); q2_at_gauss(Vy, vyg);
    double Gu[9], Gw[9], Gz[9];
#pragma unroll
    for (int g = 0; g < 9; ++g) {   // cos(lat) eps = |J| eps / (R^2 dlon dlat)
        const double c = __ldg(row + SPH_COS + g / 3), sr = __ldg(row + SPH_SINR + g / 3), ct = c * ihy;
        const double g11 = fma(ihx, dsx[g], -sr * vyg[g]);
        const double g22 = ct * dty[g];
        Gu[g] = g11 + g22;
        Gw[g] = g11 - g22;                                            // x 1/2 in the projection scale
        Gz[g] = fma(ct, dtx[g], fma(ihx, dsy[g], sr * vxg[g]));     // x 1/2 likewise
    }
    double p[6], E[6];
    proj_coeffs(Gu, 1.0, p); sph_apply_q(row, p, E); eval_gp<true, true>(E, eu);
    proj_coeffs(Gw, 0.5, p); sph_apply_q(row, p, E); eval_gp<true, true>(E, ew);
    proj_coeffs(Gz, 0.5, p); sph_apply_q(row, p, E); eval_gp<true, true>(E, e12);
}
// S11 <- fac S11 + Q (Ra + Rb), S22 <- fac S22 + Q (Ra - Rb), S12 <- fac S12 + Q Rz, with the Gauss-point
// values weighted by cos(lat) (|J_g| / (R^2 dlon dlat)); b's and z's factor 1/2 in the moments' scale
// (Ga, Gb, Gz arrive already weighted by cos(lat): the kernel folds it into p / Delta and P / 2)
__device__ __forceinline__ void sph_project(double Ga[9], double Gb[9], double Gz[9], const double* __restrict__ row,
                                            double fac, double (&S11)[6], double (&S12)[6], double (&S22)[6]) {
    double p[6], qa[6], qb[6], qz[6];
    proj_coeffs(Ga, 1.0, p); sph_apply_q(row, p, qa);
    proj_coeffs(Gb, 0.5, p); sph_apply_q(row, p, qb);
    proj_coeffs(Gz, 0.5, p); sph_apply_q(row, p, qz);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        S11[k] = fma(fac, S11[k], qa[k] + qb[k]);
        S22[k] = fma(fac, S22[k], qa[k] - qb[k]);
        S12[k] = fma(fac, S12[k], qz[k]);
    }
}
// 1D contractions over the Gauss abscissae S_q in {-a, 0, a} with the weights (5, 8, 5) / 18 of the
// Lagrange values / derivatives L_j(S) = 2S^2 - S, 1 - 4S^2, 2S^2 + S (by sums and differences):
//   val: out_j = sum_q w_q L_j(S_q) f_q,   der: out_j = sum_q w_q L_j'(S_q) f_q
__device__ __forceinline__ void lag_val3(double f0, double f1, double f2, double (&o)[3]) {
    const double s = f0 + f2, d = f2 - f0;
    const double P = (5.0 / 18.0 * 2.0 * kA * kA) * s, Q = (5.0 / 18.0 * kA) * d;
    o[0] = P - Q; o[2] = P + Q; o[1] = fma(5.0 / 18.0 * (1.0 - 4.0 * kA * kA), s, (8.0 / 18.0) * f1);
}
__device__ __forceinline__ void lag_der3(double f0, double f1, double f2, double (&o)[3]) {
    const double s = f0 + f2, d = f2 - f0;
    const double u = (5.0 / 18.0 * 4.0 * kA) * d, t = fma(5.0 / 18.0, s, (8.0 / 18.0) * f1);
    o[0] = u - t; o[2] = u + t; o[1] = -2.0 * u;
}

// F / m at this element's nodes r[jx][jy] (as div_s / div_t produce them): the weak form with the metric,
//   F^x_j = -sum_g w_g |J_g| [s11 dphi_j/dx + s12 dphi_j/dy + s12 phi_j tan/R]
//   F^y_j = -sum_g w_g |J_g| [s12 dphi_j/dx + s22 dphi_j/dy - s11 phi_j tan/R]
// over the lumped mass m_j = R^2 dlon dlat mu_j (1/mu per node row and column parity in the row table)
__device__ __forceinline__ void sph_divergence(const double (&S11)[6], const double (&S12)[6], const double (&S22)[6],
                                               const double* __restrict__ row, double ihx, double ihy,
                                               double rX[3][3], double rY[3][3]) {
    double s11[9], s12[9], s22[9];
    eval_gp<true, true>(S11, s11); eval_gp<true, true>(S12, s12); eval_gp<true, true>(S22, s22);
    // weighted 1D contractions over gx for each gy (lag_val3 / lag_der3: sum_gx w L_j G, sum_gx w L_j' G)
    double X1[3][3], X2[3][3], Y1[3][3], Y2[3][3], Y3[3][3];   // [gy][jx]
#pragma unroll
    for (int gy = 0; gy < 3; ++gy) {
        lag_der3(s11[gy * 3], s11[gy * 3 + 1], s11[gy * 3 + 2], X1[gy]);
        lag_val3(s12[gy * 3], s12[gy * 3 + 1], s12[gy * 3 + 2], X2[gy]);
        lag_der3(s12[gy * 3], s12[gy * 3 + 1], s12[gy * 3 + 2], Y1[gy]);
        lag_val3(s22[gy * 3], s22[gy * 3 + 1], s22[gy * 3 + 2], Y2[gy]);
        lag_val3(s11[gy * 3], s11[gy * 3 + 1], s11[gy * 3 + 2], Y3[gy]);
    }
    // then over gy: rX_j = sum_gy w [L_jy (ihx X1 + sr X2) + L_jy' (ihy c X2)],
    //               rY_j = sum_gy w [L_jy (ihx Y1 - sr Y3) + L_jy' (ihy c Y2)]
    double cg[3], srg[3];
#pragma unroll
    for (int gy = 0; gy < 3; ++gy) { cg[gy] = ihy * __ldg(row + SPH_COS + gy); srg[gy] = __ldg(row + SPH_SINR + gy); }
#pragma unroll
    for (int jx = 0; jx < 3; ++jx) {
        double P[3], Q[3], Py[3], Qy[3];
#pragma unroll
        for (int gy = 0; gy < 3; ++gy) {
            P[gy] = fma(ihx, X1[gy][jx], srg[gy] * X2[gy][jx]);
            Q[gy] = cg[gy] * X2[gy][jx];
            Py[gy] = fma(ihx, Y1[gy][jx], -srg[gy] * Y3[gy][jx]);
            Qy[gy] = cg[gy] * Y2[gy][jx];
        }
        double vP[3], dQ[3], vPy[3], dQy[3];
        lag_val3(P[0], P[1], P[2], vP); lag_der3(Q[0], Q[1], Q[2], dQ);
        lag_val3(Py[0], Py[1], Py[2], vPy); lag_der3(Qy[0], Qy[1], Qy[2], dQy);
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) { rX[jx][jy] = vP[jy] + dQ[jy]; rY[jx][jy] = vPy[jy] + dQy[jy]; }
    }
#pragma unroll
    for (int jx = 0; jx < 3; ++jx)
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
            const double im = -__ldg(row + SPH_IMU + 2 * jy + (jx & 1));
            rX[jx][jy] *= im; rY[jx][jy] *= im;
        }
}

// ---------------------------------------------------------------- the kernel
// LC = true (with CL = false, FP64 storage): the constants are not staged with the job; once the stress
// update has read S and P_g, lane 0 TMA-loads them (5952 B) into the stage from the start of its S region
// on a second mbarrier, and the velocity update waits for it - small stages without CL's 24 live
// registers.  For n_S = 6 the S region is 4896 B, so the constants also overwrite the start of P_g; both
// regions have been consumed by then (the static_assert below keeps them clear of the v rows, which the
// divergence / velocity still read).
// PREP (with CL, FP64, n_S = 6, single rank): the first subcycle of an outer step forms the node constants
// itself - the outer-step prep (row a1) fused into the pass that first needs it.  Instead of the six
// constants a lane loads the element's A, H coefficients and the forcing a, o at its 2 x 2 nodes; the
// velocity at its nodes (v^n) is already in the stage; the nodal means of H and A (R#17) come from its own
// element, the west one (shuffle; lane 0 is the ring column), the row below (register carry; the ring row
// of a unit is loaded like any job) - the row-marching prep's sums in its order through the same
// prep_node_calc, so the constants (also stored for the remaining subcycles) are bitwise the prep's.
// PAIR (with CL, FP64, n_S = 6, single rank): two subcycles per launch (temporal blocking).  A unit (strip
// of 29 element columns, chunk [lr0, lr1)) is processed twice: pass A runs subcycle p on rows lr0 - 2 ..
// lr1 over the columns 29 s - 2 .. 29 s + 29 (lane = column - 29 s + 2) and writes S^{p+1}, v^{p+1} to the
// scratch buffers (a.Sx, a.vxx, a.vyx; what the unit's pass B reads is all written by the same warp); pass B
// runs subcycle p + 1 on rows lr0 - 1 .. lr1 - 1 from the scratch (mapsB) and stores S^{p+2}, v^{p+2} of the
// owned columns (lanes 2 .. 30).  Lanes whose inputs come from outside the warp (pass A lane 0's west node,
// pass B lanes 0, 1, 31) compute values nobody stores.  Overlapping units write bitwise identical values
// to the scratch (the arithmetic is the one-subcycle kernel's, partition-invariant).  The new state and
// the node constants / P_g of a pass-B row were read by pass A moments before: L2 hits, so a launch reads
// S, P_g, v, the constants once from DRAM and writes S, v once for two subcycles.
// the pass-B maps exist only in the PAIR instantiation (the default kernel keeps its one-map parameter block)
struct K2NoMaps {};
template <bool PAIR> struct K2PassB { using T = K2NoMaps; };
template <> struct K2PassB<true> { using T = K2Maps; };

template <bool REPL, int STAGES, typename SF, typename CT, int NS = 6, bool CL = false, bool LC = false, bool SPH = false,
          bool PREP = false, bool PAIR = false>
__global__ void __launch_bounds__(32 * K2_WARPS, 2) k_subcycle_tma(const __grid_constant__ K2Maps maps,
                                                                   const __grid_constant__ typename K2PassB<PAIR>::T mapsB,
                                                                   SubArgs a) {
    static_assert(!(CL && LC), "one node-constant mode");
    static_assert(!PAIR || (CL && NS == 6 && sizeof(SF) == 8 && sizeof(CT) == 8 && !SPH && !PREP), "pair: FP64 box, registers");
    static_assert(!PREP || (CL && NS == 6 && sizeof(SF) == 8 && sizeof(CT) == 8 && !SPH), "fused prep: FP64 box, registers");
    static_assert(!SPH || (NS == 6 && sizeof(SF) == 8 && sizeof(CT) == 8), "sphere: FP64, n_S = 6");
    static_assert(!LC || sizeof(SF) == 8, "late constants need the FP64 S region");
    using StageNC_ = K2StageNC<SF, NS>;
    static_assert(!LC || offsetof(StageNC_, vx) >= 6 * 2 * K2_CCOLS * sizeof(double),
                  "late constants overwrite only the consumed S / P_g regions");
    constexpr bool NOBOX = CL || LC;
    using Stage = typename K2StageSel<SF, NS, NOBOX>::T;
    constexpr int AL = K2Cols<SF>::ALIGN;
    SF* const S_out = reinterpret_cast<SF*>(a.S_out);   // FP32 buffers in mixed-precision mode
    extern __shared__ __align__(1024) unsigned char k2_smem[];   // no static smem: base stays 1024-B aligned
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    Stage* stg = reinterpret_cast<Stage*>(k2_smem) + wib * STAGES;
    uint64_t* bar = reinterpret_cast<uint64_t*>(k2_smem + K2_WARPS * STAGES * sizeof(Stage)) + wib * STAGES;
    if ((su32(k2_smem) & 127u) != 0u) {                          // TMA destinations need 128-B alignment
        printf("nxsdg: dynamic smem misaligned %u\n", su32(k2_smem));
        __trap();
    }
    const int twarps = gridDim.x * K2_WARPS;
    const int gw = blockIdx.x * K2_WARPS + wib;
    const int nunits = units_total(a);
    if (gw >= nunits) return;
    // L2 policies, a.l2_hints = NXSDG_OPT_L2_POLICY bits: 1 streamed loads (S, P_g, node constants)
    // evict_first; 2 (default) stores evict_first; 4 v boxes evict_last.  The new S and v (208 B per
    // element, 3.5 GB per C4 launch) are not read again in this launch, so with bit 2 they stop
    // displacing the lines that are: the neighbouring strips' overlap and the shared v row
    const uint64_t pol_ld = l2_policy(a.l2_hints & 1 ? 1 : 0), pol_st = l2_policy(a.l2_hints & 2 ? 1 : 0);
    const uint64_t pol_v = l2_policy(a.l2_hints & 4 ? 2 : 0);
    const uint64_t pol_keep = PAIR ? l2_policy(2) : 0;           // PAIR: pass-A scratch stores (evict_last)
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
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the next subcycle may be scheduled

    // Work list: (strip, chunk) units.  A warp's first unit is gw; further units are claimed
    // from a global counter (dynamic balancing; a.work_counter is zeroed before each launch),
    // or round-robin (gw + k * twarps) when no counter is given.  Lane 0 runs the prefetch
    // cursor and records each job in the stage's descriptor slot; all lanes read it back.
    // PAIR: a unit is pass A (rows end = min(lr1 + 1, erow_end) exclusive, ring lr0 - 2) then pass B (rows up
    // to lr1, ring lr0 - 1); lr1 holds the current pass's end row, ulr0 / ulr1 the unit's own rows
    // Between the passes the cursor inserts STAGES - 1 empty positions ("gap"), so pass B's first TMA load is
    // issued only after the unit's last pass-A job has stored (and fenced) what it reads
    struct Cur { int u, lr, lr1, ix0, ulr0, ulr1, pass, gap; bool ring, first, ok; };
    auto claim = [&](int u) -> int {      // lane 0: the next unit after u
        return a.work_counter ? twarps + atomicAdd(a.work_counter, 1) : u + twarps;
    };
    auto start_pass_b = [&](Cur& c) {
        c.pass = 1; c.lr1 = c.ulr1; c.gap = 0;
        c.ring = c.ulr0 > a.erow_begin; c.lr = c.ring ? c.ulr0 - 1 : c.ulr0; c.first = true;
    };
    auto start_unit = [&](int u, Cur& c) {
        for (;;) {                        // skip empty sub-units (ragged last chunk)
            c.ok = u < nunits;
            if (!c.ok) return;
            int strip, lr0, lr1;
            unit_rows(a, u, strip, lr0, lr1);
            if (lr0 < lr1) {
                c.u = u; c.lr1 = lr1; c.ix0 = PAIR ? strip * 29 - 1 : strip * 31;
                c.ring = lr0 > 0; c.lr = c.ring ? lr0 - 1 : lr0; c.first = true;
                c.pass = 0; c.gap = 0;
                if constexpr (PAIR) {
                    c.ulr0 = lr0; c.ulr1 = lr1;
                    c.lr1 = min(lr1 + 1, a.erow_end);
                    c.ring = lr0 - 2 >= a.erow_begin;
                    c.lr = c.ring ? lr0 - 2 : max(lr0 - 1, a.erow_begin);
                }
                return;
            }
            u = claim(u);
        }
    };
    auto advance = [&](Cur& c) {          // lane 0 only
        if (PAIR && c.gap > 0) {              // inside the gap between the passes
            if (--c.gap == 0) start_pass_b(c);
            return;
        }
        ++c.lr; c.ring = false; c.first = false;
        if (c.lr >= c.lr1) {
            if (PAIR && c.pass == 0) c.gap = STAGES - 1;
            else start_unit(claim(c.u), c);
        }
    };
    int4* jobs = reinterpret_cast<int4*>(bar + K2_WARPS * STAGES - wib * STAGES) + wib * STAGES;
    auto record = [&](const Cur& c, int st) {   // lane 0
        jobs[st] = make_int4(c.ok ? c.u : -1, c.lr, c.lr1,
                             (c.ring ? 1 : 0) | (c.first ? 2 : 0) | (PAIR ? ((c.pass ? 4 : 0) | (c.gap > 0 ? 8 : 0)) : 0));
    };
    // v row carry: a continuing job (not the first of its unit) loads node rows 2lr+1, 2lr+2 into smem
    // rows 0, 1 and takes row 2lr (the previous job's top row, same lane columns) from registers
    const bool vcarry = a.vcarry != 0;
    auto issue = [&](const Cur& c, int s) {
        if (PAIR && c.gap > 0) return;       // an empty position: nothing to load
        Stage* t = stg + s;
        const bool cont = vcarry && !c.first;
        const K2Maps* Mp = &maps;
        if constexpr (PAIR) { if (c.pass) Mp = &mapsB; }       // pass B reads the pass-A scratch
        const K2Maps& M = *Mp;
        if (PAIR && c.pass) asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[s], k2_tx_bytes<SF, NS, NOBOX>() - (cont ? 2u * K2_VCOLS * 8u : 0u));
        const int xs = (c.ix0 - 1) & ~(AL - 1);   // 16-B aligned start column (arithmetic: -1 -> -2 / -4)
        tma3h(&t->S[0][0], &M.S, &bar[s], xs, c.lr, 0, pol_ld);
        tma3h(&t->Pg[0][0], &maps.Pg, &bar[s], xs, c.lr, 0, pol_ld);
        if (cont) {
            tma2h(&t->vx[0][0], &M.vx2, &bar[s], 2 * (c.ix0 - 1), 2 * c.lr + 1, pol_v);
            tma2h(&t->vy[0][0], &M.vy2, &bar[s], 2 * (c.ix0 - 1), 2 * c.lr + 1, pol_v);
        } else {
            tma2h(&t->vx[0][0], &M.vx, &bar[s], 2 * (c.ix0 - 1), 2 * c.lr, pol_v);
            tma2h(&t->vy[0][0], &M.vy, &bar[s], 2 * (c.ix0 - 1), 2 * c.lr, pol_v);
        }
        if constexpr (!NOBOX) tma3h(&t->C[0][0][0], &maps.C, &bar[s], 2 * c.ix0, 2 * c.lr, 0, pol_ld);
    };

    const double ihx = a.ihx, ihy = a.ihy, fac = a.fac, hA = 0.5 * a.ainv;
    const double mhx = -9.0 * ihx, mhy = -9.0 * ihy;   // -1 / (corner lumped mass / |K|) = -9
    const int64_t npitch = a.npitch, eplane = a.eplane;
    // Programmatic dependent launch (single-rank subcycle graphs, NXSDG_OPT_PDL): this grid may start while the
    // previous subcycle's last CTAs finish; everything above (barrier setup) overlaps that tail, and no thread
    // reads or writes S / v before the previous grid has completed and flushed (griddepcontrol.wait is a no-op
    // for a launch without the attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // prologue: jobs 0 .. STAGES-2 in flight; job j lives in stage j % STAGES
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
    uint32_t phase = 0, phaseC = 0;    // bit s = parity of stage s (LC: of its constants barrier)
    int s = 0;
    double carx[2] = {0.0, 0.0}, cary[2] = {0.0, 0.0};
    double carVx[3] = {0.0, 0.0, 0.0}, carVy[3] = {0.0, 0.0, 0.0};   // v row carry (node row 2lr of the next job)
    // PREP: the row below's DG node values on its top node row (h, a at local jx = 0, 1, 2) and whether it exists
    double pcH[3] = {0.0, 0.0, 0.0}, pcA[3] = {0.0, 0.0, 0.0};
    bool pcOK = false;
    auto okE = [&](int ex, int ey) { return ex >= 0 && ex < a.nx && ey >= 0 && ey < a.pa.elem_rows_with_nodes; };
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
            cur.pass = PAIR ? (jd.w >> 2) & 1 : 0;
            cur.ix0 = PAIR ? (cur.u % a.nstrips) * 29 - 1 : (cur.u % a.nstrips) * 31;
        }
        if (PAIR && (jobs[s].w & 8)) {       // the gap between a unit's passes: no job
            __syncwarp();
            s = (s + 1) % STAGES;
            continue;
        }
        // PAIR: pass A writes the scratch state for every lane whose value is valid (1 .. 31), pass B the
        // owned lanes 2 .. 30; the one-subcycle kernel stores lanes >= 1
        const bool passA = PAIR && cur.pass == 0;
        const bool lane_out = PAIR ? (passA ? lane >= 1 : (lane >= 2 && lane <= 30)) : lane >= 1;
        // (the one-subcycle kernel addresses its outputs from the parameter block as before: no live registers)
#define K2_SO (PAIR ? (passA ? reinterpret_cast<SF*>(a.Sx) : S_out) : S_out)
#define K2_VXO (PAIR ? (passA ? a.vxx : a.vx_out) : a.vx_out)
#define K2_VYO (PAIR ? (passA ? a.vyx : a.vy_out) : a.vy_out)
        const uint64_t pst = PAIR && passA ? pol_keep : pol_st;  // scratch: kept in L2 for pass B (evict_last hint)
        const int ix = cur.ix0 - 1 + lane, lr = cur.lr;
        // CL: this lane's node constants [field][jy][q] (only lanes that update nodes; the boundary
        // column ix = nx is forced to zero below, so it needs none)
        double cr[6][2][2];
        double pHc[6], pAc[6];             // PREP: this element's H, A coefficients
        bool pOK = false;
        if constexpr (PREP) {
            // the forcing a, o at the lane's nodes (cr[0], cr[1] <- a; cr[4], cr[5] <- o) and the element's H, A
            const bool need = lane >= 1 && ix >= 0 && ix <= a.nx && !cur.ring;
            const double* const fld[4] = {a.pa.ax, a.pa.ay, a.ox, a.oy};
            const int fi[4] = {0, 1, 4, 5};
#pragma unroll
            for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int jy = 0; jy < 2; ++jy) {
                    double2 v = make_double2(0.0, 0.0);
                    if (need) v = ldg_stream2h(fld[f] + (int64_t)(2 * lr + jy) * npitch + 2 * ix, pol_ld);
                    cr[fi[f]][jy][0] = v.x; cr[fi[f]][jy][1] = v.y;
                }
            pOK = okE(ix, lr);
            const int64_t e = (int64_t)(pOK ? lr : 0) * a.epitch + (pOK ? ix : 0);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                pHc[k] = pOK ? __ldg(a.pa.H + k * eplane + e) : 0.0;
                pAc[k] = pOK ? __ldg(a.pa.A + k * eplane + e) : 0.0;
            }
        } else if constexpr (CL) {
            const bool need = lane >= 1 && ix >= 0 && ix < a.nx && !cur.ring;
            const double* const fld[6] = {a.c1, a.rx0, a.ry0, a.cafo, a.ox, a.oy};
#pragma unroll
            for (int f = 0; f < 6; ++f)
#pragma unroll
                for (int jy = 0; jy < 2; ++jy) {
                    double2 v = make_double2(0.0, 0.0);
                    if (need) v = ldg_stream2h(fld[f] + (int64_t)(2 * lr + jy) * npitch + 2 * ix, pol_ld);
                    cr[f][jy][0] = v.x; cr[f][jy][1] = v.y;
                }
        }
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
        const Stage& t = stg[s];
        const int eo = (cur.ix0 - 1) - ((cur.ix0 - 1) & ~(AL - 1));   // lane offset inside the S / P_g box
        if (cur.first) { carx[0] = carx[1] = cary[0] = cary[1] = 0.0; }

        // ---- node values of this element (local box columns 2*lane .. 2*lane+2); node row 2lr + jy is
        //      smem row jy - ro (ro = 1 for a continuing job: its row 0 is the carried one)
        double Vx[3][3], Vy[3][3];
        const int ro = (vcarry && !cur.first) ? 1 : 0;
#pragma unroll
        for (int jy = 0; jy < 3; ++jy) {
            if (jy == 0 && ro) {
#pragma unroll
                for (int q = 0; q < 3; ++q) { Vx[0][q] = carVx[q]; Vy[0][q] = carVy[q]; }
                continue;
            }
            const int r = jy - ro;
            const double2 a2 = *reinterpret_cast<const double2*>(&t.vx[r][2 * lane]);
            const double2 b2 = *reinterpret_cast<const double2*>(&t.vy[r][2 * lane]);
            Vx[jy][0] = a2.x; Vx[jy][1] = a2.y; Vx[jy][2] = t.vx[r][2 * lane + 2];
            Vy[jy][0] = b2.x; Vy[jy][1] = b2.y; Vy[jy][2] = t.vy[r][2 * lane + 2];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) { carVx[q] = Vx[2][q]; carVy[q] = Vy[2][q]; }
        // ---- strain (Table 1 "strain"): DG coefficients, then Gauss-point values of
        //      the trace u = e11 + e22, the half difference w = (e11 - e22)/2 and e12, in which
        //      Hibler's Delta^2 = 1.25 (e11^2 + e22^2) + 1.5 e11 e22 + e12^2 is u^2 + w^2 + e12^2
        CT eu[9], ew[9], e12[9];
        const double* __restrict__ srow = SPH ? a.sph_rows + (int64_t)lr * kSphRow : nullptr;
        if constexpr (SPH) {
            sph_strain(Vx, Vy, srow, ihx, ihy, eu, ew, e12);
        } else {
            CT Es[NS], Et[NS], E[NS];
            const CT cihx = (CT)ihx, cihy = (CT)ihy;
            const CT hx2 = CT(0.5) * cihx, hy2 = CT(0.5) * cihy;
            strain_s(Vx, Es);
            strain_t(Vy, Et);
            combine(Es, Et, cihx, cihy, E);
            eval_gp<true, true>(E, eu);
            combine(Es, Et, hx2, -hy2, E);
            eval_gp<true, true>(E, ew);
            strain_t(Vx, Et);
            strain_s(Vy, Es);
            combine(Es, Et, hx2, hy2, E);
            eval_gp<true, true>(E, e12);
        }
        // ---- VP stress at the Gauss points (Listing 2), alpha^{-1} folded in: with
        //      pr = alpha^{-1} P / (2 Delta) and sub = alpha^{-1} P / 2 (REPL: P_r / 2, R#4),
        //      g11 = pr (1.25 e11 + 0.75 e22) - sub = a + b, g22 = a - b, a = pr u - sub, b = pr w / 2;
        //      g12 = alpha^{-1} P/Delta e12/4 = (pr e12) / 2 (each 1/2 goes into the projection)
        const CT cdmin2 = (CT)a.dmin2, chA = (CT)hA;
#pragma unroll
        for (int g = 0; g < 9; ++g) {
            const CT u = eu[g], w = ew[g], z = e12[g];
            const CT draw2 = fma(u, u, fma(w, w, z * z));
            const CT rD = rsqrt_t(draw2 + cdmin2);
            const CT ph = (CT)t.Pg[g][eo + lane] * chA;
            const CT pr = ph * rD;
            // replacement pressure (R#4): P_r/2 = (P/2) Draw/Delta, Draw = draw2 * rsqrt(draw2)
            const CT sub = REPL ? pr * (draw2 > CT(0) ? draw2 * rsqrt_t(draw2) : CT(0)) : ph;
            if constexpr (SPH) {   // the sphere projection weights the Gauss values by cos(lat): fold it here
                const CT c = (CT)__ldg(srow + SPH_COS + g / 3), cpr = c * pr;
                eu[g] = fma(cpr, u, -(c * sub));
                ew[g] = cpr * w;
                e12[g] = cpr * z;
            } else {
                eu[g] = fma(pr, u, -sub);
                ew[g] = pr * w;
                e12[g] = pr * z;
            }
        }
        CT C11[NS], C12[NS], C22[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            C11[k] = (CT)t.S[k][eo + lane]; C12[k] = (CT)t.S[NS + k][eo + lane];
            C22[k] = (CT)t.S[2 * NS + k][eo + lane];
        }
        const CT cfac = (CT)fac;
        if constexpr (SPH) {
            sph_project(eu, ew, e12, srow, fac, C11, C12, C22);
        } else {
            project_pair(eu, ew, cfac, C11, C22);
            project(e12, 0.5, cfac, C12);
        }
        if constexpr (LC) {   // S and P_g of this stage are consumed (their values already feed the
            if (!cur.ring) {  // projection FMAs): the node constants go there
                asm volatile("" ::: "memory");   // every lane's reads of the stage are issued before the barrier
                __syncwarp();
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&barC[s], 6u * 2u * K2_CCOLS * 8u);
                    tma3h(const_cast<SF*>(&t.S[0][0]), &maps.C, &barC[s], 2 * cur.ix0, 2 * lr, 0, pol_ld);
                }
            }
        }
        double S11[NS], S12[NS], S22[NS];   // the divergence and velocity stay FP64
#pragma unroll
        for (int k = 0; k < NS; ++k) { S11[k] = (double)C11[k]; S12[k] = (double)C12[k]; S22[k] = (double)C22[k]; }
        const bool evalid = ix >= 0 && ix < a.nx;
        if (!cur.ring && evalid && lane_out) {
            const int64_t e = (int64_t)lr * a.epitch + ix;
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                st_hint(K2_SO + k * eplane + e, (SF)S11[k], pst);
                st_hint(K2_SO + (NS + k) * eplane + e, (SF)S12[k], pst);
                st_hint(K2_SO + (2 * NS + k) * eplane + e, (SF)S22[k], pst);
            }
            if (a.peer_S_up != nullptr && lr == a.up_elem_row) {   // P2P: the neighbour's ghost element row 0
                const int64_t pe = a.peer_up_eplane;
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    a.peer_S_up[k * pe + ix] = S11[k];
                    a.peer_S_up[(NS + k) * pe + ix] = S12[k];
                    a.peer_S_up[(2 * NS + k) * pe + ix] = S22[k];
                }
            }
        }
        // ---- divergence contributions: rX = D_s S11 / hx + D_t S12 / hy, rY likewise
        double rX[3][3], rY[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) { rX[i][j] = 0.0; rY[i][j] = 0.0; }
        if constexpr (SPH) {
            sph_divergence(S11, S12, S22, srow, ihx, ihy, rX, rY);
        } else {
            div_s(S11, mhx, rX); div_t(S12, mhy, rX);      // already divided by the lumped mass
            div_s(S12, mhx, rY); div_t(S22, mhy, rY);
        }
        // ---- per-node gather (row below, W, E) + velocity update (R#11), branch-free:
        //      all four owned nodes are updated, boundary nodes select 0, stores are predicated
        const bool nvalid = lane_out && ix >= 0 && ix <= a.nx && !cur.ring;
        double sumx[2][2], sumy[2][2];                 // [jy][q]
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
        if constexpr (PREP) {
            // DG node values of this element (local (jx, jy) -> [jy * 3 + jx]) and of the west one
            double mh[9], ma[9], wh[9], wa[9];
            mh[0] = dg2_node<0, 0>(pHc); mh[1] = dg2_node<1, 0>(pHc); mh[2] = dg2_node<2, 0>(pHc);
            mh[3] = dg2_node<0, 1>(pHc); mh[4] = dg2_node<1, 1>(pHc); mh[5] = dg2_node<2, 1>(pHc);
            mh[6] = dg2_node<0, 2>(pHc); mh[7] = dg2_node<1, 2>(pHc); mh[8] = dg2_node<2, 2>(pHc);
            ma[0] = dg2_node<0, 0>(pAc); ma[1] = dg2_node<1, 0>(pAc); ma[2] = dg2_node<2, 0>(pAc);
            ma[3] = dg2_node<0, 1>(pAc); ma[4] = dg2_node<1, 1>(pAc); ma[5] = dg2_node<2, 1>(pAc);
            ma[6] = dg2_node<0, 2>(pAc); ma[7] = dg2_node<1, 2>(pAc); ma[8] = dg2_node<2, 2>(pAc);
#pragma unroll
            for (int j = 2; j < 9; j += 3) { wh[j] = __shfl_up_sync(0xffffffffu, mh[j], 1); wa[j] = __shfl_up_sync(0xffffffffu, ma[j], 1); }
            const bool wOK = __shfl_up_sync(0xffffffffu, pOK, 1);
            if (cur.first) pcOK = false;                      // a unit's first row: no row below in this warp
            const double bwH = __shfl_up_sync(0xffffffffu, pcH[2], 1), bwA = __shfl_up_sync(0xffffffffu, pcA[2], 1);
            const bool bwOK = __shfl_up_sync(0xffffffffu, pcOK, 1);
            if (nvalid) {
                PrepNodeOut o[2][2];
#pragma unroll
                for (int jy = 0; jy < 2; ++jy)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        double hs = 0.0, as = 0.0;
                        int cnt = 0;
                        // the row-marching prep's order: SW, SE, NW, NE
                        if (jy == 0 && q == 0) {
                            if (bwOK) { hs += bwH; as += bwA; ++cnt; }
                            if (pcOK) { hs += pcH[0]; as += pcA[0]; ++cnt; }
                            if (wOK) { hs += wh[2]; as += wa[2]; ++cnt; }
                            if (pOK) { hs += mh[0]; as += ma[0]; ++cnt; }
                        } else if (jy == 0) {
                            if (pcOK) { hs += pcH[1]; as += pcA[1]; ++cnt; }
                            if (pOK) { hs += mh[1]; as += ma[1]; ++cnt; }
                        } else if (q == 0) {
                            if (wOK) { hs += wh[5]; as += wa[5]; ++cnt; }
                            if (pOK) { hs += mh[3]; as += ma[3]; ++cnt; }
                        } else {
                            if (pOK) { hs += mh[4]; as += ma[4]; ++cnt; }
                        }
                        o[jy][q] = prep_node_calc(a.pa, hs, as, cnt, cr[0][jy][q], cr[1][jy][q], Vx[jy][q], Vy[jy][q],
                                                  cr[4][jy][q], cr[5][jy][q]);
                    }
#pragma unroll
                for (int jy = 0; jy < 2; ++jy) {
                    const int64_t n = (int64_t)(2 * lr + jy) * npitch + 2 * ix;
                    if (ix < a.nx) {
                        *reinterpret_cast<double2*>(a.pa.c1 + n) = make_double2(o[jy][0].c1, o[jy][1].c1);
                        *reinterpret_cast<double2*>(a.pa.rx0 + n) = make_double2(o[jy][0].rx0, o[jy][1].rx0);
                        *reinterpret_cast<double2*>(a.pa.ry0 + n) = make_double2(o[jy][0].ry0, o[jy][1].ry0);
                        *reinterpret_cast<double2*>(a.pa.cafo + n) = make_double2(o[jy][0].cafo, o[jy][1].cafo);
                    } else {                                      // ix = nx: node column 2 nx only
                        a.pa.c1[n] = o[jy][0].c1; a.pa.rx0[n] = o[jy][0].rx0;
                        a.pa.ry0[n] = o[jy][0].ry0; a.pa.cafo[n] = o[jy][0].cafo;
                    }
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        cr[0][jy][q] = o[jy][q].c1; cr[1][jy][q] = o[jy][q].rx0;
                        cr[2][jy][q] = o[jy][q].ry0; cr[3][jy][q] = o[jy][q].cafo;
                    }
                }
                if (a.top_boundary && lr == a.erow_end - 1) {   // the global top node row: elements below only
                    const int jr = 2 * a.erow_end;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int I = 2 * ix + q;
                        if (I > 2 * a.nx) continue;
                        double hs = 0.0, as = 0.0;
                        int cnt = 0;
                        if (q == 0) {
                            if (wOK) { hs += wh[8]; as += wa[8]; ++cnt; }
                            if (pOK) { hs += mh[6]; as += ma[6]; ++cnt; }
                        } else if (pOK) { hs += mh[7]; as += ma[7]; ++cnt; }
                        const int64_t n = (int64_t)jr * npitch + I;
                        const PrepNodeOut ot = prep_node_calc(a.pa, hs, as, cnt, a.pa.ax[n], a.pa.ay[n], Vx[2][q], Vy[2][q],
                                                              a.ox[n], a.oy[n]);
                        a.pa.c1[n] = ot.c1; a.pa.rx0[n] = ot.rx0; a.pa.ry0[n] = ot.ry0; a.pa.cafo[n] = ot.cafo;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 3; ++j) { pcH[j] = mh[6 + j]; pcA[j] = ma[6 + j]; }
            pcOK = pOK;
        }
        if (nvalid) {
            const bool brow0 = lr == a.erow_begin && a.bottom_boundary;
#pragma unroll
            for (int jy = 0; jy < 2; ++jy) {
                double nvx[2], nvy[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int I = 2 * ix + q;
                    const int cc = 2 * lane - 2 + q;
                    const double fx = sumx[jy][q], fy = sumy[jy][q];   // F / m (mass folded into div_s/t)
                    const double vxo = Vx[jy][q], vyo = Vy[jy][q];
                    double c1, r0x, r0y, cf, oxv, oyv;
                    if constexpr (CL) {
                        c1 = cr[0][jy][q]; r0x = cr[1][jy][q]; r0y = cr[2][jy][q];
                        cf = cr[3][jy][q]; oxv = cr[4][jy][q]; oyv = cr[5][jy][q];
                    } else if constexpr (LC) {
                        const double (*LCb)[2][K2_CCOLS] = reinterpret_cast<const double (*)[2][K2_CCOLS]>(&t.S[0][0]);
                        c1 = LCb[0][jy][cc]; r0x = LCb[1][jy][cc]; r0y = LCb[2][jy][cc];
                        cf = LCb[3][jy][cc]; oxv = LCb[4][jy][cc]; oyv = LCb[5][jy][cc];
                    } else {
                        c1 = t.C[0][jy][cc]; r0x = t.C[1][jy][cc]; r0y = t.C[2][jy][cc];
                        cf = t.C[3][jy][cc]; oxv = t.C[4][jy][cc]; oyv = t.C[5][jy][cc];
                    }
                    const double dx = oxv - vxo, dy = oyv - vyo;
                    const double w2 = fma(dx, dx, dy * dy);
                    const double w = w2 > 0.0 ? w2 * rsqrt_nr(w2) : 0.0;   // |o - v|
                    const double cw = cf * w;
                    const double rden = rcp_nr(fma(c1, a.b1, cw));
                    const double cb = c1 * a.beta, ck = c1 * a.kc;
                    const double ux = (fma(cb, vxo, r0x) + fma(cw, oxv, fma(ck, vyo, fx))) * rden;
                    const double uy = (fma(cb, vyo, r0y) + fma(cw, oyv, fma(-ck, vxo, fy))) * rden;
                    const bool bnd = (I == 0) || (I == 2 * a.nx) || (jy == 0 && brow0);
                    nvx[q] = bnd ? 0.0 : ux;
                    nvy[q] = bnd ? 0.0 : uy;
                }
                const int jr = 2 * lr + jy;
                const int64_t n = (int64_t)jr * npitch + 2 * ix;
                if (ix < a.nx) {
                    st_hint2(K2_VXO + n, nvx[0], nvx[1], pst);
                    st_hint2(K2_VYO + n, nvy[0], nvy[1], pst);
                } else {                                  // ix == nx: only the boundary column 2 nx
                    K2_VXO[n] = 0.0;
                    K2_VYO[n] = 0.0;
                }
                // P2P fused peer stores: the same values into the neighbours' ghost node rows (a strip
                // of one element row sends its bottom node row both ways)
#pragma unroll
                for (int d = 0; d < 2; ++d) {
                    double* pvx = d == 0 ? a.peer_vx_up : a.peer_vx_dn;
                    double* pvy = d == 0 ? a.peer_vy_up : a.peer_vy_dn;
                    const bool hit = pvx != nullptr && (d == 0 ? jr >= a.up_node_row0 : jr == a.dn_node_row);
                    if (!hit) continue;
                    const int64_t pn = (int64_t)(d == 0 ? jr - a.up_node_row0 : a.dn_dst_row) * npitch + 2 * ix;
                    if (ix < a.nx) {
                        *reinterpret_cast<double2*>(pvx + pn) = make_double2(nvx[0], nvx[1]);
                        *reinterpret_cast<double2*>(pvy + pn) = make_double2(nvy[0], nvy[1]);
                    } else {
                        pvx[pn] = 0.0;
                        pvy[pn] = 0.0;
                    }
                }
            }
        }
        // global top boundary row (Dirichlet) after the last owned element row
        if (a.top_boundary && lr == a.erow_end - 1 && nvalid) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int I = 2 * ix + q;
                if (I > 2 * a.nx) continue;
                K2_VXO[(int64_t)(2 * a.erow_end) * npitch + I] = 0.0;
                K2_VYO[(int64_t)(2 * a.erow_end) * npitch + I] = 0.0;
            }
        }
        if (passA) asm volatile("fence.proxy.async.global;" ::: "memory");   // the scratch feeds pass B's TMA
        __syncwarp();
        s = (s + 1) % STAGES;
    }
#undef K2_SO
#undef K2_VXO
#undef K2_VYO
}

}  // namespace nxk
