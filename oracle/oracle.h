/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, deliberately literal FP64 CPU implementation of the neXtSIM-DG
 * mEVP subcycle and DG advection as read from arXiv 2402.00466 plus
 * the readings listed in DESIGN.md §3.  It exists to prove the CUDA path
 * correct.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant generator with paper_2402_00466_b200/ (the product), and the
 * product never loads it.
 *
 * Citations "P:n" are lines of PAPER.md; "R#n" are DESIGN.md readings.
 *
 * Layouts (identical to the product ABI so one set of generated inputs
 * feeds both sides):
 *   DG field  : N_e x n row-major, element e = iy*nx + ix
 *   CG field  : (p*ny+1) x (p*nx+1) row-major, node = J*(p*nx+1)+I (R#8)
 */
#ifndef NXSDG_ORACLE_H
#define NXSDG_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int nx, ny;      /* elements per direction                      */
    double lx, ly;   /* extents [m]                                 */
    int p;           /* CG degree 1|2                               */
    int ns;          /* DG stress dofs 3|6                          */
    int na;          /* DG advection dofs 1|3|6                     */
    int bc;          /* 0 closed (Dirichlet v=0), 1 periodic (advection only) */
    const double* verts; /* NULL: axis-aligned box x_{a,b} = (a hx, b hy).  Else (ny+1) x (nx+1) x 2
                            vertex coordinates, row-major: a general (distorted) quad mesh with the
                            bilinear element map of its four vertices (R#23) */
    double radius;   /* > 0 (verts NULL): longitude-latitude mesh on the sphere of this radius [m]
                        ("quadrilateral meshes in spherical coordinates"; R#26): lx, ly are
                        the angular extents in longitude and latitude [rad], lat0 the southern edge */
    double lat0;     /* [rad], |lat0|, |lat0 + ly| < pi/2 */
} ora_mesh;

typedef struct {
    double rho_ice, rho_atm, rho_ocean, C_atm, C_ocean, f_c;
    double Pstar, DeltaMin, C_conc;
    double alpha, beta, dt;
    int replacement_pressure;
} ora_params;

/* ---- building blocks (exported so tests can pin them) ------------------ */
int    ora_ngp(int ns);
int    ora_gauss(int ngp, double* x, double* w);
void   ora_dg_basis(int n, double s, double t, double* psi);
void   ora_cg_basis(int p, double s, double t, double* phi, double* dphids, double* dphidt);
double ora_element_jacobian(const ora_mesh* m, int ix, int iy, double s, double t, double Jinv[4]);
int    ora_element_mass(const ora_mesh* m, int ix, int iy, int n, int ngp, double* M);
int    ora_solve(int n, double* A, double* b);

/* ---- the hot-path steps ------------------------------------------------ */
int ora_strain(const ora_mesh* m, const double* vx, const double* vy,
               double* E11, double* E12, double* E22);
int ora_stress(const ora_mesh* m, const ora_params* prm,
               const double* E11, const double* E12, const double* E22,
               const double* H, const double* A,
               double* S11, double* S12, double* S22);
int ora_divergence(const ora_mesh* m, const double* S11, const double* S12, const double* S22,
                   double* Fx, double* Fy);
int ora_lumped_mass(const ora_mesh* m, double* mass);
int ora_prep(const ora_mesh* m, const double* H, const double* A, double* Hn, double* An);
int ora_velocity(const ora_mesh* m, const ora_params* prm,
                 const double* Fx, const double* Fy, const double* mass,
                 const double* Hn, const double* An,
                 const double* vnx, const double* vny,
                 const double* ox, const double* oy, const double* ax, const double* ay,
                 double* vx, double* vy);
int ora_subcycles(const ora_mesh* m, const ora_params* prm, int nsub,
                  const double* H, const double* A,
                  const double* ox, const double* oy, const double* ax, const double* ay,
                  const double* vnx, const double* vny,
                  double* vx, double* vy, double* S11, double* S12, double* S22);
int ora_advect_rhs(const ora_mesh* m, const double* vx, const double* vy,
                   const double* c, double* rhs);
int ora_advect(const ora_mesh* m, double dt, const double* vx, const double* vy,
               double* A, double* H);
/* NEXT-4 (R#25): Zhang-Shu bound-preserving scaling limiter (keeps the |J|-weighted element mean)
 * and advection with it applied after every SSP-RK stage (A in [0,1], H >= 0). */
int ora_limit(const ora_mesh* m, double lo, double hi, double* c);
int ora_advect_limited(const ora_mesh* m, double dt, const double* vx, const double* vy,
                       double* A, double* H, int limiter);
int ora_outer_step(const ora_mesh* m, const ora_params* prm, int nsub, int do_advect,
                   const double* ox, const double* oy, const double* ax, const double* ay,
                   double* vx, double* vy, double* S11, double* S12, double* S22,
                   double* A, double* H);
int ora_num_threads(void);
void ora_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
