/*
 * nxsdg.h — C ABI of the B200-native neXtSIM-DG mEVP hot path (libnxsdg.so).
 *
 * What it computes (PAPER.md = arXiv 2402.00466; "P:n" = PAPER.md line n;
 * "R#n" = reading n in DESIGN.md §3):
 *   - Eq. (1): upwind DG advection of ice concentration A and
 *     thickness H with the CG velocity, explicit SSP Runge-Kutta.
 *   - Eq. (2)-(3): the mEVP pseudo-time iteration of the momentum
 *     equation with the viscous-plastic rheology, subcycled within one outer
 *     (advection) step.  One subcycle = strain (Table 1) ->
 *     stress update (Listing 1/2) -> stress divergence
 *      -> velocity update.
 *   Discretisation: structured quadrilateral mesh (the box, or general
 *   quads with the bilinear map of each cell's vertices, nxsdg_set_vertices), CG
 *   velocity of degree p (Q1|Q2), DG stress with n_S coefficients (3 with Q1; 6
 *   or 8 with Q2, R#6/R#24), DG tracers with n_A coefficients (1|3|6), Gauss rule
 *   NGP from Listing 2 line 462.
 *
 * Layouts at the ABI (logical, independent of the device layout):
 *   DG field : (owned element rows) x nx x n doubles, row-major, one element's
 *              n coefficients contiguous, element e = iy*nx + ix.
 *   CG field : (owned node rows) x (p*nx+1) doubles, row-major,
 *              node = J*(p*nx+1) + I (R#8).
 *   With nranks == 1 the owned rows are all rows: N_e = nx*ny elements,
 *   (p*ny+1)*(p*nx+1) nodes.  With nranks > 1 rank r owns element rows
 *   [r0, r1) (nxsdg_get_partition) and node rows [p*r0, p*r1), the top rank
 *   also node row p*ny.
 *
 * Ownership: the context owns all device memory.  Caller pointers are
 * borrowed for the duration of the call only (data is copied).  DEVICE
 * pointers must be on the context's device.
 *
 * Asynchrony: all work is ordered on the context stream.  HOST-memory reads
 * and writes are synchronous with respect to the host buffer; DEVICE-memory
 * reads and writes and all compute calls are asynchronous (stream-ordered);
 * nxsdg_synchronize waits.
 *
 * Errors: every call returns nxsdg_status; nothing throws across the ABI.
 * Invalid arguments never mutate state.  A CUDA or NCCL failure poisons the
 * context: every later call except nxsdg_destroy / nxsdg_last_error returns
 * NXSDG_ERR_STATE.  No CUDA device -> NXSDG_ERR_CUDA: there is no CPU
 * fallback.  A context is not thread-safe; several contexts per process are
 * allowed (used by the loopback row-strip tests).
 */
#ifndef NXSDG_ABI_INCLUDED_H_
#define NXSDG_ABI_INCLUDED_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NXSDG_ABI_VERSION 1

typedef struct nxsdg_ctx nxsdg_ctx;

typedef enum {
    NXSDG_OK = 0,
    NXSDG_ERR_INVALID_ARG = 1, /* null pointer, bad size/count, bad enum            */
    NXSDG_ERR_UNSUPPORTED = 2, /* degree combination or mode not implemented         */
    NXSDG_ERR_STATE = 3,       /* wrong call order, or context poisoned              */
    NXSDG_ERR_CUDA = 4,        /* CUDA error or no device                            */
    NXSDG_ERR_NCCL = 5,        /* NCCL error or NCCL not loadable                    */
    NXSDG_ERR_OOM = 6          /* device allocation failed                           */
} nxsdg_status;

/* HOST_ASYNC: pinned host memory, copied on the context's copy streams (one for uploads, one for read-backs,
 * so the two directions overlap on the full-duplex link); the call returns at once and
 * the caller keeps the buffer unchanged until nxsdg_synchronize.  Accepted by nxsdg_set_forcing (the
 * forcing is staged and takes effect at the next BEGIN_STEP, so the upload of step k+1's forcing
 * overlaps step k) and by nxsdg_read_state for NXSDG_VX / NXSDG_VY (a snapshot of v at that point in
 * the stream, read back while later work runs). */
typedef enum { NXSDG_MEM_HOST = 0, NXSDG_MEM_DEVICE = 1, NXSDG_MEM_HOST_ASYNC = 2 } nxsdg_mem;

typedef enum {
    NXSDG_BC_CLOSED = 0,   /* v = 0 on the box boundary, zero advective boundary flux (R#16)   */
    NXSDG_BC_PERIODIC = 1  /* advection only (tests); nxsdg_mevp_substeps -> UNSUPPORTED       */
} nxsdg_bc;

typedef enum {
    NXSDG_VX = 0, NXSDG_VY = 1,                   /* CG nodes                                  */
    NXSDG_S11 = 2, NXSDG_S12 = 3, NXSDG_S22 = 4,  /* DG n_S: stress (mEVP state)        */
    NXSDG_A = 5, NXSDG_H = 6,                     /* DG n_A: concentration, thickness  */
    NXSDG_E11 = 7, NXSDG_E12 = 8, NXSDG_E22 = 9,  /* DG n_S: strain rate, debug steps only     */
    NXSDG_FX = 10, NXSDG_FY = 11,                 /* CG: assembled -(sigma, grad phi), debug   */
    NXSDG_NFIELDS = 12
} nxsdg_field;

/* nxsdg_mevp_substeps flags */
enum {
    NXSDG_BEGIN_STEP = 1u, /* start an outer step: v^n <- v, nodal H/A, node constants, P at Gauss points */
    NXSDG_UNFUSED = 2u     /* run the 4 unfused step kernels instead of the fused subcycle kernel        */
};

/* single debug steps (nxsdg_run_step) */
typedef enum {
    NXSDG_STEP_STRAIN = 0,     /* E <- Pi_DG sym grad v                      (R#9)          */
    NXSDG_STEP_STRESS = 1,     /* S <- Listing 2 update with stored E, H, A           */
    NXSDG_STEP_DIVERGENCE = 2, /* F <- -(sigma, grad phi_j) assembled        (R#10)         */
    NXSDG_STEP_VELOCITY = 3    /* v <- mEVP velocity update with stored F    (R#11)     */
} nxsdg_step;

typedef enum {
    NXSDG_TRANSPORT_NONE = 0,     /* nranks == 1                                                  */
    NXSDG_TRANSPORT_NCCL = 1,     /* one process per GPU, ncclSend/ncclRecv halo rows              */
    NXSDG_TRANSPORT_LOOPBACK = 2, /* all ranks' contexts in one process (tests), cudaMemcpyAsync  */
    NXSDG_TRANSPORT_P2P = 3       /* halo rows copied straight into the neighbours' buffers over
                                     peer memory (NVLink / NVSwitch), device-side flag handshake;
                                     no NCCL (nxsdg_p2p_export / nxsdg_p2p_connect)                */
} nxsdg_transport;

typedef struct {
    int32_t nx, ny;       /* global elements per direction, >= 1                                  */
    double lx, ly;        /* box extents [m], > 0; hx = lx/nx, hy = ly/ny                         */
    int32_t cg_degree;    /* p: 1 | 2                                                             */
    int32_t n_stress;     /* n_S: 3 with p = 1; 6 (R#6) or 8 (full gradient space of Q2, R#24) with p = 2 */
    int32_t n_adv;        /* n_A: 1 | 3 (p = 1), 1 | 3 | 6 (p = 2) (R#7)                          */
    int32_t bc;           /* nxsdg_bc                                                             */
    int32_t rank, nranks; /* row-strip partition, 1 <= nranks <= ny                               */
    int32_t transport;    /* nxsdg_transport                                                      */
    const void* nccl_id;  /* 128-byte ncclUniqueId (NCCL transport), else NULL                    */
    int32_t device;       /* CUDA ordinal                                                         */
    void* stream;         /* cudaStream_t to run on; NULL -> library-owned stream                 */
} nxsdg_mesh_desc;

typedef struct {
    double rho_ice, rho_atm, rho_ocean; /* densities [kg m^-3] (values R#12)                 */
    double C_atm, C_ocean;              /* drag coefficients (R#11, R#12)                           */
    double f_c;                         /* Coriolis parameter [s^-1]                                */
    double Pstar, DeltaMin;             /* ice strength [N m^-2], minimal deformation [s^-1] */
    double C_conc;                      /* concentration exponent, the literal 20 of P:183          */
    double alpha, beta;                 /* mEVP, code form fac = 1 - 1/alpha (R#1); > 1, > 0 */
    double dt;                          /* outer step [s] (R#14)                                    */
    int32_t replacement_pressure;       /* 0: -P/2 as Listing 1/2; 1: -P_r/2, P_r = P Draw/Delta (R#4) */
} nxsdg_params;

/* ---- lifecycle ----------------------------------------------------------- */
/* Validate, pick the device, partition, allocate padded SoA buffers, run the
 * element-matrix precompute kernel (K0).  State starts at zero; forcing unset.
 * Errors: INVALID_ARG (null, nx/ny < 1, extents <= 0, alpha <= 1, bad rank),
 * UNSUPPORTED (degree combination, periodic with nranks > 1), CUDA, NCCL, OOM. */
nxsdg_status nxsdg_create_mesh(const nxsdg_mesh_desc* desc, const nxsdg_params* params, nxsdg_ctx** out);
nxsdg_status nxsdg_destroy(nxsdg_ctx* ctx);
const char* nxsdg_last_error(const nxsdg_ctx* ctx);
int32_t nxsdg_abi_version(void);

/* Replace the physical parameters (takes effect at the next BEGIN_STEP for the
 * node constants; alpha/beta/DeltaMin/Pstar immediately). */
nxsdg_status nxsdg_set_params(nxsdg_ctx* ctx, const nxsdg_params* params);

/* Row-strip partition of this rank: element rows [elem_row0, elem_row0+elem_rows),
 * node rows [node_row0, node_row0+node_rows).  Pure host arithmetic. */
nxsdg_status nxsdg_get_partition(const nxsdg_ctx* ctx, int64_t* elem_row0, int32_t* elem_rows,
                                 int64_t* node_row0, int32_t* node_rows);
/* Same arithmetic without a context (host only, no GPU needed). */
nxsdg_status nxsdg_partition(int32_t ny, int32_t cg_degree, int32_t nranks, int32_t rank,
                             int64_t* elem_row0, int32_t* elem_rows, int64_t* node_row0, int32_t* node_rows);

/* Tuning / A-B options (take effect at the next compute call):
 *   NXSDG_OPT_FUSED_KERNEL  0 (default): TMA-staged structured kernel for p = 2 (table-driven for p = 1);
 *                           1: table-driven register kernel k_subcycle<p> (reference-table variant)
 *   NXSDG_OPT_CHUNK_ROWS    element rows per warp work unit (one ring row each); 0 (default) = automatic: 32,
 *                           halved down to 4 while the mesh would give fewer (strip, chunk) units than the
 *                           device's resident warps (8 per SM) - small single-rank meshes such as C2 (256^2);
 *                           row strips keep 32; every height gives bitwise the same result
 *   NXSDG_OPT_CTAS_PER_SM   cap on resident CTAs per SM for the persistent TMA kernel (0 = occupancy;
 *                           -1 (default) = tuned: 4 with the node constants in registers or loaded late,
 *                           3 (n_S = 6) / 2 (n_S = 8) with them TMA-staged in FP64, 4 with FP32 storage,
 *                           4 / 3 for the fused general-quad kernel with late / boxed constants)
 *   NXSDG_OPT_STAGES        TMA pipeline depth per warp, 2..4 (default 2; 2..3 with FP32 storage)
 *   NXSDG_OPT_CONST_STAGING the fused kernels' six node constants (c1, rhs0, cAFo, o): 0 = a TMA box of each
 *                           stage; 1 = box kernel: each lane prefetches its 24 doubles into registers with
 *                           16-B loads; 2 = box kernel (FP64 storage only, else UNSUPPORTED at the launch):
 *                           a second TMA loads them into the stage's S / P_g region once the stress update has
 *                           consumed it; general-quad kernel: 1 and 2 both mean that late TMA (all: smaller
 *                           stages, more CTAs per SM); -1 (default) = tuned: box kernel 1 (FP64, n_S = 6),
 *                           2 (FP64, n_S = 8), 0 (FP32 storage); general-quad kernel late
 *   NXSDG_OPT_TAIL_SPLIT    persistent fused kernels with the work counter: 1 (default) = the last chunks of
 *                           each launch are split into ~8-row sub-units so the warps finish together; 0 = off
 *   NXSDG_OPT_L2_POLICY     fused TMA kernels' L2 eviction policies (createpolicy + .L2::cache_hint), bits:
 *                           1 = streamed loads (S, P_g, node constants) evict_first, 2 = the new S and v
 *                           stores evict_first, 4 = v boxes evict_last (bits 1 and 4: box kernel only);
 *                           default 2 (0 = evict_normal everywhere)
 *   NXSDG_OPT_V_ROW_CARRY   box TMA kernel: 1 (default) = consecutive element rows of a warp's work unit share
 *                           a v node row, which the next job takes from registers (its TMA boxes load the two
 *                           new node rows only); 0 = every job loads all three rows
 *   NXSDG_OPT_DYNAMIC       1 (default): warps claim work units from an atomic counter; 0: static round-robin
 *   NXSDG_OPT_PRECISION     0 (default): FP64 everywhere; 1 (NEXT-3): the fused CG2/DG2 subcycles keep
 *                           S and P_g in FP32 storage (arithmetic and the v state stay FP64); the FP64 S
 *                           seen through the ABI is converted at each nxsdg_mevp_substeps call (single rank);
 *                           2: as 1 and the stress update (strain, Listing 2, projection) in FP32 arithmetic
 *   NXSDG_OPT_MAP_MODE      general quads (nxsdg_set_vertices): 0 = per-element iMJwPSI pre-assembled and
 *                           stored, 1 (default) = recomputed on the fly from the 4 vertices
 *   NXSDG_OPT_P2P_FUSED_STORES  P2P transport with the TMA kernel: 1 (default) = the fused subcycle kernel stores
 *                           the halo rows (v node rows, S element row) straight into the neighbours' buffers as
 *                           it computes them, the exchange is the flag handshake alone; 0 = copy-engine copies
 *   NXSDG_OPT_LIMITER       NEXT-4 (DESIGN R#25): 0 (default, the paper's unlimited scheme) | 1 = Zhang-Shu
 *                           bound-preserving scaling limiter after every SSP-RK stage of nxsdg_advect (A in [0,1],
 *                           H >= 0 at the volume and edge Gauss points; element means, hence mass, unchanged)
 *   NXSDG_OPT_ADVECT_KERNEL 0 (default) = the persistent TMA-staged structured advection k_advect_tma for the
 *                           closed-box CG2/DG2 pair without limiter (bitwise = k_advect_q2); 1 = k_advect_q2
 *   NXSDG_OPT_ADVECT_STAGES shared-memory row slots per warp of k_advect_tma: 3 (late ring: row k+2 issued into
 *                           row k-1's slot once job k has read it; 5 CTAs / 10 warps per SM) | 4 (default) | 5
 *   NXSDG_OPT_PREP_KERNEL   CG2/DG2 outer-step prep of the node constants: 0 (default) = row-marching warps (each
 *                           element read once, neighbours by shuffle / register carry); 1 = a thread per element
 *                           gathering its 4 neighbours; 2 = formed by the first fused subcycle of the outer step,
 *                           which needs them first (single rank, FP64 box kernel with constants in registers and 2
 *                           stages; elsewhere 0): BEGIN_STEP defers the node pass and the next nxsdg_mevp_substeps
 *                           with n > 0 runs it inside its first launch (an unfused call or a VELOCITY debug step runs
 *                           it first as the separate pass).  All three are bitwise equal; 2 measured no faster than
 *                           0 plus a plain subcycle
 *   NXSDG_OPT_FUSE_PREP_PG  single rank with k_advect_tma: 1 (default) = the last advection stage also writes the
 *                           outer-step prep's P at the Gauss points of the new A, H (bitwise what the prep would
 *                           compute); 0 = the prep computes it at BEGIN_STEP
 *   NXSDG_OPT_PDL           1 = the subcycle launches of a single-rank graph use programmatic dependent launch:
 *                           a launch's CTAs set up while the previous subcycle's last CTAs finish and wait
 *                           (griddepcontrol.wait) before touching S or v; 0 (default: measured no faster) = plain
 *   NXSDG_OPT_PAIR_SUBCYCLES 1 = two subcycles per launch of the box TMA kernel (temporal blocking: a unit runs
 *                           subcycle p over a 2-row / 2-column wider halo into scratch buffers, then subcycle
 *                           p + 1 from them; single rank, FP64, n_S = 6, node constants in registers; an odd
 *                           count ends with a one-subcycle launch; bitwise equal); 0 (default) = one per launch
 *   NXSDG_OPT_MULTIRANK_GRAPH  row-strip ranks (P2P or NCCL transport): 1 = nxsdg_mevp_substeps captures its
 *                           n fused subcycles - boundary chunks, exchange (peer stores + flag handshake, or
 *                           NCCL send/recv) on the halo stream, interior chunks, join - in one CUDA graph per
 *                           (n, ping-pong and flag-slot parity) and replays it (one host crossing per call);
 *                           0 = the same work issued from the host one subcycle at a time; -1 (default) = 1 for
 *                           P2P between processes, 0 for NCCL.  Ranks connected in one process
 *                           (nxsdg_p2p_connect_local, a one-GPU test topology) always issue from the host and
 *                           advect with k_advect_q2 (graph replays / k_advect_tma launches of several ranks
 *                           sharing one context hung the device there)
 * INVALID_ARG for an unknown option or value. */
enum { NXSDG_OPT_FUSED_KERNEL = 0, NXSDG_OPT_CHUNK_ROWS = 1, NXSDG_OPT_CTAS_PER_SM = 2, NXSDG_OPT_STAGES = 3,
       NXSDG_OPT_DYNAMIC = 4, NXSDG_OPT_MAP_MODE = 5, NXSDG_OPT_PRECISION = 6, NXSDG_OPT_P2P_FUSED_STORES = 7,
       NXSDG_OPT_LIMITER = 8, NXSDG_OPT_CONST_STAGING = 9, NXSDG_OPT_TAIL_SPLIT = 10, NXSDG_OPT_L2_POLICY = 11,
       NXSDG_OPT_V_ROW_CARRY = 12, NXSDG_OPT_MULTIRANK_GRAPH = 13, NXSDG_OPT_ADVECT_KERNEL = 14,
       NXSDG_OPT_ADVECT_STAGES = 15, NXSDG_OPT_FUSE_PREP_PG = 16, NXSDG_OPT_PREP_KERNEL = 18,
       NXSDG_OPT_PAIR_SUBCYCLES = 19, NXSDG_OPT_PDL = 20 };
nxsdg_status nxsdg_set_option(nxsdg_ctx* ctx, int32_t option, int64_t value);

/* ---- state ----------------------------------------------------------------- */
/* count = number of doubles of this rank's owned part in the ABI layout.
 * Writing invalidates the outer-step constants (next substep call needs BEGIN_STEP). */
nxsdg_status nxsdg_write_state(nxsdg_ctx* ctx, nxsdg_field field, const double* src, int64_t count, nxsdg_mem mem);
nxsdg_status nxsdg_read_state(nxsdg_ctx* ctx, nxsdg_field field, double* dst, int64_t count, nxsdg_mem mem);

/* Forcing on the CG nodes (owned rows): ocean current o and wind a [m/s] ("F"). */
nxsdg_status nxsdg_set_forcing(nxsdg_ctx* ctx, const double* ox, const double* oy,
                               const double* ax, const double* ay, int64_t count, nxsdg_mem mem);

/* Synthetic VP-benchmark forcing evaluated on the device at time t [s] (DESIGN.md §5 recipe:
 * ocean gyre o, cyclone wind a moving at 51.2 km/day; global box coordinates), for multi-outer-step
 * runs without host transfers.  Same effect as nxsdg_set_forcing with those fields. */
nxsdg_status nxsdg_set_forcing_cyclone(nxsdg_ctx* ctx, double t);

/* NEXT-1: switch the context to a general quadrilateral mesh with these vertices,
 * (ny+1) x (nx+1) x 2 doubles row-major (count = 2 (nx+1)(ny+1)); elements map bilinearly from their
 * four vertices.  In this mode the stress step (Listing 2) uses per-element inverse
 * maps per NXSDG_OPT_MAP_MODE, every nxsdg_run_step step and nxsdg_advect (closed box) run the
 * general-geometry kernels, and nxsdg_mevp_substeps runs the fused general-quad subcycle kernel
 * (geometry recomputed on the fly from the vertices; CG2/DG2 with n_S = 6) or, with NXSDG_UNFUSED, the
 * unfused general-geometry steps.  Fused subcycles with CG1 or n_S = 8 on a general mesh return
 * UNSUPPORTED (use NXSDG_UNFUSED).  Single rank only. */
nxsdg_status nxsdg_set_vertices(nxsdg_ctx* ctx, const double* xy, int64_t count, nxsdg_mem mem);

/* NEXT-4 ("quadrilateral meshes in spherical coordinates"; R#26): switch the
 * context to a longitude-latitude mesh on the sphere of `radius` [m]: element (ix, iy) spans longitudes
 * [ix, ix + 1] x lon_extent / nx and latitudes lat0 + [iy, iy + 1] x lat_extent / ny [rad] (the mesh
 * descriptor's lx, ly are then unused).  Velocities are the physical (east, north) components; the strain
 * rate carries the frame's metric terms (eps11 -= v tan(lat)/R, eps12 += u tan(lat)/(2R)), the stress
 * divergence their adjoint, every integral the weight |J| = R^2 cos(lat) dlon dlat (3-point Gauss rule),
 * the advection the meridian / parallel arc lengths.  Supported: CG2 / DG2 (n_S = n_A = 6), FP64, the fused
 * TMA subcycle kernel and the structured advection (single rank or row strips); UNSUPPORTED otherwise
 * (other degrees, general quads, FP32 storage, unfused / debug steps, the limiter).  INVALID_ARG unless
 * radius, extents > 0 and both edge latitudes lie inside (-pi/2, pi/2). */
nxsdg_status nxsdg_set_sphere(nxsdg_ctx* ctx, double radius, double lat0, double lon_extent, double lat_extent);

/* ---- compute ----------------------------------------------------------------- */
/* n_sub mEVP subcycles.  flags: NXSDG_BEGIN_STEP, NXSDG_UNFUSED.
 * STATE if forcing unset, or if no BEGIN_STEP happened since the last state write. */
nxsdg_status nxsdg_mevp_substeps(nxsdg_ctx* ctx, int32_t n_sub, uint32_t flags);

/* One advection step of A and H over dt with the current v (Eq. 1, P:121 order: call before
 * the outer step's substeps).  Invalidates the outer-step constants. */
nxsdg_status nxsdg_advect(nxsdg_ctx* ctx, double dt);

/* Debug: one unfused step on the current state (needs BEGIN_STEP for STRESS/VELOCITY). */
nxsdg_status nxsdg_run_step(nxsdg_ctx* ctx, nxsdg_step step);

nxsdg_status nxsdg_synchronize(nxsdg_ctx* ctx);   /* waits for the context stream and the copy streams */
/* Make the context stream wait for every HOST_ASYNC copy issued so far (stream-ordered join). */
nxsdg_status nxsdg_stream_join(nxsdg_ctx* ctx);

/* ---- multi-rank plumbing ------------------------------------------------------- */
/* Fill 128 bytes with a fresh ncclUniqueId (rank 0; broadcast it to the others). */
nxsdg_status nxsdg_nccl_unique_id(void* out128);
/* P2P transport (SURVEY §8(e) "device-initiated peer stores").  Each halo exchange
 * copies the halo plan's send rows with the copy engine directly into the receive rows of the
 * neighbour's buffers (one 2D copy per message, no staging, no NCCL), then sets its word of flag
 * slot (k & 1) in each neighbour to 1 (cuStreamWriteValue32, fenced) and makes the context stream
 * wait on the device until both neighbours have set ours (cuStreamWaitValue32 ==, with
 * CU_STREAM_WAIT_VALUE_FLUSH where the device can flush remote writes), then clears it.  Constant
 * values: the exchange replays inside CUDA graphs.  The host never blocks.
 * nxsdg_p2p_export: an opaque blob (*needed bytes; blob == NULL: size only) with CUDA IPC handles
 *   of this rank's exchanged buffers and flag pair; give it to ranks r-1 and r+1 (e.g. with
 *   torch.distributed all_gather_object).  STATE unless the context uses NXSDG_TRANSPORT_P2P.
 * nxsdg_p2p_connect: map the neighbours' blobs (NULL where no neighbour exists); INVALID_ARG for a
 *   blob of another mesh / rank, UNSUPPORTED without peer access between the devices, CUDA when
 *   cudaIpcOpenMemHandle fails.  Every rank must connect before its first halo exchange (STATE).
 * nxsdg_p2p_connect_local: the same for all ranks' contexts living in this process (tests; each
 *   context on its own stream - ranks then run concurrently and synchronise on the device). */
nxsdg_status nxsdg_p2p_export(nxsdg_ctx* ctx, void* blob, int64_t cap, int64_t* needed);
nxsdg_status nxsdg_p2p_connect(nxsdg_ctx* ctx, const void* lower_blob, const void* upper_blob);
nxsdg_status nxsdg_p2p_connect_local(nxsdg_ctx** ctxs, int32_t n);
/* Link the contexts of a loopback partition (ctxs[r] has rank r), all in this process,
 * all on one device and one stream.  INVALID_ARG otherwise. */
nxsdg_status nxsdg_loopback_connect(nxsdg_ctx** ctxs, int32_t n);
/* Loopback partitions step in lockstep: the same semantics as nxsdg_mevp_substeps /
 * nxsdg_advect on every rank, with the halo rows copied between the contexts
 * (cudaMemcpyAsync) where the NCCL transport would send/recv them. */
nxsdg_status nxsdg_group_mevp_substeps(nxsdg_ctx** ctxs, int32_t n, int32_t n_sub, uint32_t flags);
nxsdg_status nxsdg_group_advect(nxsdg_ctx** ctxs, int32_t n, double dt);

/* Halo-exchange plan (pure host arithmetic; what the NCCL and loopback transports execute).
 * For rank `rank` of a row-strip partition: an ordered list of segments, each a contiguous run of
 * `count` doubles at `offset` doubles from the base of buffer `field` in this rank's local layout
 * (nxsdg_local_geometry).  dir 0 = send to `peer`, 1 = receive from `peer`.  Rank r's k-th send to q
 * pairs with q's k-th receive from r (ncclSend/ncclRecv matching).  With out == NULL only *n_out is
 * set.  INVALID_ARG for a bad partition or max < the plan length. */
typedef enum { NXSDG_HALO_V = 1, NXSDG_HALO_S = 2, NXSDG_HALO_AH = 4, NXSDG_HALO_AH_SCR0 = 8, NXSDG_HALO_AH_SCR1 = 16 } nxsdg_halo_what;
typedef enum { NXSDG_HF_VX = 0, NXSDG_HF_VY = 1, NXSDG_HF_S = 2, NXSDG_HF_A = 3, NXSDG_HF_H = 4, NXSDG_HF_A_SCR0 = 5,
               NXSDG_HF_H_SCR0 = 6, NXSDG_HF_A_SCR1 = 7, NXSDG_HF_H_SCR1 = 8 } nxsdg_halo_field;
typedef struct { int32_t dir, field, peer, plane; int64_t offset, count; } nxsdg_halo_seg;
nxsdg_status nxsdg_halo_plan(int32_t nx, int32_t ny, int32_t cg_degree, int32_t n_stress, int32_t n_adv, int32_t nranks,
                             int32_t rank, uint32_t what, nxsdg_halo_seg* out, int32_t max, int32_t* n_out);
/* Local layout of a rank: out8 = {elem_row0, owned elem rows, ghost rows below (0|1), stored element rows,
 * stored node rows, element row pitch, element plane stride, node row pitch} (element rows and node rows
 * in local numbering start at the ghost row below). */
nxsdg_status nxsdg_local_geometry(int32_t nx, int32_t ny, int32_t cg_degree, int32_t n_stress, int32_t n_adv,
                                  int32_t nranks, int32_t rank, int64_t* out8);

/* ---- introspection ------------------------------------------------------------- */
/* The K0 reference-element tables of degree p (1|2) as built on the device (row a0), flattened:
 * gx[ngp], gw[ngp] (Gauss rule on [0,1]), psi[nd][ng] (DG basis at the Gauss points), phi, dphi/ds,
 * dphi/dt [ncg][ng] (CG basis), mref[nd] (reference DG mass), R[nd][ng] (iMJwPSI of the reference
 * element), Ds, Dt [ncg][nd] (divergence composites); ngp = p+1, ng = ncg = ngp^2, nd = 8 when p = 2
 * and the context has n_S = 8 (R#24), else 6.  With out == NULL only *needed is set. */
nxsdg_status nxsdg_debug_reference_tables(nxsdg_ctx* ctx, int32_t p, double* out, int64_t count, int64_t* needed);
/* Number of kernels this context has launched (for the bench's gpu_launches claim). */
int64_t nxsdg_kernel_launches(const nxsdg_ctx* ctx);
/* Algorithmic HBM bytes per element-subcycle of the fused kernel. */
double nxsdg_bytes_per_element_subcycle(const nxsdg_ctx* ctx);
/* cudaStream_t the context runs on. */
void* nxsdg_stream(const nxsdg_ctx* ctx);
/* One line describing this rank's transport (for the bench's per-rank line): rank, device, transport,
 * P2P neighbours (device, IPC or in-process), whether the P2P waits flush remote writes, whether the
 * fused peer stores and the multi-rank subcycle graph are in use (and why not, if capture was refused).
 * Writes at most cap bytes including the terminating NUL into buf (truncating); returns the full
 * length (excluding NUL), or -1 for a NULL context. */
int64_t nxsdg_transport_info(const nxsdg_ctx* ctx, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* NXSDG_ABI_INCLUDED_H_ */
