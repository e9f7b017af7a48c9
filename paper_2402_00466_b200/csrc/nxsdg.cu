// libnxsdg.so — host runtime and C ABI (include/nxsdg.h).
//
// Owns: the context (partition, padded SoA device buffers, stream), the
// element-matrix precompute (K0), outer-step prep (K0p), the fused subcycle
// kernel and its CUDA-graph replay, the unfused debug steps, DG advection, the
// AoS<->SoA conversion at the ABI, and the row-strip halo exchange (NCCL
// send/recv, or a loopback transport between contexts of one process).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/nxsdg.h"
#include "kernels.cuh"
#include "subcycle_tma.cuh"
#include "subcycle_gen.cuh"
#include "advect_q2.cuh"
#include "advect_tma.cuh"
#include <nvtx3/nvToolsExt.h>     // header-only NVTX v3: ranges for nsys / ncu (--nvtx), no link dependency
#include "prep_q2.cuh"
#include "general_quads.cuh"
#include "general_steps.cuh"

using namespace nxk;

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclFloat64 = 8;

struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (api.loaded) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
                 api.GroupStart && api.GroupEnd;
    return api;
}
}  // namespace

// ---------------------------------------------------------------- context
// Local geometry of one rank's row strip.
struct Geom {
    int nx, ny, P, NS, NA, nranks, rank;
    int64_t r0, r1;
    int glo, ghi, nown, erows_local, nrows_local;
    int64_t epitch, eplane, npitch, nn;
};
static Geom make_geom(int nx, int ny, int p, int ns, int na, int nranks, int rank);

constexpr int kP2PBufs = 12;   // vx0 vx1 vy0 vy1 S0 S1 A H Asc0 Asc1 Hsc0 Hsc1

struct nxsdg_ctx {
    nxsdg_mesh_desc d{};
    nxsdg_params prm{};
    int P = 2, NS = 6, NA = 6, NG = 9;
    // partition
    Geom geom{};
    int64_t r0 = 0, r1 = 0;
    int glo = 0, ghi = 0, nown = 0, erows_local = 0, nrows_local = 0;
    int64_t eplane = 0, npitch = 0, epitch = 0;
    // device buffers
    double* S[2] = {nullptr, nullptr};
    double* Pg = nullptr;
    double* A = nullptr; double* H = nullptr;
    double* Asc[2] = {nullptr, nullptr}; double* Hsc[2] = {nullptr, nullptr};
    double* E = nullptr; double* Fx = nullptr; double* Fy = nullptr;
    double* vx[2] = {nullptr, nullptr}; double* vy[2] = {nullptr, nullptr};
    double *ox = nullptr, *oy = nullptr, *ax = nullptr, *ay = nullptr;
    double *c1 = nullptr, *rx0 = nullptr, *ry0 = nullptr, *cafo = nullptr;
    double* nodec = nullptr;   // one allocation: c1, rx0, ry0, cafo, ox, oy (6 x node grid; one TMA tensor)
    int64_t nn = 0;            // doubles per node grid
    double* staging = nullptr; size_t staging_bytes = 0;
    int cv = 0, cs = 0; // ping-pong index of v and of S
    // state flags
    bool forcing_set = false, prepped = false, poisoned = false;
    cudaStream_t stream = nullptr; bool own_stream = false;
    std::string err;
    int64_t launches = 0;
    int ty = 0;        // fused kernel chunk rows (NXSDG_OPT_CHUNK_ROWS; 0 = automatic: 32, halved down to 4
                       // while the strips x chunks work units are fewer than the resident warps)
    int nsm = 0;       // SM count of the device (cached for the automatic chunk height)
    int variant = 0;   // fused kernel: 0 = TMA-staged structured (p = 2), 1 = table-driven k_subcycle<P>
    int ctas_per_sm = -1;  // -1 = tuned default on C4: 2 (FP64 S, P_g), 4 (FP32 storage)
    int stages = 2;        // TMA pipeline depth 2..4
    int const_regs = -1;   // node constants: 0 = fifth TMA box of the stage, 1 = register prefetch, -1 = default
    int tail_split = 1;    // persistent kernels: split the last chunks into short sub-units (1) or not (0)
    int l2_policy = 2;     // fused TMA kernels: L2 eviction-policy bits (2 = stores evict_first)
    int v_carry = 1;       // box TMA kernel: a unit's next job re-uses the shared v node row from registers
    int adv_kernel = 0;    // NXSDG_OPT_ADVECT_KERNEL: 0 = TMA-staged k_advect_tma where it applies, 1 = k_advect_q2
    int adv_stages = 4;    // NXSDG_OPT_ADVECT_STAGES: slots per warp of k_advect_tma (4 | 5)
    int adv_ty = 32;       // element rows per k_advect_tma work unit
    int fuse_pg = 1;       // NXSDG_OPT_FUSE_PREP_PG: the last k_advect_tma stage also writes P_g (single rank)
    int prep_kernel = 0;   // NXSDG_OPT_PREP_KERNEL: CG2/DG2 prep nodes: 0 = row-marching, 1 = per-element threads,
                           // 2 = in the first fused subcycle where it applies (measured no faster: not the default)
    bool prep_defer = false;   // BEGIN_STEP left the node constants to the next fused subcycle (PREP launch)
    int pair = 0;              // NXSDG_OPT_PAIR_SUBCYCLES: two subcycles per launch (PAIR instantiation)
    bool pair_now = false;     // the next TMA launch is a PAIR launch
    int pdl = 0;               // NXSDG_OPT_PDL: single-rank subcycle graphs launch with programmatic dependence
                               // (measured no faster: profiles/ab_pdl_r02.log)
    bool pdl_now = false;      // the next TMA subcycle launch carries the PDL attribute
    double* Sx = nullptr; double* vxx = nullptr; double* vyx = nullptr;   // PAIR scratch (S^{p+1}, v^{p+1})
    K2Maps mapsP{};            // PAIR pass-B maps over the scratch
    bool mapsP_ok = false;
    bool prep_now = false;     // the next TMA launch is that PREP launch
    bool pg_fresh = false; // P_g already holds P of the current A, H (written by the last advection stage)
    bool adv_last = false; // the advection stage being launched is the last one
    int* counters = nullptr; int ncounters = 0;   // dynamic work counters, one per launch in a graph
    int dynamic = 1;       // TMA kernel work distribution: 1 = atomic counter, 0 = static round-robin
    double* hstage_send = nullptr; double* hstage_recv = nullptr;   // packed halo messages
    double* verts = nullptr; double* gmaps = nullptr;               // NEXT-1 general quads (stress step)
    // NXSDG_MEM_HOST_ASYNC: copies on a copy stream, forcing staged until the next BEGIN_STEP
    cudaStream_t cstream = nullptr;    // HOST_ASYNC host -> device copies (forcing uploads)
    cudaStream_t dstream = nullptr;    // HOST_ASYNC device -> host copies (velocity read-back): PCIe is full
                                       // duplex, so a step's upload and the previous step's read-back overlap
    cudaEvent_t ev_fup = nullptr, ev_fcons = nullptr, ev_vsnap[2] = {nullptr, nullptr}, ev_vdone[2] = {nullptr, nullptr};
    cudaEvent_t ev_cjoin = nullptr, ev_djoin = nullptr;
    double* fstage[4] = {nullptr, nullptr, nullptr, nullptr};
    double* vsnap[2] = {nullptr, nullptr};
    bool fpending = false;
    bool general = false, gmaps_ready = false;
    // NEXT-4 sphere (R#26): lon-lat mesh of radius R, southern edge lat0, element size dlon x dlat [rad]
    bool sphere = false;
    double sph_R = 0.0, sph_lat0 = 0.0, sph_dlon = 0.0, sph_dlat = 0.0;
    double* sph_rows = nullptr;      // kSphRow doubles per local element row
    double* mlump = nullptr; double* imlump = nullptr; double* gcontrib = nullptr;           // general quads: lumped masses, div scratch
    int map_mode = 1;      // 0: iMJwPSI pre-assembled per element, 1: on the fly from the vertices
    cudaStream_t hstream = nullptr;                                 // halo stream (NCCL overlap)
    cudaEvent_t ev_bnd = nullptr, ev_x = nullptr;
    K2Maps maps[2][2]; // [cv][cs]
    bool maps_ok = false;
    K2GenMaps gen_maps[2][2];   // NEXT-1 fused general-quad subcycle: + vertices, lumped masses
    bool gen_maps_ok = false;
    int precision = 0; // 0: FP64 storage; 1 (NEXT-3): S and P_g stored in FP32, arithmetic FP64
    float* S32[2] = {nullptr, nullptr}; float* Pg32 = nullptr;
    K2Maps maps32[2][2];
    bool maps32_ok = false, pg32_ok = false;
    // transport
    ncclComm_t comm = nullptr;
    std::vector<nxsdg_ctx*> peers;   // loopback: all ranks' contexts
    // P2P transport: the exchanged allocations in a fixed order (advection swaps A/H with its
    // scratch buffers, identically on every rank, so a field's current allocation has the same
    // index on both sides), this rank's two flag words and the neighbours' mapped buffers
    double* orig[kP2PBufs] = {};
    uint32_t* flags = nullptr;       // [slot][side]: [2k] written by the lower neighbour, [2k+1] by the upper one
    struct Peer { bool on = false, ipc = false; double* buf[kP2PBufs] = {}; uint32_t* flags = nullptr; Geom g{}; } peer[2];
    uint32_t p2p_seq = 0;            // P2P exchanges so far; exchange k uses flag slot k & 1
    unsigned p2p_wait_flags = 0;     // CU_STREAM_WAIT_VALUE_FLUSH where the device can flush remote writes
    bool p2p_ok = false;
    int mr_graph = -1;               // NXSDG_OPT_MULTIRANK_GRAPH (-1: default by transport)
    bool inproc = false;             // P2P ranks of this process on one device (nxsdg_p2p_connect_local)
    int p2p_fused = 1;               // NXSDG_OPT_P2P_FUSED_STORES
    int limiter = 0;                 // NXSDG_OPT_LIMITER (NEXT-4, R#25)
    // graphs: key = (n_sub, cv, cs + 2 precision + 8 P2P-slot parity + 16 multi-rank)
    struct Graph { cudaGraphExec_t exec; int64_t launches; };
    std::map<std::tuple<int, int, int>, Graph> graphs;
    std::string mr_graph_note;       // why multi-rank capture was given up (empty = in use)
};

static nxsdg_status fail(nxsdg_ctx* c, nxsdg_status s, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap; va_start(ap, fmt); vsnprintf(buf, sizeof buf, fmt, ap); va_end(ap);
        c->err = buf;
        if (s == NXSDG_ERR_CUDA || s == NXSDG_ERR_NCCL) c->poisoned = true;
    }
    return s;
}

#define CU(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return fail(c, NXSDG_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define LAUNCHED()                                                                            \
    do {                                                                                      \
        ++c->launches;                                                                        \
        cudaError_t e_ = cudaGetLastError();                                                  \
        if (e_ != cudaSuccess) return fail(c, NXSDG_ERR_CUDA, "launch: %s", cudaGetErrorString(e_)); \
    } while (0)

static int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// NVTX range for the host span of an API call / exchange (visible on nsys timelines, filterable in ncu)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

extern "C" nxsdg_status nxsdg_partition(int32_t ny, int32_t p, int32_t nranks, int32_t rank, int64_t* er0,
                                        int32_t* erows, int64_t* nr0, int32_t* nrows) {
    if (ny < 1 || nranks < 1 || nranks > ny || rank < 0 || rank >= nranks || (p != 1 && p != 2))
        return NXSDG_ERR_INVALID_ARG;
    int64_t base = ny / nranks, rem = ny % nranks;
    int64_t r0 = rank * base + std::min<int64_t>(rank, rem);
    int64_t n = base + (rank < rem ? 1 : 0);
    if (er0) *er0 = r0;
    if (erows) *erows = (int32_t)n;
    if (nr0) *nr0 = p * r0;
    if (nrows) *nrows = (int32_t)(p * n + (rank == nranks - 1 ? 1 : 0));
    return NXSDG_OK;
}

extern "C" int32_t nxsdg_abi_version(void) { return NXSDG_ABI_VERSION; }

static nxsdg_status check_params(nxsdg_ctx* c, const nxsdg_params* p) {
    if (!p) return fail(c, NXSDG_ERR_INVALID_ARG, "params is NULL");
    if (!(p->alpha > 1.0) || !(p->beta > 0.0) || !(p->dt > 0.0) || !(p->rho_ice > 0.0) || !(p->DeltaMin > 0.0) ||
        p->Pstar < 0.0)
        return fail(c, NXSDG_ERR_INVALID_ARG, "params out of range (alpha>1, beta>0, dt>0, rho_ice>0, DeltaMin>0, Pstar>=0)");
    return NXSDG_OK;
}

static nxsdg_status alloc(nxsdg_ctx* c, double** p, size_t n) {
    cudaError_t e = cudaMalloc((void**)p, n * sizeof(double));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, e == cudaErrorMemoryAllocation ? NXSDG_ERR_OOM : NXSDG_ERR_CUDA, "cudaMalloc(%zu doubles): %s", n,
                    cudaGetErrorString(e));
    }
    e = cudaMemsetAsync(*p, 0, n * sizeof(double), c->stream);
    if (e != cudaSuccess) return fail(c, NXSDG_ERR_CUDA, "cudaMemset: %s", cudaGetErrorString(e));
    return NXSDG_OK;
}

// Destroy the cached subcycle graphs (their captured launch arguments went stale); a replay may
// still be in flight on the stream, so wait for it first.
static void drop_graphs(nxsdg_ctx* c) {
    if (c->graphs.empty()) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second.exec);
    c->graphs.clear();
}

static void free_all(nxsdg_ctx* c) {
    drop_graphs(c);
    for (auto& pr : c->peer) {
        if (pr.ipc) {
            for (double* b : pr.buf) if (b) cudaIpcCloseMemHandle(b);
            if (pr.flags) cudaIpcCloseMemHandle(pr.flags);
        }
        pr = nxsdg_ctx::Peer{};
    }
    if (c->flags) { cudaFree(c->flags); c->flags = nullptr; }
    double** bufs[] = {&c->S[0], &c->S[1], &c->Pg, &c->A, &c->H, &c->Asc[0], &c->Asc[1], &c->Hsc[0], &c->Hsc[1],
                       &c->E, &c->Fx, &c->Fy, &c->vx[0], &c->vx[1], &c->vy[0], &c->vy[1],
                       &c->ax, &c->ay, &c->nodec, &c->staging};
    for (auto b : bufs)
        if (*b) { cudaFree(*b); *b = nullptr; }
    if (c->counters) { cudaFree(c->counters); c->counters = nullptr; c->ncounters = 0; }
    for (int k = 0; k < 2; ++k) if (c->S32[k]) { cudaFree(c->S32[k]); c->S32[k] = nullptr; }
    if (c->Pg32) { cudaFree(c->Pg32); c->Pg32 = nullptr; }
    if (c->hstage_send) { cudaFree(c->hstage_send); c->hstage_send = nullptr; }
    if (c->verts) { cudaFree(c->verts); c->verts = nullptr; }
    if (c->sph_rows) { cudaFree(c->sph_rows); c->sph_rows = nullptr; }
    for (int k = 0; k < 4; ++k) if (c->fstage[k]) { cudaFree(c->fstage[k]); c->fstage[k] = nullptr; }
    for (int k = 0; k < 2; ++k) {
        if (c->vsnap[k]) { cudaFree(c->vsnap[k]); c->vsnap[k] = nullptr; }
        if (c->ev_vsnap[k]) { cudaEventDestroy(c->ev_vsnap[k]); c->ev_vsnap[k] = nullptr; }
        if (c->ev_vdone[k]) { cudaEventDestroy(c->ev_vdone[k]); c->ev_vdone[k] = nullptr; }
    }
    if (c->ev_fup) { cudaEventDestroy(c->ev_fup); c->ev_fup = nullptr; }
    if (c->ev_fcons) { cudaEventDestroy(c->ev_fcons); c->ev_fcons = nullptr; }
    if (c->ev_cjoin) { cudaEventDestroy(c->ev_cjoin); c->ev_cjoin = nullptr; }
    if (c->ev_djoin) { cudaEventDestroy(c->ev_djoin); c->ev_djoin = nullptr; }
    if (c->cstream) { cudaStreamDestroy(c->cstream); c->cstream = nullptr; }
    if (c->dstream) { cudaStreamDestroy(c->dstream); c->dstream = nullptr; }
    if (c->gmaps) { cudaFree(c->gmaps); c->gmaps = nullptr; }
    if (c->mlump) { cudaFree(c->mlump); c->mlump = nullptr; }
    if (c->imlump) { cudaFree(c->imlump); c->imlump = nullptr; }
    if (c->Sx) { cudaFree(c->Sx); c->Sx = nullptr; }
    if (c->vxx) { cudaFree(c->vxx); c->vxx = nullptr; }
    if (c->vyx) { cudaFree(c->vyx); c->vyx = nullptr; }
    if (c->gcontrib) { cudaFree(c->gcontrib); c->gcontrib = nullptr; }
    if (c->hstage_recv) { cudaFree(c->hstage_recv); c->hstage_recv = nullptr; }
    if (c->ev_bnd) { cudaEventDestroy(c->ev_bnd); c->ev_bnd = nullptr; }
    if (c->ev_x) { cudaEventDestroy(c->ev_x); c->ev_x = nullptr; }
    if (c->hstream) { cudaStreamDestroy(c->hstream); c->hstream = nullptr; }
    c->c1 = c->rx0 = c->ry0 = c->cafo = c->ox = c->oy = nullptr;
}

extern "C" nxsdg_status nxsdg_create_mesh(const nxsdg_mesh_desc* d, const nxsdg_params* prm, nxsdg_ctx** out) {
    if (!d || !prm || !out) return NXSDG_ERR_INVALID_ARG;
    *out = nullptr;
    if (d->nx < 1 || d->ny < 1 || !(d->lx > 0) || !(d->ly > 0)) return NXSDG_ERR_INVALID_ARG;
    if (d->nranks < 1 || d->nranks > d->ny || d->rank < 0 || d->rank >= d->nranks) return NXSDG_ERR_INVALID_ARG;
    if (d->bc != NXSDG_BC_CLOSED && d->bc != NXSDG_BC_PERIODIC) return NXSDG_ERR_INVALID_ARG;
    bool ok_deg = (d->cg_degree == 1 && d->n_stress == 3 && (d->n_adv == 1 || d->n_adv == 3)) ||
                  (d->cg_degree == 2 && (d->n_stress == 6 || d->n_stress == 8) &&
                   (d->n_adv == 1 || d->n_adv == 3 || d->n_adv == 6));
    if (!ok_deg) return NXSDG_ERR_UNSUPPORTED;
    if (d->bc == NXSDG_BC_PERIODIC && d->nranks > 1) return NXSDG_ERR_UNSUPPORTED;
    if (d->nranks > 1 && d->transport != NXSDG_TRANSPORT_NCCL && d->transport != NXSDG_TRANSPORT_LOOPBACK &&
        d->transport != NXSDG_TRANSPORT_P2P)
        return NXSDG_ERR_INVALID_ARG;
    if (d->transport == NXSDG_TRANSPORT_NCCL && d->nranks > 1 && !d->nccl_id) return NXSDG_ERR_INVALID_ARG;
    if (!(prm->alpha > 1.0) || !(prm->beta > 0.0) || !(prm->dt > 0.0) || !(prm->rho_ice > 0.0) ||
        !(prm->DeltaMin > 0.0) || prm->Pstar < 0.0)
        return NXSDG_ERR_INVALID_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { cudaGetLastError(); return NXSDG_ERR_CUDA; }
    if (d->device < 0 || d->device >= ndev) return NXSDG_ERR_INVALID_ARG;

    nxsdg_ctx* c = new nxsdg_ctx();
    c->d = *d; c->prm = *prm;
    c->P = d->cg_degree; c->NS = d->n_stress; c->NA = d->n_adv; c->NG = (c->P + 1) * (c->P + 1);
    c->geom = make_geom(d->nx, d->ny, c->P, c->NS, c->NA, d->nranks, d->rank);
    c->r0 = c->geom.r0; c->r1 = c->geom.r1; c->nown = c->geom.nown;
    c->glo = c->geom.glo; c->ghi = c->geom.ghi;
    c->erows_local = c->geom.erows_local; c->nrows_local = c->geom.nrows_local;
    c->epitch = c->geom.epitch; c->eplane = c->geom.eplane; c->npitch = c->geom.npitch;
    auto bail = [&](nxsdg_status s) { nxsdg_status r = s; free_all(c); if (c->own_stream) cudaStreamDestroy(c->stream); delete c; return r; };
    if (cudaSetDevice(d->device) != cudaSuccess) { cudaGetLastError(); return bail(NXSDG_ERR_CUDA); }
    cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, d->device);
    if (d->stream) c->stream = (cudaStream_t)d->stream;
    else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(NXSDG_ERR_CUDA);
        c->own_stream = true;
    }
    const size_t ne = (size_t)c->eplane, nn = (size_t)c->npitch * c->nrows_local;
    nxsdg_status s;
#define AL(ptr, n) if ((s = alloc(c, &(ptr), (n))) != NXSDG_OK) return bail(s)
    AL(c->S[0], 3 * c->NS * ne); AL(c->S[1], 3 * c->NS * ne);
    AL(c->Pg, c->NG * ne);
    AL(c->A, c->NA * ne); AL(c->H, c->NA * ne);
    AL(c->Asc[0], c->NA * ne); AL(c->Asc[1], c->NA * ne); AL(c->Hsc[0], c->NA * ne); AL(c->Hsc[1], c->NA * ne);
    AL(c->vx[0], nn); AL(c->vx[1], nn); AL(c->vy[0], nn); AL(c->vy[1], nn);
    AL(c->ax, nn); AL(c->ay, nn);
    AL(c->nodec, 6 * nn);
    c->nn = (int64_t)nn;
    c->c1 = c->nodec; c->rx0 = c->nodec + nn; c->ry0 = c->nodec + 2 * nn; c->cafo = c->nodec + 3 * nn;
    c->ox = c->nodec + 4 * nn; c->oy = c->nodec + 5 * nn;
    {
        double* const o[kP2PBufs] = {c->vx[0], c->vx[1], c->vy[0], c->vy[1], c->S[0], c->S[1],
                                     c->A, c->H, c->Asc[0], c->Asc[1], c->Hsc[0], c->Hsc[1]};
        std::copy(o, o + kP2PBufs, c->orig);
    }
    if (d->nranks > 1 && d->transport == NXSDG_TRANSPORT_P2P) {
        if (cudaMalloc(&c->flags, 4 * sizeof(uint32_t)) != cudaSuccess) return bail(NXSDG_ERR_OOM);
        if (cudaMemset(c->flags, 0, 4 * sizeof(uint32_t)) != cudaSuccess) return bail(NXSDG_ERR_CUDA);
    }
#undef AL
    // K0: reference-element tables into __constant__ (all three spaces; tiny)
    {
        RefTab* dtab = nullptr;
        if (cudaMalloc(&dtab, sizeof(RefTab)) != cudaSuccess) return bail(NXSDG_ERR_OOM);
        cudaMemsetAsync(dtab, 0, sizeof(RefTab), c->stream);   // struct padding is never written by K0
        const int spaces[3][2] = {{1, 3}, {2, 6}, {2, 8}};
        for (const auto& sp : spaces) {
            k_build_tables<<<1, 32, 0, c->stream>>>(dtab, sp[0], sp[1]);
            ++c->launches;
            if (cudaMemcpyToSymbolAsync(c_tab, dtab, sizeof(RefTab), tab_index(sp[0], sp[1]) * sizeof(RefTab),
                                        cudaMemcpyDeviceToDevice, c->stream) != cudaSuccess) {
                cudaFree(dtab); return bail(NXSDG_ERR_CUDA);
            }
        }
        cudaError_t e = cudaStreamSynchronize(c->stream);
        cudaFree(dtab);
        if (e != cudaSuccess) return bail(NXSDG_ERR_CUDA);
    }
    if (d->nranks > 1 && d->transport == NXSDG_TRANSPORT_NCCL) {
        NcclApi& api = nccl();
        if (!api.loaded) return bail(NXSDG_ERR_NCCL);
        ncclUniqueId id; memcpy(&id, d->nccl_id, sizeof id);
        if (api.CommInitRank(&c->comm, d->nranks, id, d->rank) != 0) return bail(NXSDG_ERR_NCCL);
    }
    *out = c;
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_destroy(nxsdg_ctx* c) {
    if (!c) return NXSDG_ERR_INVALID_ARG;
    cudaSetDevice(c->d.device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm) { nccl().CommDestroy(c->comm); c->comm = nullptr; }
    free_all(c);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return NXSDG_OK;
}

extern "C" const char* nxsdg_last_error(const nxsdg_ctx* c) { return c ? c->err.c_str() : "null context"; }
extern "C" int64_t nxsdg_kernel_launches(const nxsdg_ctx* c) { return c ? c->launches : -1; }
extern "C" void* nxsdg_stream(const nxsdg_ctx* c) { return c ? (void*)c->stream : nullptr; }

static bool pair_ok(const nxsdg_ctx* c);
extern "C" double nxsdg_bytes_per_element_subcycle(const nxsdg_ctx* c) {
    if (!c) return 0.0;
    // NXSDG_OPT_PAIR_SUBCYCLES: one DRAM pass (the same bytes) per two subcycles
    if (c->pair && pair_ok(c)) return 4.0 * (2 * c->P * c->P + 6.0 * c->NS + c->NG + 8.0 * c->P * c->P);
    // one fused pass: v gather P^2*2, S read+write 2*3NS, P_g NG,
    // per node (P^2 per element): 6 constants + v write 2
    const double p2 = (double)c->P * c->P;
    if (c->general) return 8.0 * (2 * p2 + 6.0 * c->NS + c->NG + 8.0 * p2) + 8.0 * (2.0 + p2);   // + vertex, lumped masses
    if (c->precision >= 1) return 8.0 * (2 * p2 + 8.0 * p2) + 4.0 * (6.0 * c->NS + c->NG);   // S, P_g in FP32
    return 8.0 * (2 * p2 + 6.0 * c->NS + c->NG + 8.0 * p2);
}

extern "C" nxsdg_status nxsdg_get_partition(const nxsdg_ctx* c, int64_t* er0, int32_t* erows, int64_t* nr0,
                                            int32_t* nrows) {
    if (!c) return NXSDG_ERR_INVALID_ARG;
    return nxsdg_partition(c->d.ny, c->P, c->d.nranks, c->d.rank, er0, erows, nr0, nrows);
}

#define GUARD(c)                                                                   \
    do {                                                                           \
        if (!(c)) return NXSDG_ERR_INVALID_ARG;                                    \
        if ((c)->poisoned) return NXSDG_ERR_STATE;                                 \
        if (cudaSetDevice((c)->d.device) != cudaSuccess) return fail(c, NXSDG_ERR_CUDA, "cudaSetDevice"); \
    } while (0)

extern "C" nxsdg_status nxsdg_set_params(nxsdg_ctx* c, const nxsdg_params* p) {
    GUARD(c);
    nxsdg_status s = check_params(c, p);
    if (s) return s;
    c->prm = *p;
    c->prepped = false; c->prep_defer = false;
    c->pg_fresh = false;   // P depends on P*, C
    drop_graphs(c);   // captured launch arguments are stale
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_set_option(nxsdg_ctx* c, int32_t opt, int64_t value) {
    GUARD(c);
    switch (opt) {
        case NXSDG_OPT_FUSED_KERNEL:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "fused kernel variant 0|1");
            c->variant = (int)value; break;
        case NXSDG_OPT_CHUNK_ROWS:
            if (value < 0 || value > (1 << 20)) return fail(c, NXSDG_ERR_INVALID_ARG, "chunk rows >= 1 (0 = automatic)");
            c->ty = (int)value; break;
        case NXSDG_OPT_CTAS_PER_SM:
            if (value < -1 || value > 32) return fail(c, NXSDG_ERR_INVALID_ARG, "ctas per SM -1..32");
            c->ctas_per_sm = (int)value; break;
        case NXSDG_OPT_DYNAMIC:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "dynamic 0|1");
            c->dynamic = (int)value; break;
        case NXSDG_OPT_PRECISION:
            if (value < 0 || value > 2) return fail(c, NXSDG_ERR_INVALID_ARG, "precision 0|1|2");
            if (value >= 1 && (c->P != 2 || c->NS != 6 || c->d.nranks != 1 || c->general || c->sphere))
                return fail(c, NXSDG_ERR_UNSUPPORTED, "FP32 storage: CG2/DG2 (n_S = 6), single rank, plane box");
            if (value >= 1 && c->stages > 3) c->stages = 3;
            c->precision = (int)value; c->pg32_ok = false; break;
        case NXSDG_OPT_MAP_MODE:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "map mode 0|1");
            c->map_mode = (int)value; break;
        case NXSDG_OPT_LIMITER:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "limiter 0|1");
            c->limiter = (int)value; break;
        case NXSDG_OPT_P2P_FUSED_STORES:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "p2p fused stores 0|1");
            c->p2p_fused = (int)value; break;
        case NXSDG_OPT_STAGES:
            if (value < 2 || value > 4) return fail(c, NXSDG_ERR_INVALID_ARG, "stages 2..4");
            if (value > 3 && c->precision >= 1) return fail(c, NXSDG_ERR_INVALID_ARG, "stages 2..3 with FP32 storage");
            c->stages = (int)value; break;
        case NXSDG_OPT_V_ROW_CARRY:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "v row carry 0|1");
            c->v_carry = (int)value; break;
        case NXSDG_OPT_L2_POLICY:
            if (value < 0 || value > 7) return fail(c, NXSDG_ERR_INVALID_ARG, "L2 policy bits 0..7");
            c->l2_policy = (int)value; break;
        case NXSDG_OPT_TAIL_SPLIT:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "tail split 0|1");
            c->tail_split = (int)value; break;
        case NXSDG_OPT_CONST_STAGING:
            if (value < -1 || value > 2) return fail(c, NXSDG_ERR_INVALID_ARG, "node-constant staging -1|0|1|2");
            c->const_regs = (int)value; break;
        case NXSDG_OPT_ADVECT_KERNEL:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "advect kernel 0|1");
            c->adv_kernel = (int)value; break;
        case NXSDG_OPT_ADVECT_STAGES:
            if (value < 3 || value > 5) return fail(c, NXSDG_ERR_INVALID_ARG, "advect stages 3|4|5");
            c->adv_stages = (int)value; break;
        case NXSDG_OPT_FUSE_PREP_PG:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "fuse prep P_g 0|1");
            c->fuse_pg = (int)value; break;
        case NXSDG_OPT_PREP_KERNEL:
            if (value < 0 || value > 2) return fail(c, NXSDG_ERR_INVALID_ARG, "prep kernel 0|1|2");
            c->prep_kernel = (int)value; break;
        case NXSDG_OPT_PDL:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "pdl 0|1");
            c->pdl = (int)value; break;
        case NXSDG_OPT_PAIR_SUBCYCLES:
            if (value != 0 && value != 1) return fail(c, NXSDG_ERR_INVALID_ARG, "pair subcycles 0|1");
            c->pair = (int)value; break;
        case NXSDG_OPT_MULTIRANK_GRAPH:
            if (value < -1 || value > 1) return fail(c, NXSDG_ERR_INVALID_ARG, "multi-rank graph -1|0|1");
            c->mr_graph = (int)value; break;
        default: return fail(c, NXSDG_ERR_INVALID_ARG, "unknown option %d", opt);
    }
    c->pg_fresh = false;
    drop_graphs(c);
    return NXSDG_OK;
}

// ---------------------------------------------------------------- state I/O
static bool is_dg(nxsdg_field f) {
    return f == NXSDG_S11 || f == NXSDG_S12 || f == NXSDG_S22 || f == NXSDG_A || f == NXSDG_H || f == NXSDG_E11 ||
           f == NXSDG_E12 || f == NXSDG_E22;
}

static int64_t owned_node_rows(const nxsdg_ctx* c) {
    return (int64_t)c->P * c->nown + (c->r1 == c->d.ny ? 1 : 0);
}

// device pointer of plane 0 of a DG field and its coefficient count
static double* dg_base(nxsdg_ctx* c, nxsdg_field f, int* n) {
    switch (f) {
        case NXSDG_S11: *n = c->NS; return c->S[c->cs];
        case NXSDG_S12: *n = c->NS; return c->S[c->cs] + (size_t)c->NS * c->eplane;
        case NXSDG_S22: *n = c->NS; return c->S[c->cs] + (size_t)2 * c->NS * c->eplane;
        case NXSDG_A: *n = c->NA; return c->A;
        case NXSDG_H: *n = c->NA; return c->H;
        case NXSDG_E11: *n = c->NS; return c->E;
        case NXSDG_E12: *n = c->NS; return c->E ? c->E + (size_t)c->NS * c->eplane : nullptr;
        case NXSDG_E22: *n = c->NS; return c->E ? c->E + (size_t)2 * c->NS * c->eplane : nullptr;
        default: *n = 0; return nullptr;
    }
}
static double* cg_base(nxsdg_ctx* c, nxsdg_field f) {
    switch (f) {
        case NXSDG_VX: return c->vx[c->cv];
        case NXSDG_VY: return c->vy[c->cv];
        case NXSDG_FX: return c->Fx;
        case NXSDG_FY: return c->Fy;
        default: return nullptr;
    }
}

static nxsdg_status ensure_staging(nxsdg_ctx* c, size_t bytes) {
    if (c->staging_bytes >= bytes) return NXSDG_OK;
    if (c->staging) { cudaFree(c->staging); c->staging = nullptr; c->staging_bytes = 0; }
    cudaError_t e = cudaMalloc((void**)&c->staging, bytes);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(c, NXSDG_ERR_OOM, "staging alloc %zu B", bytes); }
    c->staging_bytes = bytes;
    return NXSDG_OK;
}

static nxsdg_status ensure_debug_buffers(nxsdg_ctx* c) {
    nxsdg_status s;
    const size_t nn = (size_t)c->npitch * c->nrows_local;
    if (!c->E && (s = alloc(c, &c->E, 3 * (size_t)c->NS * c->eplane))) return s;
    if (!c->Fx && (s = alloc(c, &c->Fx, nn))) return s;
    if (!c->Fy && (s = alloc(c, &c->Fy, nn))) return s;
    return NXSDG_OK;
}

static nxsdg_status copy_in_nodes(nxsdg_ctx* c, double* dst, const double* src, int64_t count, nxsdg_mem mem) {
    const int64_t rows = owned_node_rows(c), cols = (int64_t)c->P * c->d.nx + 1;
    if (count != rows * cols) return fail(c, NXSDG_ERR_INVALID_ARG, "count %lld != %lld nodes", (long long)count, (long long)(rows * cols));
    double* d0 = dst + (size_t)c->P * c->glo * c->npitch;
    CU(cudaMemcpy2DAsync(d0, c->npitch * sizeof(double), src, cols * sizeof(double), cols * sizeof(double), rows,
                         mem == NXSDG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->stream));
    if (mem == NXSDG_MEM_HOST) CU(cudaStreamSynchronize(c->stream));
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_write_state(nxsdg_ctx* c, nxsdg_field f, const double* src, int64_t count, nxsdg_mem mem) {
    GUARD(c);
    if (!src || (mem != NXSDG_MEM_HOST && mem != NXSDG_MEM_DEVICE) || f < 0 || f >= NXSDG_NFIELDS)
        return fail(c, NXSDG_ERR_INVALID_ARG, "bad argument");
    if (f == NXSDG_FX || f == NXSDG_FY || f == NXSDG_E11 || f == NXSDG_E12 || f == NXSDG_E22) {
        nxsdg_status s = ensure_debug_buffers(c);
        if (s) return s;
    }
    if (is_dg(f)) {
        int n = 0;
        double* base = dg_base(c, f, &n);
        const int64_t ne = (int64_t)c->nown * c->d.nx;
        if (count != ne * n) return fail(c, NXSDG_ERR_INVALID_ARG, "count %lld != %lld", (long long)count, (long long)(ne * n));
        const double* dsrc = src;
        if (mem == NXSDG_MEM_HOST) {
            nxsdg_status s = ensure_staging(c, count * sizeof(double));
            if (s) return s;
            CU(cudaMemcpyAsync(c->staging, src, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            dsrc = c->staging;
        }
        const int64_t tot = ne * n;
        k_aos_to_soa<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(dsrc, base, ne, n, c->eplane,
                                                                         (int64_t)c->glo, c->d.nx, c->epitch);
        LAUNCHED();
        if (mem == NXSDG_MEM_HOST) CU(cudaStreamSynchronize(c->stream));
    } else {
        nxsdg_status s = copy_in_nodes(c, cg_base(c, f), src, count, mem);
        if (s) return s;
    }
    c->prepped = false; c->prep_defer = false;
    c->pg_fresh = false;
    return NXSDG_OK;
}

static nxsdg_status ensure_async(nxsdg_ctx* c);

extern "C" nxsdg_status nxsdg_read_state(nxsdg_ctx* c, nxsdg_field f, double* dst, int64_t count, nxsdg_mem mem) {
    GUARD(c);
    if (mem == NXSDG_MEM_HOST_ASYNC) {
        if (!dst || (f != NXSDG_VX && f != NXSDG_VY)) return fail(c, NXSDG_ERR_INVALID_ARG, "HOST_ASYNC reads: vx, vy");
        const int64_t rows = owned_node_rows(c), cols = (int64_t)c->P * c->d.nx + 1;
        if (count != rows * cols) return fail(c, NXSDG_ERR_INVALID_ARG, "count mismatch");
        nxsdg_status s = ensure_async(c);
        if (s) return s;
        const int k = f == NXSDG_VX ? 0 : 1;
        const size_t nn = (size_t)c->npitch * c->nrows_local;
        if (!c->vsnap[k] && (s = alloc(c, &c->vsnap[k], nn))) return s;
        // snapshot on the context stream (after the work issued so far), D2H on the copy stream
        CU(cudaStreamWaitEvent(c->stream, c->ev_vdone[k], 0));
        CU(cudaMemcpyAsync(c->vsnap[k], cg_base(c, f), nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CU(cudaEventRecord(c->ev_vsnap[k], c->stream));
        CU(cudaStreamWaitEvent(c->dstream, c->ev_vsnap[k], 0));
        CU(cudaMemcpy2DAsync(dst, cols * sizeof(double), c->vsnap[k] + (size_t)c->P * c->glo * c->npitch,
                             c->npitch * sizeof(double), cols * sizeof(double), rows, cudaMemcpyDeviceToHost, c->dstream));
        CU(cudaEventRecord(c->ev_vdone[k], c->dstream));
        return NXSDG_OK;
    }
    if (!dst || (mem != NXSDG_MEM_HOST && mem != NXSDG_MEM_DEVICE) || f < 0 || f >= NXSDG_NFIELDS)
        return fail(c, NXSDG_ERR_INVALID_ARG, "bad argument");
    if (is_dg(f)) {
        int n = 0;
        double* base = dg_base(c, f, &n);
        if (!base) return fail(c, NXSDG_ERR_STATE, "field not computed yet");
        const int64_t ne = (int64_t)c->nown * c->d.nx;
        if (count != ne * n) return fail(c, NXSDG_ERR_INVALID_ARG, "count %lld != %lld", (long long)count, (long long)(ne * n));
        double* ddst = dst;
        if (mem == NXSDG_MEM_HOST) {
            nxsdg_status s = ensure_staging(c, count * sizeof(double));
            if (s) return s;
            ddst = c->staging;
        }
        const int64_t tot = ne * n;
        k_soa_to_aos<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(base, ddst, ne, n, c->eplane,
                                                                          (int64_t)c->glo, c->d.nx, c->epitch);
        LAUNCHED();
        if (mem == NXSDG_MEM_HOST) {
            CU(cudaMemcpyAsync(dst, c->staging, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            CU(cudaStreamSynchronize(c->stream));
        }
    } else {
        double* base = cg_base(c, f);
        if (!base) return fail(c, NXSDG_ERR_STATE, "field not computed yet");
        const int64_t rows = owned_node_rows(c), cols = (int64_t)c->P * c->d.nx + 1;
        if (count != rows * cols) return fail(c, NXSDG_ERR_INVALID_ARG, "count mismatch");
        CU(cudaMemcpy2DAsync(dst, cols * sizeof(double), base + (size_t)c->P * c->glo * c->npitch,
                             c->npitch * sizeof(double), cols * sizeof(double), rows,
                             mem == NXSDG_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream));
        if (mem == NXSDG_MEM_HOST) CU(cudaStreamSynchronize(c->stream));
    }
    return NXSDG_OK;
}

static nxsdg_status ensure_async(nxsdg_ctx* c) {
    if (c->cstream) return NXSDG_OK;
    CU(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&c->dstream, cudaStreamNonBlocking));
    cudaEvent_t* evs[] = {&c->ev_fup, &c->ev_fcons, &c->ev_vsnap[0], &c->ev_vsnap[1], &c->ev_vdone[0], &c->ev_vdone[1],
                          &c->ev_cjoin, &c->ev_djoin};
    for (auto e : evs) CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    return NXSDG_OK;
}

// BEGIN_STEP: bring a staged (HOST_ASYNC) forcing into place on the context stream
static nxsdg_status consume_forcing(nxsdg_ctx* c) {
    if (!c->fpending) return NXSDG_OK;
    CU(cudaStreamWaitEvent(c->stream, c->ev_fup, 0));
    const size_t bytes = (size_t)c->npitch * c->nrows_local * sizeof(double);
    CU(cudaMemcpyAsync(c->ox, c->fstage[0], bytes, cudaMemcpyDeviceToDevice, c->stream));   // o lives in the
    CU(cudaMemcpyAsync(c->oy, c->fstage[1], bytes, cudaMemcpyDeviceToDevice, c->stream));   // node-constant tensor
    std::swap(c->ax, c->fstage[2]);
    std::swap(c->ay, c->fstage[3]);
    CU(cudaEventRecord(c->ev_fcons, c->stream));
    c->fpending = false;
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_stream_join(nxsdg_ctx* c) {
    GUARD(c);
    if (!c->cstream) return NXSDG_OK;
    CU(cudaEventRecord(c->ev_cjoin, c->cstream));
    CU(cudaStreamWaitEvent(c->stream, c->ev_cjoin, 0));
    CU(cudaEventRecord(c->ev_djoin, c->dstream));
    CU(cudaStreamWaitEvent(c->stream, c->ev_djoin, 0));
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_set_forcing(nxsdg_ctx* c, const double* ox, const double* oy, const double* ax,
                                          const double* ay, int64_t count, nxsdg_mem mem) {
    GUARD(c);
    if (!ox || !oy || !ax || !ay || (mem != NXSDG_MEM_HOST && mem != NXSDG_MEM_DEVICE && mem != NXSDG_MEM_HOST_ASYNC))
        return fail(c, NXSDG_ERR_INVALID_ARG, "bad argument");
    const int64_t need = owned_node_rows(c) * ((int64_t)c->P * c->d.nx + 1);
    if (count != need) return fail(c, NXSDG_ERR_INVALID_ARG, "count %lld != %lld", (long long)count, (long long)need);
    nxsdg_status s;
    if (mem == NXSDG_MEM_HOST_ASYNC) {
        if ((s = ensure_async(c))) return s;
        const size_t nn = (size_t)c->npitch * c->nrows_local;
        for (int k = 0; k < 4; ++k)
            if (!c->fstage[k]) {
                if ((s = alloc(c, &c->fstage[k], nn))) return s;
            }
        CU(cudaStreamWaitEvent(c->cstream, c->ev_fcons, 0));   // the previous staging has been consumed
        const double* src[4] = {ox, oy, ax, ay};
        const int64_t rows = owned_node_rows(c), cols = (int64_t)c->P * c->d.nx + 1;
        for (int k = 0; k < 4; ++k)
            CU(cudaMemcpy2DAsync(c->fstage[k] + (size_t)c->P * c->glo * c->npitch, c->npitch * sizeof(double), src[k],
                                 cols * sizeof(double), cols * sizeof(double), rows, cudaMemcpyHostToDevice, c->cstream));
        CU(cudaEventRecord(c->ev_fup, c->cstream));
        c->fpending = true;
        c->forcing_set = true;
        c->prepped = false; c->prep_defer = false;
        return NXSDG_OK;
    }
    c->fpending = false;
    if ((s = copy_in_nodes(c, c->ox, ox, count, mem))) return s;
    if ((s = copy_in_nodes(c, c->oy, oy, count, mem))) return s;
    if ((s = copy_in_nodes(c, c->ax, ax, count, mem))) return s;
    if ((s = copy_in_nodes(c, c->ay, ay, count, mem))) return s;
    c->forcing_set = true;
    c->prepped = false; c->prep_defer = false;
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_set_forcing_cyclone(nxsdg_ctx* c, double t) {
    GUARD(c);
    if (!(t == t)) return fail(c, NXSDG_ERR_INVALID_ARG, "t is NaN");
    ForcingArgs a{};
    a.ox = c->ox; a.oy = c->oy; a.ax = c->ax; a.ay = c->ay;
    a.npitch = c->npitch; a.ncols = c->P * c->d.nx + 1;
    a.row_begin = c->P * c->glo; a.row_end = (int)(c->P * c->glo + owned_node_rows(c));
    a.global_row0 = (int)(c->P * (c->r0 - c->glo));
    a.dxn = c->d.lx / c->d.nx / c->P; a.dyn = c->d.ly / c->d.ny / c->P;
    a.lx = c->d.lx; a.ly = c->d.ly; a.t = t;
    dim3 b(128), g((unsigned)((a.ncols + 127) / 128), (unsigned)(a.row_end - a.row_begin));
    k_cyclone_forcing<<<g, b, 0, c->stream>>>(a);
    LAUNCHED();
    c->forcing_set = true;
    c->prepped = false; c->prep_defer = false;
    return NXSDG_OK;
}

// ---------------------------------------------------------------- NEXT-1: general quads (stress step)
static nxsdg_status ensure_debug_buffers(nxsdg_ctx* c);

static GenStepArgs gen_step_args(nxsdg_ctx* c) {
    GenStepArgs a{};
    a.verts = c->verts;
    a.vx_in = c->vx[c->cv]; a.vy_in = c->vy[c->cv]; a.vx_out = c->vx[c->cv ^ 1]; a.vy_out = c->vy[c->cv ^ 1];
    a.S = c->S[c->cs]; a.E = c->E; a.Fx = c->Fx; a.Fy = c->Fy; a.contrib = c->gcontrib; a.mlump = c->mlump; a.imlump = c->imlump;
    a.H = c->H; a.A = c->A;
    a.c1 = c->c1; a.rx0 = c->rx0; a.ry0 = c->ry0; a.cafo = c->cafo; a.ox = c->ox; a.oy = c->oy;
    a.eplane = c->eplane; a.epitch = c->epitch; a.npitch = c->npitch; a.nx = c->d.nx; a.ny = c->d.ny;
    a.beta = c->prm.beta; a.b1 = 1.0 + c->prm.beta; a.kc = c->prm.dt * c->prm.f_c;
    return a;
}

// one unfused step on the general mesh (strain / divergence / velocity; stress is general_stress)
static nxsdg_status general_step(nxsdg_ctx* c, nxsdg_step st) {
    GenStepArgs a = gen_step_args(c);
    dim3 be(128), ge((unsigned)((c->d.nx + 127) / 128), (unsigned)c->d.ny);
    dim3 bn(128), gn((unsigned)((c->P * c->d.nx + 1 + 127) / 128), (unsigned)(c->P * c->d.ny + 1));
    const bool p1 = c->P == 1;
    switch (st) {
        case NXSDG_STEP_STRAIN:
            if (p1) k_strain_gen<1><<<ge, be, 0, c->stream>>>(a); else k_strain_gen<2><<<ge, be, 0, c->stream>>>(a);
            break;
        case NXSDG_STEP_DIVERGENCE:
            if (p1) k_div_contrib_gen<1><<<ge, be, 0, c->stream>>>(a); else k_div_contrib_gen<2><<<ge, be, 0, c->stream>>>(a);
            LAUNCHED();
            if (p1) k_div_gather_gen<1><<<gn, bn, 0, c->stream>>>(a); else k_div_gather_gen<2><<<gn, bn, 0, c->stream>>>(a);
            break;
        case NXSDG_STEP_VELOCITY:
            if (p1) k_velocity_gen<1><<<gn, bn, 0, c->stream>>>(a); else k_velocity_gen<2><<<gn, bn, 0, c->stream>>>(a);
            break;
        default: return fail(c, NXSDG_ERR_INVALID_ARG, "bad step");
    }
    LAUNCHED();
    if (st == NXSDG_STEP_VELOCITY) c->cv ^= 1;
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_set_vertices(nxsdg_ctx* c, const double* xy, int64_t count, nxsdg_mem mem) {
    GUARD(c);
    if (!xy || (mem != NXSDG_MEM_HOST && mem != NXSDG_MEM_DEVICE)) return fail(c, NXSDG_ERR_INVALID_ARG, "bad argument");
    if (c->d.nranks != 1) return fail(c, NXSDG_ERR_UNSUPPORTED, "general quads are single-rank");
    if (c->NS == 8) return fail(c, NXSDG_ERR_UNSUPPORTED, "general quads: n_S = 3 | 6");
    if (c->precision != 0) return fail(c, NXSDG_ERR_UNSUPPORTED, "general quads: FP64 storage only");
    if (c->sphere) return fail(c, NXSDG_ERR_UNSUPPORTED, "general quads or the sphere, not both");
    const int64_t need = 2 * (int64_t)(c->d.nx + 1) * (c->d.ny + 1);
    if (count != need) return fail(c, NXSDG_ERR_INVALID_ARG, "count %lld != %lld", (long long)count, (long long)need);
    if (!c->verts) CU(cudaMalloc(&c->verts, need * sizeof(double)));
    CU(cudaMemcpyAsync(c->verts, xy, need * sizeof(double),
                       mem == NXSDG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->stream));
    if (mem == NXSDG_MEM_HOST) CU(cudaStreamSynchronize(c->stream));
    c->general = true;
    c->gmaps_ready = false;
    c->gen_maps_ok = false;
    drop_graphs(c);
    nxsdg_status st = ensure_debug_buffers(c);
    if (st) return st;
    const size_t nn = (size_t)c->npitch * c->nrows_local;
    if (!c->mlump) CU(cudaMalloc(&c->mlump, nn * sizeof(double)));
    if (!c->imlump) CU(cudaMalloc(&c->imlump, nn * sizeof(double)));
    if (!c->gcontrib) CU(cudaMalloc(&c->gcontrib, (size_t)2 * (c->P + 1) * (c->P + 1) * c->eplane * sizeof(double)));
    GenStepArgs a = gen_step_args(c);
    dim3 b(128), g((unsigned)((c->P * c->d.nx + 1 + 127) / 128), (unsigned)(c->P * c->d.ny + 1));
    if (c->P == 1) k_gen_lumped<1><<<g, b, 0, c->stream>>>(a);
    else k_gen_lumped<2><<<g, b, 0, c->stream>>>(a);
    LAUNCHED();
    return NXSDG_OK;
}

// ---------------------------------------------------------------- NEXT-4: spherical lon-lat mesh (R#26)
// Per local element row (latitudes lat0 + (gr + t) dlat, gr the global row) the fused subcycle and the
// advection need: cos(lat) and sin(lat)/R at the 3 Gauss latitudes; the blocks Q = M_row^{-1} M_ref of
// the row's DG mass M_K = R^2 dlon dlat M_row, M_row = int int psi_a psi_b cos(lat) with the 3-point rule,
// block-diagonal in the S-degree of the centred Legendre modes (S-parts orthogonal): modes {0, 2, 4} =
// 1 x {1, T, T^2 - 1/12} -> C^{-1} diag(1, 1/12, 1/180), {1, 5} = S x {1, T} -> C2^{-1} diag(1, 1/12),
// {3} -> 1 / C00, where C_ij = sum_g w_g P_i(T_g) P_j(T_g) cos(lat_g); the reciprocal lumped masses
// 1 / mu of the three node rows 2 gr + jy for even / odd node columns (m_j = R^2 dlon dlat mu_j,
// mu = (1/3 | 2/3) x sum over the touching element rows of sum_g w_g L_jy(t_g) cos(lat_g)); and
// cos(lat) of the row's south / north edge (from the node-row latitude, so a shared edge gets the
// bitwise-same factor on both sides).
static void solve3(const double A[3][3], double X[3][3]) {   // X = A^{-1} (symmetric positive definite)
    const double d = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                     A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
    X[0][0] = (A[1][1] * A[2][2] - A[1][2] * A[2][1]) / d; X[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / d;
    X[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / d; X[1][0] = (A[1][2] * A[2][0] - A[1][0] * A[2][2]) / d;
    X[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / d; X[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / d;
    X[2][0] = (A[1][0] * A[2][1] - A[1][1] * A[2][0]) / d; X[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / d;
    X[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / d;
}

static nxsdg_status sphere_tables(nxsdg_ctx* c) {
    const double ka = 0.38729833462074170, gw[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
    const double tg[3] = {0.5 - ka, 0.5, 0.5 + ka};
    const double L[3][3] = {{0.3 + ka, 0.4, 0.3 - ka}, {0.0, 1.0, 0.0}, {0.3 - ka, 0.4, 0.3 + ka}};   // L_jy(t_g) [g][jy]
    const int ny = c->d.ny;
    auto lat = [&](int64_t gr, double t) { return c->sph_lat0 + ((double)gr + t) * c->sph_dlat; };
    // T(gr, jy) = sum_g w_g L_jy(t_g) cos(lat_g) of element row gr
    auto trow = [&](int64_t gr, int jy) {
        double acc = 0.0;
        for (int g = 0; g < 3; ++g) acc += gw[g] * L[g][jy] * cos(lat(gr, tg[g]));
        return acc;
    };
    std::vector<double> tab((size_t)c->erows_local * kSphRow, 0.0);
    for (int lr = 0; lr < c->erows_local; ++lr) {
        const int64_t gr = c->r0 + (lr - c->glo);
        double* row = &tab[(size_t)lr * kSphRow];
        double C[3][3] = {};
        for (int g = 0; g < 3; ++g) {
            const double la = lat(gr, tg[g]), cg = cos(la), T = tg[g] - 0.5;
            const double P[3] = {1.0, T, T * T - 1.0 / 12.0};
            row[SPH_COS + g] = cg;
            row[SPH_SINR + g] = sin(la) / c->sph_R;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) C[i][j] += gw[g] * P[i] * P[j] * cg;
        }
        double Ci[3][3];
        solve3(C, Ci);
        const double mref[3] = {1.0, 1.0 / 12.0, 1.0 / 180.0};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) row[SPH_QA + 3 * i + j] = Ci[i][j] * mref[j];
        const double d2 = C[0][0] * C[1][1] - C[0][1] * C[1][0];
        const double C2i[2][2] = {{C[1][1] / d2, -C[0][1] / d2}, {-C[1][0] / d2, C[0][0] / d2}};
        const double mref2[2] = {1.0, 1.0 / 12.0};
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) row[SPH_QB + 2 * i + j] = C2i[i][j] * mref2[j];
        row[SPH_QC] = 1.0 / C[0][0];
        for (int jy = 0; jy < 3; ++jy) {   // node row J = 2 gr + jy, global element rows touching it
            const int64_t J = 2 * gr + jy;
            double T = 0.0;
            if (J % 2) T = trow(gr, 1);
            else {
                const int64_t r = J / 2;
                if (r - 1 >= 0 && r - 1 < ny) T += trow(r - 1, 2);
                if (r >= 0 && r < ny) T += trow(r, 0);
            }
            row[SPH_IMU + 2 * jy + 0] = T > 0.0 ? 3.0 / T : 0.0;          // even column: 2 x 1/6
            row[SPH_IMU + 2 * jy + 1] = T > 0.0 ? 1.5 / T : 0.0;          // odd column: 2/3
        }
        row[SPH_COS_S] = cos(c->sph_lat0 + (double)gr * c->sph_dlat);
        row[SPH_COS_N] = cos(c->sph_lat0 + (double)(gr + 1) * c->sph_dlat);
    }
    if (!c->sph_rows) CU(cudaMalloc(&c->sph_rows, tab.size() * sizeof(double)));
    CU(cudaMemcpyAsync(c->sph_rows, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_set_sphere(nxsdg_ctx* c, double radius, double lat0, double lon_extent, double lat_extent) {
    GUARD(c);
    const double half_pi = 1.5707963267948966;
    if (!(radius > 0.0) || !(lon_extent > 0.0) || !(lat_extent > 0.0) || !(fabs(lat0) < half_pi) ||
        !(fabs(lat0 + lat_extent) < half_pi))
        return fail(c, NXSDG_ERR_INVALID_ARG, "sphere: radius, extents > 0 and latitudes inside (-pi/2, pi/2)");
    if (c->P != 2 || c->NS != 6 || c->NA != 6 || c->general || c->precision != 0)
        return fail(c, NXSDG_ERR_UNSUPPORTED, "sphere: CG2 / DG2 (n_S = n_A = 6), FP64, box mesh");
    c->sphere = true;
    c->sph_R = radius; c->sph_lat0 = lat0;
    c->sph_dlon = lon_extent / c->d.nx; c->sph_dlat = lat_extent / c->d.ny;
    drop_graphs(c);
    c->prepped = false; c->prep_defer = false;
    return sphere_tables(c);
}

static GenArgs gen_args(nxsdg_ctx* c) {
    GenArgs a{};
    a.verts = c->verts; a.maps = c->gmaps; a.E = c->E; a.S = c->S[c->cs]; a.H = c->H; a.A = c->A;
    a.eplane = c->eplane; a.epitch = c->epitch; a.nx = c->d.nx; a.ny = c->d.ny;
    a.ainv = 1.0 / c->prm.alpha; a.fac = 1.0 - a.ainv; a.dmin2 = c->prm.DeltaMin * c->prm.DeltaMin;
    a.Pstar = c->prm.Pstar; a.C_conc = c->prm.C_conc; a.repl = c->prm.replacement_pressure;
    return a;
}

template <int P, int NA>
static nxsdg_status general_stress_t(nxsdg_ctx* c) {
    constexpr int NSG = Deg<P>::NS * Deg<P>::NG;
    if (c->map_mode == 0 && !c->gmaps_ready) {
        if (!c->gmaps) CU(cudaMalloc(&c->gmaps, (size_t)NSG * c->eplane * sizeof(double)));
        GenArgs a = gen_args(c);
        dim3 b(128), g((unsigned)((c->d.nx + 127) / 128), (unsigned)c->d.ny);
        k_gen_maps<P><<<g, b, 0, c->stream>>>(a);
        LAUNCHED();
        c->gmaps_ready = true;
    }
    GenArgs a = gen_args(c);
    dim3 b(128), g((unsigned)((c->d.nx + 127) / 128), (unsigned)c->d.ny);
    if (c->map_mode == 0) k_stress_general<P, NA, false><<<g, b, 0, c->stream>>>(a);
    else k_stress_general<P, NA, true><<<g, b, 0, c->stream>>>(a);
    LAUNCHED();
    return NXSDG_OK;
}

static nxsdg_status general_stress(nxsdg_ctx* c) {
    if (c->P == 1) return c->NA == 1 ? general_stress_t<1, 1>(c) : general_stress_t<1, 3>(c);
    if (c->NA == 1) return general_stress_t<2, 1>(c);
    if (c->NA == 3) return general_stress_t<2, 3>(c);
    return general_stress_t<2, 6>(c);
}

// ---------------------------------------------------------------- halo exchange
// Rows that cross a rank boundary:
//   up   (r -> r+1): top owned element row of element fields; top P owned node rows of node fields
//   down (r -> r-1): bottom owned node row of node fields; bottom owned element row (A/H only)
// The plan is pure host arithmetic on the local geometry (nxsdg_halo_plan exports it).  Every
// rank emits the fields in the same order and, per field, [send up, recv up, send down,
// recv down], so rank r's k-th send to q pairs with q's k-th recv from r - the matching rule
// of ncclSend/ncclRecv, and the rule the loopback transport applies explicitly.

static Geom make_geom(int nx, int ny, int p, int ns, int na, int nranks, int rank) {
    Geom g{};
    g.nx = nx; g.ny = ny; g.P = p; g.NS = ns; g.NA = na; g.nranks = nranks; g.rank = rank;
    int32_t erows = 0;
    nxsdg_partition(ny, p, nranks, rank, &g.r0, &erows, nullptr, nullptr);
    g.r1 = g.r0 + erows; g.nown = erows;
    g.glo = g.r0 > 0 ? 1 : 0;
    g.ghi = g.r1 < ny ? 1 : 0;
    g.erows_local = g.glo + g.nown + g.ghi;
    g.nrows_local = p * (g.glo + g.nown) + 1;
    g.epitch = round_up(nx, 4);     // element row pitch: 32-B aligned rows (TMA strides)
    g.eplane = round_up((int64_t)g.erows_local * g.epitch, 32);
    g.npitch = round_up((int64_t)p * nx + 2, 32);
    g.nn = g.npitch * g.nrows_local;
    return g;
}

static void halo_plan(const Geom& g, uint32_t what, std::vector<nxsdg_halo_seg>& out) {
    const bool up = g.rank + 1 < g.nranks, down = g.rank > 0;
    const int64_t top = g.glo + g.nown - 1, bot = g.glo, ghost_hi = g.glo + g.nown;
    auto seg = [&](int dir, int field, int peer, int plane, int64_t off, int64_t cnt) {
        out.push_back(nxsdg_halo_seg{dir, field, peer, plane, off, cnt});
    };
    auto node_field = [&](int f) {
        if (up) {
            seg(0, f, g.rank + 1, 0, g.P * top * g.npitch, g.P * g.npitch);       // top P owned rows
            seg(1, f, g.rank + 1, 0, g.P * ghost_hi * g.npitch, g.npitch);        // top ghost row
        }
        if (down) {
            seg(0, f, g.rank - 1, 0, g.P * bot * g.npitch, g.npitch);              // bottom owned row
            seg(1, f, g.rank - 1, 0, 0, g.P * g.npitch);                           // P bottom ghost rows
        }
    };
    auto elem_field = [&](int f, int nplanes, bool both) {
        // per kind [send up, recv up, send down, recv down], all planes: one packed message each
        auto planes = [&](int dir, int peer, int64_t row) {
            for (int k = 0; k < nplanes; ++k) seg(dir, f, peer, k, (int64_t)k * g.eplane + row * g.epitch, g.nx);
        };
        if (up) {
            planes(0, g.rank + 1, top);
            if (both) planes(1, g.rank + 1, ghost_hi);
        }
        if (down) {
            if (both) planes(0, g.rank - 1, bot);
            planes(1, g.rank - 1, 0);
        }
    };
    if (what & NXSDG_HALO_V) { node_field(NXSDG_HF_VX); node_field(NXSDG_HF_VY); }
    if (what & NXSDG_HALO_S) elem_field(NXSDG_HF_S, 3 * g.NS, false);
    if (what & NXSDG_HALO_AH) { elem_field(NXSDG_HF_A, g.NA, true); elem_field(NXSDG_HF_H, g.NA, true); }
    if (what & NXSDG_HALO_AH_SCR0) { elem_field(NXSDG_HF_A_SCR0, g.NA, true); elem_field(NXSDG_HF_H_SCR0, g.NA, true); }
    if (what & NXSDG_HALO_AH_SCR1) { elem_field(NXSDG_HF_A_SCR1, g.NA, true); elem_field(NXSDG_HF_H_SCR1, g.NA, true); }
}

extern "C" nxsdg_status nxsdg_local_geometry(int32_t nx, int32_t ny, int32_t p, int32_t ns, int32_t na, int32_t nranks,
                                             int32_t rank, int64_t* out8) {
    if (!out8 || nx < 1 || nxsdg_partition(ny, p, nranks, rank, nullptr, nullptr, nullptr, nullptr)) return NXSDG_ERR_INVALID_ARG;
    Geom g = make_geom(nx, ny, p, ns, na, nranks, rank);
    const int64_t v[8] = {g.r0, g.nown, g.glo, g.erows_local, g.nrows_local, g.epitch, g.eplane, g.npitch};
    memcpy(out8, v, sizeof v);
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_halo_plan(int32_t nx, int32_t ny, int32_t p, int32_t ns, int32_t na, int32_t nranks,
                                        int32_t rank, uint32_t what, nxsdg_halo_seg* out, int32_t max, int32_t* n_out) {
    if (!n_out || nx < 1 || nxsdg_partition(ny, p, nranks, rank, nullptr, nullptr, nullptr, nullptr)) return NXSDG_ERR_INVALID_ARG;
    std::vector<nxsdg_halo_seg> v;
    halo_plan(make_geom(nx, ny, p, ns, na, nranks, rank), what, v);
    *n_out = (int32_t)v.size();
    if (out) {
        if ((int32_t)v.size() > max) return NXSDG_ERR_INVALID_ARG;
        std::copy(v.begin(), v.end(), out);
    }
    return NXSDG_OK;
}

static double* halo_base(nxsdg_ctx* c, int field) {
    switch (field) {
        case NXSDG_HF_VX: return c->vx[c->cv];
        case NXSDG_HF_VY: return c->vy[c->cv];
        case NXSDG_HF_S: return c->S[c->cs];
        case NXSDG_HF_A: return c->A;
        case NXSDG_HF_H: return c->H;
        case NXSDG_HF_A_SCR0: return c->Asc[0];
        case NXSDG_HF_H_SCR0: return c->Hsc[0];
        case NXSDG_HF_A_SCR1: return c->Asc[1];
        default: return c->Hsc[1];
    }
}

// Messages: consecutive plan segments with the same (dir, peer, field), equal counts and a
// uniform stride (the planes of one element field) travel as one contiguous message, packed
// into / unpacked from staging buffers with 2D copies.
struct HaloMsg { int dir, peer, field; int64_t off0, count, stride, nseg, stage_off; };

static void halo_messages(const Geom& g, uint32_t what, std::vector<HaloMsg>& out) {
    std::vector<nxsdg_halo_seg> plan;
    halo_plan(g, what, plan);
    for (const auto& sg : plan) {
        if (!out.empty()) {
            HaloMsg& m = out.back();
            if (m.dir == sg.dir && m.peer == sg.peer && m.field == sg.field && m.count == sg.count) {
                const int64_t st = sg.offset - m.off0;
                if (m.nseg == 1 && st > 0) { m.stride = st; ++m.nseg; continue; }
                if (m.nseg > 1 && sg.offset == m.off0 + m.nseg * m.stride) { ++m.nseg; continue; }
            }
        }
        out.push_back(HaloMsg{sg.dir, sg.peer, sg.field, sg.offset, sg.count, sg.count, 1, 0});
    }
    int64_t so = 0, ro = 0;
    for (auto& m : out) {
        int64_t& o = m.dir == 0 ? so : ro;
        m.stage_off = o;
        o += round_up(m.count * m.nseg, 32);
    }
}

static nxsdg_status ensure_halo_staging(nxsdg_ctx* c) {
    if (c->hstage_send) return NXSDG_OK;
    std::vector<HaloMsg> msgs;
    halo_messages(c->geom, NXSDG_HALO_V | NXSDG_HALO_S | NXSDG_HALO_AH, msgs);
    int64_t need = 64;
    for (auto& m : msgs) need = std::max(need, m.stage_off + round_up(m.count * m.nseg, 32));
    CU(cudaMalloc(&c->hstage_send, need * sizeof(double)));
    CU(cudaMalloc(&c->hstage_recv, need * sizeof(double)));
    return NXSDG_OK;
}

static nxsdg_status copy2d(nxsdg_ctx* c, double* dst, int64_t dpitch, const double* src, int64_t spitch,
                           int64_t width, int64_t height, cudaStream_t st) {
    CU(cudaMemcpy2DAsync(dst, dpitch * sizeof(double), src, spitch * sizeof(double), width * sizeof(double), height,
                         cudaMemcpyDeviceToDevice, st));
    return NXSDG_OK;
}

static nxsdg_status pack_sends(nxsdg_ctx* c, const std::vector<HaloMsg>& msgs, cudaStream_t st) {
    nxsdg_status s;
    for (const auto& m : msgs)
        if (m.dir == 0 && m.nseg > 1 &&
            (s = copy2d(c, c->hstage_send + m.stage_off, m.count, halo_base(c, m.field) + m.off0, m.stride, m.count, m.nseg, st)))
            return s;
    return NXSDG_OK;
}
static nxsdg_status unpack_recvs(nxsdg_ctx* c, const std::vector<HaloMsg>& msgs, cudaStream_t st) {
    nxsdg_status s;
    for (const auto& m : msgs)
        if (m.dir == 1 && m.nseg > 1 &&
            (s = copy2d(c, halo_base(c, m.field) + m.off0, m.stride, c->hstage_recv + m.stage_off, m.count, m.count, m.nseg, st)))
            return s;
    return NXSDG_OK;
}
static double* msg_ptr(nxsdg_ctx* c, const HaloMsg& m) {
    if (m.nseg == 1) return halo_base(c, m.field) + m.off0;
    return (m.dir == 0 ? c->hstage_send : c->hstage_recv) + m.stage_off;
}

static nxsdg_status halo_nccl(nxsdg_ctx* c, uint32_t what, cudaStream_t st) {
    NvtxRange nv("nxsdg halo nccl");
    nxsdg_status s = ensure_halo_staging(c);
    if (s) return s;
    std::vector<HaloMsg> msgs;
    halo_messages(c->geom, what, msgs);
    if ((s = pack_sends(c, msgs, st))) return s;
    NcclApi& api = nccl();
    if (api.GroupStart() != 0) return fail(c, NXSDG_ERR_NCCL, "ncclGroupStart");
    for (const auto& m : msgs) {
        const size_t n = (size_t)(m.count * m.nseg);
        const int r = m.dir == 0 ? api.Send(msg_ptr(c, m), n, kNcclFloat64, m.peer, c->comm, st)
                                 : api.Recv(msg_ptr(c, m), n, kNcclFloat64, m.peer, c->comm, st);
        if (r != 0) { api.GroupEnd(); return fail(c, NXSDG_ERR_NCCL, "ncclSend/Recv: %d", r); }
    }
    if (api.GroupEnd() != 0) return fail(c, NXSDG_ERR_NCCL, "ncclGroupEnd");
    return unpack_recvs(c, msgs, st);
}

// Loopback: the NCCL data flow with cudaMemcpyAsync in place of send/recv - pack on every
// rank, copy rank r's k-th message to q into q's k-th receive from r, unpack on every rank
// (all contexts share one stream, so stream order is the exchange order).
static nxsdg_status halo_loopback_all(std::vector<nxsdg_ctx*>& ctxs, uint32_t what) {
    const int n = (int)ctxs.size();
    nxsdg_status s;
    std::vector<std::vector<HaloMsg>> msgs(n);
    for (int r = 0; r < n; ++r) {
        if ((s = ensure_halo_staging(ctxs[r]))) return s;
        halo_messages(ctxs[r]->geom, what, msgs[r]);
        if ((s = pack_sends(ctxs[r], msgs[r], ctxs[r]->stream))) return s;
    }
    for (int r = 0; r < n; ++r) {
        nxsdg_ctx* c = ctxs[r];
        std::vector<int> kth(n, 0);
        for (const auto& m : msgs[r]) {
            if (m.dir != 0) continue;
            const int q = m.peer;
            int seen = -1;
            const HaloMsg* rv = nullptr;
            for (const auto& t : msgs[q])
                if (t.dir == 1 && t.peer == r && ++seen == kth[q]) { rv = &t; break; }
            ++kth[q];
            if (!rv || rv->count * rv->nseg != m.count * m.nseg || rv->field != m.field)
                return fail(c, NXSDG_ERR_STATE, "halo plan mismatch between ranks %d and %d", r, q);
            CU(cudaMemcpyAsync(msg_ptr(ctxs[q], *rv), msg_ptr(c, m), (size_t)(m.count * m.nseg) * sizeof(double),
                               cudaMemcpyDeviceToDevice, c->stream));
        }
    }
    for (int r = 0; r < n; ++r)
        if ((s = unpack_recvs(ctxs[r], msgs[r], ctxs[r]->stream))) return s;
    return NXSDG_OK;
}

// ---- P2P transport (NXSDG_TRANSPORT_P2P): no NCCL, no staging.  Every send segment of the halo
// plan is copied by the copy engine straight from this rank's buffer into the matching receive
// rows of the neighbour's buffer (peer memory over NVLink / NVSwitch: a CUDA IPC mapping across
// processes, a plain device pointer inside one process), then this rank sets its word of slot
// k & 1 in each neighbour's flags to 1 (cuStreamWriteValue32, which fences the copies and kernel
// peer stores before it), and its stream waits, on the device, until both neighbours have set its
// own slot-(k & 1) words to 1 (cuStreamWaitValue32 EQ, with CU_STREAM_WAIT_VALUE_FLUSH where the
// device supports it, so remote writes that arrived before the flag are visible to the work after
// the wait even if the device reordered them), then clears them.  Every value is a constant, so
// the exchange can be captured in a CUDA graph and replayed (the multi-rank subcycle graphs).
// Every rank issues the same sequence of halo calls, so slots match.  A sender sets slot s again
// (exchange k + 2) only after waiting for the receiver's exchange-(k + 1) signal, which the receiver
// writes after clearing slot s (stream order + the write's fence), so no signal is lost.  Race
// freedom: an exchange writes only ghost rows of the buffer the preceding kernel produced, which
// no kernel of the receiver reads before the receiver's own wait for this exchange; and the sender
// can only reach its next exchange after waiting for the receiver's signal of this one, which the
// receiver issues after the kernels that read the previous contents of those ghost rows.
typedef CUresult (*PFN_sv32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps { PFN_sv32 write = nullptr, wait = nullptr; };
static MemOps& memops() {
    static MemOps m;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr; cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) m.write = (PFN_sv32)p;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) m.wait = (PFN_sv32)p;
    }
    return m;
}

static int p2p_index(const nxsdg_ctx* c, const double* b) {
    for (int i = 0; i < kP2PBufs; ++i) if (c->orig[i] == b) return i;
    return -1;
}

static nxsdg_status halo_p2p(nxsdg_ctx* c, uint32_t what, cudaStream_t st) {
    NvtxRange nv("nxsdg halo p2p");
    if (!c->p2p_ok) return fail(c, NXSDG_ERR_STATE, "P2P transport not connected (nxsdg_p2p_connect)");
    MemOps& mo = memops();
    if (!mo.write || !mo.wait) return fail(c, NXSDG_ERR_UNSUPPORTED, "stream memory operations unavailable");
    std::vector<HaloMsg> mine, theirs[2];
    halo_messages(c->geom, what, mine);
    for (int sd = 0; sd < 2; ++sd) if (c->peer[sd].on) halo_messages(c->peer[sd].g, what, theirs[sd]);
    int kth[2] = {0, 0};
    for (const auto& m : mine) {
        if (m.dir != 0) continue;
        const int sd = m.peer < c->d.rank ? 0 : 1;
        const nxsdg_ctx::Peer& pr = c->peer[sd];
        if (!pr.on) return fail(c, NXSDG_ERR_STATE, "P2P neighbour %d not connected", m.peer);
        const HaloMsg* rv = nullptr;
        int seen = -1;
        for (const auto& t : theirs[sd])
            if (t.dir == 1 && t.peer == c->d.rank && ++seen == kth[sd]) { rv = &t; break; }
        ++kth[sd];
        double* base = halo_base(c, m.field);
        const int bi = p2p_index(c, base);
        if (!rv || bi < 0 || rv->count != m.count || rv->nseg != m.nseg)
            return fail(c, NXSDG_ERR_STATE, "P2P halo plan mismatch with rank %d", m.peer);
        nxsdg_status s = copy2d(c, pr.buf[bi] + rv->off0, rv->stride, base + m.off0, m.stride, m.count, m.nseg, st);
        if (s) return s;
    }
    const int slot = (int)(c->p2p_seq++ & 1u) * 2;
    for (int sd = 0; sd < 2; ++sd)   // I am my lower neighbour's upper one (word 1) and vice versa
        if (c->peer[sd].on &&
            mo.write((CUstream)st, (CUdeviceptr)(c->peer[sd].flags + slot + (sd == 0 ? 1 : 0)), 1u, 0) != CUDA_SUCCESS)
            return fail(c, NXSDG_ERR_CUDA, "cuStreamWriteValue32 failed");
    for (int sd = 0; sd < 2; ++sd) {
        if (!c->peer[sd].on) continue;
        if (mo.wait((CUstream)st, (CUdeviceptr)(c->flags + slot + sd), 1u, CU_STREAM_WAIT_VALUE_EQ | c->p2p_wait_flags) !=
            CUDA_SUCCESS)
            return fail(c, NXSDG_ERR_CUDA, "cuStreamWaitValue32 failed");
        if (mo.write((CUstream)st, (CUdeviceptr)(c->flags + slot + sd), 0u, 0) != CUDA_SUCCESS)
            return fail(c, NXSDG_ERR_CUDA, "cuStreamWriteValue32 (clear) failed");
    }
    return NXSDG_OK;
}

static nxsdg_status halo_on(nxsdg_ctx* c, uint32_t what, cudaStream_t st) {
    if (c->d.transport == NXSDG_TRANSPORT_NCCL) return halo_nccl(c, what, st);
    return halo_p2p(c, what, st);
}

static nxsdg_status halo(nxsdg_ctx* c, uint32_t what) {
    if (c->d.nranks == 1) return NXSDG_OK;
    if (c->d.transport == NXSDG_TRANSPORT_NCCL || c->d.transport == NXSDG_TRANSPORT_P2P) return halo_on(c, what, c->stream);
    return NXSDG_OK;   // loopback exchanges are driven by the group calls
}

struct P2PBlob {
    uint32_t magic, version;
    int32_t rank, nranks, nx, ny, P, NS, NA, device;
    cudaIpcMemHandle_t h[kP2PBufs + 1];   // buffers, then the flag pair
};
constexpr uint32_t kP2PMagic = 0x4e585032u;   // "NXP2"

extern "C" nxsdg_status nxsdg_p2p_export(nxsdg_ctx* c, void* blob, int64_t cap, int64_t* needed) {
    GUARD(c);
    if (needed) *needed = (int64_t)sizeof(P2PBlob);
    if (c->d.transport != NXSDG_TRANSPORT_P2P || c->d.nranks < 2) return fail(c, NXSDG_ERR_STATE, "not a P2P rank");
    if (!blob) return NXSDG_OK;
    if (cap < (int64_t)sizeof(P2PBlob)) return fail(c, NXSDG_ERR_INVALID_ARG, "cap < %zu", sizeof(P2PBlob));
    P2PBlob b{};
    b.magic = kP2PMagic; b.version = 1;
    b.rank = c->d.rank; b.nranks = c->d.nranks; b.nx = c->d.nx; b.ny = c->d.ny;
    b.P = c->P; b.NS = c->NS; b.NA = c->NA; b.device = c->d.device;
    cudaSetDevice(c->d.device);
    for (int i = 0; i < kP2PBufs; ++i) CU(cudaIpcGetMemHandle(&b.h[i], c->orig[i]));
    CU(cudaIpcGetMemHandle(&b.h[kP2PBufs], c->flags));
    memcpy(blob, &b, sizeof b);
    return NXSDG_OK;
}

static bool p2p_blob_ok(const nxsdg_ctx* c, const P2PBlob& b, int rank) {
    return b.magic == kP2PMagic && b.version == 1 && b.rank == rank && b.nranks == c->d.nranks && b.nx == c->d.nx &&
           b.ny == c->d.ny && b.P == c->P && b.NS == c->NS && b.NA == c->NA;
}

static void p2p_finish_connect(nxsdg_ctx* c) {
    bool ok = true;
    if (c->d.rank > 0 && !c->peer[0].on) ok = false;
    if (c->d.rank + 1 < c->d.nranks && !c->peer[1].on) ok = false;
    for (int sd = 0; sd < 2; ++sd)
        if (c->peer[sd].on)
            c->peer[sd].g = make_geom(c->d.nx, c->d.ny, c->P, c->NS, c->NA, c->d.nranks, c->d.rank + (sd == 0 ? -1 : 1));
    int can_flush = 0;
    if (cudaDeviceGetAttribute(&can_flush, cudaDevAttrCanFlushRemoteWrites, c->d.device) != cudaSuccess) {
        cudaGetLastError();
        can_flush = 0;
    }
    c->p2p_wait_flags = can_flush ? (unsigned)CU_STREAM_WAIT_VALUE_FLUSH : 0u;
    c->p2p_ok = ok;
}

extern "C" nxsdg_status nxsdg_p2p_connect(nxsdg_ctx* c, const void* lower, const void* upper) {
    GUARD(c);
    if (c->d.transport != NXSDG_TRANSPORT_P2P || c->d.nranks < 2) return fail(c, NXSDG_ERR_STATE, "not a P2P rank");
    if (c->p2p_ok) return fail(c, NXSDG_ERR_STATE, "already connected");
    const void* blobs[2] = {lower, upper};
    const int want[2] = {c->d.rank > 0, c->d.rank + 1 < c->d.nranks};
    cudaSetDevice(c->d.device);
    for (int sd = 0; sd < 2; ++sd) {
        if (!want[sd]) continue;
        if (!blobs[sd]) return fail(c, NXSDG_ERR_INVALID_ARG, "missing %s neighbour blob", sd ? "upper" : "lower");
        P2PBlob b;
        memcpy(&b, blobs[sd], sizeof b);
        if (!p2p_blob_ok(c, b, c->d.rank + (sd == 0 ? -1 : 1)))
            return fail(c, NXSDG_ERR_INVALID_ARG, "%s neighbour blob does not match this mesh", sd ? "upper" : "lower");
        if (b.device != c->d.device) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, c->d.device, b.device);
            if (!can) return fail(c, NXSDG_ERR_UNSUPPORTED, "no peer access from device %d to %d", c->d.device, b.device);
        }
        nxsdg_ctx::Peer& pr = c->peer[sd];
        pr.ipc = true;
        for (int i = 0; i <= kP2PBufs; ++i) {
            void* ptr = nullptr;
            cudaError_t e = cudaIpcOpenMemHandle(&ptr, b.h[i], cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return fail(c, NXSDG_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
            }
            if (i < kP2PBufs) pr.buf[i] = (double*)ptr; else pr.flags = (uint32_t*)ptr;
        }
        pr.on = true;
    }
    p2p_finish_connect(c);
    return NXSDG_OK;
}

static bool p2p_fused_stores(const nxsdg_ctx* c);
static bool mr_graph_on(const nxsdg_ctx* c);
extern "C" int64_t nxsdg_transport_info(const nxsdg_ctx* c, char* buf, int64_t cap) {
    if (!c) return -1;
    static const char* names[] = {"none", "nccl", "loopback", "p2p"};
    const int t = c->d.transport >= 0 && c->d.transport < 4 ? c->d.transport : 0;
    std::string s = "rank " + std::to_string(c->d.rank) + "/" + std::to_string(c->d.nranks) + " device " +
                    std::to_string(c->d.device) + " transport " + names[t];
    if (c->d.transport == NXSDG_TRANSPORT_P2P) {
        for (int sd = 0; sd < 2; ++sd) {
            s += sd == 0 ? " lower:" : " upper:";
            if (!c->peer[sd].on) { s += "none"; continue; }
            s += c->peer[sd].ipc ? "ipc" : "in-process";
        }
        s += std::string(" wait_flush=") + (c->p2p_wait_flags ? "1" : "0");
        s += std::string(" fused_peer_stores=") + (p2p_fused_stores(c) ? "1" : "0");
    }
    if (c->d.nranks > 1)
        s += std::string(" subcycle_graph=") + (mr_graph_on(c) ? "1" : "0") +
             (c->mr_graph_note.empty() ? "" : " (" + c->mr_graph_note + ")") +
             (c->inproc ? " (in-process ranks: host-issued subcycles, k_advect_q2)" : "");
    if (buf && cap > 0) {
        const size_t n = std::min<size_t>(s.size(), (size_t)cap - 1);
        memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return (int64_t)s.size();
}

extern "C" nxsdg_status nxsdg_p2p_connect_local(nxsdg_ctx** ctxs, int32_t n) {
    if (!ctxs || n < 2) return NXSDG_ERR_INVALID_ARG;
    for (int i = 0; i < n; ++i)
        if (!ctxs[i] || ctxs[i]->d.rank != i || ctxs[i]->d.nranks != n || ctxs[i]->d.transport != NXSDG_TRANSPORT_P2P ||
            ctxs[i]->p2p_ok)
            return NXSDG_ERR_INVALID_ARG;
    for (int i = 0; i < n; ++i) {
        nxsdg_ctx* c = ctxs[i];
        for (int sd = 0; sd < 2; ++sd) {
            const int q = i + (sd == 0 ? -1 : 1);
            if (q < 0 || q >= n) continue;
            if (ctxs[q]->d.device != c->d.device) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, c->d.device, ctxs[q]->d.device);
                if (!can) return fail(c, NXSDG_ERR_UNSUPPORTED, "no peer access between devices");
                cudaSetDevice(c->d.device);
                cudaError_t e = cudaDeviceEnablePeerAccess(ctxs[q]->d.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(c, NXSDG_ERR_CUDA, "peer access");
                cudaGetLastError();
            }
            nxsdg_ctx::Peer& pr = c->peer[sd];
            std::copy(ctxs[q]->orig, ctxs[q]->orig + kP2PBufs, pr.buf);
            pr.flags = ctxs[q]->flags;
            pr.ipc = false; pr.on = true;
        }
        c->inproc = true;
        drop_graphs(c);
        p2p_finish_connect(c);
    }
    return NXSDG_OK;
}

// ---------------------------------------------------------------- launches
static PrepArgs prep_args(nxsdg_ctx* c) {
    PrepArgs a{};
    a.H = c->H; a.A = c->A; a.vx = c->vx[c->cv]; a.vy = c->vy[c->cv];
    a.ox = c->ox; a.oy = c->oy; a.ax = c->ax; a.ay = c->ay;
    a.c1 = c->c1; a.rx0 = c->rx0; a.ry0 = c->ry0; a.cafo = c->cafo; a.Pg = c->Pg;
    a.eplane = c->eplane; a.npitch = c->npitch; a.epitch = c->epitch; a.nx = c->d.nx; a.erows_local = c->erows_local;
    a.node_row_begin = c->P * c->glo;
    a.node_row_end = (int)(c->P * c->glo + owned_node_rows(c));
    a.elem_rows_with_nodes = c->glo + c->nown;
    a.rho_ice = c->prm.rho_ice; a.Fa = c->prm.rho_atm * c->prm.C_atm; a.Fo = c->prm.rho_ocean * c->prm.C_ocean;
    a.f_c = c->prm.f_c; a.dt = c->prm.dt; a.Pstar = c->prm.Pstar; a.C_conc = c->prm.C_conc;
    a.rdt = 1.0 / c->prm.dt;
    return a;
}

template <int P, int NA>
static nxsdg_status launch_prep(nxsdg_ctx* c) {
    PrepArgs a = prep_args(c);
    dim3 bn(128), gn((unsigned)((P * c->d.nx + 1 + 127) / 128), (unsigned)(a.node_row_end - a.node_row_begin));
    k_prep_nodes<P, NA><<<gn, bn, 0, c->stream>>>(a);
    LAUNCHED();
    dim3 be(128), ge((unsigned)((c->d.nx + 127) / 128), (unsigned)c->erows_local);
    k_prep_elems<P, NA><<<ge, be, 0, c->stream>>>(a);
    LAUNCHED();
    return NXSDG_OK;
}

static bool use_tma(const nxsdg_ctx* c);
static int const_mode(const nxsdg_ctx* c);
// NXSDG_OPT_PREP_KERNEL 2: the node constants are formed by the first fused subcycle (the PREP instantiation
// of the box TMA kernel: single rank, FP64, n_S = 6, constants in registers, 2 stages)
static bool prep_in_subcycle(const nxsdg_ctx* c) {
    return c->prep_kernel == 2 && c->d.nranks == 1 && c->P == 2 && c->NA == 6 && c->NS == 6 && !c->general &&
           !c->sphere && c->precision == 0 && c->variant == 0 && use_tma(c) && const_mode(c) == 1 &&
           c->stages == 2;
}

// the CG2/DG2 node pass as its own launch (kind 0 row-marching, 1 per-element threads)
static nxsdg_status launch_prep_nodes_q2(nxsdg_ctx* c, int kind) {
    PrepArgs a = prep_args(c);
    if (kind != 1) {
        const int pr_lo = a.node_row_begin >> 1, pr_hi = (a.node_row_end + 1) >> 1;
        // 64 element rows per warp; shorter on small meshes so the warps fill the device (16 resident per SM)
        int chunk = 64;
        while (chunk > 4 && (int64_t)prep_march_strips(c->d.nx) * ((pr_hi - pr_lo + chunk - 1) / chunk) <
                                (int64_t)(c->nsm > 0 ? c->nsm : 148) * 16)
            chunk /= 2;
        const int64_t warps = (int64_t)prep_march_strips(c->d.nx) * ((pr_hi - pr_lo + chunk - 1) / chunk);
        k_prep_nodes_march<<<(unsigned)((warps + 3) / 4), 128, 0, c->stream>>>(a, chunk);
    } else {
        const int rows = a.node_row_end - a.node_row_begin;
        dim3 bn(32, 4), gn((unsigned)((c->d.nx + 1 + 31) / 32), (unsigned)((rows / 2 + 1 + 3) / 4));
        k_prep_nodes_q2<<<gn, bn, 0, c->stream>>>(a);
    }
    LAUNCHED();
    return NXSDG_OK;
}
// a deferred node pass that cannot run inside a fused subcycle (unfused call, debug VELOCITY step, options
// changed since BEGIN_STEP): run it now as the separate pass (same inputs: v is still v^n)
static nxsdg_status flush_prep(nxsdg_ctx* c) {
    if (!c->prep_defer) return NXSDG_OK;
    c->prep_defer = false;
    return launch_prep_nodes_q2(c, 0);
}

static nxsdg_status dispatch_prep(nxsdg_ctx* c) {
    if (c->P == 2 && c->NA == 6) {   // structured (prep_q2.cuh); P_g only if the advection did not write it
        PrepArgs a = prep_args(c);
        if (prep_in_subcycle(c)) {   // the node pass runs in the next fused subcycle
            c->prep_defer = true;
        } else {
            nxsdg_status st = launch_prep_nodes_q2(c, c->prep_kernel == 1 ? 1 : 0);
            if (st) return st;
        }
        if (!c->pg_fresh) {
            dim3 be(128), ge((unsigned)((c->d.nx + 127) / 128), (unsigned)c->erows_local);
            k_prep_elems_q2<<<ge, be, 0, c->stream>>>(a);
            LAUNCHED();
        }
        return NXSDG_OK;
    }
    if (c->P == 1) return c->NA == 1 ? launch_prep<1, 1>(c) : launch_prep<1, 3>(c);
    if (c->NA == 1) return launch_prep<2, 1>(c);
    if (c->NA == 3) return launch_prep<2, 3>(c);
    return launch_prep<2, 6>(c);
}

static bool use_tma(const nxsdg_ctx* c);
// P2P + the TMA box kernel in FP64: the subcycle's halo rows travel as peer stores from the kernel
static bool p2p_fused_stores(const nxsdg_ctx* c) {
    return c->d.nranks > 1 && c->d.transport == NXSDG_TRANSPORT_P2P && c->p2p_ok && c->p2p_fused && use_tma(c) &&
           !c->general && c->precision == 0;
}

// Chunk height of the subcycle kernels' work units.  32 rows (tuned on C4 and its 8-GPU strips)
// unless a small mesh would then give fewer (strip, chunk) units than the 8 resident warps per SM can run at
// once: C2 (256^2) has 9 strips x 8 chunks = 72 units for 1184 warps, so each warp would march 33 rows while
// the others idle; halving down to 4 rows (one ring row each) spreads the rows over more warps.  Single rank
// only; every partition gives bitwise the same result (ring recomputation, fixed-order node sums).
static int chunk_rows(const nxsdg_ctx* c) {
    if (c->ty > 0) return c->ty;
    if (c->d.nranks > 1) return 32;   // row strips keep the tuned height (their boundary / interior split)
    const int64_t nstrips = (c->d.nx + 1 + 30) / 31, resident = (int64_t)(c->nsm > 0 ? c->nsm : 148) * 8;
    int ty = 32;
    while (ty > 4 && nstrips * ((c->nown + ty - 1) / ty) < resident) ty /= 2;
    return ty;
}

static SubArgs sub_args(nxsdg_ctx* c, int cv, int cs) {
    SubArgs a{};
    a.S_in = c->S[cs]; a.S_out = c->S[cs ^ 1]; a.Pg = c->Pg;
    a.vx_in = c->vx[cv]; a.vy_in = c->vy[cv]; a.vx_out = c->vx[cv ^ 1]; a.vy_out = c->vy[cv ^ 1];
    a.c1 = c->c1; a.rx0 = c->rx0; a.ry0 = c->ry0; a.cafo = c->cafo; a.ox = c->ox; a.oy = c->oy;
    a.eplane = c->eplane; a.npitch = c->npitch; a.epitch = c->epitch; a.nx = c->d.nx;
    a.nstrips = (c->d.nx + 1 + 30) / 31;
    a.pa = prep_args(c);
    a.ty = chunk_rows(c);
    a.erow_begin = c->glo; a.erow_end = c->glo + c->nown;
    a.bottom_boundary = c->r0 == 0;
    a.top_boundary = c->r1 == c->d.ny;
    const double hx = c->d.lx / c->d.nx, hy = c->d.ly / c->d.ny;
    a.ihx = 1.0 / hx; a.ihy = 1.0 / hy;
    if (c->sphere) {   // R#26: the row tables carry the latitude dependence
        a.ihx = 1.0 / (c->sph_R * c->sph_dlon); a.ihy = 1.0 / (c->sph_R * c->sph_dlat);
        a.sph_rows = c->sph_rows;
    }
    a.ainv = 1.0 / c->prm.alpha; a.fac = 1.0 - a.ainv;
    a.dmin2 = c->prm.DeltaMin * c->prm.DeltaMin;
    a.beta = c->prm.beta; a.b1 = 1.0 + c->prm.beta; a.kc = c->prm.dt * c->prm.f_c;
    a.repl = c->prm.replacement_pressure;
    a.chunk0 = 0; a.chunk_step = 1; a.nsel = (c->nown + a.ty - 1) / a.ty;
    if (p2p_fused_stores(c)) {   // the new state goes to v[cv ^ 1], S[cs ^ 1] on every rank
        const int iv = p2p_index(c, c->vx[cv ^ 1]), iw = p2p_index(c, c->vy[cv ^ 1]), is = p2p_index(c, c->S[cs ^ 1]);
        if (c->peer[1].on) {
            a.peer_vx_up = c->peer[1].buf[iv]; a.peer_vy_up = c->peer[1].buf[iw]; a.peer_S_up = c->peer[1].buf[is];
            a.up_node_row0 = c->P * (c->glo + c->nown - 1);
            a.up_elem_row = c->glo + c->nown - 1;
            a.peer_up_eplane = c->peer[1].g.eplane;
        }
        if (c->peer[0].on) {
            a.peer_vx_dn = c->peer[0].buf[iv]; a.peer_vy_dn = c->peer[0].buf[iw];
            a.dn_node_row = c->P * c->glo;
            a.dn_dst_row = c->P * (c->peer[0].g.glo + c->peer[0].g.nown);
        }
    }
    return a;
}

// chunk selections for the overlapped multi-rank subcycle
enum { SEL_ALL = 0, SEL_BOUNDARY = 1, SEL_INTERIOR = 2 };
static int n_chunks(const nxsdg_ctx* c) { const int ty = chunk_rows(c); return (c->nown + ty - 1) / ty; }
static void select_chunks(const nxsdg_ctx* c, int sel, SubArgs& a) {
    const int nc = n_chunks(c);
    if (sel == SEL_BOUNDARY) { a.chunk0 = 0; a.chunk_step = nc > 1 ? nc - 1 : 1; a.nsel = nc > 1 ? 2 : 1; }
    if (sel == SEL_INTERIOR) { a.chunk0 = 1; a.chunk_step = 1; a.nsel = nc - 2; }
}

// ---------------------------------------------------------------- TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// L2 sector promotion of the TMA loads: 64 B.  A box row of the S / P_g boxes is 272 B at a 16-B
// offset, so 256-B promotion fetches up to 768 B for it and relies on the neighbour strip to use the
// rest while it is still in L2; at 8 warps/SM that often fails: C4 launch DRAM reads 8.97 GB (256 B)
// vs 8.53 GB (128 B), sustained 1.910 vs 1.905 ms (profiles/tune_promo_r01.log).  Round 2: 64 B reads
// less again - DRAM traffic 1.046-1.054 x algorithmic against 1.054-1.097 x at 128 B over four ncu
// launches, sustained time and the advection / general-quad kernels unchanged
// (profiles/ab_l2_promotion_r02.log).  Experiment hook: NXSDG_TMA_L2_PROMOTION = 0 none, 1 64 B
// (default), 2 128 B, 3 256 B
static CUtensorMapL2promotion l2_promotion() {
    const char* e = getenv("NXSDG_TMA_L2_PROMOTION");
    const int v = e ? atoi(e) : 1;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

static bool encode(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                   const cuuint32_t* box) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(),
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static nxsdg_status build_maps(nxsdg_ctx* c) {
    if (c->maps_ok) return NXSDG_OK;
    const cuuint64_t nx = c->d.nx, er = c->erows_local, ncols = 2 * (cuuint64_t)c->d.nx + 1, nr = c->nrows_local;
    const cuuint64_t es[2] = {(cuuint64_t)c->epitch * 8, (cuuint64_t)c->eplane * 8};
    const cuuint64_t ns[2] = {(cuuint64_t)c->npitch * 8, (cuuint64_t)c->nn * 8};
    const cuuint64_t nS = 3 * (cuuint64_t)c->NS;
    const cuuint64_t dS[3] = {nx, er, nS}, dP[3] = {nx, er, 9}, dV[2] = {ncols, nr}, dC[3] = {ncols, nr, 6};
    const cuuint32_t bS[3] = {K2Cols<double>::E, 1, (cuuint32_t)nS}, bP[3] = {K2Cols<double>::E, 1, 9}, bV[2] = {K2_VCOLS, 3}, bV2[2] = {K2_VCOLS, 2},
                     bC[3] = {K2_CCOLS, 2, 6};
    for (int v = 0; v < 2; ++v)
        for (int s = 0; s < 2; ++s) {
            K2Maps& M = c->maps[v][s];
            bool ok = encode(&M.S, c->S[s], 3, dS, es, bS) && encode(&M.Pg, c->Pg, 3, dP, es, bP) &&
                      encode(&M.vx, c->vx[v], 2, dV, ns, bV) && encode(&M.vy, c->vy[v], 2, dV, ns, bV) &&
                      encode(&M.vx2, c->vx[v], 2, dV, ns, bV2) && encode(&M.vy2, c->vy[v], 2, dV, ns, bV2) &&
                      encode(&M.C, c->nodec, 3, dC, ns, bC);
            if (!ok) return fail(c, NXSDG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        }
    c->maps_ok = true;
    return NXSDG_OK;
}

static bool encode_f32(CUtensorMap* m, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                       const cuuint32_t* box) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(),
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NEXT-3: FP32 stress / P_g buffers and their tensor maps (v and node-constant maps as in FP64)
static nxsdg_status build_maps32(nxsdg_ctx* c) {
    nxsdg_status st = build_maps(c);
    if (st || c->maps32_ok) return st;
    const size_t ne = (size_t)c->eplane;
    for (int k = 0; k < 2; ++k)   // zeroed: the kernels never write the row / plane padding
        if (!c->S32[k]) {
            CU(cudaMalloc(&c->S32[k], 3 * (size_t)c->NS * ne * sizeof(float)));
            CU(cudaMemset(c->S32[k], 0, 3 * (size_t)c->NS * ne * sizeof(float)));
        }
    if (!c->Pg32) {
        CU(cudaMalloc(&c->Pg32, (size_t)c->NG * ne * sizeof(float)));
        CU(cudaMemset(c->Pg32, 0, (size_t)c->NG * ne * sizeof(float)));
    }
    const cuuint64_t nx = c->d.nx, er = c->erows_local;
    const cuuint64_t es[2] = {(cuuint64_t)c->epitch * 4, (cuuint64_t)c->eplane * 4};
    const cuuint64_t nS = 3 * (cuuint64_t)c->NS;
    const cuuint64_t dS[3] = {nx, er, nS}, dP[3] = {nx, er, 9};
    const cuuint32_t bS[3] = {K2Cols<float>::E, 1, (cuuint32_t)nS}, bP[3] = {K2Cols<float>::E, 1, 9};
    for (int v = 0; v < 2; ++v)
        for (int s = 0; s < 2; ++s) {
            K2Maps& M = c->maps32[v][s];
            M = c->maps[v][s];
            if (!encode_f32(&M.S, c->S32[s], dS, es, bS) || !encode_f32(&M.Pg, c->Pg32, dP, es, bP))
                return fail(c, NXSDG_ERR_CUDA, "cuTensorMapEncodeTiled (fp32) failed");
        }
    c->maps32_ok = true;
    return NXSDG_OK;
}

static nxsdg_status cvt(nxsdg_ctx* c, const double* src, float* dst, int64_t n) {
    k_cvt_d2f<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(src, dst, n);
    LAUNCHED();
    return NXSDG_OK;
}
static nxsdg_status cvt(nxsdg_ctx* c, const float* src, double* dst, int64_t n) {
    k_cvt_f2d<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(src, dst, n);
    LAUNCHED();
    return NXSDG_OK;
}

static bool use_tma(const nxsdg_ctx* c) { return c->P == 2 && c->variant == 0 && (!c->general || c->NS == 6); }
// NXSDG_OPT_PAIR_SUBCYCLES: the PAIR instantiation (single rank, FP64 box, n_S = 6, constants in registers)
static bool pair_ok(const nxsdg_ctx* c) {
    return c->pair && c->d.nranks == 1 && use_tma(c) && !c->general && !c->sphere && c->NS == 6 && c->precision == 0 &&
           const_mode(c) == 1 && c->stages <= 3;
}
// scratch state of pass A and the pass-B tensor maps over it (same geometry as S and v)
static nxsdg_status build_pair_maps(nxsdg_ctx* c) {
    if (c->mapsP_ok) return NXSDG_OK;
    const size_t ne = (size_t)c->eplane, nn = (size_t)c->npitch * c->nrows_local;
    if (!c->Sx) { CU(cudaMalloc(&c->Sx, 3 * (size_t)c->NS * ne * sizeof(double))); CU(cudaMemset(c->Sx, 0, 3 * (size_t)c->NS * ne * sizeof(double))); }
    if (!c->vxx) { CU(cudaMalloc(&c->vxx, nn * sizeof(double))); CU(cudaMemset(c->vxx, 0, nn * sizeof(double))); }
    if (!c->vyx) { CU(cudaMalloc(&c->vyx, nn * sizeof(double))); CU(cudaMemset(c->vyx, 0, nn * sizeof(double))); }
    const cuuint64_t nx = c->d.nx, er = c->erows_local, ncols = 2 * (cuuint64_t)c->d.nx + 1, nr = c->nrows_local;
    const cuuint64_t es[2] = {(cuuint64_t)c->epitch * 8, (cuuint64_t)c->eplane * 8};
    const cuuint64_t ns[2] = {(cuuint64_t)c->npitch * 8, (cuuint64_t)c->nn * 8};
    const cuuint64_t nS = 3 * (cuuint64_t)c->NS;
    const cuuint64_t dS[3] = {nx, er, nS}, dV[2] = {ncols, nr};
    const cuuint32_t bS[3] = {K2Cols<double>::E, 1, (cuuint32_t)nS}, bV[2] = {K2_VCOLS, 3}, bV2[2] = {K2_VCOLS, 2};
    K2Maps& M = c->mapsP;
    M = c->maps[0][0];   // P_g and the constants maps are the same; S and v point at the scratch
    if (!(encode(&M.S, c->Sx, 3, dS, es, bS) && encode(&M.vx, c->vxx, 2, dV, ns, bV) && encode(&M.vy, c->vyx, 2, dV, ns, bV) &&
          encode(&M.vx2, c->vxx, 2, dV, ns, bV2) && encode(&M.vy2, c->vyx, 2, dV, ns, bV2)))
        return fail(c, NXSDG_ERR_CUDA, "cuTensorMapEncodeTiled (pair scratch) failed");
    c->mapsP_ok = true;
    return NXSDG_OK;
}
// Tail split of a persistent launch with twarps warps: the last chunks become ~8-row sub-units, enough of
// them (2 x twarps) that every warp's final unit is short, so the warps finish within ~8 jobs of each
// other instead of ~ty (the idle tail of a launch is half a unit on average)
static SubArgs launch_args(const nxsdg_ctx* c, const SubArgs& a0, int64_t twarps) {
    SubArgs a = a0;
    a.ntail = 0; a.qtail = 1;
    a.l2_hints = c->l2_policy;
    a.vcarry = c->v_carry;
    const int q = a.ty / 8;
    if (!c->tail_split || !a.work_counter || q < 2 || a.nsel < 1) return a;
    const int64_t need = (2 * twarps + (int64_t)a.nstrips * q - 1) / ((int64_t)a.nstrips * q);
    a.ntail = (int)std::min<int64_t>(a.nsel, need);
    a.qtail = q;
    return a;
}
// Defaults of the box kernel, tuned on C4 under sustained load (scripts/tune_sustained.py)
// FP64 storage, n_S = 6: node constants in registers, 4 CTAs/SM (C4: 1.87-1.96 ms vs 1.95-2.11 ms per
// subcycle with the fifth TMA box at 3 or 2 CTAs/SM).  n_S = 8 (18.4 KB stages, 240 registers with the
// constants in registers): the TMA box at 2 CTAs/SM, 2.12 ms vs 2.22 ms.  FP32 storage keeps the box (its
// stages are small already: 1.48 vs 1.58 ms).  profiles/tune_sustained_r01.log, tune_l2_policy_r01.log
// n_S = 8: late constants (mode 2) at 4 CTAs/SM, 2.20 ms vs 2.31 ms with the box at 2 CTAs/SM; n_S = 6: the
// register prefetch (mode 1) stays ahead of mode 2 (1.91 vs 1.99 ms; profiles/tune_box_late_const_r01.log)
static int const_mode(const nxsdg_ctx* c) {
    if (c->const_regs >= 0) return c->const_regs;
    if (c->precision != 0) return 0;
    return c->NS == 8 ? 2 : 1;
}
// general-quad fused kernel: node constants loaded late into the consumed S / P_g region (1, default: 4 CTAs/SM,
// sustained C4 2.75 ms per subcycle) or as a box of the stage (0: 3 CTAs/SM, 2.88 ms;
// profiles/tune_gen_late_const_r01.log)
static bool gen_late_const(const nxsdg_ctx* c) { return c->const_regs < 0 ? true : c->const_regs >= 1; }
static int default_ctas(size_t sf_bytes, bool cl, int ns) { return cl ? 4 : (sf_bytes == 8 ? (ns == 8 ? 2 : 3) : 4); }

// NEXT-1: the fused general-quad subcycle stages the vertex rows and the lumped node masses too
static nxsdg_status build_gen_maps(nxsdg_ctx* c) {
    nxsdg_status st = build_maps(c);
    if (st || c->gen_maps_ok) return st;
    const cuuint64_t dX[2] = {2 * (cuuint64_t)(c->d.nx + 1), (cuuint64_t)(c->d.ny + 1)};
    const cuuint64_t sX[1] = {2 * (cuuint64_t)(c->d.nx + 1) * 8};
    const cuuint32_t bX[2] = {K2_VCOLS, 2};
    const cuuint64_t dM[2] = {2 * (cuuint64_t)c->d.nx + 1, (cuuint64_t)c->nrows_local};
    const cuuint64_t sM[1] = {(cuuint64_t)c->npitch * 8};
    const cuuint32_t bM[2] = {K2_CCOLS, 2};
    for (int v = 0; v < 2; ++v)
        for (int s2 = 0; s2 < 2; ++s2) {
            K2GenMaps& G = c->gen_maps[v][s2];
            const K2Maps& B = c->maps[v][s2];
            G.S = B.S; G.Pg = B.Pg; G.vx = B.vx; G.vy = B.vy; G.C = B.C;
            if (!encode(&G.X, c->verts, 2, dX, sX, bX) || !encode(&G.M, c->imlump, 2, dM, sM, bM))
                return fail(c, NXSDG_ERR_CUDA, "cuTensorMapEncodeTiled (general) failed");
        }
    c->gen_maps_ok = true;
    return NXSDG_OK;
}

// per-device "function attribute already set" flags (ordinals >= 64 set the attribute on every launch)
static inline bool dev_bit_test(uint64_t m, int dev) { return dev >= 0 && dev < 64 && ((m >> dev) & 1u); }
static inline void dev_bit_set(uint64_t& m, int dev) { if (dev >= 0 && dev < 64) m |= uint64_t(1) << dev; }

template <bool R, int ST, bool LC = false>
static nxsdg_status launch_gen_t(nxsdg_ctx* c, int cv, int cs, const SubArgs& a) {
    const size_t smem = (size_t)K2_WARPS * ST *
                        (sizeof(typename K2GenStageSel<LC>::T) + 2 * sizeof(uint64_t) + sizeof(int4));
    static uint64_t attr_set = 0;   // the attribute is per device: one bit per ordinal
    if (!dev_bit_test(attr_set, c->d.device)) {
        CU(cudaFuncSetAttribute(k_subcycle_gen<R, ST, LC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dev_bit_set(attr_set, c->d.device);
    }
    int nsm = 148, occ = 1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->d.device);
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_subcycle_gen<R, ST, LC>, 32 * K2_WARPS, smem));
    // tuned on C4 (profiles/tune_gen_r01.log, tune_gen_sustained_r01.log): 3 CTAs/SM with the constant box,
    // 4 with the late constants (smaller stages)
    const int cap = c->ctas_per_sm < 0 ? (LC ? 4 : 3) : c->ctas_per_sm;
    if (cap > 0) occ = std::min(occ, cap);
    const int64_t units = (int64_t)a.nstrips * a.nsel;
    const int64_t want = (units + K2_WARPS - 1) / K2_WARPS;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * std::max(occ, 1)));
    k_subcycle_gen<R, ST, LC><<<blocks, 32 * K2_WARPS, smem, c->stream>>>(c->gen_maps[cv][cs],
                                                                       launch_args(c, a, (int64_t)blocks * K2_WARPS));
    return NXSDG_OK;
}

template <bool R, int ST, typename SF, typename CT = double, int NS = 6, bool CL = false, bool LC = false, bool SPH = false,
          bool PREP = false, bool PAIR = false>
static nxsdg_status launch_tma_t(nxsdg_ctx* c, int cv, int cs, const SubArgs& a) {
    // a.work_counter must be zero when the kernel starts (memset by the caller / graph)
    using Stage = typename K2StageSel<SF, NS, CL || LC>::T;
    const size_t smem = (size_t)K2_WARPS * ST * (sizeof(Stage) + 2 * sizeof(uint64_t) + sizeof(int4));
    static uint64_t attr_set = 0;   // the attribute is per device: one bit per ordinal
    if (!dev_bit_test(attr_set, c->d.device)) {
        CU(cudaFuncSetAttribute(k_subcycle_tma<R, ST, SF, CT, NS, CL, LC, SPH, PREP, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        dev_bit_set(attr_set, c->d.device);
    }
    int nsm = 148, occ = 1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->d.device);
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_subcycle_tma<R, ST, SF, CT, NS, CL, LC, SPH, PREP, PAIR>, 32 * K2_WARPS,
                                                     smem));
    const int cap = c->ctas_per_sm < 0 ? default_ctas(sizeof(SF), CL || LC, NS) : c->ctas_per_sm;
    if (cap > 0) occ = std::min(occ, cap);
    const int64_t units = (int64_t)a.nstrips * a.nsel;
    const int64_t want = (units + K2_WARPS - 1) / K2_WARPS;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * std::max(occ, 1)));
    const K2Maps& mp = sizeof(SF) == 8 ? c->maps[cv][cs] : c->maps32[cv][cs];
    typename K2PassB<PAIR>::T mb{};
    if constexpr (PAIR) mb = c->mapsP;
    const SubArgs la = launch_args(c, a, (int64_t)blocks * K2_WARPS);
    if (c->pdl_now) {   // programmatic dependent launch: may overlap the previous subcycle's tail (run_graph)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(32 * K2_WARPS); cfg.dynamicSmemBytes = smem; cfg.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        CU(cudaLaunchKernelEx(&cfg, k_subcycle_tma<R, ST, SF, CT, NS, CL, LC, SPH, PREP, PAIR>, mp, mb, la));
    } else {
        k_subcycle_tma<R, ST, SF, CT, NS, CL, LC, SPH, PREP, PAIR><<<blocks, 32 * K2_WARPS, smem, c->stream>>>(mp, mb, la);
    }
    return NXSDG_OK;
}
// stages x replacement pressure x node-constant staging (TMA box | registers)
// stages x replacement pressure x node-constant mode (0 TMA box | 1 registers | 2 late TMA, FP64 only)
template <typename SF, typename CT, int NS, int ST>
static nxsdg_status launch_tma_mode(nxsdg_ctx* c, int cv, int cs, const SubArgs& a, int mode) {
    if (mode == 1) return a.repl ? launch_tma_t<true, ST, SF, CT, NS, true>(c, cv, cs, a)
                                 : launch_tma_t<false, ST, SF, CT, NS, true>(c, cv, cs, a);
    if constexpr (sizeof(SF) == 8) {
        if (mode == 2) return a.repl ? launch_tma_t<true, ST, SF, CT, NS, false, true>(c, cv, cs, a)
                                     : launch_tma_t<false, ST, SF, CT, NS, false, true>(c, cv, cs, a);
    }
    return a.repl ? launch_tma_t<true, ST, SF, CT, NS>(c, cv, cs, a) : launch_tma_t<false, ST, SF, CT, NS>(c, cv, cs, a);
}
template <typename SF, typename CT = double, int NS = 6>
static nxsdg_status launch_tma_sel(nxsdg_ctx* c, int cv, int cs, const SubArgs& a) {
    if constexpr (sizeof(SF) == 8 && sizeof(CT) == 8 && NS == 6) {
        if (c->sphere) {   // R#26: node constants in registers, 2 or 3 stages
            if (c->stages >= 3) return a.repl ? launch_tma_t<true, 3, SF, CT, 6, true, false, true>(c, cv, cs, a)
                                              : launch_tma_t<false, 3, SF, CT, 6, true, false, true>(c, cv, cs, a);
            return a.repl ? launch_tma_t<true, 2, SF, CT, 6, true, false, true>(c, cv, cs, a)
                          : launch_tma_t<false, 2, SF, CT, 6, true, false, true>(c, cv, cs, a);
        }
    }
    int mode = const_mode(c);
    if constexpr (sizeof(SF) == 8 && sizeof(CT) == 8 && NS == 6) {
        if (c->pair_now) {   // two subcycles in one launch (pair_ok): 29-column strips, scratch outputs of pass A
            SubArgs b = a;
            b.nstrips = c->d.nx / 29 + 1;
            b.Sx = c->Sx; b.vxx = c->vxx; b.vyx = c->vyx;
            if (c->stages >= 3) return b.repl ? launch_tma_t<true, 3, SF, CT, 6, true, false, false, false, true>(c, cv, cs, b)
                                              : launch_tma_t<false, 3, SF, CT, 6, true, false, false, false, true>(c, cv, cs, b);
            return b.repl ? launch_tma_t<true, 2, SF, CT, 6, true, false, false, false, true>(c, cv, cs, b)
                          : launch_tma_t<false, 2, SF, CT, 6, true, false, false, false, true>(c, cv, cs, b);
        }
        if (c->prep_now) {   // the outer step's first subcycle forms the node constants (prep_in_subcycle)
            if (mode != 1 || c->stages != 2) return fail(c, NXSDG_ERR_STATE, "fused prep launch without its configuration");
            return a.repl ? launch_tma_t<true, 2, SF, CT, 6, true, false, false, true>(c, cv, cs, a)
                          : launch_tma_t<false, 2, SF, CT, 6, true, false, false, true>(c, cv, cs, a);
        }
    }
    if (sizeof(SF) != 8 && mode == 2) return fail(c, NXSDG_ERR_UNSUPPORTED, "late node constants need FP64 storage");
    if (c->stages == 2) return launch_tma_mode<SF, CT, NS, 2>(c, cv, cs, a, mode);
    if (c->stages == 3) return launch_tma_mode<SF, CT, NS, 3>(c, cv, cs, a, mode);
    if constexpr (sizeof(SF) == 8) return launch_tma_mode<SF, CT, NS, 4>(c, cv, cs, a, mode);
    return fail(c, NXSDG_ERR_INVALID_ARG, "stages %d with FP32 storage", c->stages);
}

static nxsdg_status ensure_counters(nxsdg_ctx* c, int n) {
    if (c->ncounters >= n) return NXSDG_OK;
    // cached graphs captured the old buffer (memset node + kernel argument): drop them (this waits
    // for any replay still in flight) before the buffer goes away
    drop_graphs(c);
    if (c->counters) cudaFree(c->counters);
    c->counters = nullptr; c->ncounters = 0;
    CU(cudaMalloc(&c->counters, sizeof(int) * (size_t)std::max(n, 128)));
    c->ncounters = std::max(n, 128);
    return NXSDG_OK;
}

// slot < 0: direct launch, zero slot 0 first; slot >= 0: inside a graph whose first node zeroes all slots
static nxsdg_status launch_tma(nxsdg_ctx* c, int cv, int cs, int slot = -1, int sel = SEL_ALL) {
    nxsdg_status st = build_maps(c);
    if (st) return st;
    SubArgs a = sub_args(c, cv, cs);
    select_chunks(c, sel, a);
    if (a.nsel <= 0) return NXSDG_OK;
    if (slot < 0) {
        if ((st = ensure_counters(c, 1))) return st;
        CU(cudaMemsetAsync(c->counters, 0, sizeof(int), c->stream));
        slot = 0;
    }
    a.work_counter = c->dynamic ? c->counters + slot : nullptr;
    if (c->general) {
        if ((st = build_gen_maps(c))) return st;
        const bool lc = gen_late_const(c);
        const int st = std::min(c->stages, 3);   // the general kernel is instantiated for 2 and 3 stages
        switch ((st * 2 + (a.repl ? 1 : 0)) * 2 + (lc ? 1 : 0)) {
            case 8: return launch_gen_t<false, 2, false>(c, cv, cs, a);
            case 9: return launch_gen_t<false, 2, true>(c, cv, cs, a);
            case 10: return launch_gen_t<true, 2, false>(c, cv, cs, a);
            case 11: return launch_gen_t<true, 2, true>(c, cv, cs, a);
            case 12: return launch_gen_t<false, 3, false>(c, cv, cs, a);
            case 13: return launch_gen_t<false, 3, true>(c, cv, cs, a);
            case 14: return launch_gen_t<true, 3, false>(c, cv, cs, a);
            default: return launch_gen_t<true, 3, true>(c, cv, cs, a);
        }
    }
    if (c->precision == 2) {
        if ((st = build_maps32(c))) return st;
        a.S_out = reinterpret_cast<double*>(c->S32[cs ^ 1]);   // FP32 storage, FP32 stress arithmetic
        return launch_tma_sel<float, float>(c, cv, cs, a);
    }
    if (c->precision == 1) {
        if ((st = build_maps32(c))) return st;
        a.S_out = reinterpret_cast<double*>(c->S32[cs ^ 1]);   // the kernel stores FP32
        return launch_tma_sel<float>(c, cv, cs, a);
    }
    if (c->NS == 8) return launch_tma_sel<double, double, 8>(c, cv, cs, a);
    return launch_tma_sel<double>(c, cv, cs, a);
}

// One fused subcycle launch over the selected chunks (no ping-pong flip); slot: the launch's work
// counter inside a graph (-1: direct launch, the counter is zeroed first).
static nxsdg_status launch_subcycle_sel(nxsdg_ctx* c, int sel, int slot = -1) {
    if (use_tma(c)) {
        nxsdg_status st = launch_tma(c, c->cv, c->cs, slot, sel);
        if (st) return st;
    } else {
        SubArgs a = sub_args(c, c->cv, c->cs);
        select_chunks(c, sel, a);
        if (a.nsel <= 0) return NXSDG_OK;
        const int64_t warps = (int64_t)a.nstrips * a.nsel;
        const unsigned blocks = (unsigned)((warps + 3) / 4);
        if (c->P == 1) k_subcycle<1><<<blocks, 128, 0, c->stream>>>(a);
        else if (c->NS == 8) k_subcycle<2, 8><<<blocks, 128, 0, c->stream>>>(a);
        else k_subcycle<2><<<blocks, 128, 0, c->stream>>>(a);
    }
    LAUNCHED();
    return NXSDG_OK;
}

static nxsdg_status launch_subcycle(nxsdg_ctx* c, int slot = -1) {
    nxsdg_status st = launch_subcycle_sel(c, SEL_ALL, slot);
    if (st) return st;
    c->cv ^= 1; c->cs ^= 1;
    return NXSDG_OK;
}

static nxsdg_status ensure_halo_stream(nxsdg_ctx* c) {
    if (!c->hstream) {
        CU(cudaStreamCreateWithFlags(&c->hstream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&c->ev_bnd, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming));
    }
    return NXSDG_OK;
}

// Multi-rank subcycle with overlap: boundary chunks (first and last chunk rows,
// which produce every row a neighbour needs) -> event -> halo exchange on the halo stream,
// concurrently the interior chunks on the main stream -> join.  Exactly one exchange per subcycle.
// slot0 >= 0: inside a graph capture, the launches use work-counter slots slot0, slot0 + 1.
static nxsdg_status subcycle_overlapped(nxsdg_ctx* c, int slot0 = -1) {
    nxsdg_status st;
    if (n_chunks(c) < 3) {
        if ((st = launch_subcycle(c, slot0))) return st;
        return halo(c, p2p_fused_stores(c) ? 0u : (uint32_t)(NXSDG_HALO_V | NXSDG_HALO_S));
    }
    if ((st = ensure_halo_stream(c))) return st;
    if ((st = launch_subcycle_sel(c, SEL_BOUNDARY, slot0))) return st;
    c->cv ^= 1; c->cs ^= 1;                      // the exchange moves rows of the new state
    CU(cudaEventRecord(c->ev_bnd, c->stream));
    CU(cudaStreamWaitEvent(c->hstream, c->ev_bnd, 0));
    if ((st = halo_on(c, p2p_fused_stores(c) ? 0u : (uint32_t)(NXSDG_HALO_V | NXSDG_HALO_S), c->hstream))) return st;
    CU(cudaEventRecord(c->ev_x, c->hstream));
    c->cv ^= 1; c->cs ^= 1;                      // interior reads the old state
    if ((st = launch_subcycle_sel(c, SEL_INTERIOR, slot0 < 0 ? -1 : slot0 + 1))) return st;
    c->cv ^= 1; c->cs ^= 1;
    CU(cudaStreamWaitEvent(c->stream, c->ev_x, 0));
    return NXSDG_OK;
}

static StepArgs step_args(nxsdg_ctx* c) {
    StepArgs a{};
    a.vx_in = c->vx[c->cv]; a.vy_in = c->vy[c->cv]; a.vx_out = c->vx[c->cv ^ 1]; a.vy_out = c->vy[c->cv ^ 1];
    a.S = c->S[c->cs]; a.E = c->E; a.Fx = c->Fx; a.Fy = c->Fy; a.H = c->H; a.A = c->A;
    a.c1 = c->c1; a.rx0 = c->rx0; a.ry0 = c->ry0; a.cafo = c->cafo; a.ox = c->ox; a.oy = c->oy;
    a.eplane = c->eplane; a.npitch = c->npitch; a.epitch = c->epitch; a.nx = c->d.nx;
    a.erow_begin = c->glo; a.erow_end = c->glo + c->nown; a.elem_rows_with_nodes = c->glo + c->nown;
    a.node_row_begin = c->P * c->glo; a.node_row_end = (int)(c->P * c->glo + owned_node_rows(c));
    a.node_row_global0 = (int)(c->P * (c->r0 - c->glo));
    a.node_rows_global = c->P * c->d.ny + 1;
    const double hx = c->d.lx / c->d.nx, hy = c->d.ly / c->d.ny;
    a.ihx = 1.0 / hx; a.ihy = 1.0 / hy; a.area = hx * hy;
    a.ainv = 1.0 / c->prm.alpha; a.fac = 1.0 - a.ainv;
    a.dmin2 = c->prm.DeltaMin * c->prm.DeltaMin;
    a.beta = c->prm.beta; a.b1 = 1.0 + c->prm.beta; a.kc = c->prm.dt * c->prm.f_c;
    a.Pstar = c->prm.Pstar; a.C_conc = c->prm.C_conc; a.repl = c->prm.replacement_pressure;
    return a;
}

template <int P, int NA, int NS = Deg<P>::NS>
static nxsdg_status launch_step_t(nxsdg_ctx* c, nxsdg_step st) {
    StepArgs a = step_args(c);
    dim3 be(128), ge((unsigned)((c->d.nx + 127) / 128), (unsigned)c->nown);
    dim3 bn(128), gn((unsigned)((P * c->d.nx + 1 + 127) / 128), (unsigned)(a.node_row_end - a.node_row_begin));
    switch (st) {
        case NXSDG_STEP_STRAIN: k_strain<P, NS><<<ge, be, 0, c->stream>>>(a); break;
        case NXSDG_STEP_STRESS: k_stress<P, NA, NS><<<ge, be, 0, c->stream>>>(a); break;
        case NXSDG_STEP_DIVERGENCE: k_divergence<P, NS><<<gn, bn, 0, c->stream>>>(a); break;
        case NXSDG_STEP_VELOCITY: k_velocity<P><<<gn, bn, 0, c->stream>>>(a); break;
    }
    LAUNCHED();
    if (st == NXSDG_STEP_VELOCITY) c->cv ^= 1;   // S is updated in place, v ping-pongs
    return NXSDG_OK;
}

static nxsdg_status launch_step(nxsdg_ctx* c, nxsdg_step st) {
    if (c->P == 1) return c->NA == 1 ? launch_step_t<1, 1>(c, st) : launch_step_t<1, 3>(c, st);
    if (c->NS == 8) {
        if (c->NA == 1) return launch_step_t<2, 1, 8>(c, st);
        if (c->NA == 3) return launch_step_t<2, 3, 8>(c, st);
        return launch_step_t<2, 6, 8>(c, st);
    }
    if (c->NA == 1) return launch_step_t<2, 1>(c, st);
    if (c->NA == 3) return launch_step_t<2, 3>(c, st);
    return launch_step_t<2, 6>(c, st);
}

// ---------------------------------------------------------------- compute API
static nxsdg_status begin_step(nxsdg_ctx* c) {
    NvtxRange nv("nxsdg begin_step (prep)");
    if (!c->forcing_set) return fail(c, NXSDG_ERR_STATE, "forcing not set");
    nxsdg_status s;
    if ((s = consume_forcing(c))) return s;
    if ((s = halo(c, NXSDG_HALO_V | NXSDG_HALO_S | NXSDG_HALO_AH))) return s;
    if ((s = dispatch_prep(c))) return s;
    c->prepped = true;
    return NXSDG_OK;
}

static nxsdg_status check_substeps(nxsdg_ctx* c, int32_t n, uint32_t flags) {
    if (n < 0 || (flags & ~(uint32_t)(NXSDG_BEGIN_STEP | NXSDG_UNFUSED))) return fail(c, NXSDG_ERR_INVALID_ARG, "bad n/flags");
    if (c->d.bc != NXSDG_BC_CLOSED) return fail(c, NXSDG_ERR_UNSUPPORTED, "mEVP substeps need the closed box");
    if (c->general && !(flags & NXSDG_UNFUSED) && n > 0 && !use_tma(c))
        return fail(c, NXSDG_ERR_UNSUPPORTED, "general quads: the fused subcycle needs CG2/DG2 and the TMA kernel; "
                                              "use NXSDG_UNFUSED");
    if (c->sphere && n > 0 && ((flags & NXSDG_UNFUSED) || !use_tma(c) || c->precision != 0))
        return fail(c, NXSDG_ERR_UNSUPPORTED, "sphere: fused FP64 TMA subcycles only");
    if (!c->forcing_set) return fail(c, NXSDG_ERR_STATE, "forcing not set");
    if (!(flags & NXSDG_BEGIN_STEP) && !c->prepped) return fail(c, NXSDG_ERR_STATE, "first call of an outer step needs NXSDG_BEGIN_STEP");
    return NXSDG_OK;
}

static nxsdg_status one_subcycle(nxsdg_ctx* c, bool unfused) {
    nxsdg_status s;
    if (!unfused) {
        if (c->d.nranks > 1 && c->d.transport != NXSDG_TRANSPORT_LOOPBACK) return subcycle_overlapped(c);
        if ((s = launch_subcycle(c))) return s;
        return halo(c, NXSDG_HALO_V | NXSDG_HALO_S);
    }
    if ((s = ensure_debug_buffers(c))) return s;
    if (c->general) {
        if ((s = general_step(c, NXSDG_STEP_STRAIN))) return s;
        if ((s = general_stress(c))) return s;
        if ((s = general_step(c, NXSDG_STEP_DIVERGENCE))) return s;
        return general_step(c, NXSDG_STEP_VELOCITY);
    }
    if ((s = launch_step(c, NXSDG_STEP_STRAIN))) return s;
    if ((s = launch_step(c, NXSDG_STEP_STRESS))) return s;
    if ((s = halo(c, NXSDG_HALO_S))) return s;
    if ((s = launch_step(c, NXSDG_STEP_DIVERGENCE))) return s;
    if ((s = launch_step(c, NXSDG_STEP_VELOCITY))) return s;
    return halo(c, NXSDG_HALO_V);
}

// Capture n fused subcycles into a CUDA graph (nranks == 1) and replay it.
static nxsdg_status run_graph(nxsdg_ctx* c, int n) {
    const bool pr = n >= 2 && pair_ok(c);   // two subcycles per launch, an odd count ends with a single one
    const int nl = pr ? n / 2 + (n & 1) : n;
    auto key = std::make_tuple(n, c->cv, c->cs + 2 * c->precision + (pr ? 16 : 0));
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
        cudaGraph_t g;
        if (use_tma(c)) {   // descriptors and counters are created outside the capture
            nxsdg_status st = build_maps(c);
            if (!st && pr) st = build_pair_maps(c);
            if (!st) st = ensure_counters(c, n);
            if (st) return st;
        }
        CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        int cv = c->cv, cs = c->cs;
        if (use_tma(c)) {
            cudaError_t me = cudaMemsetAsync(c->counters, 0, sizeof(int) * (size_t)n, c->stream);
            if (me != cudaSuccess) {   // end (and discard) the capture so the stream stays usable
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(c->stream, &junk);
                if (junk) cudaGraphDestroy(junk);
                cudaGetLastError();
                return fail(c, NXSDG_ERR_CUDA, "graph capture memset: %s", cudaGetErrorString(me));
            }
        }
        for (int i = 0, slot = 0; i < n; ++slot) {
            if (use_tma(c)) {
                c->pair_now = pr && n - i >= 2;
                c->pdl_now = c->pdl && slot > 0;   // the previous node is a subcycle launch
                nxsdg_status st = launch_tma(c, cv, cs, slot);
                i += c->pair_now ? 2 : 1;
                c->pair_now = false;
                c->pdl_now = false;
                if (st) { cudaGraph_t junk; cudaStreamEndCapture(c->stream, &junk); if (junk) cudaGraphDestroy(junk); return st; }
            } else {
                ++i;
                SubArgs a = sub_args(c, cv, cs);
                const int nchunks = (c->nown + a.ty - 1) / a.ty;
                const unsigned blocks = (unsigned)(((int64_t)a.nstrips * nchunks + 3) / 4);
                if (c->P == 1) k_subcycle<1><<<blocks, 128, 0, c->stream>>>(a);
                else if (c->NS == 8) k_subcycle<2, 8><<<blocks, 128, 0, c->stream>>>(a);
                else k_subcycle<2><<<blocks, 128, 0, c->stream>>>(a);
            }
            cv ^= 1; cs ^= 1;
        }
        cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        if (e != cudaSuccess) return fail(c, NXSDG_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
        cudaGraphExec_t ge;
        e = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(c, NXSDG_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
        it = c->graphs.emplace(key, nxsdg_ctx::Graph{ge, nl}).first;
    }
    CU(cudaGraphLaunch(it->second.exec, c->stream));
    c->launches += it->second.launches;
    if (nl & 1) { c->cv ^= 1; c->cs ^= 1; }   // one ping-pong flip per launch (a pair flips once)
    return NXSDG_OK;
}

// The multi-rank subcycle graph: default on for the P2P transport between processes (the one-process-per-GPU
// deployment); off by default for NCCL (a captured NCCL exchange hung with the socket transport of the
// one-GPU test topology) and always off for ranks that share this process and device
// (nxsdg_p2p_connect_local: a single-GPU test topology, where graph replays of several ranks hung the device)
static bool mr_graph_on(const nxsdg_ctx* c) {
    if (c->d.nranks < 2 || c->d.transport == NXSDG_TRANSPORT_LOOPBACK || c->inproc || !c->mr_graph_note.empty())
        return false;
    if (c->mr_graph >= 0) return c->mr_graph == 1;
    return c->d.transport == NXSDG_TRANSPORT_P2P;
}

// Multi-rank (P2P / NCCL row strips): capture n overlapped subcycles - boundary launch, exchange on
// the halo stream (fused peer stores + flag handshake, copy-engine peer copies, or NCCL send/recv),
// interior launch, join - in one CUDA graph and replay it: one host crossing per call instead of
// ~8 API calls per subcycle.  The P2P handshake uses constant flag values (halo_p2p), so replays
// are exact; the graph is keyed by the ping-pong parities and the P2P slot parity it starts from.
// Returns NXSDG_ERR_UNSUPPORTED (state unchanged) if the capture itself is refused, so the caller can
// issue the subcycles from the host instead.
static nxsdg_status run_graph_multirank(nxsdg_ctx* c, int n) {
    NvtxRange nv("nxsdg multi-rank subcycle graph");
    const int par = (int)(c->p2p_seq & 1u);
    auto key = std::make_tuple(n, c->cv, c->cs + 8 * par + 16);
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
        nxsdg_status st;
        if (use_tma(c) && (st = build_maps(c))) return st;
        if ((st = ensure_counters(c, 2 * n))) return st;
        if ((st = ensure_halo_stream(c))) return st;
        if (c->d.transport == NXSDG_TRANSPORT_NCCL && (st = ensure_halo_staging(c))) return st;
        const int cv0 = c->cv, cs0 = c->cs;
        const uint32_t seq0 = c->p2p_seq;
        const int64_t l0 = c->launches;
        CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        cudaError_t me = use_tma(c) ? cudaMemsetAsync(c->counters, 0, sizeof(int) * (size_t)(2 * n), c->stream)
                                    : cudaSuccess;
        st = me == cudaSuccess ? NXSDG_OK : NXSDG_ERR_CUDA;
        for (int i = 0; i < n && !st; ++i) st = subcycle_overlapped(c, 2 * i);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        const int64_t nl = c->launches - l0;
        c->cv = cv0; c->cs = cs0; c->p2p_seq = seq0; c->launches = l0;   // nothing ran yet
        if (st || e != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            c->mr_graph_note = st ? c->err : std::string("capture: ") + cudaGetErrorString(e);
            // an API call refused inside the capture is not a device fault: un-poison; the host-issued
            // fallback reports any real error again
            c->err.clear();
            c->poisoned = false;
            return NXSDG_ERR_UNSUPPORTED;
        }
        cudaGraphExec_t ge;
        e = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            cudaGetLastError();
            c->mr_graph_note = std::string("instantiate: ") + cudaGetErrorString(e);
            return NXSDG_ERR_UNSUPPORTED;
        }
        it = c->graphs.emplace(key, nxsdg_ctx::Graph{ge, nl}).first;
    }
    CU(cudaGraphLaunch(it->second.exec, c->stream));
    c->launches += it->second.launches;
    if (n & 1) { c->cv ^= 1; c->cs ^= 1; }
    if (c->d.transport == NXSDG_TRANSPORT_P2P) c->p2p_seq += (uint32_t)n;
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_mevp_substeps(nxsdg_ctx* c, int32_t n, uint32_t flags) {
    GUARD(c);
    NvtxRange nv("nxsdg_mevp_substeps");
    nxsdg_status s = check_substeps(c, n, flags);
    if (s) return s;
    if (c->d.nranks > 1 && c->d.transport == NXSDG_TRANSPORT_LOOPBACK)
        return fail(c, NXSDG_ERR_STATE, "loopback ranks step through nxsdg_group_mevp_substeps");
    if ((flags & NXSDG_BEGIN_STEP) && (s = begin_step(c))) return s;
    const bool unfused = flags & NXSDG_UNFUSED;
    if (c->prep_defer && n > 0) {
        if (!unfused && prep_in_subcycle(c)) {   // subcycle 1 forms the node constants (direct launch)
            c->prep_now = true;
            s = launch_subcycle(c);
            c->prep_now = false;
            c->prep_defer = false;
            if (s) return s;
            if (--n == 0) return NXSDG_OK;
        } else if ((s = flush_prep(c))) return s;
    }
    if (!unfused && c->d.nranks == 1 && n > 0 && c->precision >= 1 && use_tma(c)) {
        // NEXT-3: the FP64 state is the ABI-visible copy; the subcycles run on FP32 S / P_g
        if ((s = build_maps32(c))) return s;
        const int64_t nS = 3 * (int64_t)c->NS * c->eplane;
        if ((flags & NXSDG_BEGIN_STEP) || !c->pg32_ok) {
            if ((s = cvt(c, c->Pg, c->Pg32, (int64_t)c->NG * c->eplane))) return s;
            c->pg32_ok = true;
        }
        if ((s = cvt(c, c->S[c->cs], c->S32[c->cs], nS))) return s;
        if ((s = run_graph(c, n))) return s;
        return cvt(c, c->S32[c->cs], c->S[c->cs], nS);
    }
    if (!unfused && c->d.nranks == 1 && n > 0) return run_graph(c, n);
    if (!unfused && c->d.nranks > 1 && n > 0 && mr_graph_on(c) && c->precision == 0) {
        s = run_graph_multirank(c, n);
        if (s != NXSDG_ERR_UNSUPPORTED) return s;   // else: capture refused (noted), issue from the host
    }
    for (int i = 0; i < n; ++i)
        if ((s = one_subcycle(c, unfused))) return s;
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_run_step(nxsdg_ctx* c, nxsdg_step st) {
    GUARD(c);
    if (st < NXSDG_STEP_STRAIN || st > NXSDG_STEP_VELOCITY) return fail(c, NXSDG_ERR_INVALID_ARG, "bad step");
    if (st == NXSDG_STEP_VELOCITY && !c->prepped)
        return fail(c, NXSDG_ERR_STATE, "needs a BEGIN_STEP (nxsdg_mevp_substeps(ctx, 0, NXSDG_BEGIN_STEP))");
    if (st == NXSDG_STEP_VELOCITY) {
        nxsdg_status fs = flush_prep(c);
        if (fs) return fs;
    }
    if (c->d.nranks > 1) return fail(c, NXSDG_ERR_UNSUPPORTED, "debug steps are single-rank");
    if (c->sphere) return fail(c, NXSDG_ERR_UNSUPPORTED, "sphere: no unfused debug steps");
    nxsdg_status s = ensure_debug_buffers(c);
    if (s) return s;
    if (c->general) return st == NXSDG_STEP_STRESS ? general_stress(c) : general_step(c, st);
    return launch_step(c, st);
}

// ---------------------------------------------------------------- advection
// the structured CG2/DG2 advection kernel applies the R#25 limiter in its epilogue
static bool adv_fused_limit(const nxsdg_ctx* c) { return c->limiter && !c->general && c->P == 2 && c->NA == 6 && c->variant == 0; }

// k_advect_tma applies to the configs' structured closed-box CG2/DG2 pair (no limiter, no sphere)
static bool use_adv_tma(const nxsdg_ctx* c) {
    return c->P == 2 && c->NA == 6 && c->variant == 0 && c->adv_kernel == 0 && !c->general && !c->sphere &&
           !c->limiter && c->d.bc == NXSDG_BC_CLOSED && !c->inproc;
}
// single rank: the last k_advect_tma stage writes P_g for the new A, H (the ghost rows of a strip need
// their neighbour's new A, H, so row strips keep the separate P_g pass after the BEGIN_STEP exchange)
static bool fuse_pg(const nxsdg_ctx* c) { return c->fuse_pg && c->d.nranks == 1 && use_adv_tma(c); }

template <int ST>
static nxsdg_status launch_adv_tma_t(nxsdg_ctx* c, const AdvMaps& mp, const AdvTmaArgs& ta) {
    const size_t smem = adv_smem_bytes(ST);
    static uint64_t attr_set = 0;
    if (!dev_bit_test(attr_set, c->d.device)) {
        CU(cudaFuncSetAttribute(k_advect_tma<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dev_bit_set(attr_set, c->d.device);
    }
    int nsm = 148, occ = 1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->d.device);
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_advect_tma<ST>, 32 * ADV_TMA_WARPS, smem));
    const int64_t units = (int64_t)ta.nstrips * ta.nchunks;
    const int64_t want = (units + ADV_TMA_WARPS - 1) / ADV_TMA_WARPS;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * std::max(occ, 1)));
    k_advect_tma<ST><<<blocks, 32 * ADV_TMA_WARPS, smem, c->stream>>>(mp, ta);
    return NXSDG_OK;
}

// k_advect_tma's folded coefficients: every scale between its raw Gauss sums and dt a1 mr_k L_k (advect_tma.cuh)
static void adv_coeffs(AdvArgs& a) {
    const double ka = 0.38729833462074170, f = 5.0 / 18.0, g = 5.0 * ka / 18.0;
    const double mr[6] = {1.0, 12.0, 12.0, 180.0, 180.0, 144.0};
    double U[6];
    for (int k = 0; k < 6; ++k) U[k] = a.a1 * a.dt * mr[k];
    const double hx = a.ihx, hy = a.ihy;
    const double kc[18] = {U[0] * f * hx, U[0] * f * hy,
                           U[1] * hx * f * f, -U[1] * hx * (5.0 / 36.0), U[1] * hy * g,
                           U[2] * hy * f * f, U[2] * hx * g, -U[2] * hy * (5.0 / 36.0),
                           U[3] * 2.0 * hx * f * g, U[3] * (hx / 6.0) * f, U[3] * hy / 54.0,
                           U[4] * 2.0 * hy * f * g, U[4] * hx / 54.0, U[4] * (hy / 6.0) * f,
                           U[5] * hx * f * g, U[5] * hy * f * g, -U[5] * hx * (5.0 * ka / 36.0), -U[5] * hy * (5.0 * ka / 36.0)};
    for (int k = 0; k < 18; ++k) a.kc[k] = kc[k];
}

static nxsdg_status launch_adv_tma(nxsdg_ctx* c, const AdvArgs& a0) {
    AdvArgs a = a0;
    adv_coeffs(a);
    AdvMaps mp;
    const cuuint64_t nx = c->d.nx, er = c->erows_local, ncols = 2 * (cuuint64_t)c->d.nx + 1, nr = c->nrows_local;
    const cuuint64_t es[2] = {(cuuint64_t)c->epitch * 8, (cuuint64_t)c->eplane * 8};
    const cuuint64_t ns[2] = {(cuuint64_t)c->npitch * 8, (cuuint64_t)c->nn * 8};
    const cuuint64_t dA[3] = {nx, er, 6}, dV[2] = {ncols, nr};
    const cuuint32_t bA[3] = {ADV_COLS, 1, 6}, bV[2] = {K2_VCOLS, 2};
    if (!encode(&mp.A, a.Ain, 3, dA, es, bA) || !encode(&mp.H, a.Hin, 3, dA, es, bA) ||
        !encode(&mp.vx, a.vx, 2, dV, ns, bV) || !encode(&mp.vy, a.vy, 2, dV, ns, bV) ||
        !encode(&mp.A0, a.A0, 3, dA, es, bA) || !encode(&mp.H0, a.H0, 3, dA, es, bA))
        return fail(c, NXSDG_ERR_CUDA, "cuTensorMapEncodeTiled (advection) failed");
    AdvTmaArgs ta{};
    ta.a = a;
    ta.nstrips = (c->d.nx + 1 + 30) / 31;
    ta.ty = c->adv_ty;
    if (c->d.nranks == 1 && c->ty == 0)   // small meshes: as chunk_rows, enough units for the resident warps
        while (ta.ty > 4 && (int64_t)ta.nstrips * ((c->nown + ta.ty - 1) / ta.ty) < (int64_t)(c->nsm > 0 ? c->nsm : 148) * 8)
            ta.ty /= 2;
    ta.nchunks = (c->nown + ta.ty - 1) / ta.ty;
    ta.dbg = getenv("NXSDG_DEBUG_ADV_TMA") != nullptr;
    if (c->adv_stages == 3) return launch_adv_tma_t<3>(c, mp, ta);
    return c->adv_stages == 5 ? launch_adv_tma_t<5>(c, mp, ta) : launch_adv_tma_t<4>(c, mp, ta);
}

template <int P, int NA>
static nxsdg_status launch_advect_stage(nxsdg_ctx* c, const double* Ain, const double* Hin, double* Aout,
                                        double* Hout, double dt, double a0, double a1) {
    AdvArgs a{};
    a.Ain = Ain; a.Hin = Hin; a.A0 = c->A; a.H0 = c->H; a.Aout = Aout; a.Hout = Hout;
    a.vx = c->vx[c->cv]; a.vy = c->vy[c->cv];
    a.eplane = c->eplane; a.npitch = c->npitch; a.epitch = c->epitch; a.nx = c->d.nx;
    a.erow_begin = c->glo; a.erow_end = c->glo + c->nown;
    a.has_south = c->glo; a.has_north = c->ghi;
    a.periodic = c->d.bc == NXSDG_BC_PERIODIC; a.erows_local = c->erows_local;
    a.ihx = 1.0 / (c->d.lx / c->d.nx); a.ihy = 1.0 / (c->d.ly / c->d.ny);
    if (c->sphere) {
        a.ihx = 1.0 / (c->sph_R * c->sph_dlon); a.ihy = 1.0 / (c->sph_R * c->sph_dlat);
        a.sph_rows = c->sph_rows;
    }
    a.dt = dt; a.a0 = a0; a.a1 = a1;
    a.limit = adv_fused_limit(c);
    if (c->adv_last && fuse_pg(c)) { a.Pg = c->Pg; a.Pstar = c->prm.Pstar; a.C_conc = c->prm.C_conc; }
    dim3 b(32, ADV_ROWS), g((unsigned)((c->d.nx + 31) / 32), (unsigned)((c->nown + ADV_ROWS - 1) / ADV_ROWS));
    if (c->general) {
        GenAdvArgs ga{a, c->verts, c->d.ny};
        k_advect_gen<P, NA><<<g, b, 0, c->stream>>>(ga);
    } else if (P == 2 && NA == 6 && use_adv_tma(c)) {   // persistent TMA-staged form (advect_tma.cuh)
        nxsdg_status st = launch_adv_tma(c, a);
        if (st) return st;
    } else if (P == 2 && NA == 6 && c->sphere) k_advect_q2<true><<<g, b, 0, c->stream>>>(a);   // R#26
    else if (P == 2 && NA == 6 && c->variant == 0) k_advect_q2<false><<<g, b, 0, c->stream>>>(a);   // structured
    else k_advect<P, NA><<<g, b, 0, c->stream>>>(a);
    LAUNCHED();
    return NXSDG_OK;
}

template <int P, int NA>
static nxsdg_status advect_t(nxsdg_ctx* c, double dt, int stage) {
    // stage-by-stage so the loopback group driver can exchange between stages
    switch (NA) {
        case 1:
            return launch_advect_stage<P, NA>(c, c->A, c->H, c->Asc[0], c->Hsc[0], dt, 0.0, 1.0);
        case 3:
            if (stage == 0) return launch_advect_stage<P, NA>(c, c->A, c->H, c->Asc[0], c->Hsc[0], dt, 0.0, 1.0);
            return launch_advect_stage<P, NA>(c, c->Asc[0], c->Hsc[0], c->Asc[1], c->Hsc[1], dt, 0.5, 0.5);
        default:
            if (stage == 0) return launch_advect_stage<P, NA>(c, c->A, c->H, c->Asc[0], c->Hsc[0], dt, 0.0, 1.0);
            if (stage == 1) return launch_advect_stage<P, NA>(c, c->Asc[0], c->Hsc[0], c->Asc[1], c->Hsc[1], dt, 0.75, 0.25);
            return launch_advect_stage<P, NA>(c, c->Asc[1], c->Hsc[1], c->Asc[0], c->Hsc[0], dt, 1.0 / 3.0, 2.0 / 3.0);
    }
}

static int n_stages(const nxsdg_ctx* c) { return c->NA == 1 ? 1 : (c->NA == 3 ? 2 : 3); }
static int stage_out_buf(const nxsdg_ctx* c, int stage) {
    if (c->NA == 3) return stage;           // 0 -> scr0, 1 -> scr1
    if (c->NA == 6) return stage == 1 ? 1 : 0;
    return 0;
}

template <int P, int NA>
static nxsdg_status limit_t(nxsdg_ctx* c, double* A, double* H) {
    LimArgs a{};
    a.A = A; a.H = H; a.verts = c->general ? c->verts : nullptr;
    a.eplane = c->eplane; a.epitch = c->epitch; a.nx = c->d.nx; a.erow_begin = c->glo; a.erow_end = c->glo + c->nown;
    dim3 b(128), g((unsigned)((c->d.nx + 127) / 128), (unsigned)c->nown);
    k_limit<P, NA><<<g, b, 0, c->stream>>>(a);
    LAUNCHED();
    return NXSDG_OK;
}

static nxsdg_status advect_stage(nxsdg_ctx* c, double dt, int stage) {
    nxsdg_status s;
    c->adv_last = stage == n_stages(c) - 1;
    if (c->P == 1) s = c->NA == 1 ? advect_t<1, 1>(c, dt, stage) : advect_t<1, 3>(c, dt, stage);
    else if (c->NA == 1) s = advect_t<2, 1>(c, dt, stage);
    else if (c->NA == 3) s = advect_t<2, 3>(c, dt, stage);
    else s = advect_t<2, 6>(c, dt, stage);
    if (s || !c->limiter || c->NA == 1 || adv_fused_limit(c)) return s;
    // NEXT-4 (R#25): bound-preserving limiter on the stage output, before its halo exchange
    const int ob = stage_out_buf(c, stage);
    if (c->P == 1) return limit_t<1, 3>(c, c->Asc[ob], c->Hsc[ob]);
    return c->NA == 3 ? limit_t<2, 3>(c, c->Asc[ob], c->Hsc[ob]) : limit_t<2, 6>(c, c->Asc[ob], c->Hsc[ob]);
}

// the final stage buffer becomes A, H (pointer swap; ghost rows are refreshed by the next exchange)
static nxsdg_status advect_finish(nxsdg_ctx* c) {
    const int last = stage_out_buf(c, n_stages(c) - 1);
    std::swap(c->A, c->Asc[last]);
    std::swap(c->H, c->Hsc[last]);
    c->prepped = false; c->prep_defer = false;
    c->pg_fresh = fuse_pg(c);   // the last stage wrote P of the new A, H
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_advect(nxsdg_ctx* c, double dt) {
    GUARD(c);
    NvtxRange nv("nxsdg_advect");
    if (!(dt >= 0.0)) return fail(c, NXSDG_ERR_INVALID_ARG, "dt < 0");
    if (c->sphere && c->limiter) return fail(c, NXSDG_ERR_UNSUPPORTED, "sphere: no limiter (R#25 uses the box mean)");
    c->pg_fresh = false;
    if (c->general && c->d.bc != NXSDG_BC_CLOSED) return fail(c, NXSDG_ERR_UNSUPPORTED, "general quads: closed box only");
    if (c->d.nranks > 1 && c->d.transport == NXSDG_TRANSPORT_LOOPBACK)
        return fail(c, NXSDG_ERR_STATE, "loopback ranks advect through nxsdg_group_advect");
    nxsdg_status s;
    if ((s = halo(c, NXSDG_HALO_V | NXSDG_HALO_AH))) return s;
    for (int st = 0; st < n_stages(c); ++st) {
        if ((s = advect_stage(c, dt, st))) return s;
        if (st + 1 < n_stages(c) && (s = halo(c, stage_out_buf(c, st) == 0 ? NXSDG_HALO_AH_SCR0 : NXSDG_HALO_AH_SCR1))) return s;
    }
    return advect_finish(c);
}

extern "C" nxsdg_status nxsdg_synchronize(nxsdg_ctx* c) {
    GUARD(c);
    if (c->comm && nccl().CommGetAsyncError) {   // failure detection: a broken peer surfaces here
        ncclResult_t ar = 0;
        if (nccl().CommGetAsyncError(c->comm, &ar) != 0 || ar != 0)
            return fail(c, NXSDG_ERR_NCCL, "NCCL async error %d", (int)ar);
    }
    if (c->cstream) CU(cudaStreamSynchronize(c->cstream));
    if (c->dstream) CU(cudaStreamSynchronize(c->dstream));
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaGetLastError());
    return NXSDG_OK;
}

// ---------------------------------------------------------------- multi-rank plumbing
// K0 tables for tests (a0): {gx[ngp], gw[ngp], psi[nd][ng], phi[ncg][ng], dphis[ncg][ng], dphit[ncg][ng],
// mref[nd], R[nd][ng], Ds[ncg][nd], Dt[ncg][nd]} of degree p, flattened in this order; nd = 8 for the
// (2, 8) space of a context with n_S = 8 and p = 2, else 6.
extern "C" nxsdg_status nxsdg_debug_reference_tables(nxsdg_ctx* c, int32_t p, double* out, int64_t count, int64_t* needed) {
    GUARD(c);
    if (p != 1 && p != 2) return fail(c, NXSDG_ERR_INVALID_ARG, "p 1|2");
    const int ngp = p + 1, ng = ngp * ngp, ncg = ng;
    const int nd = (p == 2 && c->NS == 8) ? 8 : 6;
    const int64_t n = 2 * ngp + nd * ng + 3 * ncg * ng + nd + nd * ng + 2 * ncg * nd;
    if (needed) *needed = n;
    if (!out) return NXSDG_OK;
    if (count < n) return fail(c, NXSDG_ERR_INVALID_ARG, "count < %lld", (long long)n);
    RefTab T;
    CU(cudaMemcpyFromSymbol(&T, c_tab, sizeof(RefTab), tab_index(p, p == 2 ? c->NS : 3) * sizeof(RefTab),
                            cudaMemcpyDeviceToHost));
    int64_t o = 0;
    for (int i = 0; i < ngp; ++i) out[o++] = T.gx[i];
    for (int i = 0; i < ngp; ++i) out[o++] = T.gw[i];
    for (int k = 0; k < nd; ++k) for (int g = 0; g < ng; ++g) out[o++] = T.psi[k][g];
    for (int j = 0; j < ncg; ++j) for (int g = 0; g < ng; ++g) out[o++] = T.phi[j][g];
    for (int j = 0; j < ncg; ++j) for (int g = 0; g < ng; ++g) out[o++] = T.dphis[j][g];
    for (int j = 0; j < ncg; ++j) for (int g = 0; g < ng; ++g) out[o++] = T.dphit[j][g];
    for (int k = 0; k < nd; ++k) out[o++] = T.mref[k];
    for (int k = 0; k < nd; ++k) for (int g = 0; g < ng; ++g) out[o++] = T.R[k][g];
    for (int j = 0; j < ncg; ++j) for (int k = 0; k < nd; ++k) out[o++] = T.Ds[j][k];
    for (int j = 0; j < ncg; ++j) for (int k = 0; k < nd; ++k) out[o++] = T.Dt[j][k];
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_nccl_unique_id(void* out128) {
    if (!out128) return NXSDG_ERR_INVALID_ARG;
    NcclApi& api = nccl();
    if (!api.loaded) return NXSDG_ERR_NCCL;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != 0) return NXSDG_ERR_NCCL;
    memcpy(out128, &id, sizeof id);
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_loopback_connect(nxsdg_ctx** ctxs, int32_t n) {
    if (!ctxs || n < 1) return NXSDG_ERR_INVALID_ARG;
    for (int i = 0; i < n; ++i) {
        if (!ctxs[i] || ctxs[i]->d.rank != i || ctxs[i]->d.nranks != n || ctxs[i]->d.transport != NXSDG_TRANSPORT_LOOPBACK)
            return NXSDG_ERR_INVALID_ARG;
        if (ctxs[i]->stream != ctxs[0]->stream || ctxs[i]->d.device != ctxs[0]->d.device) return NXSDG_ERR_INVALID_ARG;
    }
    std::vector<nxsdg_ctx*> v(ctxs, ctxs + n);
    for (int i = 0; i < n; ++i) ctxs[i]->peers = v;
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_group_mevp_substeps(nxsdg_ctx** ctxs, int32_t nr, int32_t n, uint32_t flags) {
    if (!ctxs || nr < 1) return NXSDG_ERR_INVALID_ARG;
    std::vector<nxsdg_ctx*> v(ctxs, ctxs + nr);
    nxsdg_status s;
    for (nxsdg_ctx* c : v) {
        GUARD(c);
        if (c->peers.size() != (size_t)nr && nr > 1) return fail(c, NXSDG_ERR_STATE, "not loopback-connected");
        if ((s = check_substeps(c, n, flags))) return s;
    }
    const bool unfused = flags & NXSDG_UNFUSED;
    if (flags & NXSDG_BEGIN_STEP) {
        for (nxsdg_ctx* c : v) if ((s = consume_forcing(c))) return s;
        if ((s = halo_loopback_all(v, NXSDG_HALO_V | NXSDG_HALO_S | NXSDG_HALO_AH))) return s;
        for (nxsdg_ctx* c : v) {
            cudaSetDevice(c->d.device);
            if ((s = dispatch_prep(c))) return s;
            c->prepped = true;
        }
    }
    for (int i = 0; i < n; ++i) {
        if (!unfused) {
            // same split as the NCCL path: boundary chunks, exchange, interior chunks
            for (nxsdg_ctx* c : v) {
                if ((s = launch_subcycle_sel(c, n_chunks(c) < 3 ? SEL_ALL : SEL_BOUNDARY))) return s;
                c->cv ^= 1; c->cs ^= 1;
            }
            if ((s = halo_loopback_all(v, NXSDG_HALO_V | NXSDG_HALO_S))) return s;
            for (nxsdg_ctx* c : v) {
                if (n_chunks(c) < 3) continue;
                c->cv ^= 1; c->cs ^= 1;
                if ((s = launch_subcycle_sel(c, SEL_INTERIOR))) return s;
                c->cv ^= 1; c->cs ^= 1;
            }
        } else {
            for (nxsdg_ctx* c : v) {
                if ((s = ensure_debug_buffers(c))) return s;
                if ((s = launch_step(c, NXSDG_STEP_STRAIN))) return s;
                if ((s = launch_step(c, NXSDG_STEP_STRESS))) return s;
            }
            if ((s = halo_loopback_all(v, NXSDG_HALO_S))) return s;
            for (nxsdg_ctx* c : v) {
                if ((s = launch_step(c, NXSDG_STEP_DIVERGENCE))) return s;
                if ((s = launch_step(c, NXSDG_STEP_VELOCITY))) return s;
            }
            if ((s = halo_loopback_all(v, NXSDG_HALO_V))) return s;
        }
    }
    return NXSDG_OK;
}

extern "C" nxsdg_status nxsdg_group_advect(nxsdg_ctx** ctxs, int32_t nr, double dt) {
    if (!ctxs || nr < 1) return NXSDG_ERR_INVALID_ARG;
    std::vector<nxsdg_ctx*> v(ctxs, ctxs + nr);
    nxsdg_status s;
    for (nxsdg_ctx* c : v) GUARD(c);
    if ((s = halo_loopback_all(v, NXSDG_HALO_V | NXSDG_HALO_AH))) return s;
    const int ns = n_stages(v[0]);
    for (int st = 0; st < ns; ++st) {
        for (nxsdg_ctx* c : v) if ((s = advect_stage(c, dt, st))) return s;
        if (st + 1 < ns && (s = halo_loopback_all(v, stage_out_buf(v[0], st) == 0 ? NXSDG_HALO_AH_SCR0 : NXSDG_HALO_AH_SCR1))) return s;
    }
    for (nxsdg_ctx* c : v) if ((s = advect_finish(c))) return s;
    return NXSDG_OK;
}
