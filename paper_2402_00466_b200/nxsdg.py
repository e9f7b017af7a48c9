"""Thin ctypes binding of libnxsdg.so (include/nxsdg.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels.  There is no CPU
fallback: importing this module on a machine without the built library raises,
and creating a mesh without a CUDA device returns NXSDG_ERR_CUDA.

Host arrays are numpy float64; device arrays are torch CUDA float64 tensors
(torch is used only for device memory and streams).  Function names mirror
the C ABI without the ``nxsdg_`` prefix; :class:`Mesh` is a small RAII helper.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import asdict, dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnxsdg.so")
# A/B experiments only (scripts/): load another build of the same ABI, e.g. the previous commit's kernels
if os.environ.get("NXSDG_LIB_AB"):
    LIB_PATH = os.path.join(_HERE, os.path.basename(os.environ["NXSDG_LIB_AB"]))

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_STATE, ERR_CUDA, ERR_NCCL, ERR_OOM = range(7)
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "UNSUPPORTED", 3: "STATE", 4: "CUDA", 5: "NCCL", 6: "OOM"}
MEM_HOST, MEM_DEVICE, MEM_HOST_ASYNC = 0, 1, 2
BC_CLOSED, BC_PERIODIC = 0, 1
FIELDS = {"vx": 0, "vy": 1, "S11": 2, "S12": 3, "S22": 4, "A": 5, "H": 6, "E11": 7, "E12": 8, "E22": 9,
          "Fx": 10, "Fy": 11}
CG_FIELDS = {"vx", "vy", "Fx", "Fy"}
BEGIN_STEP, UNFUSED = 1, 2
STEPS = {"strain": 0, "stress": 1, "divergence": 2, "velocity": 3}
TRANSPORT_NONE, TRANSPORT_NCCL, TRANSPORT_LOOPBACK, TRANSPORT_P2P = 0, 1, 2, 3
(OPT_FUSED_KERNEL, OPT_CHUNK_ROWS, OPT_CTAS_PER_SM, OPT_STAGES, OPT_DYNAMIC, OPT_MAP_MODE, OPT_PRECISION,
 OPT_P2P_FUSED_STORES, OPT_LIMITER, OPT_CONST_STAGING, OPT_TAIL_SPLIT, OPT_L2_POLICY, OPT_V_ROW_CARRY,
 OPT_MULTIRANK_GRAPH, OPT_ADVECT_KERNEL, OPT_ADVECT_STAGES, OPT_FUSE_PREP_PG, _OPT_17_UNUSED,
 OPT_PREP_KERNEL, OPT_PAIR_SUBCYCLES, OPT_PDL) = range(21)


class NxsdgError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str = ""):
        self.status = status
        super().__init__(f"{where}: NXSDG_ERR_{STATUS.get(status, status)} {msg}".strip())


class MeshDesc(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("lx", C.c_double), ("ly", C.c_double),
                ("cg_degree", C.c_int32), ("n_stress", C.c_int32), ("n_adv", C.c_int32), ("bc", C.c_int32),
                ("rank", C.c_int32), ("nranks", C.c_int32), ("transport", C.c_int32),
                ("nccl_id", C.c_void_p), ("device", C.c_int32), ("stream", C.c_void_p)]


class Params(C.Structure):
    _fields_ = [("rho_ice", C.c_double), ("rho_atm", C.c_double), ("rho_ocean", C.c_double),
                ("C_atm", C.c_double), ("C_ocean", C.c_double), ("f_c", C.c_double),
                ("Pstar", C.c_double), ("DeltaMin", C.c_double), ("C_conc", C.c_double),
                ("alpha", C.c_double), ("beta", C.c_double), ("dt", C.c_double),
                ("replacement_pressure", C.c_int32)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2402_00466_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u32, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double
    sig = {
        "nxsdg_create_mesh": ([C.POINTER(MeshDesc), C.POINTER(Params), C.POINTER(vp)], i32),
        "nxsdg_destroy": ([vp], i32),
        "nxsdg_last_error": ([vp], C.c_char_p),
        "nxsdg_abi_version": ([], i32),
        "nxsdg_set_params": ([vp, C.POINTER(Params)], i32),
        "nxsdg_get_partition": ([vp, C.POINTER(i64), C.POINTER(i32), C.POINTER(i64), C.POINTER(i32)], i32),
        "nxsdg_partition": ([i32, i32, i32, i32, C.POINTER(i64), C.POINTER(i32), C.POINTER(i64), C.POINTER(i32)], i32),
        "nxsdg_write_state": ([vp, i32, vp, i64, i32], i32),
        "nxsdg_read_state": ([vp, i32, vp, i64, i32], i32),
        "nxsdg_set_forcing": ([vp, vp, vp, vp, vp, i64, i32], i32),
        "nxsdg_mevp_substeps": ([vp, i32, u32], i32),
        "nxsdg_advect": ([vp, dbl], i32),
        "nxsdg_run_step": ([vp, i32], i32),
        "nxsdg_synchronize": ([vp], i32),
        "nxsdg_nccl_unique_id": ([vp], i32),
        "nxsdg_loopback_connect": ([C.POINTER(vp), i32], i32),
        "nxsdg_group_mevp_substeps": ([C.POINTER(vp), i32, i32, u32], i32),
        "nxsdg_group_advect": ([C.POINTER(vp), i32, dbl], i32),
        "nxsdg_kernel_launches": ([vp], i64),
        "nxsdg_bytes_per_element_subcycle": ([vp], dbl),
        "nxsdg_stream": ([vp], vp),
        "nxsdg_set_option": ([vp, i32, i64], i32),
        "nxsdg_set_forcing_cyclone": ([vp, dbl], i32),
        "nxsdg_set_vertices": ([vp, vp, i64, i32], i32),
        "nxsdg_stream_join": ([vp], i32),
        "nxsdg_debug_reference_tables": ([vp, i32, vp, i64, C.POINTER(i64)], i32),
        "nxsdg_halo_plan": ([i32, i32, i32, i32, i32, i32, i32, u32, vp, i32, C.POINTER(i32)], i32),
        "nxsdg_local_geometry": ([i32, i32, i32, i32, i32, i32, i32, C.POINTER(i64)], i32),
        "nxsdg_p2p_export": ([vp, vp, i64, C.POINTER(i64)], i32),
        "nxsdg_p2p_connect": ([vp, vp, vp], i32),
        "nxsdg_p2p_connect_local": ([C.POINTER(vp), i32], i32),
        "nxsdg_transport_info": ([vp, C.c_char_p, i64], i64),
        "nxsdg_set_sphere": ([vp, dbl, dbl, dbl, dbl], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


lib = _load()
EXPORTED = [
    "nxsdg_create_mesh", "nxsdg_destroy", "nxsdg_last_error", "nxsdg_abi_version", "nxsdg_set_params",
    "nxsdg_get_partition", "nxsdg_partition", "nxsdg_write_state", "nxsdg_read_state", "nxsdg_set_forcing",
    "nxsdg_mevp_substeps", "nxsdg_advect", "nxsdg_run_step", "nxsdg_synchronize", "nxsdg_nccl_unique_id",
    "nxsdg_loopback_connect", "nxsdg_group_mevp_substeps", "nxsdg_group_advect", "nxsdg_kernel_launches",
    "nxsdg_bytes_per_element_subcycle", "nxsdg_stream", "nxsdg_set_option", "nxsdg_halo_plan",
    "nxsdg_local_geometry", "nxsdg_set_forcing_cyclone", "nxsdg_set_vertices", "nxsdg_stream_join",
    "nxsdg_debug_reference_tables", "nxsdg_p2p_export", "nxsdg_p2p_connect", "nxsdg_p2p_connect_local",
    "nxsdg_transport_info", "nxsdg_set_sphere",
]
HALO_V, HALO_S, HALO_AH, HALO_AH_SCR0, HALO_AH_SCR1 = 1, 2, 4, 8, 16
HF_VX, HF_VY, HF_S, HF_A, HF_H, HF_A_SCR0, HF_H_SCR0, HF_A_SCR1, HF_H_SCR1 = range(9)


class HaloSeg(C.Structure):
    _fields_ = [("dir", C.c_int32), ("field", C.c_int32), ("peer", C.c_int32), ("plane", C.c_int32),
                ("offset", C.c_int64), ("count", C.c_int64)]


def halo_plan(nx, ny, p, ns, na, nranks, rank, what):
    """The ordered halo send/recv plan of one rank (pure host arithmetic, no GPU)."""
    n = C.c_int32()
    _chk(None, lib.nxsdg_halo_plan(nx, ny, p, ns, na, nranks, rank, what, None, 0, C.byref(n)), "halo_plan")
    arr = (HaloSeg * max(1, n.value))()
    _chk(None, lib.nxsdg_halo_plan(nx, ny, p, ns, na, nranks, rank, what, arr, n.value, C.byref(n)), "halo_plan")
    return [dict(dir=s.dir, field=s.field, peer=s.peer, plane=s.plane, offset=s.offset, count=s.count)
            for s in arr[:n.value]]


def local_geometry(nx, ny, p, ns, na, nranks, rank) -> dict:
    out = (C.c_int64 * 8)()
    _chk(None, lib.nxsdg_local_geometry(nx, ny, p, ns, na, nranks, rank, out), "local_geometry")
    keys = ("elem_row0", "elem_rows", "glo", "erows_local", "nrows_local", "epitch", "eplane", "npitch")
    return dict(zip(keys, list(out)))


def _chk(ctx, st: int, where: str):
    if st != OK:
        msg = lib.nxsdg_last_error(ctx).decode() if ctx else ""
        raise NxsdgError(st, where, msg)


@dataclass
class PhysParams:
    rho_ice: float = 900.0
    rho_atm: float = 1.3
    rho_ocean: float = 1026.0
    C_atm: float = 1.2e-3
    C_ocean: float = 5.5e-3
    f_c: float = 1.46e-4
    Pstar: float = 27500.0
    DeltaMin: float = 2e-9
    C_conc: float = 20.0
    alpha: float = 1500.0
    beta: float = 1500.0
    dt: float = 120.0
    replacement_pressure: int = 0

    def c(self) -> Params:
        return Params(**asdict(self))


def _ptr_mem(a):
    """(pointer, count, mem) of a numpy float64 array or a torch CUDA float64 tensor."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise TypeError("host arrays must be C-contiguous float64")
        return a.ctypes.data, a.size, MEM_HOST
    import torch
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise TypeError("device tensors must be contiguous float64")
        if a.is_cuda:
            return a.data_ptr(), a.numel(), MEM_DEVICE
        return a.data_ptr(), a.numel(), MEM_HOST
    raise TypeError(type(a))


# ---- functional API (same names as the C ABI) ----------------------------------------
def partition(ny: int, cg_degree: int, nranks: int, rank: int):
    r0, er, n0, nr = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int32()
    _chk(None, lib.nxsdg_partition(ny, cg_degree, nranks, rank, C.byref(r0), C.byref(er), C.byref(n0),
                                   C.byref(nr)), "partition")
    return r0.value, er.value, n0.value, nr.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(None, lib.nxsdg_nccl_unique_id(buf), "nccl_unique_id")
    return buf.raw


class Mesh:
    """One rank's context.  ``stream`` = cudaStream_t integer (e.g. torch's), 0 -> library-owned."""

    def __init__(self, nx, ny, lx=512e3, ly=512e3, p=2, ns=6, na=6, bc=BC_CLOSED, params=None,
                 rank=0, nranks=1, transport=TRANSPORT_NONE, nccl_id: bytes | None = None, device=0, stream=0):
        self.nx, self.ny, self.lx, self.ly, self.p, self.ns, self.na = nx, ny, lx, ly, p, ns, na
        self.params = params or PhysParams()
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        d = MeshDesc(nx, ny, lx, ly, p, ns, na, bc, rank, nranks, transport,
                     C.cast(self._id, C.c_void_p) if self._id else None, device, stream or None)
        h = C.c_void_p()
        st = lib.nxsdg_create_mesh(C.byref(d), C.byref(self.params.c()), C.byref(h))
        if st != OK:
            raise NxsdgError(st, "create_mesh")
        self.h = h
        r0, er, n0, nr = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int32()
        _chk(self.h, lib.nxsdg_get_partition(self.h, C.byref(r0), C.byref(er), C.byref(n0), C.byref(nr)), "partition")
        self.elem_row0, self.elem_rows, self.node_row0, self.node_rows = r0.value, er.value, n0.value, nr.value

    # shapes of this rank's owned part in the ABI layout
    def shape(self, field: str):
        if field in CG_FIELDS or field in ("ox", "oy", "ax", "ay"):
            return (self.node_rows, self.p * self.nx + 1)
        n = self.na if field in ("A", "H") else self.ns
        return (self.elem_rows * self.nx, n)

    def destroy(self):
        if getattr(self, "h", None):
            lib.nxsdg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.destroy()

    @property
    def stream(self) -> int:
        return int(lib.nxsdg_stream(self.h) or 0)

    @property
    def kernel_launches(self) -> int:
        return int(lib.nxsdg_kernel_launches(self.h))

    @property
    def bytes_per_element_subcycle(self) -> float:
        return float(lib.nxsdg_bytes_per_element_subcycle(self.h))

    @property
    def transport_info(self) -> str:
        buf = C.create_string_buffer(512)
        lib.nxsdg_transport_info(self.h, buf, len(buf))
        return buf.value.decode()

    def set_option(self, option: int, value: int):
        _chk(self.h, lib.nxsdg_set_option(self.h, int(option), int(value)), "set_option")

    def set_params(self, params: PhysParams):
        self.params = params
        _chk(self.h, lib.nxsdg_set_params(self.h, C.byref(params.c())), "set_params")

    def write_state(self, field: str, arr):
        p, n, mem = _ptr_mem(arr)
        _chk(self.h, lib.nxsdg_write_state(self.h, FIELDS[field], p, n, mem), f"write_state({field})")

    def read_state(self, field: str, out=None, asynchronous: bool = False):
        if out is None:
            out = np.empty(self.shape(field), dtype=np.float64)
        p, n, mem = _ptr_mem(out)
        if asynchronous:
            if mem != MEM_HOST:
                raise ValueError("asynchronous reads go to pinned host memory")
            mem = MEM_HOST_ASYNC
        _chk(self.h, lib.nxsdg_read_state(self.h, FIELDS[field], p, n, mem), f"read_state({field})")
        return out

    def set_forcing(self, ox, oy, ax, ay, asynchronous: bool = False):
        ps = [_ptr_mem(a) for a in (ox, oy, ax, ay)]
        if len({(n, m) for _, n, m in ps}) != 1:
            raise ValueError("forcing arrays must match in size and memory kind")
        mem = ps[0][2]
        if asynchronous:
            if mem != MEM_HOST:
                raise ValueError("asynchronous forcing comes from pinned host memory")
            mem = MEM_HOST_ASYNC
        _chk(self.h, lib.nxsdg_set_forcing(self.h, *[p for p, _, _ in ps], ps[0][1], mem), "set_forcing")

    def reference_tables(self, p: int) -> dict:
        """K0 device tables of degree p (see include/nxsdg.h), split into named arrays."""
        need = C.c_int64()
        _chk(self.h, lib.nxsdg_debug_reference_tables(self.h, p, None, 0, C.byref(need)), "tables")
        buf = np.empty(need.value)
        _chk(self.h, lib.nxsdg_debug_reference_tables(self.h, p, buf.ctypes.data, need.value, C.byref(need)), "tables")
        ngp = p + 1; ng = ngp * ngp
        nd = 8 if (p == 2 and self.ns == 8) else 6
        shapes = [("gx", (ngp,)), ("gw", (ngp,)), ("psi", (nd, ng)), ("phi", (ng, ng)), ("dphis", (ng, ng)),
                  ("dphit", (ng, ng)), ("mref", (nd,)), ("R", (nd, ng)), ("Ds", (ng, nd)), ("Dt", (ng, nd))]
        out, o = {}, 0
        for name, shp in shapes:
            n = int(np.prod(shp)); out[name] = buf[o:o + n].reshape(shp); o += n
        return out

    def p2p_export(self) -> bytes:
        """Opaque blob with CUDA IPC handles of this rank's exchanged buffers (P2P transport)."""
        need = C.c_int64()
        _chk(self.h, lib.nxsdg_p2p_export(self.h, None, 0, C.byref(need)), "p2p_export")
        buf = (C.c_char * need.value)()
        _chk(self.h, lib.nxsdg_p2p_export(self.h, buf, need.value, C.byref(need)), "p2p_export")
        return bytes(buf)

    def p2p_connect(self, lower: bytes | None, upper: bytes | None):
        lo = C.create_string_buffer(lower, len(lower)) if lower else None
        hi = C.create_string_buffer(upper, len(upper)) if upper else None
        _chk(self.h, lib.nxsdg_p2p_connect(self.h, lo, hi), "p2p_connect")

    def stream_join(self):
        _chk(self.h, lib.nxsdg_stream_join(self.h), "stream_join")

    def set_sphere(self, radius: float, lat0: float, lon_extent: float, lat_extent: float):
        """NEXT-4 (R#26): lon-lat mesh on the sphere (angles in radians)."""
        _chk(self.h, lib.nxsdg_set_sphere(self.h, float(radius), float(lat0), float(lon_extent), float(lat_extent)),
             "set_sphere")

    def set_vertices(self, xy):
        p, n, mem = _ptr_mem(xy)
        _chk(self.h, lib.nxsdg_set_vertices(self.h, p, n, mem), "set_vertices")

    def set_forcing_cyclone(self, t: float):
        _chk(self.h, lib.nxsdg_set_forcing_cyclone(self.h, float(t)), "set_forcing_cyclone")

    def load(self, st: dict):
        """Write every state field and the forcing present in ``st`` (numpy or torch)."""
        for k in ("vx", "vy", "S11", "S12", "S22", "A", "H"):
            if k in st:
                self.write_state(k, st[k])
        if "ox" in st:
            self.set_forcing(st["ox"], st["oy"], st["ax"], st["ay"])

    def state(self, keys=("vx", "vy", "S11", "S12", "S22", "A", "H")) -> dict:
        return {k: self.read_state(k) for k in keys}

    def mevp_substeps(self, n_sub: int, begin_step: bool = True, unfused: bool = False):
        flags = (BEGIN_STEP if begin_step else 0) | (UNFUSED if unfused else 0)
        _chk(self.h, lib.nxsdg_mevp_substeps(self.h, int(n_sub), flags), "mevp_substeps")

    def advect(self, dt: float):
        _chk(self.h, lib.nxsdg_advect(self.h, float(dt)), "advect")

    def run_step(self, step: str):
        _chk(self.h, lib.nxsdg_run_step(self.h, STEPS[step]), f"run_step({step})")

    def synchronize(self):
        _chk(self.h, lib.nxsdg_synchronize(self.h), "synchronize")


def _handles(meshes):
    arr = (C.c_void_p * len(meshes))(*[m.h for m in meshes])
    return arr


def p2p_connect_local(meshes):
    _chk(None, lib.nxsdg_p2p_connect_local(_handles(meshes), len(meshes)), "p2p_connect_local")


def p2p_connect_group(mesh, rank: int, world: int, all_gather_object):
    """Exchange P2P blobs with torch.distributed-style all_gather_object and connect this rank."""
    blobs = [None] * world
    all_gather_object(blobs, mesh.p2p_export())
    mesh.p2p_connect(blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank + 1 < world else None)


def loopback_connect(meshes):
    _chk(None, lib.nxsdg_loopback_connect(_handles(meshes), len(meshes)), "loopback_connect")


def group_mevp_substeps(meshes, n_sub: int, begin_step: bool = True, unfused: bool = False):
    flags = (BEGIN_STEP if begin_step else 0) | (UNFUSED if unfused else 0)
    st = lib.nxsdg_group_mevp_substeps(_handles(meshes), len(meshes), int(n_sub), flags)
    if st != OK:
        msgs = "; ".join(lib.nxsdg_last_error(m.h).decode() for m in meshes)
        raise NxsdgError(st, "group_mevp_substeps", msgs)


def group_advect(meshes, dt: float):
    st = lib.nxsdg_group_advect(_handles(meshes), len(meshes), float(dt))
    if st != OK:
        msgs = "; ".join(lib.nxsdg_last_error(m.h).decode() for m in meshes)
        raise NxsdgError(st, "group_advect", msgs)
