"""ctypes binding of libdflb200.so (include/dflb200.h).

The library is required: importing this module on a machine where it cannot
be loaded raises :class:`~paper_1710_03940_b200.errors.DeviceError` -- there is
no CPU fallback for the solve.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import DeviceError, raise_for_status

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DFL_LIB") or os.path.join(_PKG, "libdflb200.so")

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

DFL_RELAX = {"damped_jacobi": 0, "spai0": 1}
DFL_SOLVER = {"cg": 0, "bicgstab2": 1, "gmres": 2, "fgmres": 3}
PTR_HOST, PTR_DEVICE = 0, 1
LEVEL_A, LEVEL_P, LEVEL_R = 0, 1, 2
DFL_TIME_FLUSH_L2, DFL_TIME_FORMAT_BYTES = 0x100, 0x200  # dfl_ctx_time flags (include/dflb200.h)


class Csr(ctypes.Structure):
    _fields_ = [("nrows", c_i64), ("ncols", c_i64), ("row_ptr", c_vp), ("col_idx", c_vp), ("values", c_vp)]


class AmgOptions(ctypes.Structure):
    _fields_ = [("eps_strong", c_dbl), ("omega", c_dbl), ("damping", c_dbl), ("relax", c_i32),
                ("max_levels", c_i32), ("coarse_enough", c_i64)]


class SolveParams(ctypes.Structure):
    _fields_ = [("solver", c_i32), ("maxiter", c_i32), ("refresh_every", c_i32), ("deflated", c_i32),
                ("tol", c_dbl), ("restart", c_i32), ("x0_given", c_i32)]


class BlockDesc(ctypes.Structure):
    _fields_ = [("n", c_i64), ("n_u", c_i64), ("A", c_vp), ("K", c_vp), ("G", c_vp), ("D", c_vp), ("S", c_vp),
                ("u_idx", c_vp), ("p_idx", c_vp), ("wK", c_vp), ("invKdiag", c_vp)]


class BlockParams(ctypes.Structure):
    _fields_ = [("tol", c_dbl), ("maxiter", c_i32), ("restart", c_i32), ("usolver", c_i32), ("umaxiter", c_i32),
                ("utol", c_dbl), ("psolver", c_i32), ("pmaxiter", c_i32), ("ptol", c_dbl)]


class BlockReport(ctypes.Structure):
    _fields_ = [("iterations", c_i32), ("converged", c_i32), ("relative_residual", c_dbl),
                ("solve_seconds", c_dbl), ("velocity_iterations", c_i64), ("pressure_iterations", c_i64),
                ("kernel_launches", c_i64), ("breakdown_value", c_dbl)]


class Report(ctypes.Structure):
    _fields_ = [("iterations", c_i32), ("converged", c_i32), ("breakdown", c_i32), ("device_loop", c_i32),
                ("bnorm", c_dbl), ("resnorm", c_dbl), ("relative_residual", c_dbl),
                ("solve_seconds", c_dbl), ("h2d_seconds", c_dbl), ("d2h_seconds", c_dbl),
                ("kernel_launches", c_i64), ("breakdown_value", c_dbl)]


_lib = None


class GenParams(ctypes.Structure):
    _fields_ = [("shape", c_i64 * 3), ("boxes", c_i64 * 3), ("kind", c_i32), ("cells", c_i32),
                ("contrast", c_dbl), ("conv", c_dbl * 3)]


GEN_KIND = {"poisson": 0, "jump": 1, "convdiff": 2}


def gen_rows(device: int, shape, boxes, kind: str, r0: int, r1: int, contrast=1e4, cells=4, c=(0.3, 0.2, 0.1),
             coords: bool = True):
    """CSR rows [r0, r1) of a structured problem built on the GPU
    (dfl_gen_rows); returns (row_ptr, col_idx, values, coords or None)."""
    p = GenParams((c_i64 * 3)(*shape), (c_i64 * 3)(*boxes), GEN_KIND[kind], int(cells), float(contrast),
                  (c_dbl * 3)(*[float(v) for v in c]))
    nr = r1 - r0
    ptr = np.empty(nr + 1, dtype=np.int64)
    col = np.empty(7 * nr, dtype=np.int64)
    val = np.empty(7 * nr)
    xyz = np.empty((nr, 3)) if coords else None
    nnz = c_i64()
    check(lib().dfl_gen_rows(int(device), ctypes.byref(p), int(r0), int(r1), _ptr(ptr), _ptr(col), _ptr(val),
                             ctypes.byref(nnz), _ptr(xyz) if coords else None))
    return ptr, col[: nnz.value], val[: nnz.value], xyz


def gen_unknown_of_node(device: int, shape, boxes, n: int) -> np.ndarray:
    p = GenParams((c_i64 * 3)(*shape), (c_i64 * 3)(*boxes), 0, 4, 1e4, (c_dbl * 3)(0.0, 0.0, 0.0))
    uon = np.empty(n, dtype=np.int64)
    check(lib().dfl_gen_unknown_of_node(int(device), ctypes.byref(p), _ptr(uon)))
    return uon


def lib():
    """Load libdflb200.so (built in-tree by ``paper_1710_03940_b200._build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1710_03940_b200._build` "
            "(there is no CPU fallback for the solve)"
        )
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
    P = ctypes.POINTER
    sig = {
        "dfl_abi_version": ([], c_i32),
        "dfl_last_setup_error": ([], ctypes.c_char_p),
        "dfl_breakdown_string": ([c_i32], ctypes.c_char_p),
        "dfl_hier_build": ([P(Csr), P(AmgOptions), P(c_vp)], c_i32),
        "dfl_setup_device": ([c_i32], c_i32),
        "dfl_gen_rows": ([c_i32, P(GenParams), c_i64, c_i64, c_vp, c_vp, c_vp, P(c_i64), c_vp], c_i32),
        "dfl_gen_unknown_of_node": ([c_i32, P(GenParams), c_vp], c_i32),
        "dfl_hier_num_levels": ([c_vp], c_i32),
        "dfl_hier_level_shape": ([c_vp, c_i32, c_i32, P(c_i64), P(c_i64), P(c_i64)], c_i32),
        "dfl_hier_level_copy": ([c_vp, c_i32, c_i32, c_vp, c_vp, c_vp], c_i32),
        "dfl_hier_level_weights": ([c_vp, c_i32, c_vp], c_i32),
        "dfl_hier_bottom_inverse": ([c_vp, c_vp], c_i32),
        "dfl_hier_free": ([c_vp], None),
        "dfl_basis_az": ([P(Csr), c_i32, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, P(c_vp), c_vp], c_i32),
        "dfl_matrix_shape": ([c_vp, P(c_i64), P(c_i64), P(c_i64)], c_i32),
        "dfl_matrix_copy": ([c_vp, c_vp, c_vp, c_vp], c_i32),
        "dfl_matrix_free": ([c_vp], None),
        "dfl_mm_read": ([ctypes.c_char_p, P(c_vp)], c_i32),
        "dfl_vec_read": ([ctypes.c_char_p, c_i32, P(c_vp)], c_i32),
        "dfl_dense_inverse": ([c_i64, c_vp, c_vp], c_i32),
        "dfl_ctx_create": ([c_i32, P(c_vp)], c_i32),
        "dfl_ctx_destroy": ([c_vp], None),
        "dfl_last_error": ([c_vp], ctypes.c_char_p),
        "dfl_nccl_unique_id": ([c_vp], c_i32),
        "dfl_ctx_set_comm": ([c_vp, c_i32, c_i32, c_vp], c_i32),
        "dfl_fabric_create": ([c_i32, P(c_vp)], c_i32),
        "dfl_fabric_destroy": ([c_vp], None),
        "dfl_fabric_set_timeout": ([c_vp, c_dbl], c_i32),
        "dfl_ctx_set_fabric": ([c_vp, c_vp, c_i32], c_i32),
        "dfl_ctx_set_operator": ([c_vp, P(Csr), c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp], c_i32),
        "dfl_ctx_add_hierarchy": ([c_vp, c_i32, c_vp], c_i32),
        "dfl_ctx_set_deflation": ([c_vp, c_i32, c_vp, P(Csr), c_i64, c_vp, c_i32], c_i32),
        "dfl_ctx_finalize": ([c_vp], c_i32),
        "dfl_ctx_set_inexact": ([c_vp, c_vp, c_dbl], c_i32),
        "dfl_ctx_device_bytes": ([c_vp], c_i64),
        "dfl_solve": ([c_vp, P(SolveParams), c_vp, c_vp, c_i32, P(Report)], c_i32),
        "dfl_ctx_wait_stream": ([c_vp, c_vp], c_i32),
        "dfl_host_alloc": ([c_i64], c_vp),
        "dfl_host_free": ([c_vp], None),
        "dfl_op_apply": ([c_vp, c_vp, c_vp, c_i32], c_i32),
        "dfl_precond_apply": ([c_vp, c_vp, c_vp, c_i32], c_i32),
        "dfl_project": ([c_vp, c_vp, c_vp, c_i32], c_i32),
        "dfl_coarse_lift": ([c_vp, c_vp, c_vp, c_i32], c_i32),
        "dfl_dot": ([c_vp, c_vp, c_vp, c_i32, P(c_dbl)], c_i32),
        "dfl_spmv_csr": ([P(Csr), c_vp, c_vp, c_i32], c_i32),
        "dfl_ctx_time": ([c_vp, c_i32, c_i32, P(c_dbl), P(c_dbl)], c_i32),
        "dfl_ctx_profile_vcycle": ([c_vp, c_i32, c_i32, c_vp, c_vp], c_i32),
        "dfl_block_create": ([c_vp, c_i32, P(BlockDesc), P(c_vp)], c_i32),
        "dfl_block_free": ([c_vp], None),
        "dfl_block_last_error": ([c_vp], ctypes.c_char_p),
        "dfl_block_device_bytes": ([c_vp], c_i64),
        "dfl_block_solve": ([c_vp, P(BlockParams), c_vp, c_vp, c_i32, P(BlockReport)], c_i32),
        "dfl_block_precond": ([c_vp, P(BlockParams), c_vp, c_vp, c_vp, c_vp, c_i32, P(c_i64), P(c_i64)], c_i32),
        "dfl_block_schur_apply": ([c_vp, c_vp, c_vp, c_i32], c_i32),
        "dfl_block_apply": ([c_vp, c_vp, c_vp, c_i32], c_i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


EXPORTED = None  # filled lazily by exported_symbols()


def exported_symbols():
    """The dfl_* functions include/dflb200.h declares."""
    import re

    hdr = os.path.join(os.path.dirname(_PKG), "include", "dflb200.h")
    with open(hdr) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(dfl_[a-z0-9_]+)\s*\(", text)))


def pinned_empty(n: int) -> np.ndarray:
    """float64[n] in page-locked host memory from the library's block cache
    (dfl_host_alloc); the block goes back to the cache when the array (and
    every view of it) is gone.  Pageable memory if the driver refuses."""
    import weakref

    p = lib().dfl_host_alloc(8 * n) if n > 0 else None
    if not p:
        return np.empty(n)
    buf = (ctypes.c_double * n).from_address(p)
    weakref.finalize(buf, lib().dfl_host_free, c_vp(p))
    return np.frombuffer(buf, dtype=np.float64)


def _ptr(a: np.ndarray):
    return c_vp(a.ctypes.data) if a is not None else None


def setup_error() -> str:
    return (lib().dfl_last_setup_error() or b"").decode()


def check(rc: int, ctx=None) -> None:
    if rc != 0:
        msg = (lib().dfl_last_error(ctx) if ctx is not None else lib().dfl_last_setup_error()) or b""
        raise_for_status(rc, msg.decode())


class CsrArrays:
    """Keeps numpy buffers alive for a ctypes Csr view."""

    def __init__(self, nrows, ncols, row_ptr, col_idx, values):
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.s = Csr(int(nrows), int(ncols), _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(self.values))


class Hierarchy:
    """Host AMG hierarchy built by the native setup (dfl_hier_build)."""

    def __init__(self, A: CsrArrays, opts: AmgOptions, device: int | None = None):
        """device: build the products on that GPU (dfl_setup_device), else on the host."""
        h = c_vp()
        L = lib()
        if device is not None:
            check(L.dfl_setup_device(int(device)))
        try:
            check(L.dfl_hier_build(ctypes.byref(A.s), ctypes.byref(opts), ctypes.byref(h)))
        finally:
            if device is not None:
                L.dfl_setup_device(-1)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dfl_hier_free(self.h)
            self.h = None

    @property
    def nlevels(self) -> int:
        return lib().dfl_hier_num_levels(self.h)

    def level_shape(self, level: int, which: int = LEVEL_A):
        r, c, z = c_i64(), c_i64(), c_i64()
        check(lib().dfl_hier_level_shape(self.h, level, which, ctypes.byref(r), ctypes.byref(c), ctypes.byref(z)))
        return r.value, c.value, z.value

    @property
    def level_sizes(self):
        return [self.level_shape(l)[0] for l in range(self.nlevels)]

    def level_nnz(self):
        return [self.level_shape(l)[2] for l in range(self.nlevels)]

    def matrix(self, level: int, which: int = LEVEL_A):
        nr, nc, nnz = self.level_shape(level, which)
        if nnz < 0:
            return None
        ptr = np.empty(nr + 1, dtype=np.int64)
        col = np.empty(nnz, dtype=np.int64)
        val = np.empty(nnz, dtype=np.float64)
        check(lib().dfl_hier_level_copy(self.h, level, which, _ptr(ptr), _ptr(col), _ptr(val)))
        return nr, nc, ptr, col, val

    def weights(self, level: int) -> np.ndarray:
        n = self.level_shape(level)[0]
        w = np.empty(n)
        check(lib().dfl_hier_level_weights(self.h, level, _ptr(w)))
        return w

    def bottom_inverse(self) -> np.ndarray:
        n = self.level_shape(self.nlevels - 1)[0]
        inv = np.empty((n, n))
        check(lib().dfl_hier_bottom_inverse(self.h, _ptr(inv)))
        return inv


def basis_az(A: CsrArrays, k: int, zext: np.ndarray, owner: np.ndarray, rowsub: np.ndarray, K: int,
             sub0: int, nsub: int, keep_zeros: bool = False):
    zext = np.ascontiguousarray(zext, dtype=np.float64)
    owner = np.ascontiguousarray(owner, dtype=np.int32)
    rowsub = np.ascontiguousarray(rowsub, dtype=np.int32)
    E_rows = np.zeros((nsub * k, K))
    m = c_vp()
    check(lib().dfl_basis_az(ctypes.byref(A.s), k, _ptr(zext), _ptr(owner), _ptr(rowsub), K, sub0, nsub,
                             1 if keep_zeros else 0, ctypes.byref(m), _ptr(E_rows)))
    try:
        r, c, z = c_i64(), c_i64(), c_i64()
        check(lib().dfl_matrix_shape(m, ctypes.byref(r), ctypes.byref(c), ctypes.byref(z)))
        ptr = np.empty(r.value + 1, dtype=np.int64)
        col = np.empty(z.value, dtype=np.int64)
        val = np.empty(z.value)
        check(lib().dfl_matrix_copy(m, _ptr(ptr), _ptr(col), _ptr(val)))
    finally:
        lib().dfl_matrix_free(m)
    return (r.value, c.value, ptr, col, val), E_rows


def dense_inverse(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    inv = np.empty((n, n))
    check(lib().dfl_dense_inverse(n, _ptr(a), _ptr(inv)))
    return inv


class DeviceContext:
    """One rank's device state (dfl_ctx)."""

    def __init__(self, device: int = 0):
        h = c_vp()
        check(lib().dfl_ctx_create(int(device), ctypes.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dfl_ctx_destroy(self.h)
            self.h = None

    __del__ = close

    def _c(self, rc):
        check(rc, self.h)

    def set_fabric(self, fabric: "Fabric", rank: int):
        self._fabric = fabric  # keep alive
        self._c(lib().dfl_ctx_set_fabric(self.h, fabric.h, rank))

    def set_comm(self, nranks: int, rank: int, nccl_id: bytes):
        buf = ctypes.create_string_buffer(nccl_id, 128)
        self._c(lib().dfl_ctx_set_comm(self.h, nranks, rank, buf))

    def set_operator(self, A: CsrArrays, sub_offsets, nbr, recv_counts, send_counts, send_idx):
        self._keep_sub = np.ascontiguousarray(sub_offsets, dtype=np.int64)
        nbr = np.ascontiguousarray(nbr, dtype=np.int32)
        rc_ = np.ascontiguousarray(recv_counts, dtype=np.int64)
        sc_ = np.ascontiguousarray(send_counts, dtype=np.int64)
        si = np.ascontiguousarray(send_idx, dtype=np.int64)
        self._c(lib().dfl_ctx_set_operator(self.h, ctypes.byref(A.s), len(self._keep_sub) - 1,
                                           _ptr(self._keep_sub), len(nbr), _ptr(nbr), _ptr(rc_), _ptr(sc_),
                                           _ptr(si)))

    def add_hierarchy(self, sub: int, h: Hierarchy):
        self._c(lib().dfl_ctx_add_hierarchy(self.h, sub, h.h))

    def set_deflation(self, k: int, zcols, AZ: CsrArrays, K: int, Einv, first_sub: int):
        zc = np.ascontiguousarray(zcols, dtype=np.float64) if zcols is not None and k > 1 else None
        Ei = np.ascontiguousarray(Einv, dtype=np.float64)
        self._c(lib().dfl_ctx_set_deflation(self.h, k, _ptr(zc) if zc is not None else None,
                                            ctypes.byref(AZ.s), K, _ptr(Ei), first_sub))

    def set_inexact(self, E, coarse_tol: float):
        self._E = np.ascontiguousarray(E, dtype=np.float64) if E is not None else None
        self._c(lib().dfl_ctx_set_inexact(self.h, _ptr(self._E) if self._E is not None else None, float(coarse_tol)))

    def finalize(self):
        self._c(lib().dfl_ctx_finalize(self.h))

    @property
    def device_bytes(self) -> int:
        return lib().dfl_ctx_device_bytes(self.h)

    def wait_stream(self, stream: int | None):
        """Order the context after the work queued on CUDA stream `stream` (a cudaStream_t)."""
        self._c(lib().dfl_ctx_wait_stream(self.h, c_vp(stream or 0)))

    def solve(self, params: SolveParams, b, x, ptr_kind: int = PTR_HOST) -> Report:
        rep = Report()
        bp = _ptr(b) if ptr_kind == PTR_HOST else c_vp(b)
        xp = _ptr(x) if ptr_kind == PTR_HOST else c_vp(x)
        self._c(lib().dfl_solve(self.h, ctypes.byref(params), bp, xp, ptr_kind, ctypes.byref(rep)))
        return rep

    def _unary(self, fn, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self._c(fn(self.h, _ptr(v), _ptr(out), PTR_HOST))
        return out

    def op_apply(self, v):
        return self._unary(lib().dfl_op_apply, v)

    def precond_apply(self, v):
        return self._unary(lib().dfl_precond_apply, v)

    def project(self, v):
        return self._unary(lib().dfl_project, v)

    def coarse_lift(self, v):
        return self._unary(lib().dfl_coarse_lift, v)

    def dot(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = c_dbl()
        self._c(lib().dfl_dot(self.h, _ptr(a), _ptr(b), PTR_HOST, ctypes.byref(out)))
        return out.value

    def profile_vcycle(self, reps: int = 10):
        """[(label, ms)] per launch of one V-cycle."""
        cap = 256
        ms = np.zeros(cap)
        lab = ctypes.create_string_buffer(32 * cap)
        cnt = lib().dfl_ctx_profile_vcycle(self.h, reps, cap, _ptr(ms), lab)
        if cnt < 0:
            self._c(cnt)
        raw = lab.raw
        return [(raw[32 * i:32 * i + 32].split(b"\0")[0].decode(), float(ms[i])) for i in range(cnt)]

    def time(self, what: int, reps: int):
        ms, by = c_dbl(), c_dbl()
        self._c(lib().dfl_ctx_time(self.h, what, reps, ctypes.byref(ms), ctypes.byref(by)))
        return ms.value, by.value


class Fabric:
    """In-process communicator (dfl_fabric) for multi-rank tests on one device."""

    def __init__(self, nranks: int):
        h = c_vp()
        check(lib().dfl_fabric_create(nranks, ctypes.byref(h)))
        self.h = h
        self.nranks = nranks

    def set_timeout(self, seconds: float):
        check(lib().dfl_fabric_set_timeout(self.h, float(seconds)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dfl_fabric_destroy(self.h)
            self.h = None


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().dfl_nccl_unique_id(buf))
    return buf.raw


def spmv_device(A: CsrArrays, x: np.ndarray, device: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.s.nrows)
    check(lib().dfl_spmv_csr(ctypes.byref(A.s), _ptr(x), _ptr(y), device))
    return y


def breakdown_string(code: int, value: float | None = None) -> str:
    """The reference's breakdown note; CG's carry the scalar (krylov.py:124,140)."""
    s = (lib().dfl_breakdown_string(code) or b"").decode()
    if value is not None and code == 1:  # DFL_BRK_CURVATURE
        return f"{s} = {value:g}"
    if value is not None and code == 2:  # DFL_BRK_RZ
        return f"{s} to {value:g}"
    return s


class DeviceBlock:
    """A saddle-point block system on the device (dfl_block).  ``pressure`` is
    the DeviceContext of the deflated pressure solver (shares its stream) or
    None (operators only, or no pressure unknowns)."""

    def __init__(self, n, n_u, A: CsrArrays, K, G, D, S, u_idx, p_idx, wK, invKdiag, pressure=None,
                 device: int = 0):
        self._keep = [A, K, G, D, S]
        self._u = np.ascontiguousarray(u_idx, dtype=np.int32)
        self._p = np.ascontiguousarray(p_idx, dtype=np.int32)
        self._w = np.ascontiguousarray(wK, dtype=np.float64)
        self._k = np.ascontiguousarray(invKdiag, dtype=np.float64)
        ref = lambda m: ctypes.cast(ctypes.pointer(m.s), c_vp) if m is not None else None  # noqa: E731
        d = BlockDesc(int(n), int(n_u), ref(A), ref(K), ref(G), ref(D), ref(S), _ptr(self._u), _ptr(self._p),
                      _ptr(self._w), _ptr(self._k))
        self.pressure = pressure  # keep the context alive for the block's lifetime
        h = c_vp()
        check(lib().dfl_block_create(pressure.h if pressure is not None else None, int(device), ctypes.byref(d),
                                     ctypes.byref(h)))
        self.h = h
        self.n, self.n_u, self.n_p = int(n), int(n_u), int(n) - int(n_u)

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.dfl_block_free(self.h)
            self.h = None

    __del__ = close

    def _c(self, rc):
        if rc != 0:
            raise_for_status(rc, (lib().dfl_block_last_error(self.h) or b"").decode())

    @property
    def device_bytes(self) -> int:
        return lib().dfl_block_device_bytes(self.h)

    def solve(self, params: BlockParams, b, x, ptr_kind: int = PTR_HOST) -> BlockReport:
        rep = BlockReport()
        bp = _ptr(b) if ptr_kind == PTR_HOST else c_vp(b)
        xp = _ptr(x) if ptr_kind == PTR_HOST else c_vp(x)
        self._c(lib().dfl_block_solve(self.h, ctypes.byref(params), bp, xp, ptr_kind, ctypes.byref(rep)))
        return rep

    def precond(self, params: BlockParams, b_u, b_p):
        b_u = np.ascontiguousarray(b_u, dtype=np.float64)
        b_p = np.ascontiguousarray(b_p, dtype=np.float64)
        u, p = np.empty(self.n_u), np.empty(self.n_p)
        vi, pi = c_i64(), c_i64()
        self._c(lib().dfl_block_precond(self.h, ctypes.byref(params), _ptr(b_u), _ptr(b_p), _ptr(u), _ptr(p),
                                        PTR_HOST, ctypes.byref(vi), ctypes.byref(pi)))
        return u, p, vi.value, pi.value

    def schur_apply(self, p):
        p = np.ascontiguousarray(p, dtype=np.float64)
        out = np.empty(self.n_p)
        self._c(lib().dfl_block_schur_apply(self.h, _ptr(p), _ptr(out), PTR_HOST))
        return out

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.n)
        self._c(lib().dfl_block_apply(self.h, _ptr(x), _ptr(out), PTR_HOST))
        return out
