"""Thin Python binding of libnrto.so (include/nrto.h): argument marshalling only.

Every step of the inner solve runs in the CUDA kernels of libnrto.so; this
module only converts torch tensors / numpy arrays to the C structs.  There
is no CPU fallback: importing works without a GPU, but every compute call
raises if the library or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnrto.so")

NRTO_OK, NRTO_EINVAL, NRTO_ENOTSPD, NRTO_ECUDA, NRTO_ENOMEM, NRTO_ESTATE = 0, -1, -2, -3, -4, -5
NRTO_FULLADMM, NRTO_DR = 0, 1
NRTO_CONVERGED, NRTO_MAX_ITERS, NRTO_DIVERGED = 0, 1, 2
NRTO_MEM_DEVICE, NRTO_MEM_HOST = 0, 1

_dp = C.POINTER(C.c_double)


class nrto_shape(C.Structure):
    _fields_ = [("n_x", C.c_int32), ("n_u", C.c_int32), ("T", C.c_int32), ("n_g", C.c_int32),
                ("batch", C.c_int32), ("cone_knot", C.POINTER(C.c_int32)),
                ("cone_kind", C.POINTER(C.c_int8))]


class nrto_data(C.Structure):
    _fields_ = [("memory", C.c_int32)] + [(n, C.c_void_p) for n in
                ("A", "B", "grad", "g0", "Psi", "tau", "W_K", "R_u", "u_hat", "r_trust")]


PARAM_DOUBLES = ("rho", "rho_admm", "alpha_dr", "sigma_dr", "r_s", "eps_p", "eps_d", "eps_dr",
                 "rho_qp", "sigma_qp", "alpha_qp")
PARAM_INTS = ("max_iter", "max_admm_iter", "max_dr_iter", "qp_iters", "check_every", "fixed_iters")


class nrto_uncertainty(C.Structure):
    _fields_ = [("memory", C.c_int32), ("n_z", C.c_int32), ("Gamma", C.c_void_p), ("Psi", C.c_void_p)]


class nrto_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in PARAM_DOUBLES] + [(n, C.c_int32) for n in PARAM_INTS]


OUT_FIELDS = ("kv", "du", "p", "p_tilde", "lam_p", "nu", "lam_nu", "objective", "margin_cone",
              "margin_lin", "iters", "status", "r_p", "r_d", "hist")


class nrto_out(C.Structure):
    _fields_ = [("memory", C.c_int32)] + [(n, C.c_void_p) for n in OUT_FIELDS]


_lib = None


class NrtoError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libnrto error {code}: {msg}")
        self.code = code


def lib():
    """Load libnrto.so (fails loudly; no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.nrto_last_error.restype = C.c_char_p
        L.nrto_default_params.argtypes = [C.POINTER(nrto_params)]
        L.nrto_layout.argtypes = [C.POINTER(nrto_shape), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.nrto_setup.argtypes = [C.POINTER(nrto_shape), C.POINTER(nrto_data), C.POINTER(nrto_params),
                                 C.c_void_p, C.POINTER(C.c_void_p)]
        L.nrto_inner_solve.argtypes = [C.c_void_p, C.c_int32, C.POINTER(nrto_out), C.c_void_p]
        L.nrto_gain_update.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.nrto_soc_project.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_void_p]
        L.nrto_destroy.argtypes = [C.c_void_p]
        L.nrto_launch_count.argtypes = [C.c_void_p]
        L.nrto_launch_count.restype = C.c_int64
        L.nrto_refresh.argtypes = [C.c_void_p, C.POINTER(nrto_data), C.c_void_p]
        L.nrto_profile_enable.argtypes = [C.c_void_p, C.c_int32]
        L.nrto_profile_read.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_double),
                                        C.POINTER(C.c_int64)]
        L.nrto_pass_bytes.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.nrto_setup_general.argtypes = [C.POINTER(nrto_shape), C.POINTER(nrto_data),
                                         C.POINTER(nrto_uncertainty), C.POINTER(nrto_params),
                                         C.c_void_p, C.POINTER(C.c_void_p)]
        L.nrto_case_stats_enable.argtypes = [C.c_void_p, C.c_int32]
        L.nrto_case_stats_read.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]
        L.nrto_solve_begin.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.nrto_solve_iterate.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_void_p]
        L.nrto_solve_flags.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.nrto_solve_end.argtypes = [C.c_void_p, C.POINTER(nrto_out), C.c_void_p]
        for f in ("nrto_layout", "nrto_setup", "nrto_inner_solve", "nrto_gain_update",
                  "nrto_soc_project", "nrto_destroy", "nrto_refresh", "nrto_profile_enable",
                  "nrto_profile_read", "nrto_pass_bytes", "nrto_case_stats_enable",
                  "nrto_case_stats_read", "nrto_solve_begin", "nrto_solve_iterate",
                  "nrto_solve_flags", "nrto_solve_end", "nrto_setup_general", "nrto_set_allocator",
                  "nrto_shard_cones", "nrto_dr_step", "nrto_buffer"):
            getattr(L, f).restype = C.c_int
        L.nrto_set_allocator.argtypes = [ALLOC_FN, FREE_FN, C.c_void_p]
        L.nrto_shard_cones.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        L.nrto_dr_step.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        L.nrto_buffer.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
        _lib = L
    return _lib


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)
_alloc_cbs = None      # keeps the ctypes callbacks alive while registered


def nrto_set_allocator(alloc, release):
    """Register Python callables alloc(bytes, stream_ptr) -> device ptr (int) and
    release(ptr, stream_ptr) as the workspace allocator of new handles (nrto.h);
    alloc=None restores cudaMalloc / cudaFree."""
    global _alloc_cbs
    if alloc is None:
        _check(lib().nrto_set_allocator(ALLOC_FN(), FREE_FN(), None))
        _alloc_cbs = None
        return

    def a(ctx, nbytes, stream):
        try:
            return int(alloc(int(nbytes), stream or 0)) or None
        except Exception:
            return None

    def r(ctx, ptr, stream):
        try:
            release(int(ptr), stream or 0)
        except Exception:
            pass

    cbs = (ALLOC_FN(a), FREE_FN(r))
    _check(lib().nrto_set_allocator(cbs[0], cbs[1], None))
    _alloc_cbs = cbs


def nrto_shard_cones(handle, cone_lo, cone_hi):
    _check(lib().nrto_shard_cones(C.c_void_p(handle), int(cone_lo), int(cone_hi)))


def nrto_dr_step(handle, phase, l=0, stream=None):
    _check(lib().nrto_dr_step(C.c_void_p(handle), int(phase), int(l), _stream_ptr(stream)))


class _DevBuf:
    """__cuda_array_interface__ view of a handle-owned float64 device buffer."""
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3}


def nrto_buffer(handle, which):
    """torch tensor aliasing handle buffer `which` (0 Z, 1 pi, 2 r_dr partials)."""
    import torch
    ptr, n = C.c_void_p(), C.c_int64()
    _check(lib().nrto_buffer(C.c_void_p(handle), int(which), C.byref(ptr), C.byref(n)))
    return torch.as_tensor(_DevBuf(ptr.value, n.value), device="cuda")


def use_torch_allocator(enable=True):
    """Back the workspace of new handles with torch's CUDA caching allocator."""
    if not enable:
        nrto_set_allocator(None, None)
        return
    import torch

    def a(nbytes, stream):
        return torch.cuda.caching_allocator_alloc(nbytes, stream=stream or None)

    def r(ptr, stream):
        torch.cuda.caching_allocator_delete(ptr)

    nrto_set_allocator(a, r)


def _check(code):
    if code != NRTO_OK:
        raise NrtoError(code, nrto_last_error())


def nrto_last_error() -> str:
    return lib().nrto_last_error().decode()


def nrto_default_params(**overrides) -> nrto_params:
    p = nrto_params()
    lib().nrto_default_params(C.byref(p))
    for k, v in overrides.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p


def _shape_struct(shape, batch):
    knot = np.ascontiguousarray(shape.cone_knot, np.int32)
    kind = np.ascontiguousarray(shape.cone_kind, np.int8)
    s = nrto_shape(shape.n_x, shape.n_u, shape.T, shape.n_g, batch,
                   knot.ctypes.data_as(C.POINTER(C.c_int32)), kind.ctypes.data_as(C.POINTER(C.c_int8)))
    s._keep = (knot, kind)
    return s


def nrto_layout(shape, batch=1):
    """(E, offsets[n_g+1]) of the ragged cone rows (host only)."""
    s = _shape_struct(shape, batch)
    E = C.c_int64()
    off = np.zeros(shape.n_g + 1, np.int64)
    _check(lib().nrto_layout(C.byref(s), C.byref(E), off.ctypes.data_as(C.POINTER(C.c_int64))))
    return int(E.value), off


def _ptr(t):
    if t is None:
        return None
    if not t.is_contiguous():
        # the C ABI reads plain row-major arrays: a strided view (e.g. a transposed
        # numpy array wrapped by torch.tensor, which keeps its strides) would be read
        # in storage order
        raise ValueError("nrto: array arguments must be contiguous (row-major)")
    return C.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


DATA_KEYS = ("A", "B", "grad", "g0", "Psi", "tau", "W_K", "R_u", "u_hat", "r_trust")


def to_tensors(batch_np: dict, device="cuda", pinned=False):
    """numpy batch dict (gen.make_batch) -> contiguous float64 torch tensors."""
    import torch
    out = {}
    for k in DATA_KEYS:
        a = np.ascontiguousarray(np.asarray(batch_np[k], np.float64))
        t = torch.from_numpy(a)
        if device == "cpu":
            out[k] = t.pin_memory() if pinned else t
        else:
            out[k] = t.to(device)
    return out


def nrto_setup(shape, data: dict, params: nrto_params, stream=None, memory=NRTO_MEM_DEVICE):
    """Returns an opaque handle (int).  data: tensors [b][...] (device or host)."""
    batch = int(data["tau"].shape[0])
    s = _shape_struct(shape, batch)
    dd = nrto_data(memory, *[_ptr(data[k]) for k in DATA_KEYS])
    h = C.c_void_p()
    _check(lib().nrto_setup(C.byref(s), C.byref(dd), C.byref(params), _stream_ptr(stream), C.byref(h)))
    return h.value


def nrto_setup_general(shape, data: dict, Gamma, Psi, params: nrto_params, stream=None,
                       memory=NRTO_MEM_DEVICE):
    """General uncertainty set (zeta = Gamma z, Psi^T Psi = S^-1): tensors
    Gamma [b][(T+1) n_x][n_z], Psi [b][n_z][n_z] in the same memory as data."""
    batch = int(data["tau"].shape[0])
    s = _shape_struct(shape, batch)
    dd = nrto_data(memory, *[_ptr(data[k]) for k in DATA_KEYS])
    Gamma, Psi = Gamma.contiguous(), Psi.contiguous()
    un = nrto_uncertainty(memory, int(Gamma.shape[-1]), _ptr(Gamma), _ptr(Psi))
    h = C.c_void_p()
    _check(lib().nrto_setup_general(C.byref(s), C.byref(dd), C.byref(un), C.byref(params),
                                    _stream_ptr(stream), C.byref(h)))
    return h.value


def nrto_refresh(handle, data: dict, stream=None, memory=NRTO_MEM_DEVICE):
    dd = nrto_data(memory, *[_ptr(data[k]) for k in DATA_KEYS])
    _check(lib().nrto_refresh(C.c_void_p(handle), C.byref(dd), _stream_ptr(stream)))


NRTO_K_PASS, NRTO_K_ADJOINT, NRTO_K_GAIN, NRTO_K_QP, NRTO_K_OTHER = 0, 1, 2, 3, 4
KERNEL_CLASSES = ("pass", "adjoint", "gain", "qp", "other", "ctrl")


def nrto_profile_enable(handle, enable=True):
    _check(lib().nrto_profile_enable(C.c_void_p(handle), int(bool(enable))))


def nrto_profile_read(handle, kclass):
    """(total_ms, launches) of one kernel class since the last read."""
    ms, n = C.c_double(), C.c_int64()
    _check(lib().nrto_profile_read(C.c_void_p(handle), int(kclass), C.byref(ms), C.byref(n)))
    return float(ms.value), int(n.value)


def nrto_pass_bytes(handle) -> int:
    """Algorithmic bytes moved by the fused state-cone pass since the last call."""
    n = C.c_int64()
    _check(lib().nrto_pass_bytes(C.c_void_p(handle), C.byref(n)))
    return int(n.value)


def nrto_case_stats_enable(handle, enable=True):
    _check(lib().nrto_case_stats_enable(C.c_void_p(handle), int(bool(enable))))


def nrto_case_stats_read(handle, L) -> np.ndarray:
    """[L, 3] int64 counts of projection cases 1/2/3 per iteration of the last FullADMM solve."""
    out = np.zeros((int(L), 3), np.int64)
    _check(lib().nrto_case_stats_read(C.c_void_p(handle), out.ctypes.data_as(C.POINTER(C.c_int64)),
                                      int(L)))
    return out


def nrto_solve_begin(handle, engine, stream=None):
    _check(lib().nrto_solve_begin(C.c_void_p(handle), int(engine), _stream_ptr(stream)))


def nrto_solve_iterate(handle, n_iters, stream=None) -> int:
    done = C.c_int32()
    _check(lib().nrto_solve_iterate(C.c_void_p(handle), int(n_iters), C.byref(done), _stream_ptr(stream)))
    return int(done.value)


def nrto_solve_flags(handle, flags, stream=None):
    """flags: device float64 tensor [4] <- [max r_p/eps_p, max r_d/eps_d, #active, any diverged]."""
    _check(lib().nrto_solve_flags(C.c_void_p(handle), _ptr(flags), _stream_ptr(stream)))


def nrto_solve_end(handle, out: dict, stream=None, memory=NRTO_MEM_DEVICE):
    o = nrto_out(memory, *[_ptr(out.get(k)) for k in OUT_FIELDS])
    _check(lib().nrto_solve_end(C.c_void_p(handle), C.byref(o), _stream_ptr(stream)))


def nrto_inner_solve(handle, engine, out: dict, stream=None, memory=NRTO_MEM_DEVICE):
    o = nrto_out(memory, *[_ptr(out.get(k)) for k in OUT_FIELDS])
    _check(lib().nrto_inner_solve(C.c_void_p(handle), int(engine), C.byref(o), _stream_ptr(stream)))


def nrto_gain_update(handle, nu, kv_prev, kv_next, stream=None):
    _check(lib().nrto_gain_update(C.c_void_p(handle), _ptr(nu), _ptr(kv_prev), _ptr(kv_next),
                                  _stream_ptr(stream)))


def nrto_soc_project(t, y, offsets, t_out, y_out, stream=None):
    n = int(t.shape[0])
    _check(lib().nrto_soc_project(_ptr(t), _ptr(y), _ptr(offsets), n, _ptr(t_out), _ptr(y_out),
                                  _stream_ptr(stream)))


def nrto_launch_count(handle) -> int:
    return int(lib().nrto_launch_count(C.c_void_p(handle)))


def nrto_destroy(handle):
    _check(lib().nrto_destroy(C.c_void_p(handle)))


# ------------------------------------------------------------------ convenience
def alloc_out(shape, batch, E, device="cuda", pinned=False, full=True, ragged=True):
    """Output tensors for nrto_inner_solve (all fields when full=True; the ragged
    [batch][E] nu / lam_nu only when ragged=True as well)."""
    import torch
    f64, i32 = torch.float64, torch.int32
    kw = dict(device=device)
    if device == "cpu" and pinned:
        kw["pin_memory"] = True
    NK = shape.T * shape.n_u * shape.n_x
    o = dict(kv=torch.empty(batch, NK, dtype=f64, **kw),
             du=torch.empty(batch, shape.T * shape.n_u, dtype=f64, **kw),
             p=torch.empty(batch, shape.n_g, dtype=f64, **kw),
             p_tilde=torch.empty(batch, shape.n_g, dtype=f64, **kw),
             lam_p=torch.empty(batch, shape.n_g, dtype=f64, **kw),
             iters=torch.empty(batch, dtype=i32, **kw), status=torch.empty(batch, dtype=i32, **kw),
             r_p=torch.empty(batch, dtype=f64, **kw), r_d=torch.empty(batch, dtype=f64, **kw),
             objective=torch.empty(batch, dtype=f64, **kw))
    if full:
        o.update(margin_cone=torch.empty(batch, shape.n_g, dtype=f64, **kw),
                 margin_lin=torch.empty(batch, shape.n_g, dtype=f64, **kw))
        if ragged:
            o.update(nu=torch.empty(batch, E, dtype=f64, **kw), lam_nu=torch.empty(batch, E, dtype=f64, **kw))
    return o


class InnerSolver:
    """Owns one nrto handle for a batch of instances sharing a cone structure.
    With Gamma / Psi given: a general uncertainty set (nrto_setup_general); the
    ragged nu / lam_nu outputs are then dense [b][n_g][n_z] rows."""

    def __init__(self, shape, data: dict, params=None, stream=None, memory=NRTO_MEM_DEVICE,
                 Gamma=None, Psi=None, **pkw):
        self.shape = shape
        self.params = params if params is not None else nrto_default_params(**pkw)
        self.batch = int(data["tau"].shape[0])
        self.E, self.offsets = nrto_layout(shape, self.batch)
        self.stream = stream
        if Gamma is not None:
            self.E = shape.n_g * int(Gamma.shape[-1])
            self.handle = nrto_setup_general(shape, data, Gamma, Psi, self.params, stream, memory)
        else:
            self.handle = nrto_setup(shape, data, self.params, stream, memory)

    def solve(self, engine=NRTO_FULLADMM, out=None, full=True, memory=NRTO_MEM_DEVICE):
        if out is None:
            out = alloc_out(self.shape, self.batch, self.E,
                            device="cpu" if memory == NRTO_MEM_HOST else "cuda",
                            pinned=memory == NRTO_MEM_HOST, full=full)
        nrto_inner_solve(self.handle, engine, out, self.stream, memory)
        return out

    def refresh(self, data: dict, memory=NRTO_MEM_DEVICE):
        nrto_refresh(self.handle, data, self.stream, memory)

    def profile(self, enable=True):
        nrto_profile_enable(self.handle, enable)

    def profile_read(self):
        return {n: nrto_profile_read(self.handle, i) for i, n in enumerate(KERNEL_CLASSES)}

    def pass_bytes(self):
        return nrto_pass_bytes(self.handle)

    def case_stats(self, enable=True):
        nrto_case_stats_enable(self.handle, enable)

    def case_stats_read(self, L=None):
        return nrto_case_stats_read(self.handle, self.params.max_iter if L is None else L)

    def gain_update(self, nu, kv_prev, kv_next):
        nrto_gain_update(self.handle, nu, kv_prev, kv_next, self.stream)

    def launches(self):
        return nrto_launch_count(self.handle)

    def close(self):
        if self.handle:
            nrto_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
