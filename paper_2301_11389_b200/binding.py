"""Thin ctypes binding over libstencil_b200.so (include/stencil.h).

Argument marshalling only: every step of the stencil path runs in the CUDA
kernels behind the C ABI.  Device buffers are torch tensors (PyTorch supplies
device memory and streams); their ``data_ptr()`` values are passed as plain
pointers.  There is no fallback: if the library is missing or fails to load,
``lib()`` raises.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# STB200_LIB: an experiment build (build.build_experiment) for A/B runs
LIB_PATH = os.environ.get("STB200_LIB") or os.path.join(PKG, "libstencil_b200.so")

KINDS = {"jacobi2d5": 1, "jacobi2d9": 2, "gaussblur5x5": 3, "gameoflife": 4,
         "laplacian3d7": 5, "jacobi3d7": 6, "wave13pt": 7, "divergence": 8,
         "gradient": 9, "tricubic": 10, "tricubic2": 11, "uxx1": 12, "lapgsrb": 13, "whispering": 14}
DTYPES = {"f32": 1, "f64": 2, "i32": 3}
VARIANTS = {"shuffle": 0, "plain": 1, "paper_original": 2, "paper_ptxasw": 3,
            "paper_noload": 4, "paper_nocorner": 5, "paper_uniform": 6,
            "auto": 7}
STATUS = {0: "ST_OK", -1: "ST_EARG", -2: "ST_EUNSUPPORTED", -3: "ST_EALIGN",
          -4: "ST_ECUDA", -5: "ST_ENCCL", -6: "ST_ESTATE"}

# Every symbol include/stencil.h declares (checked by tests/test_abi.py).
EXPORTS = ["stencil_create", "stencil_set_variant", "stencil_get_variant", "stencil_set_fusion", "stencil_arity",
           "stencil_info", "stencil_step", "stencil_step_range", "stencil_run", "stencil_run_host", "stencil_run_host_async",
           "stencil_destroy", "stencil_last_error", "stencil_version", "stencil_slab_plan",
           "stencil_dist_get_id", "stencil_dist_attach", "stencil_dist_attach_host",
           "stencil_dist_attach_p2p", "stencil_p2p_export", "stencil_p2p_import"]

# int fn(int peer, const void* send, size_t send_bytes, void* recv, size_t recv_bytes, void* user)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                               ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


class StencilError(RuntimeError):
    def __init__(self, code: int, where: str, detail: str):
        super().__init__(f"{where}: {STATUS.get(code, code)}: {detail}")
        self.code = code


class stencil_info_t(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("dtype", ctypes.c_int), ("ndims", ctypes.c_int),
                ("variant", ctypes.c_int), ("dims", ctypes.c_int64 * 3),
                ("local_dims", ctypes.c_int64 * 3), ("lo", ctypes.c_int), ("hi", ctypes.c_int),
                ("interior_points", ctypes.c_int64), ("bytes_per_point", ctypes.c_double),
                ("launches_per_step", ctypes.c_int), ("sweeps_per_launch", ctypes.c_int),
                ("rank", ctypes.c_int),
                ("nranks", ctypes.c_int)]


_lib = None


def lib():
    """Load the C-ABI library (raises if it is not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, vpp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)
        i64p, ip = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)
        L.stencil_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, i64p,
                                     ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        L.stencil_set_variant.argtypes = [vp, ctypes.c_int]
        L.stencil_get_variant.argtypes = [vp, ip]
        L.stencil_set_fusion.argtypes = [vp, ctypes.c_int]
        L.stencil_arity.argtypes = [vp, ip, ip, ip]
        L.stencil_info.argtypes = [vp, ctypes.POINTER(stencil_info_t)]
        L.stencil_step.argtypes = [vp, vpp, vpp, vp]
        L.stencil_step_range.argtypes = [vp, vpp, vpp, ctypes.c_int64, ctypes.c_int64, vp]
        L.stencil_run.argtypes = [vp, vpp, ctypes.c_int, vp, ip]
        L.stencil_run_host.argtypes = [vp, vpp, vpp, vpp, ctypes.c_int, vp]
        L.stencil_run_host_async.argtypes = [vp, vpp, vpp, vpp, ctypes.c_int, vp]
        L.stencil_destroy.argtypes = [vp]
        L.stencil_last_error.restype = ctypes.c_char_p
        L.stencil_version.restype = ctypes.c_char_p
        L.stencil_slab_plan.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, i64p]
        L.stencil_dist_get_id.argtypes = [ctypes.c_char_p]
        L.stencil_dist_attach.argtypes = [vp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int]
        L.stencil_dist_attach_host.argtypes = [vp, ctypes.c_int, ctypes.c_int, EXCHANGE_FN, vp]
        L.stencil_dist_attach_p2p.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        L.stencil_p2p_export.argtypes = [vp, vpp, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t,
                                         ctypes.POINTER(ctypes.c_size_t)]
        L.stencil_p2p_import.argtypes = [vp, vpp, ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p]
        _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != 0:
        raise StencilError(rc, where, lib().stencil_last_error().decode())


def _ptrs(ts):
    return (ctypes.c_void_p * len(ts))(*[t if isinstance(t, int) else t.data_ptr() for t in ts])


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def slab_plan(n: int, lo: int, hi: int, rank: int, nranks: int) -> dict:
    """Host-only slab decomposition plan (stencil_slab_plan)."""
    p = (ctypes.c_int64 * 8)()
    _check(lib().stencil_slab_plan(n, lo, hi, rank, nranks, p), "stencil_slab_plan")
    keys = ["own_begin", "own_end", "local_n", "recv_lo_at", "send_lo_from", "recv_hi_at",
            "send_hi_from", "n_planes"]
    d = dict(zip(keys, list(p)))
    d["n_lo"], d["n_hi"] = d["n_planes"] & 0xFFFF, d["n_planes"] >> 16
    return d


def dist_get_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().stencil_dist_get_id(buf), "stencil_dist_get_id")
    return buf.raw


class Stencil:
    """Owner of one stencil_t handle.

    ``dims`` are (nx, ny[, nz]) with x fastest, boundary ring included; a
    torch tensor for it has shape (ny, nx) or (nz, ny, nx).
    """

    def __init__(self, kind: str, dims, dtype: str = "f32", coeffs=None,
                 variant: str = "shuffle"):
        self.kind, self.dtype, self.dims = kind, dtype, tuple(int(d) for d in dims)
        h = ctypes.c_void_p()
        d = (ctypes.c_int64 * len(self.dims))(*self.dims)
        if coeffs is None:
            cp, nc = None, 0
        else:
            cs = [float(c) for c in coeffs]
            cp, nc = (ctypes.c_double * len(cs))(*cs), len(cs)
        _check(lib().stencil_create(ctypes.byref(h), KINDS[kind], len(self.dims), d,
                                    DTYPES[dtype], cp, nc), "stencil_create")
        self._h = h
        self.set_variant(variant)

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().stencil_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- queries
    def set_variant(self, variant: str):
        """A variant name; "auto" resolves (in the library) to the kind's
        measured-faster register-cache variant, reported in self.variant."""
        _check(lib().stencil_set_variant(self._h, VARIANTS[variant]), "stencil_set_variant")
        v = ctypes.c_int()
        _check(lib().stencil_get_variant(self._h, ctypes.byref(v)), "stencil_get_variant")
        self.variant = next(n for n, i in VARIANTS.items() if i == v.value)

    def set_fusion(self, sweeps_per_launch: int):
        """0 auto (fuse L2-resident 2-D runs), 1 off, S >= 2 sweeps per launch."""
        _check(lib().stencil_set_fusion(self._h, int(sweeps_per_launch)), "stencil_set_fusion")

    def arity(self):
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().stencil_arity(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
               "stencil_arity")
        return a.value, b.value, c.value

    def info(self) -> dict:
        s = stencil_info_t()
        _check(lib().stencil_info(self._h, ctypes.byref(s)), "stencil_info")
        d = {f: getattr(s, f) for f, _ in s._fields_}
        d["dims"], d["local_dims"] = tuple(s.dims), tuple(s.local_dims)
        return d

    # -- compute
    def step(self, ins, outs, stream=None):
        _check(lib().stencil_step(self._h, _ptrs(ins), _ptrs(outs), _stream(stream)),
               "stencil_step")

    def step_range(self, ins, outs, s_begin: int, s_end: int, stream=None):
        _check(lib().stencil_step_range(self._h, _ptrs(ins), _ptrs(outs), int(s_begin),
                                        int(s_end), _stream(stream)), "stencil_step_range")

    def run(self, bufs, n_iters: int, stream=None) -> int:
        r = ctypes.c_int(-1)
        _check(lib().stencil_run(self._h, _ptrs(bufs), int(n_iters), _stream(stream),
                                 ctypes.byref(r)), "stencil_run")
        return r.value

    def run_host(self, host_ins, host_outs, dev_bufs, n_iters: int, stream=None):
        """End-to-end: host arrays (numpy or pinned torch CPU tensors) in and out."""
        def hp(a):
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        hin = (ctypes.c_void_p * len(host_ins))(*[hp(a) for a in host_ins])
        hout = (ctypes.c_void_p * len(host_outs))(*[hp(a) for a in host_outs])
        _check(lib().stencil_run_host(self._h, hin, hout, _ptrs(dev_bufs), int(n_iters),
                                      _stream(stream)), "stencil_run_host")

    def run_host_async(self, host_ins, host_outs, dev_bufs, n_iters: int, stream=None):
        """run_host without the final synchronisation (pinned host buffers)."""
        hin = (ctypes.c_void_p * len(host_ins))(*[a.data_ptr() for a in host_ins])
        hout = (ctypes.c_void_p * len(host_outs))(*[a.data_ptr() for a in host_outs])
        _check(lib().stencil_run_host_async(self._h, hin, hout, _ptrs(dev_bufs), int(n_iters),
                                            _stream(stream)), "stencil_run_host_async")

    def attach(self, uid: bytes, rank: int, nranks: int):
        _check(lib().stencil_dist_attach(self._h, uid, rank, nranks), "stencil_dist_attach")

    def attach_p2p(self, rank: int, nranks: int):
        """Fused peer-store halo transport (see stencil.h)."""
        _check(lib().stencil_dist_attach_p2p(self._h, rank, nranks), "stencil_dist_attach_p2p")
        self._rank, self._nranks = rank, nranks

    def p2p_register(self, bufs, allgather):
        """Export this rank's buffers, all-gather the blobs with
        allgather(bytes) -> list of bytes (one per rank), import the
        neighbours'.  Call on every rank with the run's buffers."""
        cap = 8 + 72 * (len(bufs) + 1)
        blob = ctypes.create_string_buffer(cap)
        n = ctypes.c_size_t()
        _check(lib().stencil_p2p_export(self._h, _ptrs(bufs), len(bufs), blob, cap, ctypes.byref(n)),
               "stencil_p2p_export")
        blobs = allgather(blob.raw[: n.value])
        r, w = self._rank, self._nranks
        lo = blobs[r - 1] if r > 0 else None
        hi = blobs[r + 1] if r < w - 1 else None
        _check(lib().stencil_p2p_import(self._h, _ptrs(bufs), len(bufs), lo, hi), "stencil_p2p_import")

    def attach_host(self, rank: int, nranks: int, exchange):
        """Host-transport slab decomposition; exchange(peer, send, recv) gets
        two uint8 numpy arrays (recv to be filled) and moves the planes, e.g.
        with torch.distributed over gloo."""
        import numpy as np

        def _fn(peer, send, send_bytes, recv, recv_bytes, user):
            try:
                s_arr = np.empty(send_bytes, np.uint8)
                ctypes.memmove(s_arr.ctypes.data, send, send_bytes)
                r_arr = np.empty(recv_bytes, np.uint8)
                exchange(peer, s_arr, r_arr)
                ctypes.memmove(recv, r_arr.ctypes.data, recv_bytes)
                return 0
            except Exception:
                import traceback
                traceback.print_exc()
                return 1
        self._exchange_cb = EXCHANGE_FN(_fn)     # keep alive as long as the handle
        _check(lib().stencil_dist_attach_host(self._h, rank, nranks, self._exchange_cb, None),
               "stencil_dist_attach_host")
