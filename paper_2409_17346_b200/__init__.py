"""B200-native DMTz hot path: thin Python binding over libdmtz.so (include/dmtz.h).

Argument marshalling only: every step of the C-loop and the traces runs in the
CUDA kernels of ``csrc/``.  PyTorch provides device memory and streams.  There is
no CPU fallback: importing this package on a machine without the built library
raises, and every call needs CUDA tensors.

Fields are torch float32 tensors shaped (nz, ny, nx) (3D) or (ny, nx) (2D), x
contiguous.  P:<n> cites line n of the paper text (see include/dmtz.h).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DMTZ_LIB") or os.path.join(_HERE, "libdmtz.so")   # DMTZ_LIB: experiment builds


OK, E_ARG, E_DIMS, E_NONFINITE, E_BOUND, E_CAPACITY, E_ITER_CAP, E_STUCK, E_CUDA, E_NCCL, E_OOM, \
    E_INTERNAL = range(12)
KIND_DESC, KIND_ASC, KIND_CONN = 1, 2, 4
BOUNDARY = 0xFFFFFFFFFFFFFFFF
EDIT_DTYPE = np.dtype([("v", "<u8"), ("q", "<u2"), ("lossless", "u1"), ("pad", "u1"), ("value", "<f4")])


class DmtzError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"dmtz status {status}: {msg}")
        self.status = status


class _Dims(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64)]


class _Opts(ctypes.Structure):
    _fields_ = [("xi", ctypes.c_float), ("q_max", ctypes.c_int32), ("q_cap", ctypes.c_int32),
                ("tier", ctypes.c_int32), ("max_rounds", ctypes.c_int64), ("full_sweeps", ctypes.c_int32),
                ("profile", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("n_edited", ctypes.c_int64), ("n_quantized", ctypes.c_int64),
                ("n_lossless", ctypes.c_int64), ("n_false_round0", ctypes.c_int64),
                ("false_by_kind_round0", ctypes.c_int64 * 8), ("status", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("sweeps", ctypes.c_int64), ("anchors_swept", ctypes.c_int64),
                ("launches", ctypes.c_int64), ("sweep_ms", ctypes.c_double), ("screen_ms", ctypes.c_double),
                ("decode_ms", ctypes.c_double), ("screen_ms_full", ctypes.c_double), ("n_screen_full", ctypes.c_int64),
                ("anchors_recomputed", ctypes.c_int64), ("anchors_decoded", ctypes.c_int64),
                ("cells_evaluated", ctypes.c_int64), ("anchors_replayed", ctypes.c_int64),
                ("halo_faces_sent", ctypes.c_int64), ("halo_faces_skipped", ctypes.c_int64),
                ("edit_ms", ctypes.c_double)]


class _SStats(ctypes.Structure):
    _fields_ = [("c_rounds", ctypes.c_int64), ("s_rounds", ctypes.c_int64), ("troublemakers", ctypes.c_int64),
                ("tm_by_kind", ctypes.c_int64 * 3), ("sep_branches", ctypes.c_int64), ("sep_cells", ctypes.c_int64),
                ("tm_round1", ctypes.c_int64), ("trace_ms", ctypes.c_double), ("s_ms", ctypes.c_double),
                ("cells_checked", ctypes.c_int64), ("pad", ctypes.c_int64 * 4)]


class _Prf(ctypes.Structure):
    _fields_ = [("n_orig", ctypes.c_int64), ("n_rec", ctypes.c_int64), ("n_match", ctypes.c_int64)]


def _prf(p):
    return dict(n_orig=p.n_orig, n_rec=p.n_rec, n_match=p.n_match,
                recall=p.n_match / p.n_orig if p.n_orig else 1.0,
                precision=p.n_match / p.n_rec if p.n_rec else 1.0)


class _Seps(ctypes.Structure):
    _fields_ = [("branch_offsets", ctypes.c_void_p), ("cells", ctypes.c_void_p), ("origin", ctypes.c_void_p),
                ("terminal", ctypes.c_void_p), ("kind", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python paper_2409_17346_b200/build.py` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.dmtz_ctx_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(_Dims), i32, i32, P, i32]
    L.dmtz_ctx_destroy.argtypes = [P]
    L.dmtz_ctx_destroy.restype = None
    L.dmtz_workspace_bytes.argtypes = [P, ctypes.POINTER(_Opts)]
    L.dmtz_workspace_bytes.restype = ctypes.c_size_t
    L.dmtz_compute_gradient.argtypes = [P, P, P, P, P]
    L.dmtz_critical_mask.argtypes = [P, P, P, P]
    L.dmtz_correct.argtypes = [P, P, P, ctypes.POINTER(_Opts), P, ctypes.c_size_t, P, P, i64,
                               ctypes.POINTER(i64), ctypes.POINTER(_Stats), P]
    L.dmtz_correct_host.argtypes = [P, P, P, ctypes.POINTER(_Opts), P, ctypes.c_size_t, P, P, P, P, i64, P, P,
                                    ctypes.POINTER(i64), ctypes.POINTER(_Stats), P]
    L.dmtz_correct_host_stream.argtypes = [P, P, P, ctypes.POINTER(_Opts), P, ctypes.c_size_t, P, P, P, P, i64, P,
                                           ctypes.c_size_t, P, P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
                                           ctypes.POINTER(i64), ctypes.POINTER(_Stats), P]
    L.dmtz_correct_host_stream.restype = ctypes.c_int
    L.dmtz_trace_separatrices.argtypes = [P, P, ctypes.c_uint32, P, ctypes.c_size_t, ctypes.POINTER(_Seps),
                                          i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64), P]
    SZ = ctypes.c_size_t
    L.dmtz_slab_begin.argtypes = [P, P, P, ctypes.POINTER(_Opts), P, P, SZ, P, P]
    L.dmtz_slab_round.argtypes = [P, P, P, ctypes.POINTER(_Opts), P, P, SZ, P, i64, P, P, P]
    L.dmtz_slab_round_async.argtypes = [P, P, P, ctypes.POINTER(_Opts), P, P, SZ, P, i64, P, P]
    L.dmtz_slab_end.argtypes = [P, P, P, SZ, P, P, i64, ctypes.POINTER(i64), ctypes.POINTER(i64), P]
    L.dmtz_slab_halo.argtypes = [P, P, P, SZ, P, P, i64, i64, i64, P]
    L.dmtz_trace_separatrices_range.argtypes = [P, P, ctypes.c_uint32, i64, i64, P, ctypes.c_size_t,
                                                ctypes.POINTER(_Seps), i64, i64, ctypes.POINTER(i64),
                                                ctypes.POINTER(i64), P]
    L.dmtz_preserve_sep_bytes.argtypes = [P, ctypes.POINTER(_Opts), i64, i64]
    L.dmtz_preserve_sep_bytes.restype = ctypes.c_size_t
    L.dmtz_preserve.argtypes = [P, P, P, ctypes.POINTER(_Opts), P, SZ, P, SZ, i64, i64, P, P, i64,
                                ctypes.POINTER(i64), ctypes.POINTER(_Stats), ctypes.POINTER(_SStats), P]
    L.dmtz_edit_stream_bound.argtypes = [i64]
    L.dmtz_edit_stream_bound.restype = SZ
    L.dmtz_encode_edits.argtypes = [P, P, i64, ctypes.c_float, i32, P, P, SZ, P, SZ, ctypes.POINTER(SZ), P]
    L.dmtz_decode_edits.argtypes = [P, P, SZ, P, P, i64, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_float),
                                    ctypes.POINTER(i32), P, SZ, P]
    L.dmtz_apply_edits.argtypes = [P, P, ctypes.c_float, i32, P, i64, P, P, SZ, P]
    L.dmtz_critical_prf.argtypes = [P, P, P, ctypes.POINTER(_Prf), P, SZ, P]
    L.dmtz_separatrix_prf.argtypes = [P, ctypes.POINTER(_Seps), i64, ctypes.POINTER(_Seps), i64,
                                      ctypes.POINTER(_Prf), P, SZ, P]
    L.dmtz_status_string.argtypes = [i32]
    L.dmtz_status_string.restype = ctypes.c_char_p
    L.dmtz_last_error.restype = ctypes.c_char_p
    L.dmtz_last_trace_levels.argtypes = [P, i32]
    L.dmtz_last_trace_levels.restype = ctypes.c_int
    L.dmtz_local_slab.argtypes = [i64, i32, i32, P, P, P, P]
    L.dmtz_local_slab.restype = ctypes.c_int
    L.dmtz_ctx_set_transport.argtypes = [P, P]
    L.dmtz_ctx_set_transport.restype = ctypes.c_int
    L.dmtz_ctx_set_dist_sync.argtypes = [P, ctypes.c_int]
    L.dmtz_ctx_set_dist_sync.restype = ctypes.c_int
    L.dmtz_ctx_set_dist_graph.argtypes = [P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    L.dmtz_ctx_set_dist_graph.restype = ctypes.c_int
    L.dmtz_nccl_unique_id.argtypes = [P]
    L.dmtz_nccl_unique_id.restype = ctypes.c_int
    for fn in ("dmtz_ctx_create", "dmtz_compute_gradient", "dmtz_critical_mask", "dmtz_correct", "dmtz_correct_host",
               "dmtz_trace_separatrices", "dmtz_version", "dmtz_slab_begin", "dmtz_slab_round", "dmtz_slab_end",
               "dmtz_slab_halo", "dmtz_trace_separatrices_range", "dmtz_preserve", "dmtz_slab_round_async",
               "dmtz_encode_edits", "dmtz_decode_edits", "dmtz_apply_edits",
               "dmtz_critical_prf", "dmtz_separatrix_prf"):
        getattr(L, fn).restype = ctypes.c_int
    return L


class _LazyLib:
    """libdmtz.so, loaded on first use (so that the package can be imported to build it);
    every call raises if the library is missing -- there is no CPU fallback."""

    _L = None

    def __getattr__(self, name):
        if _LazyLib._L is None:
            _LazyLib._L = _load()
        return getattr(_LazyLib._L, name)


_lib = _LazyLib()
EXPORTED = ("dmtz_ctx_create", "dmtz_ctx_destroy", "dmtz_workspace_bytes", "dmtz_compute_gradient",
            "dmtz_critical_mask", "dmtz_correct", "dmtz_correct_host", "dmtz_trace_separatrices", "dmtz_status_string",
            "dmtz_last_error", "dmtz_version", "dmtz_slab_begin", "dmtz_slab_round", "dmtz_slab_end",
            "dmtz_slab_halo", "dmtz_trace_separatrices_range", "dmtz_slab_round_async", "dmtz_preserve_sep_bytes",
            "dmtz_preserve",
            "dmtz_edit_stream_bound", "dmtz_encode_edits", "dmtz_decode_edits", "dmtz_apply_edits",
            "dmtz_critical_prf", "dmtz_separatrix_prf", "dmtz_last_trace_levels", "dmtz_local_slab",
            "dmtz_ctx_set_transport", "dmtz_ctx_set_dist_sync", "dmtz_nccl_unique_id", "dmtz_correct_host_stream",
            "dmtz_ctx_set_dist_graph")


def pack_edit_stream(stream: torch.Tensor, level: int = 1) -> bytes:
    """The stored artifact of the edits ("the quantized edits are losslessly
    compressed"): the device edit stream (dmtz_encode_edits) copied to the host and put
    through a general-purpose lossless coder (zlib).  Not on the hot path."""
    import zlib
    return zlib.compress(stream.cpu().numpy().tobytes(), level)


def unpack_edit_stream(blob: bytes, device=None) -> torch.Tensor:
    """Inverse of pack_edit_stream: the edit stream as a uint8 tensor (for dmtz_decode_edits)."""
    import zlib
    a = np.frombuffer(zlib.decompress(blob), dtype=np.uint8).copy()
    t = torch.from_numpy(a)
    return t.to(device) if device is not None else t


def last_trace_levels() -> list:
    """Connectors per escalation level of this thread's last trace (dmtz_last_trace_levels)."""
    out = (ctypes.c_int64 * 10)()
    _check(_lib.dmtz_last_trace_levels(out, 10))
    return list(out)


def lib():
    if _LazyLib._L is None:
        _LazyLib._L = _load()
    return _LazyLib._L


def _check(st):
    if st != OK:
        raise DmtzError(st, _lib.dmtz_last_error().decode())


def _dims_of(shape):
    if len(shape) == 2:
        return int(shape[1]), int(shape[0]), 1
    if len(shape) == 3:
        return int(shape[2]), int(shape[1]), int(shape[0])
    raise ValueError(f"field must be 2D or 3D, got shape {tuple(shape)}")


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if not (isinstance(t, torch.Tensor) and t.is_cuda):
            raise TypeError("dmtz needs CUDA tensors (no CPU fallback)")


def _stats_dict(st, status):
    return dict(rounds=st.rounds, n_edited=st.n_edited, n_quantized=st.n_quantized, n_lossless=st.n_lossless,
                n_false_round0=st.n_false_round0, false_by_kind_round0=list(st.false_by_kind_round0),
                status=status, sweeps=st.sweeps, anchors_swept=st.anchors_swept, launches=st.launches,
                sweep_ms=st.sweep_ms, screen_ms=st.screen_ms, decode_ms=st.decode_ms,
                screen_ms_full=st.screen_ms_full, n_screen_full=st.n_screen_full,
                anchors_recomputed=st.anchors_recomputed, anchors_decoded=st.anchors_decoded,
                cells_evaluated=st.cells_evaluated, anchors_replayed=st.anchors_replayed,
                halo_faces_sent=st.halo_faces_sent, halo_faces_skipped=st.halo_faces_skipped, edit_ms=st.edit_ms)


class Context:
    """A dmtz_ctx for one grid plus its device workspace (a torch uint8 tensor)."""

    def __init__(self, shape, device=None):
        self.shape = tuple(int(s) for s in shape)
        self.nx, self.ny, self.nz = _dims_of(self.shape)
        self.D = 2 if self.nz == 1 else 3
        self.N = self.nx * self.ny * self.nz
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        h = ctypes.c_void_p()
        d = _Dims(self.nx, self.ny, self.nz)
        _check(_lib.dmtz_ctx_create(ctypes.byref(h), ctypes.byref(d), 0, 1, None, self.device.index or 0))
        self._h = h
        self.ws_bytes = int(_lib.dmtz_workspace_bytes(h, None))
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)

    def close(self):
        if getattr(self, "_h", None):
            _lib.dmtz_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def code_dtype(self):
        return torch.int64 if self.D == 3 else torch.int16

    # ---------------------------------------------------------------- gradient
    def compute_gradient(self, field: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        """Discrete gradient codes, layout of include/dmtz.h."""
        _need_cuda(field)
        assert field.dtype == torch.float32 and tuple(field.shape) == self.shape and field.is_contiguous()
        if out is None:
            out = torch.empty(self.shape, dtype=self.code_dtype, device=field.device)
        _check(_lib.dmtz_compute_gradient(self._h, ctypes.c_void_p(field.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr()), None, _stream_ptr(stream)))
        return out

    def critical_mask(self, codes: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        _need_cuda(codes)
        if out is None:
            out = torch.empty(self.shape, dtype=torch.int32, device=codes.device)
        _check(_lib.dmtz_critical_mask(self._h, ctypes.c_void_p(codes.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                       _stream_ptr(stream)))
        return out

    # ---------------------------------------------------------------- C-loop
    def correct(self, f: torch.Tensor, fhat: torch.Tensor, xi: float, q_max: int = 6, q_cap: int | None = None,
                tier: int = 2, max_rounds: int = 0, full_sweeps: bool = False, g_out: torch.Tensor | None = None,
                edits: torch.Tensor | None = None, edits_capacity: int | None = None, stream=None,
                raise_on_error: bool = True, profile: bool = False):
        """The C-loop with Eq. 2 edits.  Returns a Result."""
        _need_cuda(f, fhat)
        for t in (f, fhat):
            assert t.dtype == torch.float32 and tuple(t.shape) == self.shape and t.is_contiguous()
        if g_out is None:
            g_out = torch.empty_like(f)
        if edits is None:
            cap = self.N if edits_capacity is None else int(edits_capacity)
            edits = torch.empty((max(cap, 1), 16), dtype=torch.uint8, device=f.device)
        else:
            if (edits.dtype != torch.uint8 or edits.dim() != 2 or edits.shape[1] != 16 or not edits.is_contiguous()
                    or edits.device != f.device):
                raise ValueError("edits must be a contiguous (n, 16) uint8 tensor on f's device")
            cap = edits.shape[0] if edits_capacity is None else min(int(edits_capacity), edits.shape[0])
        if g_out.dtype != torch.float32 or tuple(g_out.shape) != self.shape or g_out.device != f.device \
                or not g_out.is_contiguous():
            raise ValueError("g_out must be a contiguous float32 tensor of the field's shape on f's device")
        opts = _Opts(float(xi), int(q_max), int(q_max if q_cap is None else q_cap), int(tier), int(max_rounds),
                     1 if full_sweeps else 0, 1 if profile else 0)
        ne = ctypes.c_int64()
        st = _Stats()
        status = _lib.dmtz_correct(self._h, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(fhat.data_ptr()),
                                   ctypes.byref(opts), ctypes.c_void_p(self.workspace.data_ptr()),
                                   self.ws_bytes, ctypes.c_void_p(g_out.data_ptr()),
                                   ctypes.c_void_p(edits.data_ptr()), cap, ctypes.byref(ne), ctypes.byref(st),
                                   _stream_ptr(stream))
        stats = _stats_dict(st, status)
        msg = _lib.dmtz_last_error().decode() if status != OK else ""
        if raise_on_error and status not in (OK, E_STUCK, E_ITER_CAP, E_CAPACITY):
            raise DmtzError(status, msg)
        return Result(status=status, g=g_out, edits=edits[:min(ne.value, cap)], n_edits=ne.value, stats=stats,
                      message=msg)

    def correct_host(self, f_host: torch.Tensor, fhat_host: torch.Tensor, xi: float, q_max: int = 6,
                     q_cap: int | None = None, tier: int = 2, max_rounds: int = 0, full_sweeps: bool = False,
                     bufs: dict | None = None, g_host: torch.Tensor | None = None,
                     edits_host: torch.Tensor | None = None, stream=None, raise_on_error: bool = True):
        """The end-to-end call (dmtz_correct_host): f and fhat from HOST tensors (pinned
        for full bandwidth), g and the edit list back into host tensors, every copy
        inside the library call.  ``bufs`` (from host_buffers) holds the device
        buffers; g_host / edits_host default to new pinned tensors.  Returns a Result
        whose g / edits are the HOST tensors."""
        for t in (f_host, fhat_host):
            assert t.device.type == "cpu" and t.dtype == torch.float32 and tuple(t.shape) == self.shape
            assert t.is_contiguous()
        dev = self.workspace.device
        if bufs is None:
            bufs = self.host_buffers(dev)
        if g_host is None:
            g_host = torch.empty(self.shape, dtype=torch.float32).pin_memory()
        if edits_host is None:
            edits_host = torch.empty((max(self.N, 1), 16), dtype=torch.uint8).pin_memory()
        cap = min(bufs["edits"].shape[0], edits_host.shape[0])
        opts = _Opts(float(xi), int(q_max), int(q_max if q_cap is None else q_cap), int(tier), int(max_rounds),
                     1 if full_sweeps else 0, 0)
        ne = ctypes.c_int64()
        st = _Stats()
        status = _lib.dmtz_correct_host(
            self._h, ctypes.c_void_p(f_host.data_ptr()), ctypes.c_void_p(fhat_host.data_ptr()), ctypes.byref(opts),
            ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes, ctypes.c_void_p(bufs["f"].data_ptr()),
            ctypes.c_void_p(bufs["fhat"].data_ptr()), ctypes.c_void_p(bufs["g"].data_ptr()),
            ctypes.c_void_p(bufs["edits"].data_ptr()), cap, ctypes.c_void_p(g_host.data_ptr()),
            ctypes.c_void_p(edits_host.data_ptr()), ctypes.byref(ne), ctypes.byref(st), _stream_ptr(stream))
        stats = _stats_dict(st, status)
        msg = _lib.dmtz_last_error().decode() if status != OK else ""
        if raise_on_error and status not in (OK, E_STUCK, E_ITER_CAP, E_CAPACITY):
            raise DmtzError(status, msg)
        return Result(status=status, g=g_host, edits=edits_host[:min(ne.value, cap)], n_edits=ne.value,
                      stats=stats, message=msg)

    def correct_host_stream(self, f_host: torch.Tensor, fhat_host: torch.Tensor, xi: float, q_max: int = 6,
                            q_cap: int | None = None, tier: int = 2, max_rounds: int = 0, full_sweeps: bool = False,
                            bufs: dict | None = None, stream_host: torch.Tensor | None = None,
                            g_host: torch.Tensor | None = None, stream=None, raise_on_error: bool = True):
        """The end-to-end call that returns the storable artifact
        (dmtz_correct_host_stream): f and fhat from HOST tensors, the C-loop, the edit
        list encoded on the device (version 2), and only the stream's bytes back to the
        host (plus g into g_host when given).  ``bufs`` from host_buffers(device,
        stream=True).  Returns (Result with g = g_host or None and edits = the device
        edit list, the host stream bytes as a uint8 tensor view)."""
        for t in (f_host, fhat_host):
            assert t.device.type == "cpu" and t.dtype == torch.float32 and tuple(t.shape) == self.shape
            assert t.is_contiguous()
        dev = self.workspace.device
        if bufs is None or "stream" not in bufs:
            bufs = self.host_buffers(dev, stream=True)
        if stream_host is None:
            stream_host = torch.empty(bufs["stream"].numel(), dtype=torch.uint8).pin_memory()
        cap = bufs["edits"].shape[0]
        opts = _Opts(float(xi), int(q_max), int(q_max if q_cap is None else q_cap), int(tier), int(max_rounds),
                     1 if full_sweeps else 0, 0)
        ne, nbytes, st = ctypes.c_int64(), ctypes.c_size_t(), _Stats()
        status = _lib.dmtz_correct_host_stream(
            self._h, ctypes.c_void_p(f_host.data_ptr()), ctypes.c_void_p(fhat_host.data_ptr()), ctypes.byref(opts),
            ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes, ctypes.c_void_p(bufs["f"].data_ptr()),
            ctypes.c_void_p(bufs["fhat"].data_ptr()), ctypes.c_void_p(bufs["g"].data_ptr()),
            ctypes.c_void_p(bufs["edits"].data_ptr()), cap, ctypes.c_void_p(bufs["stream"].data_ptr()),
            bufs["stream"].numel(), ctypes.c_void_p(g_host.data_ptr()) if g_host is not None else None,
            ctypes.c_void_p(stream_host.data_ptr()), stream_host.numel(), ctypes.byref(nbytes), ctypes.byref(ne),
            ctypes.byref(st), _stream_ptr(stream))
        stats = _stats_dict(st, status)
        msg = _lib.dmtz_last_error().decode() if status != OK else ""
        if raise_on_error and status not in (OK, E_STUCK, E_ITER_CAP):
            raise DmtzError(status, msg)
        return (Result(status=status, g=g_host, edits=bufs["edits"][:min(ne.value, cap)], n_edits=ne.value,
                       stats=stats, message=msg), stream_host[:nbytes.value])

    def host_buffers(self, device, stream: bool = False) -> dict:
        """Device buffers of correct_host: f, fhat, g (float[N]) and the edit list (and,
        with stream=True, the edit-stream buffer of correct_host_stream)."""
        if stream:
            d = self.host_buffers(device)
            d["stream"] = torch.empty(max(int(_lib.dmtz_edit_stream_bound(self.N)), 1), dtype=torch.uint8,
                                      device=device)
            return d
        return dict(f=torch.empty(self.shape, dtype=torch.float32, device=device),
                    fhat=torch.empty(self.shape, dtype=torch.float32, device=device),
                    g=torch.empty(self.shape, dtype=torch.float32, device=device),
                    edits=torch.empty((max(self.N, 1), 16), dtype=torch.uint8, device=device))

    # ---------------------------------------------------------------- tiers 3-4
    def preserve(self, f: torch.Tensor, fhat: torch.Tensor, xi: float, tier: int = 4, q_max: int = 6,
                 q_cap: int | None = None, max_rounds: int = 0, full_sweeps: bool = False,
                 g_out: torch.Tensor | None = None, edits_capacity: int | None = None, sep_caps=None, stream=None,
                 raise_on_error: bool = True):
        """The alternating C-/S-loop workflow for tiers 1-4.  The
        separatrix CSR of f is sized with a trace of f's gradient (sep_caps = (branches,
        cells) overrides; tier 3 also traces its candidate branches in g and gets 12.5 % headroom on the cells)."""
        _need_cuda(f, fhat)
        for t in (f, fhat):
            assert t.dtype == torch.float32 and tuple(t.shape) == self.shape and t.is_contiguous()
        if g_out is None:
            g_out = torch.empty_like(f)
        cap = self.N if edits_capacity is None else int(edits_capacity)
        edits = torch.empty((max(cap, 1), 16), dtype=torch.uint8, device=f.device)
        opts = _Opts(float(xi), int(q_max), int(q_max if q_cap is None else q_cap), int(tier), int(max_rounds),
                     1 if full_sweeps else 0, 0)
        cb = cc = 0
        sep = None
        if tier >= 3:
            if sep_caps is None:
                sz = self.trace_sizes(self.compute_gradient(f), stream=stream)
                cb, cc = sz["n_branches"], sz["n_cells"]
                if tier == 3:
                    cc = cc + cc // 8 + 1024
            else:
                cb, cc = (int(x) for x in sep_caps)
            nbytes = int(_lib.dmtz_preserve_sep_bytes(self._h, ctypes.byref(opts), cb, cc))
            sep = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=f.device)
        else:
            nbytes = 0
        ne = ctypes.c_int64()
        st, ss = _Stats(), _SStats()
        status = _lib.dmtz_preserve(self._h, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(fhat.data_ptr()),
                                    ctypes.byref(opts), ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                                    ctypes.c_void_p(sep.data_ptr()) if sep is not None else None, nbytes, cb, cc,
                                    ctypes.c_void_p(g_out.data_ptr()), ctypes.c_void_p(edits.data_ptr()), cap,
                                    ctypes.byref(ne), ctypes.byref(st), ctypes.byref(ss), _stream_ptr(stream))
        stats = _stats_dict(st, status)
        stats.update(c_rounds=ss.c_rounds, s_rounds=ss.s_rounds, troublemakers=ss.troublemakers,
                     tm_by_kind=list(ss.tm_by_kind), sep_branches=ss.sep_branches, sep_cells=ss.sep_cells,
                     tm_round1=ss.tm_round1, trace_ms=ss.trace_ms, s_ms=ss.s_ms,
                     cells_checked=ss.cells_checked)
        msg = _lib.dmtz_last_error().decode() if status != OK else ""
        if raise_on_error and status not in (OK, E_STUCK, E_ITER_CAP, E_CAPACITY):
            raise DmtzError(status, msg)
        return Result(status=status, g=g_out, edits=edits[:min(ne.value, cap)], n_edits=ne.value, stats=stats,
                      message=msg)

    # ---------------------------------------------------------------- edits as an artifact
    def encode_edits(self, edits: torch.Tensor, xi: float, q_max: int = 6, fhat: torch.Tensor | None = None,
                     stream=None) -> torch.Tensor:
        """Edit list (n, 16) uint8 rows -> the edit stream (uint8 CUDA tensor); with fhat,
        version 2 (lossless values relative to fhat), else version 1."""
        _need_cuda(edits)
        n = int(edits.shape[0])
        cap = int(_lib.dmtz_edit_stream_bound(n))
        out = torch.empty(max(cap, 1), dtype=torch.uint8, device=edits.device)
        nb = ctypes.c_size_t()
        _check(_lib.dmtz_encode_edits(self._h, ctypes.c_void_p(edits.data_ptr()) if n else None, n, float(xi),
                                      int(q_max), ctypes.c_void_p(fhat.data_ptr()) if fhat is not None else None,
                                      ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                                      ctypes.c_void_p(out.data_ptr()), cap, ctypes.byref(nb), _stream_ptr(stream)))
        return out[:nb.value]

    def decode_edits(self, stream_bytes: torch.Tensor, fhat: torch.Tensor | None = None, stream=None):
        """Edit stream (uint8 CUDA tensor) -> (edits (n, 16) uint8, xi, q_max); version 2
        needs fhat."""
        _need_cuda(stream_bytes)
        cap = self.N
        edits = torch.empty((max(cap, 1), 16), dtype=torch.uint8, device=stream_bytes.device)
        n, xi, qm = ctypes.c_int64(), ctypes.c_float(), ctypes.c_int32()
        _check(_lib.dmtz_decode_edits(self._h, ctypes.c_void_p(stream_bytes.data_ptr()), int(stream_bytes.numel()),
                                      ctypes.c_void_p(fhat.data_ptr()) if fhat is not None else None,
                                      ctypes.c_void_p(edits.data_ptr()), cap, ctypes.byref(n), ctypes.byref(xi),
                                      ctypes.byref(qm), ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                                      _stream_ptr(stream)))
        return edits[:n.value], xi.value, qm.value

    def apply_edits(self, fhat: torch.Tensor, xi: float, edits: torch.Tensor, q_max: int = 6,
                    g_out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Decompression side: fhat with the edits applied (bit-exact with correct()'s g)."""
        _need_cuda(fhat, edits)
        assert fhat.dtype == torch.float32 and tuple(fhat.shape) == self.shape and fhat.is_contiguous()
        if g_out is None:
            g_out = torch.empty_like(fhat)
        n = int(edits.shape[0])
        _check(_lib.dmtz_apply_edits(self._h, ctypes.c_void_p(fhat.data_ptr()), float(xi), int(q_max),
                                     ctypes.c_void_p(edits.data_ptr()) if n else None, n,
                                     ctypes.c_void_p(g_out.data_ptr()), ctypes.c_void_p(self.workspace.data_ptr()),
                                     self.ws_bytes, _stream_ptr(stream)))
        return g_out

    # ---------------------------------------------------------------- metrics (§5.1)
    def critical_prf(self, crit_orig: torch.Tensor, crit_rec: torch.Tensor, stream=None) -> dict:
        """Critical-cell recall / precision from two critical masks."""
        _need_cuda(crit_orig, crit_rec)
        p = _Prf()
        _check(_lib.dmtz_critical_prf(self._h, ctypes.c_void_p(crit_orig.data_ptr()),
                                      ctypes.c_void_p(crit_rec.data_ptr()), ctypes.byref(p),
                                      ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes, _stream_ptr(stream)))
        return _prf(p)

    def separatrix_prf(self, tr_orig: dict, tr_rec: dict, stream=None) -> dict:
        """Separatrix recall / precision from two trace_separatrices() results."""
        def seps(t):
            return _Seps(*(ctypes.c_void_p(t[k].data_ptr()) for k in ("offsets", "cells", "origin", "terminal", "kind")))
        a, b = seps(tr_orig), seps(tr_rec)
        p = _Prf()
        _check(_lib.dmtz_separatrix_prf(self._h, ctypes.byref(a), int(tr_orig["origin"].shape[0]), ctypes.byref(b),
                                        int(tr_rec["origin"].shape[0]), ctypes.byref(p),
                                        ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                                        _stream_ptr(stream)))
        return _prf(p)

    # ---------------------------------------------------------------- traces
    def _trace(self, codes, kinds, seps, cb, cc, nb, nc, stream, z_range):
        if z_range is None:
            return _lib.dmtz_trace_separatrices(self._h, ctypes.c_void_p(codes.data_ptr()), kinds,
                                                ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                                                ctypes.byref(seps), cb, cc, ctypes.byref(nb), ctypes.byref(nc),
                                                _stream_ptr(stream))
        return _lib.dmtz_trace_separatrices_range(self._h, ctypes.c_void_p(codes.data_ptr()), kinds,
                                                  int(z_range[0]), int(z_range[1]),
                                                  ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                                                  ctypes.byref(seps), cb, cc, ctypes.byref(nb), ctypes.byref(nc),
                                                  _stream_ptr(stream))

    def trace_sizes(self, codes: torch.Tensor, kinds: int = KIND_DESC | KIND_ASC | KIND_CONN, stream=None,
                    z_range=None):
        """Branch and cell counts of the traces (two sizing calls: branches, then cells);
        z_range = (z0, z1): only branches whose origin is anchored in those planes."""
        _need_cuda(codes)
        nb, nc = ctypes.c_int64(), ctypes.c_int64()
        seps = _Seps(None, None, None, None, None)
        one = torch.empty(8, dtype=torch.int64, device=codes.device)
        seps.branch_offsets = ctypes.c_void_p(one.data_ptr())
        st = self._trace(codes, kinds, seps, 0, 0, nb, nc, stream, z_range)
        if st not in (OK, E_CAPACITY):
            _check(st)
        n_b = nb.value
        bufs = [torch.empty(max(n_b, 1) + 1, dtype=torch.int64, device=codes.device) for _ in range(3)]
        kb = torch.empty(max(n_b, 1), dtype=torch.uint8, device=codes.device)
        seps = _Seps(ctypes.c_void_p(bufs[0].data_ptr()), None, ctypes.c_void_p(bufs[1].data_ptr()),
                     ctypes.c_void_p(bufs[2].data_ptr()), ctypes.c_void_p(kb.data_ptr()))
        st = self._trace(codes, kinds, seps, n_b, 0, nb, nc, stream, z_range)
        if st not in (OK, E_CAPACITY):
            _check(st)
        return {"n_branches": n_b, "n_cells": nc.value}

    @staticmethod
    def trace_buffers(cap_branches: int, cap_cells: int, device):
        """Output buffers for trace_separatrices(out=...)."""
        return dict(offsets=torch.empty(cap_branches + 1, dtype=torch.int64, device=device),
                    cells=torch.empty(max(cap_cells, 1), dtype=torch.int64, device=device),
                    origin=torch.empty(max(cap_branches, 1), dtype=torch.int64, device=device),
                    terminal=torch.empty(max(cap_branches, 1), dtype=torch.int64, device=device),
                    kind=torch.empty(max(cap_branches, 1), dtype=torch.uint8, device=device))

    def trace_separatrices(self, codes: torch.Tensor, kinds: int = KIND_DESC | KIND_ASC | KIND_CONN,
                           cap_branches: int | None = None, cap_cells: int | None = None, stream=None,
                           out: dict | None = None, z_range=None):
        """V-path traces -> dict of CUDA tensors (CSR).  ``out`` (from
        trace_buffers) avoids allocating the outputs."""
        _need_cuda(codes)
        dev = codes.device

        def run(cb, cc):
            bufs = out if out is not None else self.trace_buffers(cb, cc, dev)
            seps = _Seps(*(ctypes.c_void_p(bufs[k].data_ptr()) for k in ("offsets", "cells", "origin", "terminal", "kind")))
            nb, nc = ctypes.c_int64(), ctypes.c_int64()
            st = self._trace(codes, kinds, seps, cb, cc, nb, nc, stream, z_range)
            return st, nb.value, nc.value, bufs

        if out is not None:
            cb, cc = out["origin"].shape[0], out["cells"].shape[0]
        else:
            cb = cap_branches if cap_branches is not None else 1 << 16
            cc = cap_cells if cap_cells is not None else 1 << 20
        st, nb, nc, bufs = run(cb, cc)
        tries = 0
        while st == E_CAPACITY and cap_branches is None and cap_cells is None and out is None and tries < 2:
            # the branch count is known first; the cell count once the branches fit
            cb, cc = max(nb, cb), max(nc, cc)
            st, nb, nc, bufs = run(cb, cc)
            tries += 1
        _check(st)
        return dict(offsets=bufs["offsets"][:nb + 1], cells=bufs["cells"][:nc], origin=bufs["origin"][:nb],
                    terminal=bufs["terminal"][:nb], kind=bufs["kind"][:nb])


@dataclass
class Result:
    status: int
    g: torch.Tensor
    edits: torch.Tensor          # (n, 16) uint8 rows in dmtz_edit layout, sorted by v
    n_edits: int
    stats: dict = dc_field(default_factory=dict)
    message: str = ""

    def edits_numpy(self) -> np.ndarray:
        return self.edits.cpu().numpy().view(EDIT_DTYPE).reshape(-1)


_ctx_cache: dict = {}


def context(shape, device=None) -> Context:
    key = (tuple(shape), str(device))
    c = _ctx_cache.get(key)
    if c is None:
        c = _ctx_cache[key] = Context(shape, device)
    return c


def compute_gradient(field: torch.Tensor, stream=None):
    return context(field.shape, field.device).compute_gradient(field, stream=stream)


def critical_mask(codes: torch.Tensor, stream=None):
    return context(codes.shape, codes.device).critical_mask(codes, stream=stream)


def correct(f: torch.Tensor, fhat: torch.Tensor, xi: float, **kw) -> Result:
    return context(f.shape, f.device).correct(f, fhat, xi, **kw)


def preserve(f: torch.Tensor, fhat: torch.Tensor, xi: float, **kw) -> Result:
    return context(f.shape, f.device).preserve(f, fhat, xi, **kw)


def trace_separatrices(codes: torch.Tensor, kinds: int = KIND_DESC | KIND_ASC | KIND_CONN, **kw):
    return context(codes.shape, codes.device).trace_separatrices(codes, kinds, **kw)


def correct_host(f: np.ndarray, fhat: np.ndarray, xi: float, device="cuda", **kw):
    """End-to-end call from HOST arrays: H2D of f and fhat, the C-loop, D2H of g and
    the edit list.  Returns (g numpy, edits numpy, stats)."""
    fp = torch.from_numpy(np.ascontiguousarray(f, np.float32)).pin_memory()
    fhp = torch.from_numpy(np.ascontiguousarray(fhat, np.float32)).pin_memory()
    r = context(f.shape, torch.device(device)).correct_host(fp, fhp, xi, **kw)
    return r.g.numpy(), r.edits.numpy().view(EDIT_DTYPE).reshape(-1), r.stats
