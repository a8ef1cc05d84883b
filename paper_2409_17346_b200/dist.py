"""Multi-GPU C-loop through the library (dmtz_correct on a world > 1 context).

Argument marshalling only: the halo exchange, the rounds, the counter reduction and the
stop rule run inside libdmtz (csrc/dmtz_dist.cuh).  The transport is the context's own
NCCL communicator (``nccl_id`` = the same 128-byte id on every rank), or callbacks
installed with ``set_transport`` -- ``gloo_transport`` stages through host memory over
torch.distributed gloo (tests: two processes sharing one GPU, whose kernels never wait
on each other: every exchange completes on the host between rounds).
"""
from __future__ import annotations

import ctypes

import torch

from . import (DmtzError, Result, _Dims, _Opts, _Stats, _check, _lib, _need_cuda, _stats_dict, _stream_ptr,
               E_CAPACITY, E_ITER_CAP, E_STUCK, OK)

_EXCH = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                         ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t),
                         ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t), ctypes.c_void_p)
_AR = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)


class _Transport(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("exchange", _EXCH), ("allreduce_sum_i64", _AR)]


def local_slab(nz: int, world: int, rank: int):
    """(z0, z1, lz0, lz1): owned and local planes of a rank (dmtz_local_slab)."""
    v = [ctypes.c_int64() for _ in range(4)]
    _check(_lib.dmtz_local_slab(int(nz), int(world), int(rank), *(ctypes.byref(x) for x in v)))
    return tuple(x.value for x in v)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.dmtz_nccl_unique_id(buf))
    return buf.raw


class _DevBytes:
    """A raw device pointer as a torch uint8 tensor (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(n),), "typestr": "|u1",
                                         "version": 3}


def _dev(ptr, n):
    return torch.as_tensor(_DevBytes(ptr, n), device="cuda")


def gloo_transport(group=None):
    """(exchange, allreduce) callables for set_transport: host-staged torch.distributed
    point-to-point and all_reduce (a gloo process group)."""
    import torch.distributed as dist

    def exchange(n, peers, send, sbytes, recv, rbytes):
        torch.cuda.synchronize()
        reqs, incoming = [], []
        for i in range(n):
            if sbytes[i]:
                reqs.append(dist.isend(_dev(send[i], sbytes[i]).cpu(), peers[i], group=group))
            if rbytes[i]:
                buf = torch.empty(int(rbytes[i]), dtype=torch.uint8)
                incoming.append((recv[i], buf))
                reqs.append(dist.irecv(buf, peers[i], group=group))
        for r in reqs:
            r.wait()
        for ptr, buf in incoming:
            _dev(ptr, buf.numel()).copy_(buf)
        torch.cuda.synchronize()

    def allreduce(ptr, n):
        torch.cuda.synchronize()
        v = _dev(ptr, 8 * n).view(torch.int64)
        h = v.cpu()
        dist.all_reduce(h, group=group)
        v.copy_(h)
        torch.cuda.synchronize()

    return exchange, allreduce


class DistContext:
    """One rank of the multi-GPU C-loop: a dmtz_ctx over the rank's slab of a global
    grid (numpy shape (nz, ny, nx)); correct() takes and returns the OWNED planes."""

    def __init__(self, global_shape, rank: int, world: int, device=None, nccl_id: bytes | None = None,
                 rounds_per_sync: int = 8, graph: bool = False):
        self.global_shape = tuple(int(x) for x in global_shape)
        nz, ny, nx = self.global_shape
        self.rank, self.world = int(rank), int(world)
        self.z0, self.z1, self.lz0, self.lz1 = local_slab(nz, world, rank)
        self.owned_shape = (self.z1 - self.z0, ny, nx)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        h = ctypes.c_void_p()
        d = _Dims(nx, ny, nz)
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(_lib.dmtz_ctx_create(ctypes.byref(h), ctypes.byref(d), self.rank, self.world, idbuf,
                                    self.device.index or 0))
        self._h = h
        _check(_lib.dmtz_ctx_set_dist_sync(h, int(rounds_per_sync)))
        _check(_lib.dmtz_ctx_set_dist_graph(h, 1 if graph else 0, None))
        self.ws_bytes = int(_lib.dmtz_workspace_bytes(h, None))
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self._cb = None

    def set_transport(self, exchange, allreduce):
        """exchange(n, peers, send_ptrs, send_bytes, recv_ptrs, recv_bytes) and
        allreduce(dev_ptr, n) in Python (see gloo_transport); errors -> nonzero status."""
        def ex(user, n, peers, send, sb, recv, rb, stream):
            try:
                exchange(n, [peers[i] for i in range(n)], [send[i] for i in range(n)], [sb[i] for i in range(n)],
                         [recv[i] for i in range(n)], [rb[i] for i in range(n)])
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def ar(user, buf, n, stream):
            try:
                allreduce(buf, n)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self._cb = _Transport(None, _EXCH(ex), _AR(ar))   # kept alive with the context
        _check(_lib.dmtz_ctx_set_transport(self._h, ctypes.byref(self._cb)))

    def correct(self, f: torch.Tensor, fhat: torch.Tensor, xi: float, q_max: int = 6, q_cap: int | None = None,
                tier: int = 2, max_rounds: int = 0, full_sweeps: bool = False, stream=None,
                raise_on_error: bool = True) -> Result:
        _need_cuda(f, fhat)
        for t in (f, fhat):
            assert t.dtype == torch.float32 and tuple(t.shape) == self.owned_shape and t.is_contiguous()
        g = torch.empty_like(f)
        cap = f.numel()
        edits = torch.empty((max(cap, 1), 16), dtype=torch.uint8, device=f.device)
        opts = _Opts(float(xi), int(q_max), int(q_max if q_cap is None else q_cap), int(tier), int(max_rounds),
                     1 if full_sweeps else 0, 0)
        ne, st = ctypes.c_int64(), _Stats()
        status = _lib.dmtz_correct(self._h, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(fhat.data_ptr()),
                                   ctypes.byref(opts), ctypes.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                                   ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(edits.data_ptr()), cap,
                                   ctypes.byref(ne), ctypes.byref(st), _stream_ptr(stream))
        stats = _stats_dict(st, status)
        msg = _lib.dmtz_last_error().decode() if status != OK else ""
        if raise_on_error and status not in (OK, E_STUCK, E_ITER_CAP, E_CAPACITY):
            raise DmtzError(status, msg)
        return Result(status=status, g=g, edits=edits[:min(ne.value, cap)], n_edits=ne.value, stats=stats,
                      message=msg)

    def graph_used(self) -> bool:
        """Whether the last correct() replayed its batches from a CUDA graph."""
        u = ctypes.c_int()
        _check(_lib.dmtz_ctx_set_dist_graph(self._h, -1, ctypes.byref(u)))
        return bool(u.value)

    def close(self):
        if getattr(self, "_h", None):
            _lib.dmtz_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
