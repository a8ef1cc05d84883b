"""Seeded synthetic inputs shared by tests, bench.py and smoke().

Holds none of the method's arithmetic (see gen.c's header): original fields f
shaped like the paper's datasets, the absolute bound xi for a relative bound,
and the decompressed field fhat from a built-in error-bounded quantizer that
stands in for SZ3.  The recipe is documented in DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libdmtz_inputs.so")

FAMILIES = {"gauss2d": 0, "climate": 1, "hurricane": 2, "lognormal": 3, "multiscale": 4, "noise": 5}


@dataclass(frozen=True)
class Config:
    name: str
    family: str
    shape: tuple          # numpy shape, slowest first: (ny, nx) or (nz, ny, nx)
    eps: float            # value-range-relative error bound
    seed: int
    q_max: int = 6
    gpus: tuple = (1,)


# BASELINE.json "configs", in order (dims read slowest -> fastest, x contiguous)
CONFIGS = {
    "C1": Config("C1", "gauss2d", (64, 64), 1e-3, 101),
    "C2": Config("C2", "climate", (1800, 3600), 1e-3, 102),
    "C3": Config("C3", "hurricane", (100, 500, 500), 1e-3, 103, gpus=(1, 2)),
    "C4": Config("C4", "lognormal", (512, 512, 512), 1e-4, 104, gpus=(1, 2, 4, 8)),
    "C5": Config("C5", "multiscale", (1024, 1024, 1024), 1e-3, 105, gpus=(8,)),
}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC",
                               "-shared", "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P, i64 = ctypes.c_void_p, ctypes.c_int64
        L.dmtz_gen_raw.argtypes = [ctypes.c_int, i64, i64, i64, ctypes.c_uint64, P]
        L.dmtz_gen_normalize.argtypes = [P, i64, P]
        L.dmtz_gen_xi.argtypes = [P, i64, ctypes.c_double]
        L.dmtz_gen_xi.restype = ctypes.c_float
        L.dmtz_gen_lorenzo.argtypes = [P, i64, i64, i64, ctypes.c_float, P]
        L.dmtz_gen_lorenzo_codes.argtypes = [P, i64, i64, i64, ctypes.c_float, P, P]
        L.dmtz_gen_uniform_noise.argtypes = [P, i64, ctypes.c_float, ctypes.c_uint64, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _nxyz(shape):
    if len(shape) == 2:
        return shape[1], shape[0], 1
    return shape[2], shape[1], shape[0]


def field(family: str, shape, seed: int) -> np.ndarray:
    """Original field f (float32, values in [1, 2)) of the given family."""
    nx, ny, nz = _nxyz(shape)
    raw = np.empty(int(np.prod(shape)), np.float64)
    if _L().dmtz_gen_raw(FAMILIES[family], nx, ny, nz, seed, _p(raw)):
        raise ValueError(family)
    f = np.empty(raw.size, np.float32)
    _L().dmtz_gen_normalize(_p(raw), raw.size, _p(f))
    return f.reshape(shape)


def xi_for(f: np.ndarray, eps: float) -> float:
    """xi = RN32(eps * (max f - min f)) computed in f64 (reading A12)."""
    f = np.ascontiguousarray(f, np.float32)
    return float(_L().dmtz_gen_xi(_p(f), f.size, eps))


def lorenzo(f: np.ndarray, xi: float) -> np.ndarray:
    """Closed-loop Lorenzo error-bounded quantizer -> fhat with |fhat - f| <= xi."""
    f = np.ascontiguousarray(f, np.float32)
    nx, ny, nz = _nxyz(f.shape)
    out = np.empty_like(f)
    _L().dmtz_gen_lorenzo(_p(f), nx, ny, nz, ctypes.c_float(xi), _p(out))
    return out


LORENZO_RAW = 0x7FFFFFFF


def lorenzo_codes(f: np.ndarray, xi: float):
    """(fhat, codes): the Lorenzo quantizer's integer codes (LORENZO_RAW = stored verbatim)."""
    f = np.ascontiguousarray(f, np.float32)
    nx, ny, nz = _nxyz(f.shape)
    out = np.empty_like(f)
    codes = np.empty(f.shape, np.int32)
    _L().dmtz_gen_lorenzo_codes(_p(f), nx, ny, nz, ctypes.c_float(xi), _p(out), _p(codes))
    return out, codes


def base_compressed_bytes(f: np.ndarray, xi: float) -> dict:
    """Size model of the SZ3 stand-in's compressed stream (for CR and OCR): the
    entropy of its integer quantization codes (the ideal size of SZ3's Huffman stage)
    plus the verbatim float32 values, plus a 4 B per distinct code table."""
    _, codes = lorenzo_codes(f, xi)
    raw = codes == LORENZO_RAW
    _, cnt = np.unique(codes[~raw], return_counts=True)
    p = cnt / max(cnt.sum(), 1)
    bits = float(-(cnt * np.log2(p)).sum()) if cnt.size else 0.0
    nbytes = int(np.ceil(bits / 8)) + 4 * int(raw.sum()) + 4 * int(cnt.size)
    return {"bytes": nbytes, "n_verbatim": int(raw.sum()), "bits_per_value": bits / max(codes.size, 1),
            "model": "entropy of the Lorenzo codes + verbatim floats + code table"}


def uniform_noise(f: np.ndarray, xi: float, seed: int) -> np.ndarray:
    f = np.ascontiguousarray(f, np.float32)
    out = np.empty_like(f)
    _L().dmtz_gen_uniform_noise(_p(f), f.size, ctypes.c_float(xi), seed, _p(out))
    return out


def config_inputs(name: str, shape=None, perturb: str = "lorenzo"):
    """(f, fhat, xi, cfg) for a BASELINE config; ``shape`` overrides the size
    (same family, eps and seed) for small parity cases."""
    cfg = CONFIGS[name]
    shp = tuple(shape) if shape is not None else cfg.shape
    f = field(cfg.family, shp, cfg.seed)
    xi = xi_for(f, cfg.eps)
    if perturb == "lorenzo":
        fhat = lorenzo(f, xi)
    else:
        fhat = uniform_noise(f, xi, cfg.seed ^ 0xABCDEF)
    return f, fhat, xi, cfg


def random_case(shape, seed: int, eps: float = 1e-2, ties: bool = False, perturb="lorenzo",
                family: str = "noise"):
    """Small case for parity tests (white noise by default); ``ties`` quantises f to
    force SoS ties; ``perturb`` is "lorenzo" or "noise" (uniform in [-xi, xi])."""
    f = field(family, tuple(shape), seed)
    if ties:
        f = (np.floor((f - 1.0) * 8.0) / 8.0 + 1.0).astype(np.float32)
    xi = xi_for(f, eps)
    fhat = lorenzo(f, xi) if perturb == "lorenzo" else uniform_noise(f, xi, seed + 7)
    return f, fhat, xi
