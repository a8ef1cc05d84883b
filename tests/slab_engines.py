"""Test engine for the slab driver: each rank's round is the literal oracle round
(oracle.slab_round) on its local grid -- lets the multi-rank host logic run on CPU
with gloo and be compared against the single-domain oracle."""
import numpy as np
import torch

import oracle


class OracleSlabEngine:
    def __init__(self, p, ny, nx):
        self.p = p

    def begin(self, f, fhat, xi, q_max=6, q_cap=None, tier=2):
        self.f = np.ascontiguousarray(f.numpy() if isinstance(f, torch.Tensor) else f, np.float32)
        self.fhat = np.ascontiguousarray(fhat.numpy() if isinstance(fhat, torch.Tensor) else fhat, np.float32)
        self.xi, self.q_max, self.q_cap, self.tier = xi, q_max, q_cap, tier
        self.g = torch.from_numpy(self.fhat.copy())
        self.state = np.zeros(self.f.shape, np.uint32)

    def round(self, r):
        nF, nch, nt, kinds = oracle.slab_round(self.f, self.fhat, self.xi, self.g.numpy(), self.state,
                                               self.p.anchor_local, self.p.own_local, self.q_max, self.q_cap,
                                               self.tier)
        return np.array([nF, nch, nt, 0], np.int64), (kinds if r == 1 else np.zeros(8, np.int64))

    def halo(self, r, a, b, planes):
        self.g[a:b] = torch.as_tensor(planes)

    def end(self):
        o0, o1 = self.p.own_local
        plane = self.f.shape[1] * self.f.shape[2]
        st = self.state[o0:o1].ravel()
        g = self.g.numpy()[o0:o1].ravel()
        idx = np.nonzero(st)[0]
        e = np.zeros(len(idx), dtype=oracle.EDIT_DTYPE)
        e["v"] = idx + (self.p.lz0 + o0) * plane
        e["q"] = st[idx] & 0xFFFF
        e["lossless"] = st[idx] >> 16
        e["value"] = g[idx]
        return e, int((st[idx] >> 16).sum())
