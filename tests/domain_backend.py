"""A numpy force backend for the domain-decomposition tests (test infrastructure).

Same interface as ``paper_2507_11172_b200.domain_run.GpuBackend``, computing
on the rank's local set exactly what the C01 reference does for owned base
particles (containers.py:282-370, :373-535): the force on each owned
particle from all local partners, phi/2 per owned pair visit and phi/3 per
owned triplet visit.  Used with gloo on CPU, so the exchange logic of
domain.py is exercised without a GPU.
"""

from __future__ import annotations

import numpy as np
import torch


def _lj(r2, eps, sig2):
    x = sig2 / r2
    r6 = x * x * x
    r12 = r6 * r6
    return 4.0 * eps * (r12 - r6), 24.0 * eps * (2.0 * r12 - r6) / r2


def _atm(a, b, c, nu):
    u = a + b - c
    v = a + c - b
    w = b + c - a
    p = u * v * w
    s = a * b * c
    inv_s = 1.0 / s
    s32 = inv_s / np.sqrt(s)
    s52 = s32 * inv_s
    s72 = s52 * inv_s
    e = nu * (s32 + 0.375 * p * s52)
    uv, uw, vw = u * v, u * w, v * w
    bc, ac, ab = b * c, a * c, a * b
    da = nu * ((0.375 * (vw + uw - uv) - 1.5 * bc) * s52 - 0.9375 * p * bc * s72)
    db = nu * ((0.375 * (vw - uw + uv) - 1.5 * ac) * s52 - 0.9375 * p * ac * s72)
    dc = nu * ((0.375 * (uw + uv - vw) - 1.5 * ab) * s52 - 0.9375 * p * ab * s72)
    return e, da, db, dc


class NumpyBackend:
    def __init__(self, ff, box):
        self.ff = ff
        self.box = np.asarray(box, dtype=np.float64)
        self.half = 0.5 * self.box
        self.device = torch.device("cpu")
        rc3 = ff.cutoff if getattr(ff, "cutoff_3b", None) is None else ff.cutoff_3b
        self.rc2, self.rc3 = float(ff.cutoff), float(rc3)

    def _disp(self, a, b):
        d = a - b
        d = np.where(d > self.half, d - self.box, np.where(d < -self.half, d + self.box, d))
        return d

    def set_local(self, local, n_own, window, rebuild):
        self.pos = local.detach().cpu().numpy().copy()
        self.n_own = int(n_own)

    def pair(self, scalars=True):
        pos, n = self.pos, self.n_own
        f = np.zeros((n, 3))
        e = w = 0.0
        for i in range(n):
            d = self._disp(pos[i][None, :], pos)
            r2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
            m = r2 <= self.rc2 * self.rc2
            m[i] = False
            en, sc = _lj(r2[m], self.ff.epsilon, self.ff.sigma ** 2)
            f[i] = (sc[:, None] * d[m]).sum(axis=0)
            e += float(np.sum(0.5 * en))
            w += float(np.sum(0.5 * sc * r2[m]))
        return torch.as_tensor(f), torch.tensor([e, w], dtype=torch.float64)

    def triplet(self, scalars=True):
        pos, n = self.pos, self.n_own
        f = np.zeros((n, 3))
        e = w = 0.0
        rc2 = self.rc3 * self.rc3
        nu = float(self.ff.nu)
        if nu == 0.0:
            return torch.as_tensor(f), torch.zeros(2, dtype=torch.float64)
        for i in range(n):
            d = self._disp(pos[i][None, :], pos)
            r2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
            m = r2 <= rc2
            m[i] = False
            idx = np.nonzero(m)[0]
            if idx.size < 2:
                continue
            jj, kk = np.triu_indices(idx.size, 1)
            j, k = idx[jj], idx[kk]
            djk = self._disp(pos[j], pos[k])
            c = (djk[:, 0] * djk[:, 0] + djk[:, 1] * djk[:, 1]) + djk[:, 2] * djk[:, 2]
            ok = c <= rc2
            j, k, c = j[ok], k[ok], c[ok]
            a, b = r2[j], r2[k]
            en, da, db, dc = _atm(a, b, c, nu)
            f[i] = (-2.0 * (da[:, None] * d[j] + db[:, None] * d[k])).sum(axis=0)
            e += float(np.sum(en / 3.0))
            w += float(np.sum(-2.0 * (da * a + db * b + dc * c) / 3.0))
        return torch.as_tensor(f), torch.tensor([e, w], dtype=torch.float64)

    def check(self):
        return None
