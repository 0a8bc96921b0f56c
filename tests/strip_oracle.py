"""Window operations of a strip-partitioned hierarchy restated from the oracle's GLOBAL level
operators (test infrastructure): A, D^-1 and P restricted to the rows/columns of one rank's
local window.  Used as the local backend of StripMG in the gloo tests and as the checker of
the device window kernels (DeviceStripBackend) in the GPU tests."""

import numpy as np
import scipy.sparse as sp

from oracle import hdg_oracle as O


class OracleWindowBackend:
    """Window ops from the oracle's global CSR operators (A, D^-1, P) restricted to rows/cols of
    each rank's local window."""

    def __init__(self, levels, layouts, d, omega=0.8):
        import torch
        self.t, self.levels, self.layouts, self.d, self.w = torch, levels, layouts, d, omega
        self.A, self.Dinv, self.P = [], [], []
        for l in range(d + 1):
            loc = layouts[l].local_to_global
            A = levels[l].operator.tocsr()
            self.A.append(A[loc][:, loc])
            sm = levels[l].smoother
            n1 = levels[l].p + 1
            blocks = loc.reshape(-1, n1)[:, 0] // n1
            nb = blocks.size
            self.Dinv.append(sp.bsr_matrix((np.ascontiguousarray(sm.Dinv[blocks]), np.arange(nb), np.arange(nb + 1)),
                                           shape=(nb * n1, nb * n1)).tocsr())
            locc = layouts[l + 1].local_to_global
            self.P.append(levels[l].prolong.tocsr()[loc][:, locc])

    def _T(self, a):
        return self.t.from_numpy(np.ascontiguousarray(a))

    def link(self, l):
        return "p" if self.levels[l + 1].grid.n_x == self.levels[l].grid.n_x else "h"

    def bj_zero(self, l, b, k, steps):
        return self._T(self.w * (self.Dinv[l] @ b.numpy()))

    def bj_sweep(self, l, b, x, k, steps):
        xn = x.numpy()
        return self._T(xn + self.w * (self.Dinv[l] @ (b.numpy() - self.A[l] @ xn)))

    def residual(self, l, b, x):
        return self._T(b.numpy() - self.A[l] @ x.numpy())

    def residual_restrict_p(self, l, b, x):
        return self._T(self.P[l].T @ (b.numpy() - self.A[l] @ x.numpy()))

    def restrict_h(self, l, r):
        return self._T(self.P[l].T @ r.numpy())

    def prolong_add(self, l, ec, x):
        return self._T(x.numpy() + self.P[l] @ ec.numpy())

    def global_cycle(self, bg, xg, nu1, nu2, visits):
        sub = self.levels[self.d + 1:]
        bgn = bg.numpy()
        x0 = np.zeros_like(bgn) if xg is None else xg.numpy()
        return self._T(O.cycle(sub, 0, bgn, x0, nu1, nu2, visits))
