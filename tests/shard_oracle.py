"""CPU stand-in for the GPU shard context (test infrastructure): the same
interface as paper_1603_08114_b200.sharded.CudaShard, computed with the
oracle, so the host-side sharding logic (partition, halo exchange,
fixed-order combination, Metropolis decision) can be tested with gloo on
CPUs."""
import ctypes

import numpy as np

import oracle as O
from paper_1603_08114_b200.sharded import TOTALS, W_ENDS, W_FLAG, W_SN, W_SO, W_U, fix128, local_range, put128


class OracleShard:
    def __init__(self, T, lo, hi, margin):
        self.T, self.lo, self.hi = T, lo, hi
        ls, le = local_range(T, lo, hi, margin)
        self.local_start, self.local_len = ls, le - ls
        self.st = O.Stream("philox", 0)

    def set_data(self, y, lrv):
        self.y = np.ascontiguousarray(y, dtype=np.float64)
        self.lrv = np.ascontiguousarray(lrv, dtype=np.float64)

    def set_params(self, params):
        self.params = params

    def set_latent(self, h):
        self.h = np.array(h, dtype=np.float64)

    def get_latent(self):
        return self.h.copy()

    def set_stream(self, st):
        kinds = {0: "philox", 1: "minstd", 2: "pcg32", 3: "sfc64"}
        self.st = O.Stream(kinds[st.kind], 0)
        self.st._st.kind = st.kind
        for i in range(4):
            self.st._st.s[i] = st.s[i]
        self.st._st.pos = st.pos
        self.st._st.cache_ok = 0

    def get_stream(self):
        from paper_1603_08114_b200 import _native as N
        out = N.PrngState()
        out.kind = self.st._st.kind
        for i in range(4):
            out.s[i] = self.st._st.s[i]
        out.pos = self.st._st.pos
        return out

    def _copy_stream(self):
        c = O.Stream("philox", 0)
        ctypes.memmove(ctypes.byref(c._st), ctypes.byref(self.st._st), ctypes.sizeof(c._st))
        return c

    def slice_out(self, offset, n):
        return self.h[offset:offset + n].copy()

    def slice_in(self, offset, buf):
        self.h[offset:offset + len(buf)] = buf

    def _site_terms(self, h, p):
        """per-site potential and kinetic energy (variable parts, d-space) and
        statistics; the owned slice"""
        P = self.params
        ls = self.local_start
        d = h - P.mu
        g = np.arange(ls, ls + h.size)
        ar = np.empty_like(d)
        ar[1:] = (d[1:] - P.phi * d[:-1]) ** 2 / (2 * P.sigma_eta_sq)
        ar[0] = (d[0] - P.phi * 0.0) ** 2 / (2 * P.sigma_eta_sq)  # overwritten below if global site 0
        first = g == 0
        ar[first] = (1 - P.phi ** 2) * d[first] ** 2 / (2 * P.sigma_eta_sq)
        e = self.lrv - P.xi - h
        V = 0.5 * d + 0.5 * self.y * self.y * np.exp(-h) + e * e / (2 * P.sigma_u_sq) + ar
        K = 0.5 * p * p
        own = slice(self.lo - ls, self.hi - ls)
        dprev = np.concatenate([[0.0], d[:-1]])
        cross = d * dprev
        cross[first] = 0.0
        stats = [d[own].sum(), (d * d)[own].sum(), cross[own].sum(), e[own].sum(), (e * e)[own].sum()]
        return V, K, own, d, stats

    def _groups(self, V, K):
        """per-group H (4-aligned groups of global sites, owned part): the sum
        of the group's potentials then of its kinetic terms, as the device
        forms it, one fixed-point integer per group"""
        ls = self.local_start
        out = []
        for g0 in range(self.lo, self.hi, 4):
            sl = slice(g0 - ls, min(g0 + 4, self.hi) - ls)
            pot = 0.0
            for x in V[sl]:
                pot += float(x)
            kin = 0.0
            for x in K[sl]:
                kin += float(x)
            out.append(pot + kin)
        return out

    def propose(self, dt, n_steps, fuse, stats):
        s = self._copy_stream()
        normals = s.normals(self.T)
        used = s.pos - self.st.pos
        u_word = int(s.raw(1)[0])
        ls = self.local_start
        p = normals[ls:ls + self.local_len]
        hn, pn, div = O.integrate(self.h, p, self.params, self.y, self.lrv, dt, n_steps, fuse=fuse)
        self._prop = hn
        V0, K0, own, d_old, s_old = self._site_terms(self.h, p)
        V1, K1, _, d_new, s_new = self._site_terms(hn, pn)
        g_old, g_new = self._groups(V0, K0), self._groups(V1, K1)
        v = np.zeros(TOTALS)
        put128(v, 0, sum(fix128(b - a) for a, b in zip(g_old, g_new)))
        put128(v, 2, sum(fix128(a) for a in g_old))
        put128(v, 4, sum(fix128(b) for b in g_new))
        v[W_SO:W_SO + 5] = s_old
        v[W_SN:W_SN + 5] = s_new
        v[W_FLAG] = 1.0 if div else 0.0
        if self.lo == 0:
            v[W_ENDS + 0], v[W_ENDS + 2] = d_old[0 - ls], d_new[0 - ls]
        if self.hi == self.T:
            v[W_ENDS + 1], v[W_ENDS + 3] = d_old[self.T - 1 - ls], d_new[self.T - 1 - ls]
        v[W_U:W_U + 2] = np.array([u_word, used], dtype=np.uint64).view(np.float64)
        self._used = used
        return v

    def apply(self, accept, drew):
        self.st.raw(self._used + (1 if drew else 0))
        if accept:
            self.h = self._prop.copy()
