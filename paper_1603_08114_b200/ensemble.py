"""Ensembles of independent chains on one GPU (BASELINE.json config 4).

The reference runs one chain per process (`sampler.py:291-358`); its spec
allows chain parallelism but ships no driver for it (SURVEY §2, K-ens).  An
``Ensemble`` holds ``n_chains`` chains of ``T_chain`` sites each, chain-major
in HBM, one shared parameter set, and one numpy ``SFC64`` stream per chain.
A round is, for every chain at once, exactly the reference's
``hmc_update_volatility`` (`sampler.py:144-167`) on that chain with that
chain's ``Generator(SFC64(...))``: ziggurat momenta from its own stream,
an L-step leapfrog trajectory, dH, and the Metropolis test with the next
raw word of its stream.  Chains never interact: the trajectory kernel cuts
the AR(1) coupling at chain boundaries and every chain takes its own
decision (`ens_decide_kernel` in csrc/leapfrog.cu).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .model import Params


def sfc64_states(seed: int, n_chains: int, start: int = 0) -> np.ndarray:
    """State words (a, b, c, counter) of ``SFC64(SeedSequence([seed, c]))``
    for c = start .. start+n_chains-1 (the config-4 seeding)."""
    out = np.empty((n_chains, 4), dtype=np.uint64)
    for i in range(n_chains):
        out[i] = np.random.SFC64(np.random.SeedSequence([seed, start + i])).state["state"]["state"]
    return out


class Ensemble:
    """``n_chains`` independent chains of ``T_chain`` sites on one GPU."""

    def __init__(self, n_chains: int, T_chain: int, device: int = 0):
        self.n_chains, self.T_chain = int(n_chains), int(T_chain)
        self.T = self.n_chains * self.T_chain
        self._lib = N.lib()
        h = ctypes.c_void_p()
        N.check(self._lib.rsv_ens_create(ctypes.byref(h), int(device), self.n_chains, self.T_chain))
        self.ctx = h.value

    def close(self):
        if self.ctx:
            self._lib.rsv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _ck(self, code):
        N.check(code, self.ctx)

    def _shape(self, a: np.ndarray, name: str) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.shape == (self.T_chain,):  # one series for every chain
            a = np.ascontiguousarray(np.broadcast_to(a, (self.n_chains, self.T_chain)))
        if a.shape != (self.n_chains, self.T_chain):
            raise ValueError(f"{name} must have shape ({self.n_chains}, {self.T_chain}) or ({self.T_chain},), "
                             f"got {a.shape}")
        return a

    # -- state --
    def set_data(self, returns: np.ndarray, log_rv: np.ndarray):
        y, lrv = self._shape(returns, "returns"), self._shape(log_rv, "log_rv")
        self._ck(self._lib.rsv_set_data(self.ctx, y.ctypes.data, lrv.ctypes.data, 0))

    def set_params(self, params: Params):
        self._ck(self._lib.rsv_set_params(self.ctx, ctypes.byref(N.to_params(params))))

    def set_latent(self, h: np.ndarray):
        h = self._shape(h, "latent")
        self._ck(self._lib.rsv_set_latent(self.ctx, h.ctypes.data, 0))

    def latent(self) -> np.ndarray:
        out = np.empty((self.n_chains, self.T_chain))
        self._ck(self._lib.rsv_get_latent(self.ctx, out.ctypes.data, 0))
        return out

    def set_streams(self, states: np.ndarray):
        st = np.ascontiguousarray(states, dtype=np.uint64)
        if st.shape != (self.n_chains, 4):
            raise ValueError(f"states must have shape ({self.n_chains}, 4), got {st.shape}")
        self._ck(self._lib.rsv_ens_set_streams(self.ctx, st.ctypes.data))

    def seed(self, seed: int):
        """Chain c draws from SFC64(SeedSequence([seed, c]))."""
        self.set_streams(sfc64_states(seed, self.n_chains))

    def streams(self) -> np.ndarray:
        out = np.empty((self.n_chains, 4), dtype=np.uint64)
        self._ck(self._lib.rsv_ens_get_streams(self.ctx, out.ctypes.data))
        return out

    # -- the hot path --
    def refresh_momenta(self, copy: bool = True) -> np.ndarray | None:
        """sampler.py:136-141 for every chain (advances each stream); with
        copy=False the normals stay on the device."""
        out = np.empty((self.n_chains, self.T_chain)) if copy else None
        self._ck(self._lib.rsv_ens_refresh_momenta(self.ctx, out.ctypes.data if copy else None))
        return out

    def hmc_update(self, step_size: float, n_steps: int, fuse: bool = False, rounds: int = 1):
        """``rounds`` volatility updates of every chain; returns the last
        round's (accept[bool], delta_h[+inf when diverged]) per chain."""
        acc = np.empty(self.n_chains, dtype=np.int32)
        dh = np.empty(self.n_chains)
        self._ck(self._lib.rsv_ens_hmc_update(self.ctx, float(step_size), int(n_steps), int(bool(fuse)), int(rounds),
                                              acc.ctypes.data, dh.ctypes.data))
        return acc.astype(bool), dh

    def counts(self):
        """(accepted, diverged) proposals per chain since the streams were set."""
        a = np.empty(self.n_chains, dtype=np.int32)
        d = np.empty(self.n_chains, dtype=np.int32)
        self._ck(self._lib.rsv_ens_counts(self.ctx, a.ctypes.data, d.ctypes.data))
        return a, d

    # -- benchmark helpers --
    def set_timing(self, level):
        self._ck(self._lib.rsv_set_timing(self.ctx, int(level)))

    def timing_ms(self) -> float:
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        self._ck(self._lib.rsv_get_timing(self.ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return c.value

    def set_l2_flush(self, nbytes: int):
        self._ck(self._lib.rsv_set_l2_flush(self.ctx, int(nbytes)))

    def launch_count(self) -> int:
        return int(self._lib.rsv_launch_count(self.ctx))
