"""Synthetic RSV data (mirror of the reference's ``data.py:72-95 simulate_rsv``).

Input generation only: it runs on the host with the
reference's fixed draw order -- initial deviation, latent innovations, return
shocks, measurement noise -- from ``make_rng(seed)`` (numpy Philox), so a
given seed gives the reference's dataset bit for bit.  The AR(1) recursion
out[t+1] = phi * out[t] + eta[t] (_kernels.py:70-76) is evaluated by
scipy.signal.lfilter, which performs the same two roundings per step.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.signal import lfilter

from .model import Dataset, Params
from .rng import make_rng


@dataclass
class SyntheticTruth:
    params: Params
    latent: np.ndarray
    dataset: Dataset


def ar1_path(dev0: float, innovations: np.ndarray, phi: float) -> np.ndarray:
    x = np.empty(innovations.size + 1)
    x[0] = dev0
    x[1:] = innovations
    zi = np.zeros(1)
    # y[n] = x[n] + phi * y[n-1] with y[-1] = 0  ->  y[0] = dev0
    return lfilter([1.0], [1.0, -phi], x, zi=zi)[0]


def simulate_rsv(params: Params, t_len: int, seed: int, backend=None) -> SyntheticTruth:
    """data.py:72-95.  Host (default): bit for bit the reference's dataset.
    backend=<CudaBackend>: on the GPU (rsv_simulate) -- the same normals bit
    for bit, the AR(1) path by a parallel scan (equal to rounding), for very
    long series (2^26 sites in milliseconds instead of seconds)."""
    if t_len < 2:
        raise ValueError(f"need t_len >= 2, got {t_len}")
    rng = make_rng(seed)
    if backend is not None:
        return _simulate_device(params, t_len, rng, getattr(backend, "device", 0))
    se = math.sqrt(params.sigma_eta_sq)
    dev0 = math.sqrt(params.sigma_eta_sq / (1.0 - params.phi ** 2)) * rng.standard_normal()
    eta = se * rng.standard_normal(t_len - 1)
    eps = rng.standard_normal(t_len)
    u = math.sqrt(params.sigma_u_sq) * rng.standard_normal(t_len)
    dev = ar1_path(dev0, eta, params.phi)
    h = params.mu + dev
    returns = np.exp(0.5 * h) * eps
    log_rv = params.xi + h + u
    dataset = Dataset.from_log_rv(returns, log_rv)
    return SyntheticTruth(params=params, latent=h, dataset=dataset)


def _simulate_device(params: Params, t_len: int, rng, device: int) -> SyntheticTruth:
    import ctypes

    from . import _native as N
    from .rng import store_stream_state, stream_state
    st = stream_state(rng)
    h = np.empty(t_len)
    y = np.empty(t_len)
    lrv = np.empty(t_len)
    N.check(N.lib().rsv_simulate(int(device), ctypes.byref(N.to_params(params)), int(t_len), ctypes.byref(st),
                                 h.ctypes.data, y.ctypes.data, lrv.ctypes.data, 0))
    store_stream_state(rng, st)
    return SyntheticTruth(params=params, latent=h, dataset=Dataset.from_log_rv(y, lrv))
