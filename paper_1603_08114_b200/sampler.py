"""MCMC driver: HMC for the latent path on the B200, Gibbs draws for theta.

Mirror of the reference's ``sampler.py``.  Each sweep (sampler.py:327-344):

    1. hmc_update_volatility   -- momenta, trajectory, dH, Metropolis: device
    2. update_mu               -- scalar draws on the host from the device's
    3. update_phi                 sufficient statistics of the kept path
    4. update_sigma_eta_sq        (computed inside the fused trajectory
    5. update_xi                  kernel), with numpy's Generator continuing
    6. update_sigma_u_sq          the same raw-word stream the device used

so a chain consumes the same random stream, in the same order, as the
reference's (bitwise for the momenta; the theta draws see statistics that
agree with numpy's sums to ~1e-15 relative).
"""
from __future__ import annotations

import logging
import math
from collections import deque
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as N
from .integrator import MDConfig, _resolve
from .model import PARAM_NAMES, Dataset, Params
from .rng import make_rng, store_stream_state, stream_state

logger = logging.getLogger(__name__)

DIVERGENT_DELTA_H = math.inf   # dH sentinel of a divergent proposal (sampler.py:31)
_STORM_WINDOW, _STORM_LIMIT = 100, 50  # abort when > 50 of the last 100 proposals diverged


class DivergenceStormError(RuntimeError):
    """The HMC proposals keep diverging (sampler.py:39)."""


def _positive(obj, names):
    for n in names:
        v = getattr(obj, n)
        if not v > 0.0:
            raise ValueError(f"{n} must be positive, got {v}")


@dataclass(frozen=True)
class PriorSpec:
    """Priors of theta (sampler.py:43-63): normal for mu and xi, one
    inverse-gamma (shape, scale) for both variances, Beta(phi_a, phi_b) on
    (phi + 1) / 2."""

    mu_mean: float = 0.0
    mu_var: float = 100.0
    xi_mean: float = 0.0
    xi_var: float = 100.0
    var_shape: float = 2.5
    var_scale: float = 0.025
    phi_a: float = 20.0
    phi_b: float = 1.5

    def __post_init__(self):
        _positive(self, ("mu_var", "xi_var", "var_shape", "var_scale", "phi_a", "phi_b"))


@dataclass(frozen=True)
class SamplerConfig:
    """run_chain settings (sampler.py:66-81), plus the raw-word generator
    kind (`prng`: philox -- the reference's -- minstd, pcg32 or sfc64)."""

    seed: int = 0
    md: MDConfig = field(default_factory=lambda: MDConfig(step_size=0.02, n_steps=50))
    n_burnin: int = 1000
    n_samples: int = 4000
    thin: int = 1
    store_latent: bool = False
    prng: str = "philox"

    def __post_init__(self):
        for name, low in (("n_burnin", 0), ("n_samples", 1), ("thin", 1)):
            v = getattr(self, name)
            if v < low:
                raise ValueError(f"{name} must be >= {low}, got {v}")


@dataclass
class ChainSample:
    """One stored sweep."""

    params: Params
    accept: bool
    delta_h: float
    latent: np.ndarray | None = None


@dataclass
class Chain:
    """The stored sweeps of a run, column by column (sampler.py:93-128)."""

    iters: np.ndarray
    phi: np.ndarray
    mu: np.ndarray
    xi: np.ndarray
    sigma_eta_sq: np.ndarray
    sigma_u_sq: np.ndarray
    accept: np.ndarray
    delta_h: np.ndarray
    latent: np.ndarray | None = None

    def __len__(self) -> int:
        return int(np.shape(self.iters)[0])

    def param_series(self, name: str) -> np.ndarray:
        if name in PARAM_NAMES:
            return getattr(self, name)
        raise KeyError(f"unknown parameter {name!r}")

    def sample(self, i: int) -> ChainSample:
        theta = Params(**{n: float(getattr(self, n)[i]) for n in PARAM_NAMES})
        return ChainSample(params=theta, accept=bool(self.accept[i]), delta_h=float(self.delta_h[i]),
                           latent=self.latent[i] if self.latent is not None else None)

    @property
    def n_divergent(self) -> int:
        return int(np.isinf(self.delta_h).sum())


def refresh_momenta(rng: np.random.Generator, t_len: int, dtype=np.float64, backend=None) -> np.ndarray:
    """sampler.py:136-141 on the device: numpy-ziggurat normals, bit-exact,
    drawn from ``rng``'s stream (whose position is advanced)."""
    if t_len < 2:
        raise ValueError(f"need at least 2 sites, got {t_len}")
    if np.dtype(dtype) != np.float64:
        raise NotImplementedError("the B200 path computes in float64 only")
    ch = _resolve(backend).chain(T=t_len)
    ch.set_stream(stream_state(rng))
    p = ch.refresh_momenta()
    store_stream_state(rng, ch.get_stream())
    return p


def hmc_update_volatility(h: np.ndarray, params: Params, data: Dataset, md: MDConfig, rng: np.random.Generator,
                          backend=None, fuse_half_steps: bool = False) -> tuple[np.ndarray, bool, float]:
    """sampler.py:144-167: one HMC proposal for the whole path, on the GPU.

    Returns (path, accept, delta_h); a divergent trajectory or an
    out-of-bounds dH rejects with the +inf sentinel and draws no uniform.
    An accepted path comes back read-only: it mirrors the device's copy, and
    passed back unchanged it is not sent over the link again (np.array(path)
    for a writable copy)."""
    ch = _resolve(backend).chain(data, params)
    h64 = np.ascontiguousarray(h, dtype=np.float64)
    st = stream_state(rng)
    r, h_new = ch.hmc_update_host(h64, st, md.step_size, md.n_steps, fuse_half_steps)
    store_stream_state(rng, st)
    if r.diverged:
        return h, False, DIVERGENT_DELTA_H
    if r.accept:
        return h_new, True, float(r.delta_h)
    return h, False, float(r.delta_h)


# ---- theta full conditionals (host; scalar draws) ---------------------------
# Each update has two forms: the reference signature on a host path h
# (sampler.py:170-272, same formulas), and a `_from_stats` form driven by the
# device statistics of the kept path (what run_chain uses).

def update_mu(h: np.ndarray, params: Params, prior: PriorSpec, rng: np.random.Generator) -> float:
    """sampler.py:170-188."""
    return update_mu_from_stats(path_stats(h, params.mu, 0.0, None), h.shape[0], params.mu, params, prior, rng)


def update_xi(h: np.ndarray, data: Dataset, params: Params, prior: PriorSpec, rng: np.random.Generator) -> float:
    """sampler.py:191-202."""
    st = path_stats(h, 0.0, params.xi, data.log_rv)
    return update_xi_from_stats(st, h.shape[0], params.xi, params, prior, rng)


def _inverse_gamma(rng: np.random.Generator, shape: float, scale: float) -> float:
    return scale / rng.gamma(shape)


def update_sigma_u_sq(h: np.ndarray, data: Dataset, xi: float, prior: PriorSpec, rng: np.random.Generator) -> float:
    """sampler.py:209-215."""
    st = path_stats(h, 0.0, xi, data.log_rv)
    return update_sigma_u_sq_from_stats(st, h.shape[0], xi, xi, prior, rng)


def update_sigma_eta_sq(h: np.ndarray, params: Params, prior: PriorSpec, rng: np.random.Generator) -> float:
    """sampler.py:218-230."""
    st = path_stats(h, params.mu, 0.0, None)
    return update_sigma_eta_sq_from_stats(st, h.shape[0], params.mu, params, prior, rng)


def phi_log_accept_ratio(prop: float, phi: float, h1_sq: float, se2: float, prior: PriorSpec) -> float:
    """sampler.py:233-246."""
    return (0.5 * (math.log1p(-prop * prop) - math.log1p(-phi * phi))
            - h1_sq * ((1.0 - prop * prop) - (1.0 - phi * phi)) / (2.0 * se2)
            + (prior.phi_a - 1.0) * (math.log1p(prop) - math.log1p(phi))
            + (prior.phi_b - 1.0) * (math.log1p(-prop) - math.log1p(-phi)))


def update_phi(h: np.ndarray, params: Params, prior: PriorSpec, rng: np.random.Generator) -> tuple[float, bool]:
    """sampler.py:249-272."""
    st = path_stats(h, params.mu, 0.0, None)
    return update_phi_from_stats(st, h.shape[0], params.mu, params, prior, rng)


def path_stats(h: np.ndarray, c_mu: float, c_xi: float, log_rv) -> np.ndarray:
    """Host statistics of a host path, same layout as rsv_suff_stats (used
    only by the reference-signature wrappers above)."""
    h = np.asarray(h, dtype=np.float64)
    d = h - c_mu
    st = np.zeros(7)
    st[0], st[1] = d[0], d[-1]
    st[2] = float(np.sum(d))
    st[3] = float(np.sum(d * d))
    st[4] = float(np.sum(d[1:] * d[:-1]))
    if log_rv is not None:
        e = np.asarray(log_rv) - h - c_xi
        st[5] = float(np.sum(e))
        st[6] = float(np.sum(e * e))
    return st


def _recentre(st, T, c, mu):
    """Moments of d' = h - mu from moments of d = h - c."""
    delta = mu - c
    d0, dl, s1, s2, sx = st[0], st[1], st[2], st[3], st[4]
    d0n = d0 - delta
    sum_head = (s1 - dl) - (T - 1) * delta          # sum_{t<=T-2} d'
    sum_tail = (s1 - d0) - (T - 1) * delta          # sum_{t>=1} d'
    sxx = (s2 - dl * dl) - 2.0 * delta * (s1 - dl) + (T - 1) * delta * delta    # sum_{t<=T-2} d'^2
    sall = s2 - 2.0 * delta * s1 + T * delta * delta                           # sum d'^2
    sxz = sx - delta * ((s1 - d0) + (s1 - dl)) + (T - 1) * delta * delta        # sum d'_t d'_{t-1}
    return d0n, sum_head, sum_tail, sxx, sall, sxz


def update_mu_from_stats(st, T, c_mu, params: Params, prior: PriorSpec, rng) -> float:
    phi, se2 = params.phi, params.sigma_eta_sq
    prec = ((1.0 - phi * phi) + (T - 1) * (1.0 - phi) ** 2) / se2 + 1.0 / prior.mu_var
    d0, dl, s1 = st[0], st[1], st[2]
    h0 = d0 + c_mu
    trans_sum = (s1 - d0) - phi * (s1 - dl) + (T - 1) * (1.0 - phi) * c_mu   # sum h[1:] - phi h[:-1]
    num = (1.0 - phi * phi) * h0 / se2 + (1.0 - phi) * trans_sum / se2 + prior.mu_mean / prior.mu_var
    if not (math.isfinite(prec) and prec > 0.0):
        raise ValueError(f"degenerate full-conditional precision for mu: {prec}")
    sd = math.sqrt(1.0 / prec)
    return num / prec + sd * rng.standard_normal()


def update_phi_from_stats(st, T, c_mu, params: Params, prior: PriorSpec, rng) -> tuple[float, bool]:
    phi, mu, se2 = params.phi, params.mu, params.sigma_eta_sq
    d0n, _, _, sxx, _, sxz = _recentre(st, T, c_mu, mu)
    sxx = max(sxx, 1e-300)
    phi_hat = sxz / sxx
    sd = math.sqrt(se2 / sxx)
    prop = phi_hat + sd * rng.standard_normal()
    if not -1.0 < prop < 1.0:
        return phi, False
    log_ratio = phi_log_accept_ratio(prop, phi, d0n * d0n, se2, prior)
    u = rng.random()
    if log_ratio >= 0.0 or u < math.exp(log_ratio):
        return prop, True
    return phi, False


def update_sigma_eta_sq_from_stats(st, T, c_mu, params: Params, prior: PriorSpec, rng) -> float:
    phi, mu = params.phi, params.mu
    d0n, _, _, sxx, sall, sxz = _recentre(st, T, c_mu, mu)
    tail_sq = sall - d0n * d0n
    q = (1.0 - phi * phi) * d0n * d0n + (tail_sq - 2.0 * phi * sxz + phi * phi * sxx)
    shape = prior.var_shape + 0.5 * T
    scale = prior.var_scale + 0.5 * q
    return _inverse_gamma(rng, shape, scale)


def update_xi_from_stats(st, T, c_xi, params: Params, prior: PriorSpec, rng) -> float:
    su2 = params.sigma_u_sq
    sum_r = st[5] + T * c_xi   # sum (log_rv - h)
    prec = T / su2 + 1.0 / prior.xi_var
    num = sum_r / su2 + prior.xi_mean / prior.xi_var
    if not (math.isfinite(prec) and prec > 0.0):
        raise ValueError(f"degenerate full-conditional precision for xi: {prec}")
    sd = math.sqrt(1.0 / prec)
    return num / prec + sd * rng.standard_normal()


def update_sigma_u_sq_from_stats(st, T, c_xi, xi, prior: PriorSpec, rng) -> float:
    delta = xi - c_xi
    ss = st[6] - 2.0 * delta * st[5] + T * delta * delta
    shape = prior.var_shape + 0.5 * T
    scale = prior.var_scale + 0.5 * ss
    return _inverse_gamma(rng, shape, scale)


def default_init(data: Dataset) -> tuple[Params, np.ndarray]:
    """sampler.py:275-288."""
    anchor = float(np.mean(data.log_rv))
    h0 = 0.9 * (data.log_rv - anchor)
    params = Params(phi=0.9, mu=float(np.mean(h0)), xi=0.0, sigma_eta_sq=0.1, sigma_u_sq=0.1)
    return params, h0


def run_chain(data: Dataset, config: SamplerConfig, prior: PriorSpec | None = None,
              init_params: Params | None = None, init_h: np.ndarray | None = None, backend=None,
              rng: np.random.Generator | None = None, theta_on: str = "device") -> Chain:
    """sampler.py:291-358 with the path resident on the GPU for the whole run.

    theta_on="device" (default): every sweep -- proposal and the five theta
    draws -- runs on the GPU with no host round trip (rsv_run_chain); the
    draws restate numpy's on the same raw-word stream.  theta_on="host": the
    proposal on the GPU, the theta draws with numpy on the host from the
    device's statistics (also used when the latent paths are stored)."""
    if theta_on not in ("device", "host"):
        raise ValueError(f"theta_on must be 'device' or 'host', got {theta_on!r}")
    prior = prior or PriorSpec()
    params, h = (init_params, init_h)
    if params is None or h is None:
        d_params, d_h = default_init(data)
        params = params or d_params
        h = h if h is not None else d_h
    h = np.asarray(h, dtype=np.float64).copy()
    if h.shape[0] != data.length:
        raise ValueError("initial path length does not match dataset")

    rng = rng if rng is not None else make_rng(config.seed, config.prng)
    n_sweeps = config.n_burnin + config.n_samples * config.thin
    n_store = config.n_samples
    T = data.length

    iters = np.empty(n_store, dtype=np.int64)
    cols = {name: np.empty(n_store) for name in PARAM_NAMES}
    accept = np.empty(n_store, dtype=bool)
    delta_h = np.empty(n_store)
    latent = np.empty((n_store, T)) if config.store_latent else None

    ch = _resolve(backend).chain(data, params)
    ch.set_latent(h)
    if theta_on == "device" and not config.store_latent:
        ch.set_params(params)
        ch.set_stream(stream_state(rng))
        try:
            it, par, acc, dh = ch.run_chain_device(config.md.step_size, config.md.n_steps, False, prior,
                                                   config.n_burnin, n_store, config.thin)
        except N.StormError as e:
            raise DivergenceStormError(
                f"more than {_STORM_LIMIT} of the last {_STORM_WINDOW} HMC proposals diverged at sweep {e.sweep}; "
                f"reduce the step size (current {config.md.step_size})") from None
        finally:
            store_stream_state(rng, ch.get_stream())
        cols = {name: np.ascontiguousarray(par[:, k]) for k, name in
                enumerate(("phi", "mu", "xi", "sigma_eta_sq", "sigma_u_sq"))}
        return Chain(iters=it, accept=acc, delta_h=dh, latent=None, **cols)
    recent: deque[bool] = deque(maxlen=_STORM_WINDOW)
    log_every = max(1, n_sweeps // 10)
    stored = 0
    for sweep in range(n_sweeps):
        ch.set_params(params)
        ch.set_stream(stream_state(rng))
        r = ch.hmc_update(config.md.step_size, config.md.n_steps)
        store_stream_state(rng, ch.get_stream())
        acc = bool(r.accept)
        dh = DIVERGENT_DELTA_H if r.diverged else float(r.delta_h)
        recent.append(math.isinf(dh))
        if len(recent) == _STORM_WINDOW and sum(recent) > _STORM_LIMIT:
            raise DivergenceStormError(
                f"{sum(recent)} of the last {_STORM_WINDOW} HMC proposals diverged at sweep {sweep}; "
                f"reduce the step size (current {config.md.step_size})")
        st = ch.last_stats()          # kept path, shifted by (params.mu, params.xi)
        c_mu, c_xi = params.mu, params.xi
        params = replace(params, mu=update_mu_from_stats(st, T, c_mu, params, prior, rng))
        new_phi, _ = update_phi_from_stats(st, T, c_mu, params, prior, rng)
        params = replace(params, phi=new_phi)
        params = replace(params, sigma_eta_sq=update_sigma_eta_sq_from_stats(st, T, c_mu, params, prior, rng))
        params = replace(params, xi=update_xi_from_stats(st, T, c_xi, params, prior, rng))
        params = replace(params, sigma_u_sq=update_sigma_u_sq_from_stats(st, T, c_xi, params.xi, prior, rng))

        if sweep >= config.n_burnin and (sweep - config.n_burnin) % config.thin == 0:
            iters[stored] = sweep
            for name in PARAM_NAMES:
                cols[name][stored] = getattr(params, name)
            accept[stored] = acc
            delta_h[stored] = dh
            if latent is not None:
                ch.get_latent(latent[stored])
            stored += 1
        if (sweep + 1) % log_every == 0:
            logger.info("sweep %d/%d", sweep + 1, n_sweeps)
    return Chain(iters=iters, accept=accept, delta_h=delta_h, latent=latent, **cols)
