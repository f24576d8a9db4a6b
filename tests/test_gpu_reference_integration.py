"""The unmodified reference (`rsvhmc`, installed into baseline/_ref) driven
through this package's CudaBackend -- INTEGRATION.md levels 1 and 2 -- against
the reference's own SerialBackend run on the same seeds.

Level 1: rsvhmc.run_chain(..., backend=CudaBackend()) -- the reference's
kernel protocol (integrator.py:50-105, :111-146) executes its three kernels
on the GPU.  Level 2: the two-line hook of INTEGRATION.md (sampler.py:144)
applied to the reference at run time; every proposal is one fused launch.

Bars: the chains agree to 1e-9 relative in every parameter and have the same
accept flags (momentum_update differs from numba only through exp, the
fused trajectory by rounding).  Skipped, with the reason, only when the
reference cannot be imported (no baseline/_ref or no numba)."""
import os
import sys

import numpy as np
import pytest

import paper_1603_08114_b200 as P

pytestmark = pytest.mark.gpu
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def rsvhmc():
    if not os.path.isdir(os.path.join(REF, "rsvhmc")):
        pytest.skip("reference not installed in baseline/_ref (DESIGN.md 5)")
    sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rsvhmc_numba_cache")
    try:
        import rsvhmc as R
    except ImportError as e:  # numba / numpy missing
        pytest.skip(f"reference not importable: {e}")
    assert os.path.abspath(R.__file__).startswith(REF)
    return R


def _setup(R, T=300, seed=2):
    theta = R.Params(phi=0.97, mu=-9.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)
    truth = R.simulate_rsv(theta, T, seed=seed)
    cfg = R.SamplerConfig(seed=4, md=R.MDConfig(0.02, 20), n_burnin=2, n_samples=10)
    return theta, truth, cfg


def _compare(a, b):
    for name in ("phi", "mu", "xi", "sigma_eta_sq", "sigma_u_sq"):
        np.testing.assert_allclose(getattr(a, name), getattr(b, name), rtol=1e-9, atol=0, err_msg=name)
    assert np.array_equal(np.asarray(a.accept), np.asarray(b.accept))


def test_level1_reference_run_chain_with_cuda_kernels(rsvhmc):
    R = rsvhmc
    theta, truth, cfg = _setup(R)
    ref = R.run_chain(truth.dataset, cfg, init_params=theta, init_h=truth.latent)
    with P.CudaBackend(0) as be:
        got = R.run_chain(truth.dataset, cfg, init_params=theta, init_h=truth.latent, backend=be)
    _compare(got, ref)


def test_level2_hook_runs_fused_proposals(rsvhmc, monkeypatch):
    R = rsvhmc
    import rsvhmc.sampler as RS
    theta, truth, cfg = _setup(R)
    ref = R.run_chain(truth.dataset, cfg, init_params=theta, init_h=truth.latent)
    original = RS.hmc_update_volatility
    calls = []

    def hooked(h, params, data, md, rng, backend=RS.SERIAL):
        # the maintainer's two lines (level 2)
        if hasattr(backend, "hmc_update_volatility"):
            calls.append(1)
            return backend.hmc_update_volatility(h, params, data, md, rng)
        return original(h, params, data, md, rng, backend)

    monkeypatch.setattr(RS, "hmc_update_volatility", hooked)
    with P.CudaBackend(0) as be:
        got = R.run_chain(truth.dataset, cfg, init_params=theta, init_h=truth.latent, backend=be)
    assert len(calls) == cfg.n_burnin + cfg.n_samples * cfg.thin
    _compare(got, ref)
