"""Host-side logic of the package and the C ABI library (no GPU needed)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1603_08114_b200 as P
from conftest import ROOT, golden
from paper_1603_08114_b200 import _native as N


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.lib()
    hdr = open(os.path.join(ROOT, "include", "rsvhmc_b200.h")).read()
    declared = set(re.findall(r"\b(rsv_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 30
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(N.EXPORTED) <= declared | {"rsv_debug_stamps"}
    assert b"sm_100a" in lib.rsv_version()


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    code = N.lib().rsv_create(ctypes.byref(h), 0, 1000)
    assert code == N.RSV_E_CUDA
    assert b"CUDA" in N.lib().rsv_last_error(None) or b"device" in N.lib().rsv_last_error(None)
    with pytest.raises(N.NativeError):
        P.DeviceChain(1000)


@pytest.mark.parametrize("kind", ["philox", "minstd", "pcg32", "sfc64"])
def test_host_bit_generators_match_oracle(kind):
    z = golden("prng.npz")
    g = P.make_rng(12345, kind)
    got = g.standard_normal(4096)
    assert np.array_equal(got.view(np.uint64), z[f"normal_{kind}_12345"].view(np.uint64))
    if kind in ("minstd", "pcg32"):
        bg = P.RsvBitGenerator(kind, 1)
        assert np.array_equal(bg.random_raw(64), z[f"raw_{kind}_1"])


@pytest.mark.parametrize("kind", ["philox", "sfc64", "minstd", "pcg32"])
def test_stream_state_roundtrip(kind):
    rng = P.make_rng(3, kind)
    rng.standard_normal(77)
    st = P.stream_state(rng)
    ref = O.Stream(kind, 3)
    ref.normals(77)
    s, pos = ref.state_words()
    if kind == "sfc64":
        assert [int(x) for x in st.s] == s
    else:
        assert int(st.pos) == pos
    # advance by hand and write back: the Generator continues from there
    for extra in (1, 2, 3, 4, 5, 9):
        rng2 = P.make_rng(3, kind)
        rng2.standard_normal(77)
        st2 = P.stream_state(rng2)
        if kind == "sfc64":
            continue
        st2.pos += extra
        P.store_stream_state(rng2, st2)
        r3 = O.Stream(kind, 3)
        r3.normals(77)
        r3.raw(extra)
        assert rng2.random() == r3.next_double()


def test_params_and_dataset_validation():
    with pytest.raises(ValueError):
        P.Params(1.0, 0, 0, 1, 1)
    with pytest.raises(ValueError):
        P.Params(0.5, 0, 0, 0.0, 1)
    with pytest.raises(ValueError):
        P.Dataset(returns=np.zeros(1), rv=np.ones(1))
    with pytest.raises(ValueError):
        P.Dataset(returns=np.zeros(3), rv=np.array([1.0, -1.0, 1.0]))
    with pytest.raises(ValueError):
        P.PhaseState(np.zeros(4), np.zeros(5))
    with pytest.raises(ValueError):
        P.MDConfig(0.0, 5)
    with pytest.raises(ValueError):
        P.SamplerConfig(n_samples=0)


def test_simulate_rsv_matches_reference_fixture():
    z = golden("model_T2000.npz")
    theta = P.Params(*[float(v) for v in z["theta"]])
    tr = P.simulate_rsv(theta, 2000, seed=0)
    assert np.array_equal(tr.latent, z["h_true"])
    assert np.array_equal(tr.dataset.returns, z["y"])
    assert np.array_equal(tr.dataset.log_rv, z["lrv"])


def _ref_updates(h, lrv, params, prior, rng):
    """sampler.py:170-230 restated with numpy sums (test oracle)."""
    phi, se2 = params.phi, params.sigma_eta_sq
    T = h.size
    prec = ((1.0 - phi * phi) + (T - 1) * (1.0 - phi) ** 2) / se2 + 1.0 / prior.mu_var
    num = ((1.0 - phi * phi) * h[0] / se2 + (1.0 - phi) * float(np.sum(h[1:] - phi * h[:-1])) / se2
           + prior.mu_mean / prior.mu_var)
    mu = num / prec + math.sqrt(1.0 / prec) * rng.standard_normal()
    d = h - mu
    q = (1.0 - phi * phi) * d[0] * d[0] + float(np.sum((d[1:] - phi * d[:-1]) ** 2))
    se2n = (prior.var_scale + 0.5 * q) / rng.gamma(prior.var_shape + 0.5 * T)
    r = lrv - h
    prec = T / params.sigma_u_sq + 1.0 / prior.xi_var
    xi = (float(np.sum(r)) / params.sigma_u_sq + prior.xi_mean / prior.xi_var) / prec + \
        math.sqrt(1.0 / prec) * rng.standard_normal()
    resid = lrv - xi - h
    su2 = (prior.var_scale + 0.5 * float(np.sum(resid * resid))) / rng.gamma(prior.var_shape + 0.5 * T)
    return mu, se2n, xi, su2


def test_theta_updates_from_statistics_match_direct_sums():
    z = golden("chain_pcg32.npz")
    h = z["latent_last"]
    lrv = z["lrv"]
    params = P.Params(0.95, -1.0, -0.3, 0.05, 0.1)
    prior = P.PriorSpec()
    T = h.size
    # statistics shifted by the *old* (mu, xi), then re-centred inside the updates
    st = O.suff_stats(h, lrv, params.mu, params.xi)
    g1, g2 = P.make_rng(4), P.make_rng(4)
    mu = P.sampler.update_mu_from_stats(st, T, params.mu, params, prior, g1)
    p1 = P.Params(params.phi, mu, params.xi, params.sigma_eta_sq, params.sigma_u_sq)
    se2 = P.sampler.update_sigma_eta_sq_from_stats(st, T, params.mu, p1, prior, g1)
    p2 = P.Params(params.phi, mu, params.xi, se2, params.sigma_u_sq)
    xi = P.sampler.update_xi_from_stats(st, T, params.xi, p2, prior, g1)
    su2 = P.sampler.update_sigma_u_sq_from_stats(st, T, params.xi, xi, prior, g1)
    want = _ref_updates(h, lrv, params, prior, g2)
    assert np.allclose([mu, se2, xi, su2], want, rtol=1e-11, atol=0)


def test_phi_update_from_statistics():
    z = golden("chain_pcg32.npz")
    h = z["latent_last"]
    params = P.Params(0.9, -1.02, -0.3, 0.05, 0.1)
    prior = P.PriorSpec()
    st = O.suff_stats(h, z["lrv"], -1.0, 0.0)   # shifted by a different centre
    a = P.sampler.update_phi_from_stats(st, h.size, -1.0, params, prior, P.make_rng(8))
    b = P.update_phi(h, params, prior, P.make_rng(8))
    assert a[1] == b[1] and abs(a[0] - b[0]) <= 1e-12


def test_prior_and_config_defaults_mirror_reference():
    pr = P.PriorSpec()
    assert (pr.mu_var, pr.var_shape, pr.var_scale, pr.phi_a, pr.phi_b) == (100.0, 2.5, 0.025, 20.0, 1.5)
    cfg = P.SamplerConfig()
    assert cfg.md.step_size == 0.02 and cfg.md.n_steps == 50


def test_ensemble_seeding_is_numpy_seedsequence():
    st = P.sfc64_states(5, 3)
    for c in range(3):
        want = np.random.SFC64(np.random.SeedSequence([5, c])).state["state"]["state"]
        assert [int(x) for x in st[c]] == [int(x) for x in want]


def test_protocol_fit_matches_reference_formulas():
    from paper_1603_08114_b200 import bench_protocol as BP
    pts = [(1, 3.0), (2, 5.0), (4, 9.0)]
    f = BP.fit_linear(pts)
    assert abs(f.intercept_a - 1.0) < 1e-12 and abs(f.slope_c - 2.0) < 1e-12 and abs(f.r_squared - 1.0) < 1e-12
    slow = BP.TimingFit(0.0, 10.0, 1.0)
    assert abs(BP.compute_gain(slow, f, 4) - 40.0 / 9.0) < 1e-12
    assert abs(BP.asymptotic_gain(slow, f) - 5.0) < 1e-12
    with pytest.raises(BP.NumericError):
        BP.fit_linear([(2, 1.0), (2, 2.0)])


def test_dataset_arrays_are_private_and_read_only():
    # a device context reuses its upload only while the data cannot change
    # (integrator.DeviceChain.set_data); the caller's arrays stay writable
    import paper_1603_08114_b200 as P
    from paper_1603_08114_b200.model import is_frozen
    y = np.linspace(-0.01, 0.01, 16)
    rv = np.full(16, 1e-4)
    d = P.Dataset(returns=y, rv=rv)
    assert is_frozen(d.returns) and is_frozen(d.rv) and is_frozen(d.log_rv)
    assert y.flags.writeable and d.returns is not y
    y[0] = 1.0                       # the caller's array is not aliased
    assert d.returns[0] == -0.01
    with pytest.raises(ValueError):
        d.log_rv[0] = 0.0
    assert not is_frozen(np.zeros(3)) and not is_frozen(np.zeros(3)[1:])
    v = np.zeros(3)
    ro = v[:]
    ro.setflags(write=False)
    assert not is_frozen(ro)         # a read-only view of a writable base can still change


def test_read_only_lease_cannot_be_made_writable():
    # a returned path is an array over a read-only lease of a pooled buffer:
    # neither it nor any view of it can be made writable, which is what lets
    # hmc_update_host trust that a path passed back is the one the device holds
    import gc
    import weakref
    from paper_1603_08114_b200.integrator import _Lease
    buf = np.arange(16, dtype=np.float64)
    lease = _Lease(buf, readonly=True)
    a = np.asarray(lease)
    assert a.base is lease and not a.flags.writeable and a.ctypes.data == buf.ctypes.data
    for v in (a, a[:4], a.view(), a.reshape(4, 4)):
        with pytest.raises(ValueError):
            v.flags.writeable = True
        with pytest.raises(ValueError):
            v[0] = 1.0
    assert a.view().base is a  # a view is not the returned array itself
    w = np.asarray(_Lease(buf))  # the writable hand-out (get_latent)
    assert w.flags.writeable
    # the lease lives as long as any array over it
    ref = weakref.ref(lease)
    v = a[2:]
    del a, lease
    gc.collect()
    assert ref() is not None and v[0] == 2.0
    del v
    gc.collect()
    assert ref() is None
