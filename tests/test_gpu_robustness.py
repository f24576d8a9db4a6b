"""GPU tests of the failure paths: non-finite states flag divergence
(_kernels.py:50-51), a divergence storm in the device run_chain stops exactly
where the reference raises (sampler.py:329-337), returned paths are never
recycled while referenced, and data edits reach the device."""
import gc
import math

import numpy as np
import pytest

import oracle as O
import paper_1603_08114_b200 as P
from conftest import TRUE

pytestmark = pytest.mark.gpu
THETA = P.Params(**TRUE)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf, 1e200])
def test_nonfinite_or_huge_momenta_flag_divergence(backend, bad):
    # the reference flags any kick-time h outside [-50, 50] or NaN; here the
    # range test on the exp reduction must also catch NaN / inf / huge states
    tr = P.simulate_rsv(THETA, 3000, seed=4)
    p = np.zeros(3000)
    p[1234] = bad
    for L in (1, 7, 20):
        _, div = P.integrate_trajectory(P.PhaseState(tr.latent, p), P.MDConfig(0.02, L), THETA, tr.dataset,
                                        backend=backend)
        assert div, (bad, L)
    rng = P.make_rng(3, "pcg32")
    pos = P.stream_state(rng).pos
    h = tr.latent.copy()
    h[10] = bad
    h2, acc, dh = P.hmc_update_volatility(h, THETA, tr.dataset, P.MDConfig(0.02, 20), rng, backend=backend)
    assert not acc and math.isinf(dh) and h2 is h
    assert P.stream_state(rng).pos - pos < 3000 * 1.1  # momenta only: no uniform drawn


@pytest.mark.parametrize("kind", ["pcg32", "sfc64"])
def test_device_run_chain_storm_stops_like_the_reference(backend, kind):
    # every proposal diverges (huge step): the storm fires at sweep 99; the
    # device run must raise there with the generator exactly where the
    # host-driven (reference-ordered) run leaves it -- no theta draws on the
    # storm sweep, nothing after it
    tr = P.simulate_rsv(THETA, 256, seed=2)
    cfg = P.SamplerConfig(seed=7, md=P.MDConfig(2.0, 20), n_burnin=0, n_samples=300, prng=kind)
    states = {}
    for theta_on in ("host", "device"):
        rng = P.make_rng(7, kind)
        with pytest.raises(P.DivergenceStormError, match="sweep 99"):
            P.run_chain(tr.dataset, cfg, backend=backend, init_params=THETA, init_h=tr.latent, rng=rng,
                        theta_on=theta_on)
        st = P.stream_state(rng)
        states[theta_on] = (int(st.pos), [int(x) for x in st.s])
    assert states["host"] == states["device"]
    # the context works normally afterwards (the stop is re-armed)
    ch = backend.chain(tr.dataset, THETA)
    ch.set_latent(tr.latent)
    r = ch.hmc_update(0.02, 20)
    assert not r.diverged


def test_returned_paths_are_not_recycled_while_referenced(backend):
    T = 1 << 16
    tr = P.simulate_rsv(THETA, T, seed=6)
    ch = backend.chain(tr.dataset, THETA)
    ch.set_latent(tr.latent)
    held = [ch.get_latent() for _ in range(5)]   # more than the pool holds
    addrs = {a.ctypes.data for a in held}
    assert len(addrs) == 5
    for a in held:
        assert np.array_equal(a, tr.latent)
    sub = held[0][100:200]                        # a derived view keeps its buffer alive
    base_addr = held[0].ctypes.data
    del held[0]
    gc.collect()
    again = [ch.get_latent() for _ in range(4)]
    assert base_addr not in {a.ctypes.data for a in again}
    assert np.array_equal(sub, tr.latent[100:200])
    del sub, again
    gc.collect()
    assert ch.get_latent().ctypes.data in addrs   # buffers come back once nothing refers to them


def test_data_edits_reach_the_device(backend):
    T = 2000
    tr = P.simulate_rsv(THETA, T, seed=8)
    data = tr.dataset
    with pytest.raises(ValueError):
        data.returns[3] = 1.0                     # frozen: no silent in-place edit
    lp0 = P.log_posterior(tr.latent, THETA, data, backend=backend)
    y = np.array(data.returns)
    y[3] = 0.5
    data.returns = y                              # writable array: uploaded on every call
    lp1 = P.log_posterior(tr.latent, THETA, data, backend=backend)
    y[4] = 0.7                                    # in-place edit of the writable array
    lp2 = P.log_posterior(tr.latent, THETA, data, backend=backend)
    assert lp0 != lp1 and lp1 != lp2
    ref = P.log_posterior(tr.latent, THETA, P.Dataset(returns=y, rv=data.rv), backend=backend)
    assert lp2 == ref


# ---------------------------------------------------------------- inter-CTA protocols under contention
@pytest.mark.parametrize("T", [300007, 1 << 20, 3000017])
def test_momenta_exact_while_other_kernels_hold_the_sms(backend, T):
    """The momenta draw's look-back (decoupled, by scheduling ticket) must
    make progress and stay bit-exact when its grid cannot be co-resident
    because other kernels occupy the SMs (long matmuls on another stream are
    launched right before every draw).  compute-sanitizer is closed on this
    pool; this and the checked build (tools/checked_run.sh) exercise the
    protocols instead."""
    import torch
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.float64)
    for kind in ("pcg32", "philox"):
        st = O.Stream(kind, T + 1)
        want = st.normals(T)
        rng = P.make_rng(T + 1, kind)
        with torch.cuda.stream(side):
            for _ in range(3):
                a = (a @ a) * 1e-3
        got = P.refresh_momenta(rng, T, backend=backend)
        torch.cuda.synchronize()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), kind


def test_trajectory_tiles_exact_while_other_kernels_hold_the_sms(backend):
    """Dynamic tile scheduling and the fixed-point totals under contention:
    proposals with a concurrent FP64 matmul equal the oracle's."""
    import torch
    T, L, n = 1 << 18, 20, 4
    truth = P.simulate_rsv(THETA, T, seed=21)
    y, lrv = truth.dataset.returns, truth.dataset.log_rv
    ch = backend.chain(truth.dataset, THETA)
    ch.set_latent(truth.latent)
    ch.set_stream(P.stream_state(P.make_rng(3, "pcg32")))
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.float64)
    st = O.Stream("pcg32", 3)
    h = truth.latent.copy()
    H = abs(O.hamiltonian(h, np.zeros(T), THETA, y, lrv)) + T
    for i in range(n):
        with torch.cuda.stream(side):
            a = (a @ a) * 1e-3
        r = ch.hmc_update(0.02, L)
        h, acc, dh = O.hmc_update(h, THETA, y, lrv, 0.02, L, st, nthreads=O.max_threads())
        assert bool(r.accept) == acc and abs(r.delta_h - dh) <= 1e-13 * H, i
    torch.cuda.synchronize()
    assert np.max(np.abs(ch.get_latent() - h)) <= 1e-12 * np.max(np.abs(h))


@pytest.mark.parametrize("T", [4096, 1 << 16])
@pytest.mark.parametrize("kind", ["pcg32", "philox", "sfc64", "minstd"])
def test_returned_path_stays_resident_and_matches_the_oracle(backend, T, kind):
    # a chain loop passing the returned path back (sampler.py:327-344 does):
    # after the first accept the proposal runs from the device's copy (only
    # the stream state crosses the link); every step equals the oracle's, the
    # returned path cannot be made writable, and any other call that moves
    # the device's path (here set_latent) makes the next call read the host
    # path again
    truth = P.simulate_rsv(THETA, T, seed=21)
    data = truth.dataset
    md = P.MDConfig(0.02, 20)
    rng = P.make_rng(6, kind)
    st = O.Stream(kind, 6)
    h_gpu, h_orc = truth.latent.copy(), truth.latent.copy()
    H = abs(O.hamiltonian(h_orc, np.zeros(T), THETA, data.returns, data.log_rv)) + T
    ch = backend.chain(data, THETA)
    seen_resident = link = False  # link: the device holds the path last returned
    for i in range(16):
        if i == 10:
            ch.set_latent(np.zeros(T))  # the device's path moves: the link is dropped
            link = False
        h_gpu, acc, dh = P.hmc_update_volatility(h_gpu, THETA, data, md, rng, backend=backend)
        assert ch.last_update_resident == link, i
        seen_resident |= link
        link = bool(acc) or link
        h_orc, acc_o, dh_o = O.hmc_update(h_orc, THETA, data.returns, data.log_rv, md.step_size, md.n_steps, st,
                                          nthreads=O.max_threads())
        assert acc == acc_o and abs(dh - dh_o) <= 1e-13 * H, (i, dh, dh_o)
        assert np.max(np.abs(h_gpu - h_orc)) <= 1e-10 * max(1.0, np.max(np.abs(h_orc))), i
        if acc:
            assert not h_gpu.flags.writeable
            with pytest.raises(ValueError):
                h_gpu.flags.writeable = True
            with pytest.raises(ValueError):
                h_gpu[:1].flags.writeable = True
    assert seen_resident
    assert int(rng.bit_generator.random_raw()) == int(st.raw(1)[0])
    # a writable copy of a returned path is the caller's own: read from the host
    hc = np.array(h_gpu)
    P.hmc_update_volatility(hc, THETA, data, md, rng, backend=backend)
    assert not ch.last_update_resident


@pytest.mark.parametrize("head", [None, "8", "40000", str(1 << 17)])
def test_zero_copy_with_copied_head_matches_the_oracle(monkeypatch, head):
    # a page-locked path sent every step (a view of the returned array is not
    # the chain's own): the copy engine brings the path's head in beside the
    # momenta kernel and the trajectory kernel reads the rest in place; any
    # head size (none, one group, mid-tile, the whole path) gives the oracle's
    # decisions and paths
    import torch
    if head is None:
        monkeypatch.delenv("RSV_ZC_HEAD", raising=False)
    else:
        monkeypatch.setenv("RSV_ZC_HEAD", head)
    T = 1 << 17
    truth = P.simulate_rsv(THETA, T, seed=8)
    data = truth.dataset
    md = P.MDConfig(0.02, 20)
    rng = P.make_rng(9, "pcg32")
    st = O.Stream("pcg32", 9)
    h_gpu = torch.empty(T, dtype=torch.float64, pin_memory=True).numpy()
    h_gpu[:] = truth.latent
    h_orc = truth.latent.copy()
    H = abs(O.hamiltonian(h_orc, np.zeros(T), THETA, data.returns, data.log_rv)) + T
    with P.CudaBackend(0) as be:
        n_acc = 0
        for i in range(6):
            h_gpu, acc, dh = P.hmc_update_volatility(h_gpu.view(), THETA, data, md, rng, backend=be)
            ch = be.chain(data, THETA)
            assert ch.last_update_zero_copy and not ch.last_update_resident, i
            h_orc, acc_o, dh_o = O.hmc_update(h_orc, THETA, data.returns, data.log_rv, md.step_size, md.n_steps,
                                              st, nthreads=O.max_threads())
            assert acc == acc_o and abs(dh - dh_o) <= 1e-13 * H, (i, dh, dh_o)
            assert np.max(np.abs(h_gpu - h_orc)) <= 1e-10 * max(1.0, np.max(np.abs(h_orc))), i
            n_acc += acc
    assert int(rng.bit_generator.random_raw()) == int(st.raw(1)[0])
