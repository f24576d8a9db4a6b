"""GPU parity: the CUDA path (through the C ABI) against the golden fixtures
produced by the reference itself and against the CPU oracle.

Tolerances: PRNG words and normals bit-exact; trajectories
<= 1e-12 relative; H and dH <= 1e-13 |H| absolute (the reference's own dH
error is ~3e-16 |H|, so no exact implementation can beat this bound);
accept sequences identical."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1603_08114_b200 as P
from conftest import TRUE, golden

pytestmark = pytest.mark.gpu

THETA = P.Params(**TRUE)


def _data_T2000():
    z = golden("model_T2000.npz")
    return z, P.Dataset.from_log_rv(z["y"], z["lrv"])


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


# ---------------------------------------------------------------- momenta
@pytest.mark.parametrize("kind", ["philox", "minstd", "pcg32", "sfc64"])
@pytest.mark.parametrize("seed", [0, 1, 12345])
def test_momenta_bit_exact_vs_numpy(backend, kind, seed):
    z = golden("prng.npz")
    want = z[f"normal_{kind}_{seed}"]
    rng = P.make_rng(seed, kind)
    got = P.refresh_momenta(rng, want.size, backend=backend)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    # the generator continues where numpy's would be after standard_normal(n)
    st = O.Stream(kind, seed)
    st.normals(want.size)
    _same_position(rng, st)


def _same_position(rng, st):
    got = P.stream_state(rng)
    s, pos = st.state_words()
    if st.kind == "sfc64":   # numpy's SFC64 state carries no counter: compare the words
        assert [int(x) for x in got.s] == s
    else:
        assert int(got.pos) == pos


def test_momenta_numpy_philox_object_is_continued(backend):
    z = golden("prng.npz")
    rng = np.random.Generator(np.random.Philox(7))
    got = P.refresh_momenta(rng, 8192, backend=backend)
    assert np.array_equal(got, z["np_philox_normal_7"])
    ref = np.random.Generator(np.random.Philox(7))
    ref.standard_normal(8192)
    assert rng.random() == ref.random()          # stream state written back exactly


def test_momenta_with_tail_draws(backend):
    z = golden("prng.npz")
    want = z["normal_philox_2024"]
    assert len(z["tail_word_idx_philox_2024"]) >= 10   # exponential-tail attempts inside
    got = P.refresh_momenta(P.make_rng(2024), want.size, backend=backend)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("T", [2, 3, 7, 2047, 2048, 2049, 100003, 1 << 20, 3000017])
def test_momenta_sizes_vs_oracle(backend, T):
    # 126 K .. 1.16 M normals use the co-resident grid's publication count,
    # longer draws the decoupled look-back (3000017)
    for kind in ("pcg32", "sfc64"):
        st = O.Stream(kind, T)
        want = st.normals(T)
        rng = P.make_rng(T, kind)
        got = P.refresh_momenta(rng, T, backend=backend)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), kind
        _same_position(rng, st)


# ---------------------------------------------------------------- model
def test_log_posterior_and_hamiltonian(backend):
    z, data = _data_T2000()
    h, p = z["h_true"], z["p0"]
    lp = P.log_posterior(h, THETA, data, backend=backend)
    assert abs(lp - float(z["log_post"])) <= 1e-13 * abs(float(z["log_post"]))
    H = P.hamiltonian(P.PhaseState(h, p), THETA, data, backend=backend)
    assert abs(H - float(z["ham"])) <= 1e-13 * abs(float(z["ham"]))


def test_gradient(backend):
    z, data = _data_T2000()
    g = P.grad_neg_log_posterior(z["h_true"], THETA, data, backend=backend)
    assert _rel(g, z["grad"]) <= 1e-14


# ---------------------------------------------------------------- integrator
@pytest.mark.parametrize("fuse", [False, True])
def test_trajectory_vs_reference(backend, fuse):
    z, data = _data_T2000()
    st = P.PhaseState(z["h_true"].copy(), z["p0"].copy())
    fin, div = P.integrate_trajectory(st, P.MDConfig(0.02, 20), THETA, data, backend=backend,
                                      fuse_half_steps=fuse)
    assert not div
    assert _rel(fin.h, z[f"traj_h_fuse{int(fuse)}"]) <= 1e-12
    assert _rel(fin.p, z[f"traj_p_fuse{int(fuse)}"]) <= 1e-12
    assert np.array_equal(st.h, z["h_true"])  # input untouched (integrator.py:160 copy)


def test_elementary_step_vs_reference(backend):
    z, data = _data_T2000()
    st = P.PhaseState(z["h_true"].copy(), z["p0"].copy())
    _, div = P.elementary_step(st, P.MDConfig(0.02, 1), THETA, data, backend=backend)
    assert not div
    assert _rel(st.h, z["estep_h"]) <= 1e-14
    assert _rel(st.p, z["estep_p"]) <= 1e-14


def test_divergence_flag(backend):
    z, data = _data_T2000()
    st = P.PhaseState(z["h_true"].copy(), np.full(2000, 1e4))
    _, div = P.integrate_trajectory(st, P.MDConfig(0.5, 20), THETA, data, backend=backend)
    assert div == bool(z["div_flag"]) and div


# ---------------------------------------------------------------- HMC proposals
@pytest.mark.parametrize("kind,seed", [("minstd", 1), ("philox", 11)])
def test_hmc_sequence_vs_reference(backend, kind, seed):
    z, data = _data_T2000()
    g = golden(f"hmc_{kind}.npz")
    rng = P.make_rng(seed, kind)
    h = g["h_start"].copy()
    H = abs(float(z["ham"]))
    for i in range(len(g["accept"])):
        h, acc, dh = P.hmc_update_volatility(h, THETA, data, P.MDConfig(0.02, 20), rng, backend=backend)
        want = float(g["delta_h"][i])
        assert abs(dh - want) <= 1e-13 * H, (i, dh, want)
        assert acc == bool(g["accept"][i]), i
        assert P.stream_state(rng).pos == int(g["pos"][i]), i
        if i == 0:
            assert _rel(h, g["h_first"]) <= 1e-10
    assert _rel(h, g["h_last"]) <= 1e-10


@pytest.mark.parametrize("T,kind,pinned", [(300008, "pcg32", True), (1 << 17, "sfc64", True),
                                           (300007, "philox", True), (1 << 17, "pcg32", False)])
def test_zero_copy_host_proposals_vs_oracle(backend, T, kind, pinned):
    # from T = 2^16 a page-locked path (T % 8 == 0) is read in place by the
    # trajectory kernel: same decisions, stream positions and paths as the
    # oracle (and as the copy-in path for pageable or ragged inputs)
    import torch
    truth = P.simulate_rsv(THETA, T, seed=11)
    data = truth.dataset
    md = P.MDConfig(0.02, 20)
    rng = P.make_rng(4, kind)
    st = O.Stream(kind, 4)
    if pinned:
        h_gpu = torch.empty(T, dtype=torch.float64, pin_memory=True).numpy()
        h_gpu[:] = truth.latent
    else:
        h_gpu = truth.latent.copy()
    h_orc = truth.latent.copy()
    H = abs(O.hamiltonian(h_orc, np.zeros(T), THETA, data.returns, data.log_rv)) + T
    accs = []
    for i in range(4):
        # an accepted path comes back read-only and stays on the device: passed
        # back, it is proposed from the device's copy; before that the path is
        # read in place (page-locked) or copied in
        resident = any(accs)
        h_gpu, acc, dh = P.hmc_update_volatility(h_gpu, THETA, data, md, rng, backend=backend)
        ch = backend.chain(data, THETA)
        assert ch.last_update_resident == resident, i
        # (a pageable path is staged into page-locked memory by host threads first)
        assert ch.last_update_zero_copy == (not resident and T % 8 == 0), i
        h_orc, acc_o, dh_o = O.hmc_update(h_orc, THETA, data.returns, data.log_rv, md.step_size, md.n_steps, st,
                                          nthreads=O.max_threads())
        assert acc == acc_o and abs(dh - dh_o) <= 1e-13 * H, (i, dh, dh_o)
        assert _rel(h_gpu, h_orc) <= 1e-10, i
        accs.append(acc)
    assert int(rng.bit_generator.random_raw()) == int(st.raw(1)[0])
    assert any(accs)


def test_hmc_divergent_sentinel(backend):
    g = golden("hmc_divergent.npz")
    data = P.Dataset.from_log_rv(g["y"], g["lrv"])
    rng = P.make_rng(9, "pcg32")
    for i in range(3):
        h, acc, dh = P.hmc_update_volatility(g["h"].copy(), THETA, data, P.MDConfig(0.9, 30), rng, backend=backend)
        assert not acc and math.isinf(dh)
    assert P.stream_state(rng).pos == int(g["pos"])   # no uniform drawn on divergence


# ---------------------------------------------------------------- chains
@pytest.mark.parametrize("kind,seed", [("pcg32", 3), ("philox", 5)])
@pytest.mark.parametrize("theta_on", ["host", "device"])
def test_run_chain_vs_reference(backend, kind, seed, theta_on):
    # the reference's own chain (tests/golden/make_golden.py); with theta_on
    # "device" every sweep, theta draws included, runs on the GPU
    g = golden(f"chain_{kind}.npz")
    data = P.Dataset.from_log_rv(g["y"], g["lrv"])
    store = theta_on == "host"
    cfg = P.SamplerConfig(seed=seed, md=P.MDConfig(0.05, 10), n_burnin=0, n_samples=len(g["accept"]), thin=1,
                          store_latent=store, prng=kind)
    ch = P.run_chain(data, cfg, backend=backend, theta_on=theta_on)
    assert np.array_equal(ch.accept, g["accept"])
    for name in ("phi", "mu", "xi", "sigma_eta_sq", "sigma_u_sq"):
        assert np.allclose(getattr(ch, name), g[name], rtol=1e-9, atol=1e-12), name
    if store:
        assert _rel(ch.latent[-1], g["latent_last"]) <= 1e-9
    else:
        assert _rel(backend.chain(data, THETA).get_latent(), g["latent_last"]) <= 1e-9


@pytest.mark.parametrize("kind", ["minstd", "sfc64"])
def test_run_chain_device_theta_equals_host_theta(backend, kind):
    z = golden("model_T2000.npz")
    data = P.Dataset.from_log_rv(z["y"], z["lrv"])
    cfg = P.SamplerConfig(seed=4, md=P.MDConfig(0.02, 20), n_burnin=10, n_samples=40, thin=2, prng=kind)
    a = P.run_chain(data, cfg, backend=backend, theta_on="host")
    b = P.run_chain(data, cfg, backend=backend, theta_on="device")
    assert np.array_equal(a.iters, b.iters) and np.array_equal(a.accept, b.accept)
    for name in ("phi", "mu", "xi", "sigma_eta_sq", "sigma_u_sq"):
        assert np.allclose(getattr(a, name), getattr(b, name), rtol=1e-11, atol=1e-13), name
    fin = np.isfinite(a.delta_h)
    assert np.array_equal(fin, np.isfinite(b.delta_h))
    assert np.allclose(a.delta_h[fin], b.delta_h[fin], rtol=1e-8, atol=1e-9)


# ---------------------------------------------------------------- large-T properties
def test_large_T_reversibility_and_determinism(backend):
    T = 1 << 20
    truth = P.simulate_rsv(THETA, T, seed=5)
    data = truth.dataset
    p = P.refresh_momenta(P.make_rng(6, "pcg32"), T, backend=backend)
    md = P.MDConfig(0.02, 20)
    fwd, div = P.integrate_trajectory(P.PhaseState(truth.latent, p), md, THETA, data, backend=backend)
    assert not div
    fwd2, _ = P.integrate_trajectory(P.PhaseState(truth.latent, p), md, THETA, data, backend=backend)
    assert np.array_equal(fwd.h, fwd2.h) and np.array_equal(fwd.p, fwd2.p)
    back, _ = P.integrate_trajectory(P.PhaseState(fwd.h, -fwd.p), md, THETA, data, backend=backend)
    assert np.max(np.abs(back.h - truth.latent)) <= 1e-9
    assert np.max(np.abs(-back.p - p)) <= 1e-9
    # a window of the large trajectory against the oracle (sites far from edges
    # only depend on a 2L+1 neighbourhood, so a slice with margins suffices)
    lo, hi = 300000, 300000 + 4096
    m = 64
    hh, pp, _ = O.integrate(truth.latent[lo - m:hi + m], p[lo - m:hi + m], THETA, data.returns[lo - m:hi + m],
                            data.log_rv[lo - m:hi + m], 0.02, 20)
    assert _rel(fwd.h[lo:hi], hh[m:-m]) <= 1e-12
    assert _rel(fwd.p[lo:hi], pp[m:-m]) <= 1e-12


@pytest.mark.parametrize("T", [2, 3, 5, 41, 42, 43, 2006, 2007, 4096, 65537])
@pytest.mark.parametrize("L", [1, 3, 20])
def test_trajectory_edge_sizes_vs_oracle(backend, T, L):
    truth = P.simulate_rsv(THETA, T, seed=T)
    data = truth.dataset
    p = O.Stream("pcg32", T + L).normals(T)
    fin, div = P.integrate_trajectory(P.PhaseState(truth.latent, p), P.MDConfig(0.02, L), THETA, data,
                                      backend=backend)
    hh, pp, dd = O.integrate(truth.latent, p, THETA, data.returns, data.log_rv, 0.02, L)
    assert div == dd
    assert _rel(fin.h, hh) <= 1e-12 and _rel(fin.p, pp) <= 1e-12


def test_long_trajectory_streamed_fallback(backend):
    # n_steps beyond one tile's halo budget runs one streamed step per launch
    T = 3000
    truth = P.simulate_rsv(THETA, T, seed=1)
    p = O.Stream("philox", 3).normals(T)
    fin, div = P.integrate_trajectory(P.PhaseState(truth.latent, p), P.MDConfig(0.002, 900), THETA,
                                      truth.dataset, backend=backend)
    hh, pp, dd = O.integrate(truth.latent, p, THETA, truth.dataset.returns, truth.dataset.log_rv, 0.002, 900)
    assert div == dd
    assert _rel(fin.h, hh) <= 1e-11


@pytest.mark.parametrize("kind,seed", [("pcg32", 2), ("sfc64", 7)])
def test_long_trajectory_hmc_proposals_vs_oracle(backend, kind, seed):
    # L beyond a tile's halo budget: the proposal graph streams the steps
    # (momenta, energies, L step kernels, Metropolis) -- same draws and decisions
    T = 3000
    truth = P.simulate_rsv(THETA, T, seed=2)
    data = truth.dataset
    md = P.MDConfig(0.003, 500)
    rng = P.make_rng(seed, kind)
    st = O.Stream(kind, seed)
    h_gpu = truth.latent.copy()
    h_orc = truth.latent.copy()
    H = abs(O.hamiltonian(h_orc, np.zeros(T), THETA, data.returns, data.log_rv)) + T
    n_acc = 0
    for i in range(5):
        h_gpu, acc, dh = P.hmc_update_volatility(h_gpu, THETA, data, md, rng, backend=backend)
        h_orc, acc_o, dh_o = O.hmc_update(h_orc, THETA, data.returns, data.log_rv, md.step_size, md.n_steps, st)
        assert acc == acc_o, i
        assert abs(dh - dh_o) <= 1e-12 * H, (i, dh, dh_o)
        assert _rel(h_gpu, h_orc) <= 1e-10, i
        n_acc += acc
    assert n_acc >= 1
    assert int(rng.bit_generator.random_raw()) == int(st.raw(1)[0])   # both streams at the same word


def test_long_trajectory_run_chain_device_equals_host(backend):
    T = 2000
    truth = P.simulate_rsv(THETA, T, seed=8)
    cfg = P.SamplerConfig(seed=3, md=P.MDConfig(0.004, 420), n_burnin=2, n_samples=6, thin=1, prng="minstd")
    a = P.run_chain(truth.dataset, cfg, backend=backend, theta_on="host")
    b = P.run_chain(truth.dataset, cfg, backend=backend, theta_on="device")
    assert np.array_equal(a.accept, b.accept) and a.accept.any()
    for name in ("phi", "mu", "xi", "sigma_eta_sq", "sigma_u_sq"):
        assert np.allclose(getattr(a, name), getattr(b, name), rtol=1e-11, atol=1e-13), name


# ---------------------------------------------------------------- kernel-level plug-in
def test_backend_run_protocol_matches_reference_kernels(backend):
    z, data = _data_T2000()
    h, p = z["h_true"].copy(), z["p0"].copy()
    c = np.float64(0.5) * np.float64(0.02)
    h_ref = h + c * p
    P.kernel1_half_position(P.PhaseState(h, p), 0.02, backend=backend)
    assert np.array_equal(h, h_ref)                       # exact reference arithmetic
    g, _ = O.gradient(h, THETA, data.returns, data.log_rv)
    st = P.PhaseState(h.copy(), p.copy())
    _, div = P.kernel2_momentum(st, 0.02, THETA, data, backend=backend)
    assert not div
    assert _rel(st.p, p - 0.02 * g) <= 1e-14


def test_suff_stats_vs_oracle(backend):
    z, data = _data_T2000()
    ch = backend.chain(data, THETA)
    ch.set_latent(z["h_true"])
    got = ch.suff_stats(-9.0, -0.3)
    want = O.suff_stats(z["h_true"], data.log_rv, -9.0, -0.3)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-9)


# ---------------------------------------------------------------- time sharding
@pytest.mark.parametrize("world,T", [(2, 5000), (3, 70001), (4, 1 << 18)])
def test_sharded_chain_on_one_gpu_matches_single_context(backend, world, T):
    truth = P.simulate_rsv(THETA, T, seed=9)
    data = truth.dataset
    shards = [P.ShardedChain(data, THETA, r, world, margin=32) for r in range(world)]
    st0 = P.stream_state(P.make_rng(21, "pcg32"))
    for c in shards:
        c.set_latent_global(truth.latent)
        c.set_stream(st0)
    single = backend.chain(data, THETA)
    single.set_latent(truth.latent)
    single.set_stream(st0)
    H = abs(P.hamiltonian(P.PhaseState(truth.latent, np.zeros(T)), THETA, data, backend=backend))
    for i in range(8):
        d = P.hmc_update_local(shards, 0.01, 20)
        r = single.hmc_update(0.01, 20)
        assert d.accept == bool(r.accept), i
        if r.diverged:
            assert math.isinf(d.delta_h)
        else:
            # fixed-point group sums: the same dH bits for any world size
            assert d.delta_h == r.delta_h, (i, d.delta_h, r.delta_h)
    h = np.concatenate([c.owned_latent() for c in shards])
    assert np.array_equal(h, single.get_latent())
    assert all(int(c.get_stream().pos) == int(single.get_stream().pos) for c in shards)
    for c in shards:
        c.shard.close()


@pytest.mark.parametrize("world,kind", [(2, "pcg32"), (3, "sfc64"), (4, "philox")])
def test_sharded_device_orchestration_matches_single_context(backend, world, kind):
    # the device-side driver: totals gathered in device memory, decisions on
    # the GPU, margins exchanged only every K proposals (margin >= (K+1)(L+1))
    T, L, n = 20000, 12, 14
    truth = P.simulate_rsv(THETA, T, seed=19)
    data = truth.dataset
    margin = 3 * (L + 1) + 3
    assert P.sharded.halo_period(margin, L) == 2
    shards = [P.ShardedChain(data, THETA, r, world, margin=margin) for r in range(world)]
    st0 = P.stream_state(P.make_rng(23, kind))
    for c in shards:
        c.set_latent_global(truth.latent)
        c.set_stream(st0)
    single = backend.chain(data, THETA)
    single.set_latent(truth.latent)
    single.set_stream(st0)
    res = P.sharded.hmc_update_local_device(shards, 0.02, L, n)
    ref = single.hmc_update_many(0.02, L, n)
    H = abs(P.hamiltonian(P.PhaseState(truth.latent, np.zeros(T)), THETA, data, backend=backend))
    assert [bool(x.accept) for x in res] == [bool(x.accept) for x in ref]
    assert 0 < sum(bool(x.accept) for x in ref) < n  # both outcomes exercised
    for a, b in zip(res, ref):
        if b.diverged:
            assert a.diverged
        else:
            assert a.delta_h == b.delta_h and a.h_old == b.h_old and a.h_new == b.h_new
    h = np.concatenate([c.owned_latent() for c in shards])
    assert np.array_equal(h, single.get_latent())
    for c in shards:
        s, s1 = c.get_stream(), single.get_stream()
        assert int(s.pos) == int(s1.pos) and [int(x) for x in s.s] == [int(x) for x in s1.s]
        c.shard.close()


def test_sharded_distributed_device_driver_nccl_world_of_one(backend):
    # the NCCL path of the device-orchestrated driver (all_gather of totals,
    # decisions on the GPU) with a process group of one rank
    import os
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        T, L, n = 30000, 20, 10
        truth = P.simulate_rsv(THETA, T, seed=29)
        data = truth.dataset
        chain = P.ShardedChain(data, THETA, 0, 1, margin=8 * (L + 1))
        st0 = P.stream_state(P.make_rng(31, "pcg32"))
        chain.set_latent_global(truth.latent)
        chain.set_stream(st0)
        single = backend.chain(data, THETA)
        single.set_latent(truth.latent)
        single.set_stream(st0)
        res = P.sharded.hmc_update_distributed_device(chain, 0.02, L, n)
        ref = single.hmc_update_many(0.02, L, n)
        assert [bool(x.accept) for x in res] == [bool(x.accept) for x in ref]
        for a, b in zip(res, ref):
            assert a.diverged == b.diverged and (b.diverged or abs(a.delta_h - b.delta_h) <= 1e-9)
        assert _rel(chain.owned_latent(), single.get_latent()) <= 1e-12
        chain.shard.close()
    finally:
        if own:
            dist.destroy_process_group()


# ---------------------------------------------------------------- decomposition independence
@pytest.mark.parametrize("fuse", [False, True])
def test_trajectory_bitwise_independent_of_tile_shape(backend, monkeypatch, fuse):
    # the device analogue of test_integrator.py:55 (worker-count independence):
    # every site's update uses only its neighbours with the same operations,
    # so the tile / window shape (RSV_TRAJ_VARIANT, read at context creation)
    # must not change a single bit of h' or p'
    from paper_1603_08114_b200.integrator import DeviceChain
    T = 50021
    truth = P.simulate_rsv(THETA, T, seed=13)
    p = O.Stream("pcg32", 17).normals(T)
    outs = {}
    for v in (11, 12, 13, 14, 17):
        monkeypatch.setenv("RSV_TRAJ_VARIANT", str(v))
        ch = DeviceChain(T, 0)
        try:
            ch.set_data(truth.dataset)
            ch.set_params(THETA)
            outs[v] = ch.integrate(truth.latent, p, 0.02, 20, fuse)
        finally:
            ch.close()
    h0, p0, d0 = outs[11]
    for v, (h, pp, d) in outs.items():
        assert d == d0 and np.array_equal(h, h0) and np.array_equal(pp, p0), v


def test_single_site_step_is_the_kernel_matrix_product(backend):
    # test_integrator.py:229-250: with y = 0 and phi = 0 a site's step is
    # affine, its linear part k1 k2 k1 (det 1) with w2 = 1/su2 + 1/se2
    params = P.Params(phi=0.0, mu=-1.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)
    data = P.Dataset.from_log_rv(np.zeros(2), np.array([-1.2, -1.4]))
    dt = 0.05
    w2 = 1.0 / params.sigma_u_sq + 1.0 / params.sigma_eta_sq
    k1 = np.array([[1.0, dt / 2], [0.0, 1.0]])
    k2 = np.array([[1.0, 0.0], [-dt * w2, 1.0]])
    m = k1 @ k2 @ k1
    assert abs(np.linalg.det(m) - 1.0) <= 1e-12

    def step(h0, p0):
        st = P.PhaseState(np.array([h0, 0.0]), np.array([p0, 0.0]))
        P.elementary_step(st, P.MDConfig(dt, 1), params, data, backend=backend)
        return np.array([st.h[0], st.p[0]])

    base = step(0.0, 0.0)
    cols = np.column_stack([step(1.0, 0.0) - base, step(0.0, 1.0) - base])
    assert np.allclose(cols, m, rtol=0, atol=1e-12)
    # the fused trajectory kernel gives the same one-step map
    st, _ = P.integrate_trajectory(P.PhaseState(np.array([1.0, 0.0]), np.array([0.0, 0.0])), P.MDConfig(dt, 1),
                                   params, data, backend=backend)
    assert np.allclose(np.array([st.h[0], st.p[0]]) - base, m[:, 0], rtol=0, atol=1e-12)


# ---------------------------------------------------------------- contract violations (C ABI -> Python errors)
def test_contract_violations_raise_like_the_reference(backend):
    # model.py / integrator.py conventions: ValueError for contract
    # violations (checked again by the C ABI: RSV_E_INVALID), a flag, never an
    # exception, for divergence
    import ctypes
    from paper_1603_08114_b200 import _native as N
    from paper_1603_08114_b200.integrator import DeviceChain
    truth = P.simulate_rsv(THETA, 64, seed=2)
    data = truth.dataset
    rng = P.make_rng(3, "pcg32")
    with pytest.raises(ValueError):
        P.hmc_update_volatility(truth.latent[:-1], THETA, data, P.MDConfig(0.02, 5), rng, backend=backend)
    with pytest.raises(ValueError):
        P.MDConfig(0.0, 5)
    with pytest.raises(ValueError):
        P.MDConfig(0.02, 0)
    with pytest.raises(NotImplementedError):
        P.integrate_trajectory(P.PhaseState(truth.latent.astype(np.float32), np.zeros(64, np.float32)),
                               P.MDConfig(0.02, 5), THETA, data, backend=backend)
    ch = DeviceChain(64, 0)
    try:
        lib = N.lib()
        with pytest.raises(ValueError):  # dt <= 0 through the C ABI itself
            N.check(lib.rsv_hmc_update(ch.ctx, ctypes.c_double(-1.0), 5, 0, ctypes.byref(N.Result())), ch.ctx)
        with pytest.raises(RuntimeError):  # nothing set on the context yet
            N.check(lib.rsv_hmc_update(ch.ctx, ctypes.c_double(0.02), 5, 0, ctypes.byref(N.Result())), ch.ctx)
        ch.set_data(data)
        ch.set_params(THETA)
        st = N.PrngState()
        st.kind = N.KINDS["minstd"]
        st.s[0] = 0  # not a minstd state
        with pytest.raises(ValueError):
            ch.hmc_update_host(truth.latent, st, 0.02, 5)
        bad = N.to_params(THETA)
        bad.phi = 1.0  # not stationary
        with pytest.raises(ValueError):
            N.check(lib.rsv_set_params(ch.ctx, ctypes.byref(bad)), ch.ctx)
    finally:
        ch.close()
    # divergence is a flag / sentinel, not an exception
    st, div = P.integrate_trajectory(P.PhaseState(truth.latent, np.full(64, 1e3)), P.MDConfig(0.5, 5), THETA, data,
                                     backend=backend)
    assert div


@pytest.mark.parametrize("T,kind", [(1024, "pcg32"), (70001, "minstd"), (1 << 18, "philox"), (3001, "sfc64")])
def test_batched_proposals_equal_one_by_one(backend, T, kind):
    """rsv_hmc_update_many without per-proposal timing or L2 flush runs the
    proposals in graphs of 8 (programmatic dependent launches, the result
    ring written by the Metropolis step): the same bits as proposals
    launched one by one."""
    truth = P.simulate_rsv(P.Params(**TRUE), T, seed=5)
    theta = P.Params(**TRUE)
    st0 = P.stream_state(P.make_rng(23, kind))
    other = P.CudaBackend(0)  # a second context (a backend keeps one chain per length)
    a, b = backend.chain(truth.dataset, theta), other.chain(truth.dataset, theta)
    assert a is not b
    for ch in (a, b):
        ch.set_latent(truth.latent)
        ch.set_stream(st0)
    # the third call grows the result ring (the batched graph must follow it)
    ra = (list(a.hmc_update_many(0.02, 20, 20)) + list(a.hmc_update_many(0.02, 20, 9))
          + list(a.hmc_update_many(0.02, 20, 40)))
    rb = []
    for _ in range(69):
        rb += list(b.hmc_update_many(0.02, 20, 1))
    assert [bool(x.accept) for x in ra] == [bool(x.accept) for x in rb]
    assert [x.delta_h for x in ra] == [x.delta_h for x in rb]
    assert [x.words_used for x in ra] == [x.words_used for x in rb]
    assert np.array_equal(a.get_latent(), b.get_latent())
    assert int(a.get_stream().pos) == int(b.get_stream().pos)
    other.close()


def test_batched_divergent_proposals_equal_one_by_one(backend):
    """Batches whose proposals all diverge (no uniform drawn, sampler.py:157-158)
    between batches that accept: stream positions and paths stay those of
    proposals launched one by one."""
    truth = P.simulate_rsv(P.Params(**TRUE), 2048, seed=5)
    theta = P.Params(**TRUE)
    st0 = P.stream_state(P.make_rng(23, "pcg32"))
    other = P.CudaBackend(0)
    a, b = backend.chain(truth.dataset, theta), other.chain(truth.dataset, theta)
    for ch in (a, b):
        ch.set_latent(truth.latent)
        ch.set_stream(st0)
    plan = [(0.02, 16), (0.3, 9), (0.02, 8), (0.6, 8), (0.02, 11)]
    ra, rb = [], []
    for dt, n in plan:
        ra += list(a.hmc_update_many(dt, 20, n))
        for _ in range(n):
            rb += list(b.hmc_update_many(dt, 20, 1))
    assert sum(bool(x.diverged) for x in ra) >= 17 and sum(bool(x.accept) for x in ra) > 0
    assert [(bool(x.accept), bool(x.diverged)) for x in ra] == [(bool(x.accept), bool(x.diverged)) for x in rb]
    assert [x.delta_h for x in ra] == [x.delta_h for x in rb]
    assert [x.words_used for x in ra] == [x.words_used for x in rb]
    assert np.array_equal(a.get_latent(), b.get_latent())
    assert int(a.get_stream().pos) == int(b.get_stream().pos)
    other.close()
