"""GPU parity at the sizes bench.py times (BASELINE configs 3, 4 and 5).

Every benchmarked path is checked against the oracle at the size and with the
switches the benchmark uses: the config-3 proposal graph at T=2^20 with the
256 MiB L2 flush and the per-proposal event pairs on, a full 4096 x 4096
ensemble round (every chain), and the config-5 blocked layout over 64 blocks
and at T=2^26 itself.

Tolerances: normals bit-exact, identical accept flags and stream
positions, |dH - dH_oracle| <= 1e-13 |H|, h within 1e-12 relative.
Reference: sampler.py:136-167 (momenta, proposal, Metropolis)."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1603_08114_b200 as P
from conftest import TRUE
from paper_1603_08114_b200.integrator import DeviceChain

pytestmark = pytest.mark.gpu
THETA = P.Params(**TRUE)
L2_FLUSH = 256 << 20


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def _H(h, y, lrv):
    return abs(O.hamiltonian(h, np.zeros(h.size), THETA, y, lrv)) + h.size


# ---------------------------------------------------------------- config 3
def test_config3_timed_proposals_vs_oracle():
    """bench.py's timed region: DeviceChain.hmc_update_many at T=2^20, L=20,
    dt=0.02, pcg32, data simulate_rsv(seed 0), L2 flush + timing level 1."""
    T, L, dt, n = 1 << 20, 20, 0.02, 8
    truth = P.simulate_rsv(THETA, T, seed=0)
    y, lrv = truth.dataset.returns, truth.dataset.log_rv
    ch = DeviceChain(T)
    try:
        ch.set_data(truth.dataset)
        ch.set_params(THETA)
        ch.set_latent(truth.latent)
        ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
        ch.set_l2_flush(L2_FLUSH)
        ch.set_timing(1)
        res = ch.hmc_update_many(dt, L, n, results=True)
        ch.set_timing(0)
        ch.set_l2_flush(0)
        st = O.Stream("pcg32", 1)
        h = truth.latent.copy()
        H = _H(h, y, lrv)
        nth = O.max_threads()
        for i in range(n):
            h, acc, dh = O.hmc_update(h, THETA, y, lrv, dt, L, st, nthreads=nth)
            assert bool(res[i].accept) == acc, i
            assert not res[i].diverged and math.isfinite(dh)
            assert abs(res[i].delta_h - dh) <= 1e-13 * H, (i, res[i].delta_h, dh)
        assert any(bool(r.accept) for r in res)
        assert _rel(ch.get_latent(np.empty(T)), h) <= 1e-12
        assert int(ch.get_stream().pos) == st.pos
    finally:
        ch.close()


# ---------------------------------------------------------------- config 4
def _ens_oracle_round(h, y, lrv, dt, L, streams, chains):
    out = {}
    for c in chains:
        out[c] = O.hmc_update(h[c], THETA, y, lrv, dt, L, streams[c])
    return out


@pytest.mark.parametrize("C", [64, 4096])
def test_config4_ensemble_every_chain_vs_oracle(C):
    """bench.py's ensemble_run: C chains x 4096 sites, one simulate_rsv series
    (seed 5) shared by every chain, latent at the true path, chain c on
    SFC64(SeedSequence([1, c])), L=20, dt=0.02.  C=64 is three CTAs of the
    29-chain momenta kernel; C=4096 is the benchmarked round (142 CTAs)."""
    Tc, L, dt, seed = 4096, 20, 0.02, 1
    rounds = 3 if C == 64 else 1
    tr = P.simulate_rsv(THETA, Tc, seed=5)
    y, lrv = tr.dataset.returns, tr.dataset.log_rv
    streams = [O.Stream("sfc64", np.random.SeedSequence([seed, c])) for c in range(C)]
    h = np.ascontiguousarray(np.broadcast_to(tr.latent, (C, Tc)))
    H = _H(tr.latent, y, lrv)
    with P.Ensemble(C, Tc) as ens:
        ens.set_data(y, lrv)
        ens.set_params(THETA)
        ens.set_latent(tr.latent)
        ens.seed(seed)
        for r in range(rounds):
            acc, dh = ens.hmc_update(dt, L)
            want = _ens_oracle_round(h, y, lrv, dt, L, streams, range(C))
            for c in range(C):
                hc, a, d = want[c]
                assert bool(acc[c]) == a, (r, c)
                assert abs(dh[c] - d) <= 1e-13 * H, (r, c, dh[c], d)
                h[c] = hc
        assert _rel(ens.latent(), h) <= 1e-12
        st = ens.streams()
        for c in range(C):
            assert [int(x) for x in st[c]] == streams[c].state_words()[0], c


# ---------------------------------------------------------------- config 5
def _blocked_normals(seed, nb, B, gens=None):
    gens = gens or [np.random.Generator(np.random.SFC64(np.random.SeedSequence([seed, j]))) for j in range(nb)]
    return np.concatenate([g.standard_normal(B) for g in gens]), gens


def test_config5_blocked_64_blocks_bit_exact_and_proposals():
    """The config-5 layout (4096-site blocks, SFC64(SeedSequence([1, j])),
    sfc64 main stream, dt=0.005, L=20) over 64 blocks: normals bit-exact per
    block across sweeps, proposals against the CPU trajectory + Metropolis."""
    B, nb, L, dt = 4096, 64, 20, 0.005
    T = B * nb
    tr = P.simulate_rsv(THETA, T, seed=11)
    y, lrv = tr.dataset.returns, tr.dataset.log_rv
    ch = DeviceChain(T)
    try:
        ch.set_data(tr.dataset)
        ch.set_params(THETA)
        ch.set_latent(tr.latent)
        main = P.make_rng(1, "sfc64")
        ch.set_stream(P.stream_state(main))
        ch.set_blocked_streams(1, B)
        gens = None
        for _ in range(2):  # momenta only: bit-exact, streams continue
            got = ch.refresh_momenta()
            want, gens = _blocked_normals(1, nb, B, gens)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        h = tr.latent.copy()
        H = _H(h, y, lrv)
        n_acc = 0
        for i in range(4):
            r = ch.hmc_update(dt, L, stats=False)
            p, gens = _blocked_normals(1, nb, B, gens)
            h2, p2, div = O.integrate(h, p, THETA, y, lrv, dt, L, nthreads=O.max_threads())
            assert not div
            dh = O.hamiltonian(h2, p2, THETA, y, lrv) - O.hamiltonian(h, p, THETA, y, lrv)
            u = main.random()  # drawn whenever dH is finite (sampler.py:163)
            acc = dh <= 0.0 or u < math.exp(-dh)
            assert bool(r.accept) == acc, i
            assert abs(r.delta_h - dh) <= 1e-13 * H, (i, r.delta_h, dh)
            if acc:
                h = h2
                n_acc += 1
        assert n_acc > 0
        assert _rel(ch.get_latent(np.empty(T)), h) <= 1e-12
        st = ch.blocked_streams()
        for j in range(nb):
            assert [int(x) for x in st[j]] == [int(x) for x in gens[j].bit_generator.state["state"]["state"]], j
        assert [int(x) for x in ch.get_stream().s] == [int(x) for x in P.stream_state(main).s]
    finally:
        ch.close()


def test_config5_full_size_proposal_vs_oracle():
    """One config-5 proposal at T=2^26 itself (16 384 blocks): every block's
    normals bit-exact, dH and the decision against the oracle, the kept path
    and the theta statistics of the kept path."""
    B, L, dt = 4096, 20, 0.005
    T = 1 << 26
    nb = T // B
    be = P.CudaBackend(0)
    try:
        tr = P.simulate_rsv(THETA, T, seed=11, backend=be)  # as bench.py config5_run
        y, lrv = tr.dataset.returns, tr.dataset.log_rv
        ch = be.chain(tr.dataset, THETA)
        ch.set_latent(tr.latent)
        main = P.make_rng(1, "sfc64")
        ch.set_stream(P.stream_state(main))
        ch.set_blocked_streams(1, B)
        r = ch.hmc_update(dt, L, stats=True)
        p, gens = _blocked_normals(1, nb, B)
        nth = O.max_threads()
        h2, p2, div = O.integrate(tr.latent, p, THETA, y, lrv, dt, L, nthreads=nth)
        assert not div
        dh = O.hamiltonian(h2, p2, THETA, y, lrv) - O.hamiltonian(tr.latent, p, THETA, y, lrv)
        u = main.random()
        acc = dh <= 0.0 or u < math.exp(-dh)
        H = _H(tr.latent, y, lrv)
        assert bool(r.accept) == acc
        assert abs(r.delta_h - dh) <= 1e-13 * H, (r.delta_h, dh)
        kept = h2 if acc else tr.latent
        got = ch.get_latent(np.empty(T))
        assert _rel(got, kept) <= 1e-12
        st = ch.blocked_streams()
        for j in (0, 1, 4095, 8192, nb - 1):
            assert [int(x) for x in st[j]] == [int(x) for x in gens[j].bit_generator.state["state"]["state"]], j
        want = O.suff_stats(kept, lrv, THETA.mu, THETA.xi)
        assert np.allclose(ch.last_stats(), want, rtol=1e-10, atol=1e-6 * math.sqrt(T))
        ch.set_blocked_streams(None)
    finally:
        be.close()
