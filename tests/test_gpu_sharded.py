"""Time-sharded chains on one GPU (several shard contexts in one process,
the same device-orchestrated driver the NCCL ranks run): windowed momenta,
blocked streams per shard, and run_chain across shards, against the single
context on the same stream.

Bars: the decisions, dH, the owned path and the stream state are the SAME
BITS as the single context's (dH / H are fixed-point group sums, the momenta
the whole-series draw's); run_chain's theta agrees to 1e-12 relative (the
FP64 moments are combined across shards in a different order).
Reference: sampler.py:136-167 (proposal), :291-358 (run_chain)."""
import math

import numpy as np
import pytest

import paper_1603_08114_b200 as P
from conftest import TRUE
from paper_1603_08114_b200 import sharded as S

pytestmark = pytest.mark.gpu
THETA = P.Params(**TRUE)


def _shards(data, world, margin, st0, h0, windowed=False):
    shards = [P.ShardedChain(data, THETA, r, world, margin=margin) for r in range(world)]
    for c in shards:
        c.set_stream(st0)
        c.set_latent_global(h0)
        if windowed:
            c.set_windowed_momenta(True)
    return shards


def _close(shards):
    for c in shards:
        c.shard.close()


@pytest.mark.parametrize("world,T,kind", [(2, 5000, "pcg32"), (3, 70001, "philox"), (4, 1 << 18, "minstd"),
                                          (4, 1 << 20, "pcg32"), (2, 300007, "minstd")])
def test_windowed_momenta_shards_equal_single_context(backend, world, T, kind):
    L, n = 20, 10
    truth = P.simulate_rsv(THETA, T, seed=31)
    data = truth.dataset
    margin = 3 * (L + 1)
    st0 = P.stream_state(P.make_rng(41, kind))
    shards = _shards(data, world, margin, st0, truth.latent, windowed=True)
    single = backend.chain(data, THETA)
    single.set_latent(truth.latent)
    single.set_stream(st0)
    try:
        res = S.hmc_update_local_device(shards, 0.02, L, n)
        ref = single.hmc_update_many(0.02, L, n)
        assert [bool(x.accept) for x in res] == [bool(x.accept) for x in ref]
        for a, b in zip(res, ref):
            assert a.diverged == b.diverged
            assert a.delta_h == b.delta_h and a.words_used == b.words_used
            assert math.isnan(b.u) or a.u == b.u
        h = np.concatenate([c.owned_latent() for c in shards])
        assert np.array_equal(h, single.get_latent())
        s1 = single.get_stream()
        for c in shards:
            s = c.get_stream()
            assert int(s.pos) == int(s1.pos)
    finally:
        _close(shards)


def test_windowed_momenta_refuses_sfc64(backend):
    truth = P.simulate_rsv(THETA, 4000, seed=2)
    st0 = P.stream_state(P.make_rng(1, "sfc64"))
    shards = _shards(truth.dataset, 2, 32, st0, truth.latent)
    try:
        with pytest.raises(ValueError):
            shards[0].set_windowed_momenta(True)
    finally:
        _close(shards)


@pytest.mark.parametrize("world", [2, 3])
def test_blocked_streams_per_shard_equal_single_context(backend, world):
    B, nb, L, n = 512, 24, 12, 8
    T = B * nb
    truth = P.simulate_rsv(THETA, T, seed=33)
    data = truth.dataset
    st0 = P.stream_state(P.make_rng(7, "sfc64"))
    shards = _shards(data, world, 3 * (L + 1), st0, truth.latent)
    for c in shards:
        c.set_blocked_streams(5, B)
    single = backend.chain(data, THETA)
    single.set_latent(truth.latent)
    single.set_stream(st0)
    single.set_blocked_streams(5, B)
    try:
        res = S.hmc_update_local_device(shards, 0.02, L, n)
        ref = single.hmc_update_many(0.02, L, n)
        assert [bool(x.accept) for x in res] == [bool(x.accept) for x in ref]
        assert 0 < sum(bool(x.accept) for x in ref)
        for a, b in zip(res, ref):
            assert a.delta_h == b.delta_h
        h = np.concatenate([c.owned_latent() for c in shards])
        assert np.array_equal(h, single.get_latent())
    finally:
        single.set_blocked_streams(None)
        _close(shards)


@pytest.mark.parametrize("world,kind,windowed", [(2, "pcg32", True), (3, "philox", False), (2, "sfc64", False)])
def test_sharded_run_chain_matches_single_context(backend, world, kind, windowed):
    T, L, dt = 6000, 20, 0.02
    truth = P.simulate_rsv(THETA, T, seed=35)
    data = truth.dataset
    prior = P.PriorSpec()
    st0 = P.stream_state(P.make_rng(13, kind))
    shards = _shards(data, world, 3 * (L + 1), st0, truth.latent, windowed=windowed)
    single = backend.chain(data, THETA)
    single.set_latent(truth.latent)
    single.set_params(THETA)
    single.set_stream(st0)
    try:
        it, par, acc, dh = S.run_chain_sharded(shards, dt, L, prior, n_burnin=3, n_samples=12, thin=1)
        it1, par1, acc1, dh1 = single.run_chain_device(dt, L, False, prior, 3, 12, 1)
        assert np.array_equal(it, it1)
        assert np.array_equal(acc, acc1)
        assert np.allclose(par, par1, rtol=1e-12, atol=0)
        fin = np.isfinite(dh1)
        assert np.array_equal(fin, np.isfinite(dh))
        assert np.allclose(dh[fin], dh1[fin], rtol=1e-8, atol=1e-10)
        p_shard = shards[0].shard.get_params()
        p_single = single.get_params() if hasattr(single, "get_params") else None
        if p_single is not None:
            assert abs(p_shard.mu - p_single.mu) <= 1e-12 * abs(p_single.mu)
        assert all(int(c.get_stream().pos) == int(single.get_stream().pos) for c in shards)
    finally:
        _close(shards)


@pytest.mark.parametrize("windowed", [True, False])
def test_captured_halo_periods_equal_single_context(backend, windowed):
    """graph=True: whole halo periods (halo exchange, windowed momenta,
    trajectories, records, gathers, decisions) recorded as one CUDA graph and
    replayed -- the same bits as the single context."""
    T, L, n, world = 40000, 12, 23, 3
    truth = P.simulate_rsv(THETA, T, seed=37)
    data = truth.dataset
    margin = 4 * (L + 1)  # halo period 3
    st0 = P.stream_state(P.make_rng(17, "pcg32"))
    shards = _shards(data, world, margin, st0, truth.latent, windowed=windowed)
    single = backend.chain(data, THETA)
    single.set_latent(truth.latent)
    single.set_stream(st0)
    try:
        res = S.hmc_update_local_device(shards, 0.02, L, n, graph=True)
        ref = single.hmc_update_many(0.02, L, n)
        assert len(res) == n
        assert [bool(x.accept) for x in res] == [bool(x.accept) for x in ref]
        assert [x.delta_h for x in res] == [x.delta_h for x in ref]
        h = np.concatenate([c.owned_latent() for c in shards])
        assert np.array_equal(h, single.get_latent())
        assert all(int(c.get_stream().pos) == int(single.get_stream().pos) for c in shards)
    finally:
        _close(shards)


@pytest.mark.parametrize("world,windowed,graph", [(2, True, False), (3, True, True), (4, False, True),
                                                  (3, False, False)])
def test_peer_memory_exchange_equals_single_context(backend, world, windowed, graph):
    """The records exchanged through the peer-memory boxes (each shard's
    record stored into every shard's box, flags released after the records,
    each shard collecting its own box) instead of the all-gather: the same
    bits as the single context, eager and in captured halo periods."""
    T, L, n = 50000, 12, 23
    truth = P.simulate_rsv(THETA, T, seed=43)
    data = truth.dataset
    st0 = P.stream_state(P.make_rng(19, "pcg32"))
    shards = _shards(data, world, 4 * (L + 1), st0, truth.latent, windowed=windowed)
    single = backend.chain(data, THETA)
    single.set_latent(truth.latent)
    single.set_stream(st0)
    try:
        res = S.hmc_update_local_device(shards, 0.02, L, n, graph=graph, p2p=True)
        res += S.hmc_update_local_device(shards, 0.02, L, 5, p2p=True)  # the boxes' epochs carry over calls
        ref = single.hmc_update_many(0.02, L, n + 5)
        assert [bool(x.accept) for x in res] == [bool(x.accept) for x in ref]
        assert [x.delta_h for x in res] == [x.delta_h for x in ref]
        h = np.concatenate([c.owned_latent() for c in shards])
        assert np.array_equal(h, single.get_latent())
        assert all(int(c.get_stream().pos) == int(single.get_stream().pos) for c in shards)
    finally:
        _close(shards)


def test_peer_memory_run_chain_matches_single_context(backend):
    T, L, dt, world = 6000, 20, 0.02, 3
    truth = P.simulate_rsv(THETA, T, seed=35)
    data = truth.dataset
    prior = P.PriorSpec()
    st0 = P.stream_state(P.make_rng(13, "pcg32"))
    shards = _shards(data, world, 3 * (L + 1), st0, truth.latent, windowed=True)
    single = backend.chain(data, THETA)
    single.set_latent(truth.latent)
    single.set_params(THETA)
    single.set_stream(st0)
    try:
        it, par, acc, dh = S.run_chain_sharded(shards, dt, L, prior, n_burnin=3, n_samples=12, thin=1, p2p=True)
        it1, par1, acc1, dh1 = single.run_chain_device(dt, L, False, prior, 3, 12, 1)
        assert np.array_equal(it, it1)
        assert np.array_equal(acc, acc1)
        assert np.allclose(par, par1, rtol=1e-12, atol=0)
    finally:
        _close(shards)


def test_peer_memory_missing_peer_is_an_error_not_a_hang(backend, monkeypatch):
    """A shard whose peer never publishes its record: the collect kernel
    gives up after RSV_P2P_TIMEOUT_MS and the next result read raises
    (bench.py then falls back to NCCL on every rank)."""
    monkeypatch.setenv("RSV_P2P_TIMEOUT_MS", "50")
    truth = P.simulate_rsv(THETA, 4000, seed=3)
    st0 = P.stream_state(P.make_rng(1, "pcg32"))
    shards = _shards(truth.dataset, 2, 63, st0, truth.latent)
    try:
        comm = S._LocalP2PComm(shards)
        import torch
        rec = torch.zeros(S.TOTALS, dtype=torch.float64, device="cuda")
        out = torch.zeros((2, S.TOTALS), dtype=torch.float64, device="cuda")
        c0 = shards[0].shard
        c0._ck(c0._lib.rsv_shard_p2p_push_async(c0.ctx, rec.data_ptr(), S.TOTALS))  # shard 1 never pushes
        c0._ck(c0._lib.rsv_shard_p2p_collect_async(c0.ctx, out.data_ptr(), S.TOTALS))
        with pytest.raises(P._native.NativeError, match="peer"):
            S._results(shards[0], 1)
        assert comm.world == 2
    finally:
        _close(shards)
