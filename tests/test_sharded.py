"""Time-sharded chain: host-side logic with gloo on CPUs (world size 2) and
in-process shards, against a single-process run of the oracle."""
import math
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_1603_08114_b200 as P
from paper_1603_08114_b200.sharded import combine, hmc_update_local, shard_bounds
from shard_oracle import OracleShard

THETA = P.Params(phi=0.97, mu=-9.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)


def _reference_run(truth, n, kind, seed, dt, L):
    st = O.Stream(kind, seed)
    h = truth.latent.copy()
    out = []
    for _ in range(n):
        h, acc, dh = O.hmc_update(h, THETA, truth.dataset.returns, truth.dataset.log_rv, dt, L, st)
        out.append((acc, dh))
    return h, out, st.pos


def test_shard_bounds():
    b = shard_bounds(1000, 4)
    assert b[0][0] == 0 and b[-1][1] == 1000
    assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
    assert all(lo % 8 == 0 for lo, _ in b)
    with pytest.raises(ValueError):
        shard_bounds(5, 4)


def test_combine_is_order_independent():
    rng = np.random.default_rng(0)
    parts = [np.concatenate([rng.normal(size=18) * 1e6, np.array([7, 3], dtype=np.uint64).view(np.float64)])
             for _ in range(5)]
    for p in parts:
        p[13] = 0.0
    a = combine(parts, THETA, 1000)
    b = combine(parts[::-1], THETA, 1000)
    assert a.delta_h == b.delta_h and a.accept == b.accept and a.h_old == b.h_old


@pytest.mark.parametrize("world", [2, 3])
def test_in_process_shards_match_single_chain(world):
    T, n, dt, L = 700, 12, 0.02, 10
    truth = P.simulate_rsv(THETA, T, seed=3)
    chains = [P.ShardedChain(truth.dataset, THETA, r, world, margin=24,
                             shard_factory=lambda T_, lo, hi, m: OracleShard(T_, lo, hi, m)) for r in range(world)]
    st0 = P.stream_state(P.make_rng(5, "pcg32"))
    for c in chains:
        c.set_latent_global(truth.latent)
        c.set_stream(st0)
    ref_h, ref, ref_pos = _reference_run(truth, n, "pcg32", 5, dt, L)
    H = abs(O.hamiltonian(truth.latent, np.zeros(T), THETA, truth.dataset.returns, truth.dataset.log_rv))
    for i in range(n):
        d = hmc_update_local(chains, dt, L)
        assert d.accept == ref[i][0], i
        if math.isinf(ref[i][1]):
            assert math.isinf(d.delta_h)
        else:
            assert abs(d.delta_h - ref[i][1]) <= 1e-12 * H
    h = np.concatenate([c.owned_latent() for c in chains])
    assert np.max(np.abs(h - ref_h)) <= 1e-12 * np.max(np.abs(ref_h))
    assert all(int(c.get_stream().pos) == ref_pos for c in chains)


def _worker(rank, world, port, T, n, dt, L, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    truth = P.simulate_rsv(THETA, T, seed=3)
    chain = P.ShardedChain(truth.dataset, THETA, rank, world, margin=24,
                           shard_factory=lambda T_, lo, hi, m: OracleShard(T_, lo, hi, m))
    chain.set_latent_global(truth.latent)
    chain.set_stream(P.stream_state(P.make_rng(5, "pcg32")))
    chain.halo_valid = False
    res = []
    for _ in range(n):
        d = P.hmc_update_distributed(chain, dt, L)
        res.append((d.accept, d.delta_h))
    q.put((rank, res, chain.owned_latent(), int(chain.get_stream().pos)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_match_single_chain():
    import torch.multiprocessing as mp
    T, n, dt, L, world = 640, 10, 0.02, 10, 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, n, dt, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res, h, pos = q.get(timeout=300)
        out[r] = (res, h, pos)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    truth = P.simulate_rsv(THETA, T, seed=3)
    ref_h, ref, ref_pos = _reference_run(truth, n, "pcg32", 5, dt, L)
    H = abs(O.hamiltonian(truth.latent, np.zeros(T), THETA, truth.dataset.returns, truth.dataset.log_rv))
    for r in range(world):
        assert [a for a, _ in out[r][0]] == [a for a, _ in ref]       # same decisions on every rank
        assert out[r][2] == ref_pos
        for (_, dh), (_, rd) in zip(out[r][0], ref):
            assert (math.isinf(dh) and math.isinf(rd)) or abs(dh - rd) <= 1e-12 * H
    h = np.concatenate([out[0][1], out[1][1]])
    assert np.max(np.abs(h - ref_h)) <= 1e-12 * np.max(np.abs(ref_h))


def test_halo_period_keeps_owned_sites_exact():
    from paper_1603_08114_b200.sharded import halo_period
    assert halo_period(8 * 21, 20) == 7
    assert halo_period(42, 12) == 2
    with pytest.raises(ValueError):
        halo_period(30, 20)
