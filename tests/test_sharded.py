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
    from paper_1603_08114_b200.sharded import TOTALS, W_FLAG, W_U, fix128, put128
    rng = np.random.default_rng(0)
    parts = []
    for _ in range(5):
        p = np.zeros(TOTALS)
        p[6:21] = rng.normal(size=15) * 1e6
        p[W_FLAG] = 0.0
        for at in (0, 2, 4):
            put128(p, at, sum(fix128(x) for x in rng.normal(size=50) * 10.0))
        p[W_U:W_U + 2] = np.array([7, 3], dtype=np.uint64).view(np.float64)
        parts.append(p)
    a = combine(parts, THETA, 1000)
    b = combine(parts[::-1], THETA, 1000)
    assert a.delta_h == b.delta_h and a.accept == b.accept and a.h_old == b.h_old


def test_fixed_point_roundtrip_and_exactness():
    from paper_1603_08114_b200.sharded import fix128, unfix128
    for v in (0.0, 1.0, -1.0, 0.1, -3.25e-7, 1234.5678, 2.0 ** 61, -(2.0 ** -64)):
        q = fix128(v)
        assert q == int(v * 2.0 ** 64)
        assert abs(unfix128(q) - v) <= abs(v) * 2 ** -52 + 2.0 ** -64
    # sums are associative: any grouping gives the same integer
    xs = np.random.default_rng(1).normal(size=1000) * 50
    qs = [fix128(x) for x in xs]
    assert sum(qs) == sum(qs[::-1]) == sum(sum(qs[i:i + 7]) for i in range(0, 1000, 7))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_dh_bitwise_independent_of_world(world):
    """SURVEY 8e / the reference's worker-count independence
    (test_acceptance.py:269-309): the per-group fixed-point dH makes the
    combined dH the same bits for 1..4 shards."""
    T, n, dt, L = 640, 6, 0.02, 10
    truth = P.simulate_rsv(THETA, T, seed=4)
    runs = {}
    for w in (1, world):
        chains = [P.ShardedChain(truth.dataset, THETA, r, w, margin=24,
                                 shard_factory=lambda T_, lo, hi, m: OracleShard(T_, lo, hi, m)) for r in range(w)]
        st0 = P.stream_state(P.make_rng(9, "philox"))
        for c in chains:
            c.set_latent_global(truth.latent)
            c.set_stream(st0)
        runs[w] = [hmc_update_local(chains, dt, L) for _ in range(n)]
        runs[w] = ([d.delta_h for d in runs[w]], [d.accept for d in runs[w]],
                   np.concatenate([c.owned_latent() for c in chains]))
    assert runs[1][0] == runs[world][0] and runs[1][1] == runs[world][1]
    assert np.array_equal(runs[1][2], runs[world][2])


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


class _FakeP2PLib:
    """Stand-in for the peer-memory entry points (rank `fail_rank` cannot
    allocate / map): exercises the collective, agreed set-up of
    sharded._P2PComm on CPU ranks."""

    def __init__(self, rank, fail_rank, fail_at):
        self.rank, self.fail_rank, self.fail_at = rank, fail_rank, fail_at
        self.connected_with = None

    def rsv_shard_p2p_init(self, ctx, world, rank, handle, box):
        if self.rank == self.fail_rank and self.fail_at == "init":
            return -2
        for i in range(64):
            handle[i] = (rank * 64 + i) % 256
        return 0

    def rsv_shard_p2p_connect(self, ctx, handles, boxes):
        if self.rank == self.fail_rank and self.fail_at == "connect":
            return -2
        self.connected_with = bytes(handles)
        return 0


def _p2p_worker(rank, world, port, fail_rank, fail_at, q):
    import types
    import torch.distributed as dist
    from paper_1603_08114_b200 import sharded as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = _FakeP2PLib(rank, fail_rank, fail_at)
    chain = types.SimpleNamespace(rank=rank, world=world, shard=types.SimpleNamespace(_lib=lib, ctx=None))
    comm = S._comm_for([chain], dist.group.WORLD, True)
    q.put((rank, type(comm).__name__, lib.connected_with))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank,fail_at", [(-1, None), (1, "init"), (0, "connect")])
def test_gloo_peer_memory_setup_is_agreed(fail_rank, fail_at):
    """Every rank takes the peer-memory exchange only if every rank could
    allocate its box and map every peer's; otherwise every rank falls back
    to the NCCL exchange (none is left waiting in a collective)."""
    import torch.multiprocessing as mp
    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, fail_rank, fail_at, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict((r, (kind, hb)) for r, kind, hb in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = "_P2PComm" if fail_rank < 0 else "_NcclComm"
    assert [out[r][0] for r in range(world)] == [want] * world
    if fail_rank < 0:  # every rank received every rank's handle, in rank order
        every = bytes((r * 64 + i) % 256 for r in range(world) for i in range(64))
        assert all(out[r][1] == every for r in range(world))
