"""One long chain split over several GPUs along the time axis.

The reference runs one chain on one CPU (`sampler.py:144-167`, `run_chain`
`sampler.py:291-358`); for long series (configs 3 and 5 of BASELINE.json) the
time axis is partitioned across the ranks of a process group:

* rank r owns the contiguous sites [lo_r, hi_r) and keeps a local copy of
  [lo_r - M, hi_r + M) with a margin M >= n_steps + 1 (clamped at the ends);
* before a proposal the margins are refreshed from the neighbours' owned sites
  (one halo exchange of M doubles per neighbour per *trajectory*: the
  trajectory kernel's tiles already carry an (L+1)-site halo, so the owned
  sites come out exactly as a per-step exchange would give them);
* every rank draws the momenta of the whole series from the same stream, runs
  the trajectory on its local range and publishes its partial sums of
  dH, H_old, H_new and the theta statistics;
* the partials are all-gathered and combined with an exactly rounded sum
  (math.fsum), so every rank takes the same Metropolis decision with the same
  uniform and the result does not depend on the number of ranks' reduction
  order; every rank then applies it (flip current path / advance stream).

`ShardedChain` is the per-rank object.  `hmc_update_distributed` drives it
over a `torch.distributed` process group (NCCL on GPUs, gloo on CPUs);
`hmc_update_local` drives several shards held by one process (tests, or a
single GPU emulating a sharded layout).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .integrator import DH_DIVERGENCE_THRESHOLD
from .model import Dataset, Params

# one shard's record (rsv_shard_totals, 23 8-byte words, viewed as float64):
# dh, H_old, H_new as 128-bit fixed point (2 words each), 5 + 5 moments, the
# flag, 4 end values, u_word, words_used (bit patterns)
TOTALS = 23
W_DH, W_HOLD, W_HNEW, W_SO, W_SN, W_FLAG, W_ENDS, W_U, W_USED = 0, 2, 4, 6, 11, 16, 17, 21, 22
FIX_SCALE = 2.0 ** 64


def fix128(v: float) -> int:
    """v * 2^64 rounded toward zero (exactly the device's fix128): per-group
    values become integers whose sums are independent of the grouping."""
    return int(float(v) * FIX_SCALE)


def unfix128(q: int) -> float:
    """The device's conversion back (unfix128 in leapfrog.cu): nearest doubles
    of the high and low 64-bit halves, combined in one rounded addition."""
    a = -q if q < 0 else q
    r = float(a >> 64) + float(a & 0xFFFFFFFFFFFFFFFF) * 2.0 ** -64
    return -r if q < 0 else r


def rec128(words: np.ndarray, at: int) -> int:
    """The int128 stored as {low, high} 64-bit words at `at` of a record."""
    lo = int(words[at:at + 1].view(np.uint64)[0])
    hi = int(words[at + 1:at + 2].view(np.int64)[0])
    return (hi << 64) | lo


def put128(words: np.ndarray, at: int, q: int):
    words[at:at + 1] = np.array([q & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64).view(np.float64)
    words[at + 1:at + 2] = np.array([q >> 64], dtype=np.int64).view(np.float64)


def shard_bounds(T: int, world: int, align: int = 8) -> list[tuple[int, int]]:
    """Contiguous owned ranges [lo, hi) of nearly equal size (boundaries on
    multiples of `align` sites except the last)."""
    if world < 1 or T < 2 * world:
        raise ValueError(f"cannot split {T} sites over {world} ranks")
    edges = [0]
    for r in range(1, world):
        e = (T * r // world) // align * align
        edges.append(max(e, edges[-1] + 1))
    edges.append(T)
    return [(edges[r], edges[r + 1]) for r in range(world)]


def local_range(T: int, lo: int, hi: int, margin: int) -> tuple[int, int]:
    """Same rule as rsv_create_shard: start rounded down to a multiple of 8."""
    ls = lo - margin
    ls = 0 if ls < 0 else ls // 8 * 8
    return ls, min(T, hi + margin)


class CudaShard:
    """Shard context on a GPU (rsv_create_shard / rsv_shard_* of the C ABI)."""

    def __init__(self, T: int, lo: int, hi: int, margin: int, device: int = 0):
        self._lib = N.lib()
        h = ctypes.c_void_p()
        ls, ln = ctypes.c_int64(), ctypes.c_int64()
        N.check(self._lib.rsv_create_shard(ctypes.byref(h), int(device), int(T), int(lo), int(hi), int(margin),
                                           ctypes.byref(ls), ctypes.byref(ln)))
        self.ctx = h.value
        self.local_start, self.local_len = int(ls.value), int(ln.value)

    def _ck(self, code):
        N.check(code, self.ctx)

    def close(self):
        if self.ctx:
            self._lib.rsv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launch_count(self) -> int:
        return int(self._lib.rsv_launch_count(self.ctx))

    def set_data(self, y, lrv):
        y = np.ascontiguousarray(y, dtype=np.float64)
        lrv = np.ascontiguousarray(lrv, dtype=np.float64)
        self._ck(self._lib.rsv_set_data(self.ctx, y.ctypes.data, lrv.ctypes.data, 0))

    def set_params(self, params: Params):
        self._ck(self._lib.rsv_set_params(self.ctx, ctypes.byref(N.to_params(params))))

    def set_latent(self, h):
        h = np.ascontiguousarray(h, dtype=np.float64)
        self._ck(self._lib.rsv_set_latent(self.ctx, h.ctypes.data, 0))

    def get_latent(self) -> np.ndarray:
        out = np.empty(self.local_len)
        self._ck(self._lib.rsv_get_latent(self.ctx, out.ctypes.data, 0))
        return out

    def set_stream(self, st):
        self._ck(self._lib.rsv_set_prng_state(self.ctx, ctypes.byref(st)))

    def get_stream(self):
        st = N.PrngState()
        self._ck(self._lib.rsv_get_prng_state(self.ctx, ctypes.byref(st)))
        return st

    def slice_out(self, offset: int, n: int) -> np.ndarray:
        out = np.empty(n)
        if n:
            self._ck(self._lib.rsv_latent_slice(self.ctx, int(offset), int(n), out.ctypes.data, 0, 0))
        return out

    def slice_in(self, offset: int, buf: np.ndarray):
        buf = np.ascontiguousarray(buf, dtype=np.float64)
        if buf.size:
            self._ck(self._lib.rsv_latent_slice(self.ctx, int(offset), int(buf.size), buf.ctypes.data, 1, 0))

    def propose(self, step_size: float, n_steps: int, fuse: bool, stats: bool) -> np.ndarray:
        t = N.ShardTotals()
        self._ck(self._lib.rsv_shard_propose(self.ctx, float(step_size), int(n_steps), int(bool(fuse)),
                                             int(bool(stats)), ctypes.byref(t)))
        return np.frombuffer(bytes(t), dtype=np.float64).copy()

    def apply(self, accept: bool, drew: bool):
        self._ck(self._lib.rsv_shard_apply(self.ctx, int(bool(accept)), int(bool(drew))))

    def set_momenta(self, windowed: bool):
        self._ck(self._lib.rsv_shard_set_momenta(self.ctx, int(bool(windowed))))

    def set_blocked_streams(self, block_len: int, first_block: int, states):
        if states is None:
            self._ck(self._lib.rsv_shard_set_blocked_streams(self.ctx, 0, 0, 0, None))
            return
        states = np.ascontiguousarray(states, dtype=np.uint64)
        self._ck(self._lib.rsv_shard_set_blocked_streams(self.ctx, int(block_len), int(first_block),
                                                         int(states.shape[0]), states.ctypes.data))

    def get_params(self) -> Params:
        out = N.Params()
        self._ck(self._lib.rsv_get_params(self.ctx, ctypes.byref(out)))
        return Params(phi=out.phi, mu=out.mu, xi=out.xi, sigma_eta_sq=out.sigma_eta_sq, sigma_u_sq=out.sigma_u_sq)


@dataclass
class Decision:
    accept: bool
    diverged: bool
    delta_h: float
    h_old: float
    h_new: float
    drew: bool
    u: float
    stats_kept: np.ndarray  # 7 moments of the kept path (layout of rsv_suff_stats)


def h_constant(params: Params, T: int) -> float:
    """theta-only part of H (model.py:134-163 log terms and 0.5*T*mu)."""
    phi, se2, su2 = params.phi, params.sigma_eta_sq, params.sigma_u_sq
    return (0.5 * T * params.mu + 0.5 * T * math.log(su2) + 0.5 * math.log(se2 / (1.0 - phi * phi))
            + 0.5 * (T - 1) * math.log(se2))


def combine(totals: list[np.ndarray], params: Params, T: int) -> Decision:
    """Metropolis step of sampler.py:155-167 on the shards' records.  dH,
    H_old and H_new are exact integer sums of the fixed-point parts (the same
    bits for any number or order of shards, and as a single context); the
    moments and end values use math.fsum (exactly rounded, order-free)."""
    tot = [np.asarray(t, dtype=np.float64) for t in totals]
    q = [sum(rec128(t, at) for t in tot) for at in (W_DH, W_HOLD, W_HNEW)]
    fl = max(float(t[W_FLAG]) for t in tot)
    mom = [math.fsum(float(t[W_SO + k]) for t in tot) for k in range(10)]
    ends = [math.fsum(float(t[W_ENDS + k]) for t in tot) for k in range(4)]
    u_word = int(tot[0][W_U:W_U + 1].view(np.uint64)[0])
    if any(int(t[W_U:W_U + 1].view(np.uint64)[0]) != u_word for t in tot):
        raise RuntimeError("shards drew different momenta streams")
    c = h_constant(params, T)
    dh = unfix128(q[0])
    drew = False
    u = float("nan")
    accept = False
    if fl > 0.0 or not math.isfinite(dh) or abs(dh) > DH_DIVERGENCE_THRESHOLD:
        diverged, delta_h = True, math.inf
    else:
        diverged, delta_h = False, dh
        u = float(u_word >> 11) * (1.0 / 9007199254740992.0)
        drew = True
        accept = dh <= 0.0 or u < math.exp(-dh)
    ends_old, ends_new = ends[0:2], ends[2:4]
    kept = np.array([*(ends_new if accept else ends_old), *(mom[5:10] if accept else mom[0:5])])
    return Decision(accept, diverged, delta_h, unfix128(q[1]) + c, unfix128(q[2]) + c, drew, u, kept)


class ShardedChain:
    """Rank-local part of a time-sharded chain."""

    def __init__(self, data: Dataset, params: Params, rank: int, world: int, margin: int = 64, device: int = 0,
                 shard_factory=None):
        self.T = data.length
        self.rank, self.world = rank, world
        self.bounds = shard_bounds(self.T, world)
        self.lo, self.hi = self.bounds[rank]
        self.margin = margin
        factory = shard_factory or (lambda T, lo, hi, m: CudaShard(T, lo, hi, m, device))
        self.shard = factory(self.T, self.lo, self.hi, margin)
        self.ls = self.shard.local_start
        self.le = self.ls + self.shard.local_len
        self.shard.set_data(data.returns[self.ls:self.le], data.log_rv[self.ls:self.le])
        self.params = params
        self.shard.set_params(params)
        self.halo_valid = False
        self.windowed = False

    # -- momenta layout --
    def set_windowed_momenta(self, on: bool = True):
        """Draw only this shard's window of the momenta stream (jump-ahead
        generators; device-orchestrated drivers): the normals are the
        whole-series draw's, bit for bit (rsv_shard_set_momenta)."""
        self.shard.set_momenta(on)
        self.windowed = bool(on)

    def set_blocked_streams(self, seed: int | None, block_len: int = 4096):
        """Config-5 layout on a shard: the streams SFC64(SeedSequence([seed,
        j])) of the blocks j its local range touches (DeviceChain's layout,
        per shard)."""
        if seed is None:
            self.shard.set_blocked_streams(0, 0, None)
            return
        if self.T % block_len:
            raise ValueError(f"block length {block_len} does not divide T={self.T}")
        from .ensemble import sfc64_states
        j0, j1 = self.ls // block_len, -(-self.le // block_len)
        states = sfc64_states(seed, j1 - j0, j0)
        self.shard.set_blocked_streams(block_len, j0, states)

    # -- state --
    def set_params(self, params: Params):
        self.params = params
        self.shard.set_params(params)

    def set_latent_global(self, h: np.ndarray):
        self.shard.set_latent(np.asarray(h, dtype=np.float64)[self.ls:self.le])
        self.halo_valid = True

    def owned_latent(self) -> np.ndarray:
        return self.shard.get_latent()[self.lo - self.ls:self.hi - self.ls]

    def set_stream(self, st):
        self.shard.set_stream(st)

    def get_stream(self):
        return self.shard.get_stream()

    # -- halo exchange --
    def halo_sizes(self, r: int) -> tuple[int, int]:
        lo, hi = self.bounds[r]
        ls, le = local_range(self.T, lo, hi, self.margin)
        return lo - ls, le - hi

    def halo_out(self) -> tuple[np.ndarray, np.ndarray]:
        """(to the left neighbour, to the right neighbour): my owned sites
        that fall in their margins."""
        left = right = np.empty(0)
        if self.rank > 0:
            n = self.halo_sizes(self.rank - 1)[1]
            left = self.shard.slice_out(self.lo - self.ls, n)
        if self.rank < self.world - 1:
            n = self.halo_sizes(self.rank + 1)[0]
            right = self.shard.slice_out(self.hi - self.ls - n, n)
        return left, right

    def halo_in(self, from_left: np.ndarray, from_right: np.ndarray):
        if self.rank > 0:
            self.shard.slice_in(0, from_left)
        if self.rank < self.world - 1:
            self.shard.slice_in(self.hi - self.ls, from_right)
        self.halo_valid = True

    # -- proposal phases --
    def propose(self, step_size: float, n_steps: int, fuse: bool = False, stats: bool = True) -> np.ndarray:
        if n_steps + 1 > self.margin:
            raise ValueError(f"n_steps={n_steps} needs a margin of at least {n_steps + 1} (have {self.margin})")
        return self.shard.propose(step_size, n_steps, fuse, stats)

    def apply(self, d: Decision):
        self.shard.apply(d.accept, d.drew)
        if d.accept:
            self.halo_valid = False


def hmc_update_local(chains: list[ShardedChain], step_size: float, n_steps: int, fuse: bool = False,
                     stats: bool = True) -> Decision:
    """One proposal of a sharded chain whose shards live in this process."""
    if not all(c.halo_valid for c in chains):
        outs = [c.halo_out() for c in chains]
        for r, c in enumerate(chains):
            c.halo_in(outs[r - 1][1] if r > 0 else np.empty(0),
                      outs[r + 1][0] if r < len(chains) - 1 else np.empty(0))
    totals = [c.propose(step_size, n_steps, fuse, stats) for c in chains]
    d = combine(totals, chains[0].params, chains[0].T)
    for c in chains:
        c.apply(d)
    return d


def hmc_update_distributed(chain: ShardedChain, step_size: float, n_steps: int, fuse: bool = False,
                           stats: bool = True, group=None, device=None) -> Decision:
    """One proposal of a sharded chain over a torch.distributed process group.
    Halo: point-to-point send/recv with the neighbours; totals: all_gather."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cpu") if device is None else torch.device(device)
    r, w = chain.rank, chain.world
    flag = torch.tensor([0 if chain.halo_valid else 1], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if int(flag.item()):
        left, right = chain.halo_out()
        reqs = []
        recv_l = recv_r = None
        if r > 0:
            reqs.append(dist.isend(torch.from_numpy(left).to(dev), r - 1, group=group))
            recv_l = torch.empty(chain.halo_sizes(r)[0], dtype=torch.float64, device=dev)
            reqs.append(dist.irecv(recv_l, r - 1, group=group))
        if r < w - 1:
            reqs.append(dist.isend(torch.from_numpy(right).to(dev), r + 1, group=group))
            recv_r = torch.empty(chain.halo_sizes(r)[1], dtype=torch.float64, device=dev)
            reqs.append(dist.irecv(recv_r, r + 1, group=group))
        for q in reqs:
            q.wait()
        chain.halo_in(recv_l.cpu().numpy() if recv_l is not None else np.empty(0),
                      recv_r.cpu().numpy() if recv_r is not None else np.empty(0))
    mine = torch.from_numpy(chain.propose(step_size, n_steps, fuse, stats)).to(dev)
    allt = [torch.empty_like(mine) for _ in range(w)]
    dist.all_gather(allt, mine, group=group)
    d = combine([t.cpu().numpy() for t in allt], chain.params, chain.T)
    chain.apply(d)
    return d


# ---------------------------------------------------------------------------
# Device-side orchestration: the host only enqueues work.  Per proposal every
# shard writes its 20 totals to device memory, the totals are all-gathered
# (NCCL between GPUs; one buffer for shards sharing a process), and each
# shard takes the (identical) Metropolis decision on the device.  The margins
# are refreshed every `halo_every` proposals without knowing the decisions:
# a margin of M >= (K + 1)(L + 1) sites keeps the owned sites exact for K
# proposals after an exchange, whatever was accepted in between (each
# trajectory can corrupt at most L + 1 sites inward from the margin's outer
# edge).

_RING = 1024  # decisions buffered on the device between two result reads (rsv_shard_decide_async)


def halo_period(margin: int, n_steps: int) -> int:
    """Proposals between two halo exchanges that keep the owned sites exact."""
    k = margin // (n_steps + 1) - 1
    if k < 1:
        raise ValueError(f"margin {margin} too small for n_steps={n_steps}: need >= {2 * (n_steps + 1)}")
    return k


def _cuda_shard_ptrs(chains):
    for c in chains:
        if not isinstance(c.shard, CudaShard):
            raise TypeError("device orchestration needs CUDA shards")


def _results(chain, n):
    if n == 0:
        return []
    out = (N.Result * max(1, n))()
    got = ctypes.c_int(0)
    chain.shard._ck(chain.shard._lib.rsv_shard_results(chain.shard.ctx, out, int(n), ctypes.byref(got)))
    return [out[i] for i in range(min(n, got.value))]


WIN_W = 8  # 8-byte words of a momenta window record (WinInfo)


class _LocalComm:
    """All shards of the chain in this process (one GPU, one stream): the
    records are gathered by device copies, the halos by direct slices."""

    def __init__(self, chains):
        self.chains = chains
        self.world = len(chains)

    def gather(self, out, mine):
        for r, m in enumerate(mine):
            out[r].copy_(m)

    def halo(self, chains, sends, recvs):
        for r, c in enumerate(chains):  # my left margin <- left neighbour's right send, and vice versa
            recvs[r][0].copy_(sends[r - 1][1]) if r > 0 else None
            recvs[r][1].copy_(sends[r + 1][0]) if r < len(chains) - 1 else None

    def agree(self, ok: bool) -> bool:
        return ok


class _NcclComm:
    """One shard per rank of a torch.distributed (NCCL) group: records by
    all_gather_into_tensor, halos by batched send/recv with the neighbours."""

    def __init__(self, chain, group):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = chain.rank, chain.world

    def gather(self, out, mine):
        self.dist.all_gather_into_tensor(out, mine[0], group=self.group)

    def halo(self, chains, sends, recvs):
        dist, r, w = self.dist, self.rank, self.world
        (send_l, send_r), (recv_l, recv_r) = sends[0], recvs[0]
        ops = []
        if r > 0:
            ops += [dist.P2POp(dist.isend, send_l, r - 1, self.group), dist.P2POp(dist.irecv, recv_l, r - 1, self.group)]
        if r < w - 1:
            ops += [dist.P2POp(dist.isend, send_r, r + 1, self.group), dist.P2POp(dist.irecv, recv_r, r + 1, self.group)]
        for q in dist.batch_isend_irecv(ops) if ops else []:
            q.wait()  # orders the copies on the current stream (no host block)

    def _device(self):
        """Where the group's collectives take their tensors (NCCL: the GPU; gloo: the host)."""
        import torch
        if self.dist.get_backend(self.group) == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def agree(self, ok: bool) -> bool:
        """True on every rank iff true on every rank (eager, outside any capture)."""
        import torch
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=self._device())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return bool(t.item())


def _p2p_push_collect(chains, out, mine):
    """The records of one exchange through the peer-memory boxes: every
    shard of this process pushes its record into every shard's box, then
    every shard waits for and collects its own box (into `out`, rank order:
    the layout of the all-gather)."""
    words = out.shape[1]
    for c, m in zip(chains, mine):
        c.shard._ck(c.shard._lib.rsv_shard_p2p_push_async(c.shard.ctx, m.data_ptr(), words))
    for c in chains:
        c.shard._ck(c.shard._lib.rsv_shard_p2p_collect_async(c.shard.ctx, out.data_ptr(), words))


class _LocalP2PComm(_LocalComm):
    """In-process shards (one GPU) exchanging their records through the
    peer-memory boxes -- the multi-GPU protocol with same-device addresses."""

    def __init__(self, chains):
        super().__init__(chains)
        boxes = (ctypes.c_uint64 * len(chains))()
        handle = (ctypes.c_ubyte * 64)()
        for r, c in enumerate(chains):
            v = ctypes.c_uint64()
            c.shard._ck(c.shard._lib.rsv_shard_p2p_init(c.shard.ctx, len(chains), r, handle, ctypes.byref(v)))
            boxes[r] = v.value
        for c in chains:
            c.shard._ck(c.shard._lib.rsv_shard_p2p_connect(c.shard.ctx, None, boxes))

    def gather(self, out, mine):
        _p2p_push_collect(self.chains, out, mine)


class P2PUnavailable(RuntimeError):
    """Some rank could not set up the peer-memory exchange (every rank gets it)."""


class _P2PComm(_NcclComm):
    """One shard per rank, the per-proposal records exchanged by NVLink
    stores into every rank's box (CUDA IPC mappings, set up once over the
    NCCL group); the margins still go by NCCL send/recv (every K proposals).
    The set-up is collective and agreed: if any rank fails (allocation, IPC
    mapping), every rank raises P2PUnavailable and none is left waiting."""

    def __init__(self, chain, group):
        import torch
        super().__init__(chain, group)
        self.chain = chain
        lib, ctx = chain.shard._lib, chain.shard.ctx
        handle = (ctypes.c_ubyte * 64)()
        box = ctypes.c_uint64()
        ok = lib.rsv_shard_p2p_init(ctx, self.world, self.rank, handle, ctypes.byref(box)) == 0
        dev = self._device()
        mine = torch.tensor([1 if ok else 0] + list(bytes(handle)), dtype=torch.uint8, device=dev)
        every = torch.empty(self.world * 65, dtype=torch.uint8, device=dev)
        self.dist.all_gather_into_tensor(every, mine, group=group)
        rows = every.cpu().numpy().reshape(self.world, 65)
        ok = bool(rows[:, 0].all())
        if ok:
            hb = rows[:, 1:].tobytes()
            ok = lib.rsv_shard_p2p_connect(ctx, hb, None) == 0
        if not self.agree(ok):
            raise P2PUnavailable("peer-memory exchange unavailable on some rank; use NCCL")

    def gather(self, out, mine):
        _p2p_push_collect([self.chain], out, mine)


def _comm_for(chains, group, p2p):
    """The exchange for this process's shards: in-process (all shards here)
    or one shard per rank; by peer memory (p2p) or NCCL / device copies.
    The connection is made once per chain and group."""
    local = group is None and len(chains) == chains[0].world
    key = ("local" if local else id(group), bool(p2p))
    c0 = chains[0]
    cache = c0.__dict__.setdefault("_comms", {})
    if key not in cache:
        if local:
            cache[key] = _LocalP2PComm(chains) if p2p else _LocalComm(chains)
        elif p2p:
            try:
                cache[key] = _P2PComm(c0, group)
            except P2PUnavailable:  # agreed by every rank: all of them take the NCCL exchange
                cache[key] = _NcclComm(c0, group)
        else:
            cache[key] = _NcclComm(c0, group)
    return cache[key]


def exchange_kind(chain, group=None) -> str:
    """'p2p' or 'nccl': the record exchange the last distributed call used."""
    comms = chain.__dict__.get("_comms", {})
    for (k, _), comm in comms.items():
        if k != "local" and k == id(group):
            return "p2p" if isinstance(comm, _P2PComm) else "nccl"
    return "nccl"


def _p2p_default(world):
    return world > 1 and os.environ.get("RSV_P2P", "1") != "0"


def _drive(chains, comm, step_size, n_steps, n, fuse, stats, halo_every, dev, stream, l2_flush=None, times=None,
           theta=False, graph=False):
    """n proposals (or sweeps with theta=True) of the chain whose shards
    `chains` live in this process, every step enqueued on `stream`:
    [margins every K proposals] -> [windowed momenta: window parse,
    all-gather of the window records, placement] -> trajectory + this
    shard's record -> all-gather of the records -> the same decision on
    every shard -> [theta draws].  The host synchronises only to read the
    result ring.  graph=True records one halo period (K proposals, with the
    collectives) as a CUDA graph and replays it: one host launch per K
    proposals instead of ~15 library calls per proposal."""
    import torch
    world = comm.world
    c0 = chains[0]
    lib = c0.shard._lib
    for c in chains:
        c.shard._ck(lib.rsv_set_stream(c.shard.ctx, ctypes.c_void_p(stream.cuda_stream)))
    K = halo_every or halo_period(c0.margin, n_steps)
    f64 = dict(dtype=torch.float64, device=dev)
    rec_mine = [torch.zeros(TOTALS, **f64) for _ in chains]
    rec_all = torch.zeros((world, TOTALS), **f64)
    windowed = c0.windowed
    win_mine = [torch.zeros(WIN_W, **f64) for _ in chains] if windowed else None
    win_all = torch.zeros((world, WIN_W), **f64) if windowed else None
    sends, recvs = [], []
    for c in chains:
        r = c.rank
        nl_recv, nr_recv = c.halo_sizes(r)
        sends.append((torch.empty(c.halo_sizes(r - 1)[1] if r > 0 else 0, **f64),
                      torch.empty(c.halo_sizes(r + 1)[0] if r < world - 1 else 0, **f64)))
        recvs.append((torch.empty(nl_recv if r > 0 else 0, **f64), torch.empty(nr_recv if r < world - 1 else 0, **f64)))

    def halo():
        for c, (sl, sr) in zip(chains, sends):
            c.shard._ck(lib.rsv_shard_halo_async(c.shard.ctx, sl.data_ptr(), sl.numel(), sr.data_ptr(), sr.numel(), 0))
        comm.halo(chains, sends, recvs)
        for c, (fl, fr) in zip(chains, recvs):
            c.shard._ck(lib.rsv_shard_halo_async(c.shard.ctx, fl.data_ptr(), fl.numel(), fr.data_ptr(),
                                                 fr.numel(), 1))
            c.halo_valid = True

    def proposal(i, ev=None, halo_here=True):
        if l2_flush is not None:
            l2_flush.fill_(i & 0xff)
        if ev is not None:
            ev[0].record(stream)
        if halo_here and world > 1 and (i % K == 0 or not all(c.halo_valid for c in chains)):
            halo()
        if windowed:
            for c, w in zip(chains, win_mine):
                c.shard._ck(lib.rsv_shard_momenta_async(c.shard.ctx, w.data_ptr()))
            comm.gather(win_all, win_mine)
            for c in chains:
                c.shard._ck(lib.rsv_shard_place_async(c.shard.ctx, win_all.data_ptr(), world, c.rank))
        for c, m in zip(chains, rec_mine):
            c.shard._ck(lib.rsv_shard_propose_async(c.shard.ctx, float(step_size), int(n_steps), int(bool(fuse)),
                                                    int(bool(stats or theta)), m.data_ptr()))
        comm.gather(rec_all, rec_mine)
        for c in chains:
            c.shard._ck(lib.rsv_shard_decide_async(c.shard.ctx, rec_all.data_ptr(), world))
            if theta:
                c.shard._ck(lib.rsv_shard_theta_async(c.shard.ctx))
        if ev is not None:
            ev[1].record(stream)

    def events(external=False):  # external: recorded as event nodes when captured in a graph
        return (torch.cuda.Event(enable_timing=True, external=external),
                torch.cuda.Event(enable_timing=True, external=external))

    out = [[] for _ in chains]

    def drain(k):
        for c, acc in zip(chains, out):
            acc.extend(_results(c, k))

    direct = []  # event pairs of the proposals enqueued one by one
    try:
        i = 0
        pending = 0
        if graph and n >= 2 * K:
            # align to a halo period, then replay captured periods
            while i % K:
                ev = events() if times is not None else None
                proposal(i, ev)
                if ev is not None:
                    direct.append(ev)
                i += 1
                pending += 1
            for c in chains:
                c.shard._ck(lib.rsv_shard_prepare(c.shard.ctx, float(step_size), int(n_steps), int(bool(fuse)),
                                                  int(bool(stats or theta))))
            # the captured period: K proposals with their collectives; the
            # margin exchange that opens each period (NCCL send/recv between
            # neighbours) stays eager, before every replay.  If any rank cannot
            # capture, every rank stays on the eager path.
            evs = [events(True) for _ in range(K)] if times is not None else [None] * K
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
                    for j in range(K):
                        proposal(j, evs[j], halo_here=False)
                captured = True
            except Exception:  # noqa: BLE001 -- any capture failure means the eager path
                captured = False
            if not comm.agree(captured):
                g = None
            hev = events() if times is not None and world > 1 else None
            while g is not None and n - i >= K:
                if pending + K > _RING:
                    drain(pending)
                    pending = 0
                if world > 1:
                    if hev is not None:
                        hev[0].record(stream)
                    halo()
                    if hev is not None:
                        hev[1].record(stream)
                g.replay()
                i += K
                pending += K
                if times is not None:  # the captured events are re-recorded by the next replay
                    stream.synchronize()
                    t = [a.elapsed_time(b) for a, b in evs]
                    if hev is not None:  # the period's margin exchange belongs to its first proposal
                        t[0] += hev[0].elapsed_time(hev[1])
                    times.extend(t)
        while i < n:
            ev = events() if times is not None else None
            proposal(i, ev)
            if ev is not None:
                direct.append(ev)
            i += 1
            pending += 1
            if pending == _RING:
                drain(pending)
                pending = 0
        drain(pending)
        if times is not None:
            stream.synchronize()
            times.extend(a.elapsed_time(b) for a, b in direct)
    finally:
        for c in chains:
            lib.rsv_set_stream(c.shard.ctx, None)
    for r in range(1, len(chains)):  # every shard recorded the same decisions
        if [x.accept for x in out[r]] != [x.accept for x in out[0]]:
            raise RuntimeError("shards took different decisions")
    return out[0]


def hmc_update_local_device(chains: list[ShardedChain], step_size: float, n_steps: int, n: int,
                            fuse: bool = False, stats: bool = False, halo_every: int | None = None,
                            graph: bool = False, p2p: bool = False):
    """n proposals of a chain whose shards all live in this process (one
    GPU), orchestrated on the device: no host synchronisation until the
    results are read back.  Returns the per-proposal rsv_result records."""
    import torch
    _cuda_shard_ptrs(chains)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream(dev)  # one ordered stream for every shard and every buffer
    with torch.cuda.stream(stream):
        return _drive(chains, _comm_for(chains, None, p2p), step_size, n_steps, n, fuse, stats, halo_every, dev,
                      stream, graph=graph)


def hmc_update_distributed_device(chain: ShardedChain, step_size: float, n_steps: int, n: int, fuse: bool = False,
                                  stats: bool = False, group=None, halo_every: int | None = None,
                                  l2_flush=None, times: list | None = None, graph: bool = False,
                                  p2p: bool | None = None):
    """n proposals of a sharded chain over a torch.distributed (NCCL) group,
    orchestrated on the device: window records and shard records
    all-gathered on the GPU, decisions on the GPU, periodic halo exchange;
    the host synchronises once at the end.  Benchmarking: `l2_flush` (a
    device tensor larger than L2) is overwritten before every proposal, and
    `times` collects each proposal's milliseconds between a CUDA event
    pair recorded after the flush and after the decision.  graph=True
    replays captured halo periods (see _drive)."""
    import torch
    _cuda_shard_ptrs([chain])
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream(dev)  # the kernels and the NCCL collectives share one ordered stream
    with torch.cuda.stream(stream):
        comm = _comm_for([chain], group, _p2p_default(chain.world) if p2p is None else p2p)
        return _drive([chain], comm, step_size, n_steps, n, fuse, stats, halo_every, dev, stream, l2_flush, times,
                      graph=graph)


def run_chain_sharded(chains: list[ShardedChain], step_size: float, n_steps: int, prior, n_burnin: int,
                      n_samples: int, thin: int = 1, group=None, halo_every: int | None = None,
                      p2p: bool | None = None):
    """run_chain (sampler.py:291-358) of a time-sharded chain, every sweep on
    the devices: the proposal protocol of _drive with the statistics of the
    kept path, then the theta draws (sampler.py:339-344) on every shard from
    the all-gathered statistics -- the same parameters on every shard.
    `chains` are this process's shards (all of them, or one per rank with
    `group`).  Returns (iters, params [n x 5], accept, delta_h) as
    DeviceChain.run_chain_device; raises NativeError subclass StormError on a
    divergence storm (with .sweep)."""
    import torch
    _cuda_shard_ptrs(chains)
    pr = N.Prior(*(float(getattr(prior, f)) for f, _ in N.Prior._fields_))
    for c in chains:
        c.shard._ck(c.shard._lib.rsv_shard_run_begin(c.shard.ctx, float(step_size), ctypes.byref(pr), int(n_burnin),
                                                       int(n_samples), int(thin)))
    n_sweeps = n_burnin + n_samples * thin
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream(dev)
    local = group is None and len(chains) == chains[0].world
    comm = _comm_for(chains, group, (not local and _p2p_default(chains[0].world)) if p2p is None else p2p)
    err = None
    with torch.cuda.stream(stream):
        try:
            _drive(chains, comm, step_size, n_steps, n_sweeps, False, True, halo_every, dev, stream, theta=True)
        except N.NativeError as e:  # a storm stops the device loop; the run's end reports it
            err = e
    outs = []
    for c in chains:
        iters = np.empty(n_samples, dtype=np.int64)
        par = np.empty((n_samples, 5))
        acc = np.empty(n_samples, dtype=np.int32)
        dh = np.empty(n_samples)
        stored, storm = ctypes.c_int64(0), ctypes.c_int64(-1)
        code = c.shard._lib.rsv_shard_run_end(c.shard.ctx, iters.ctypes.data, par.ctypes.data, acc.ctypes.data,
                                              dh.ctypes.data, ctypes.byref(stored), ctypes.byref(storm))
        try:
            c.shard._ck(code)
        except N.StormError as e:
            e.sweep = int(storm.value)
            raise
        outs.append((iters, par, acc.astype(bool), dh))
    if err is not None:
        raise err
    for o in outs[1:]:
        if not (np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])):
            raise RuntimeError("shards drew different parameters")
    return outs[0]
