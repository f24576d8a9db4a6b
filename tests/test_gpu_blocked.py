"""Blocked momenta layout (BASELINE config 5, SURVEY §7(ii) -- a documented
deviation from the reference's single stream): sites [j*B, (j+1)*B) draw
their momenta from SFC64(SeedSequence([seed, j])); the chain's own stream
supplies only the Metropolis uniform and the theta draws.  The oracle is
numpy itself (per-block standard_normal) plus the CPU trajectory."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1603_08114_b200 as P
from conftest import TRUE

pytestmark = pytest.mark.gpu
THETA = P.Params(**TRUE)


def _block_normals(gens, B):
    return np.concatenate([g.standard_normal(B) for g in gens])


def test_blocked_momenta_bit_exact_and_streams_advance():
    B, nb, seed = 512, 8, 21
    ch = P.DeviceChain(B * nb)
    ch.set_stream(P.stream_state(P.make_rng(3, "pcg32")))
    ch.set_blocked_streams(seed, B)
    gens = [np.random.Generator(np.random.SFC64(np.random.SeedSequence([seed, j]))) for j in range(nb)]
    pos0 = ch.get_stream().pos
    for _ in range(2):
        got = ch.refresh_momenta()
        want = _block_normals(gens, B)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    st = ch.blocked_streams()
    for j in range(nb):
        assert [int(x) for x in st[j]] == [int(x) for x in gens[j].bit_generator.state["state"]["state"]]
    assert ch.get_stream().pos == pos0  # the main stream is not used by the momenta
    ch.set_blocked_streams(None)
    ch.close()


@pytest.mark.parametrize("kind", ["sfc64", "philox"])
def test_blocked_proposals_match_oracle(kind):
    B, nb, seed, L, dt = 256, 8, 4, 12, 0.03
    T = B * nb
    tr = P.simulate_rsv(THETA, T, seed=9)
    y, lrv = tr.dataset.returns, tr.dataset.log_rv
    ch = P.DeviceChain(T)
    ch.set_data(tr.dataset)
    ch.set_params(THETA)
    h = tr.latent.copy()
    ch.set_latent(h)
    main = P.make_rng(8, kind)
    ch.set_stream(P.stream_state(main))
    ch.set_blocked_streams(seed, B)
    gens = [np.random.Generator(np.random.SFC64(np.random.SeedSequence([seed, j]))) for j in range(nb)]
    ref_main = P.make_rng(8, kind)
    for _ in range(4):
        r = ch.hmc_update(dt, L, stats=False)
        p = _block_normals(gens, B)
        h2, p2, div = O.integrate(h, p, THETA, y, lrv, dt, L)
        assert not div
        dh = O.hamiltonian(h2, p2, THETA, y, lrv) - O.hamiltonian(h, p, THETA, y, lrv)
        u = ref_main.random()
        acc = dh <= 0.0 or u < math.exp(-dh)
        assert bool(r.accept) == acc
        assert abs(r.delta_h - dh) <= 1e-9 * max(1.0, abs(dh))
        if acc:
            h = h2
    got = ch.get_latent()
    assert np.max(np.abs(got - h)) <= 1e-10 * np.max(np.abs(h))
    st = P.stream_state(ref_main)
    dev = ch.get_stream()
    if kind == "sfc64":
        assert [int(x) for x in dev.s] == [int(x) for x in st.s]
    else:
        assert int(dev.pos) == int(st.pos)
    ch.close()


def test_blocked_run_chain_on_device():
    # a short device run_chain in the blocked layout: runs, keeps the stream
    # bookkeeping consistent, and its theta draws use the main stream only
    B, nb = 512, 8
    tr = P.simulate_rsv(THETA, B * nb, seed=2)
    be = P.CudaBackend(0)
    ch = be.chain(tr.dataset, THETA)
    ch.set_blocked_streams(5, B)
    cfg = P.SamplerConfig(seed=1, md=P.MDConfig(0.02, 20), n_burnin=5, n_samples=20, prng="sfc64")
    out = P.run_chain(tr.dataset, cfg, backend=be, init_params=THETA, init_h=tr.latent)
    assert len(out) == 20 and np.all(np.isfinite(out.mu)) and out.accept.mean() > 0.3
    ch.set_blocked_streams(None)
    be.close()
