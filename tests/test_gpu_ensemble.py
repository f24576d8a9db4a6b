"""GPU parity of the chain ensemble (BASELINE config 4): every chain of an
``Ensemble`` must do exactly what the reference's single-chain
hmc_update_volatility (sampler.py:144-167) does with that chain's own
``Generator(SFC64(SeedSequence([seed, c])))`` -- bit-exact momenta and
stream positions, the same accept sequence, h and dH to the tolerances of
test_gpu_parity.py."""
import numpy as np
import pytest

import oracle as O
import paper_1603_08114_b200 as P
from conftest import TRUE

pytestmark = pytest.mark.gpu

THETA = P.Params(**TRUE)


def _sims(C, Tc, base=100):
    sims = [P.simulate_rsv(THETA, Tc, seed=base + c) for c in range(C)]
    y = np.stack([s.dataset.returns for s in sims])
    lrv = np.stack([s.dataset.log_rv for s in sims])
    h = np.stack([s.latent for s in sims])
    return y, lrv, h


def test_ensemble_momenta_bit_exact_per_chain():
    C, Tc, seed = 5, 200, 7
    gens = [np.random.Generator(np.random.SFC64(np.random.SeedSequence([seed, c]))) for c in range(C)]
    with P.Ensemble(C, Tc) as ens:
        ens.seed(seed)
        for _ in range(2):  # two draws: the streams continue exactly
            got = ens.refresh_momenta()
            st = ens.streams()
            for c in range(C):
                want = gens[c].standard_normal(Tc)
                assert np.array_equal(got[c].view(np.uint64), want.view(np.uint64)), c
                assert [int(x) for x in st[c]] == [int(x) for x in gens[c].bit_generator.state["state"]["state"]]


@pytest.mark.parametrize("C,Tc", [(1, 64), (29, 64), (30, 1032), (61, 200), (59, 4096)])
def test_ensemble_momenta_pipeline_shapes(C, Tc):
    """The ensemble momenta kernel's chunk pipeline (29 chains per CTA,
    64-word chunks): partial CTAs, chains shorter than a chunk, chains ending
    mid-chunk, three consecutive draws -- every chain bit-exact against
    numpy's own SFC64 stream, and the streams continue exactly."""
    seed = 3
    gens = [np.random.Generator(np.random.SFC64(np.random.SeedSequence([seed, c]))) for c in range(C)]
    with P.Ensemble(C, Tc) as ens:
        ens.seed(seed)
        for _ in range(3):
            got = ens.refresh_momenta()
            st = ens.streams()
            for c in range(C):
                want = gens[c].standard_normal(Tc)
                assert np.array_equal(got[c].view(np.uint64), want.view(np.uint64)), c
                assert [int(x) for x in st[c]] == [int(x) for x in gens[c].bit_generator.state["state"]["state"]]


@pytest.mark.parametrize("fuse", [False, True])
def test_ensemble_matches_single_chain_oracle(fuse):
    C, Tc, L, dt, seed = 6, 256, 12, 0.03, 11
    y, lrv, h0 = _sims(C, Tc)
    streams = [O.Stream("sfc64", np.random.SeedSequence([seed, c])) for c in range(C)]
    h = h0.copy()
    with P.Ensemble(C, Tc) as ens:
        ens.set_data(y, lrv)
        ens.set_params(THETA)
        ens.set_latent(h0)
        ens.seed(seed)
        n_acc = np.zeros(C, dtype=int)
        # |H| of each chain bounds the dH error (the reference's own dH error is ~3e-16 |H|)
        Hc = [abs(O.hamiltonian(h0[c], np.zeros(Tc), THETA, y[c], lrv[c])) + Tc for c in range(C)]
        for _ in range(4):
            acc, dh = ens.hmc_update(dt, L, fuse=fuse)
            for c in range(C):
                # the oracle's proposal in the same grouping (fuse_half_steps, integrator.py:149)
                hc, a, d = O.hmc_update(h[c], THETA, y[c], lrv[c], dt, L, streams[c], fuse=fuse)
                assert abs(dh[c] - d) <= 1e-13 * Hc[c], (c, dh[c], d)
                assert bool(acc[c]) == a, c
                h[c] = hc
                n_acc[c] += int(a)
        got = ens.latent()
        assert np.max(np.abs(got - h)) <= 1e-12 * max(1.0, float(np.max(np.abs(h))))
        st = ens.streams()
        for c in range(C):
            assert [int(x) for x in st[c]] == streams[c].state_words()[0]
        a, d = ens.counts()
        assert np.array_equal(a, n_acc) and not d.any()


def test_ensemble_divergent_chain_rejects_without_uniform():
    # chain 1 gets a step size so large that it diverges; the other chains
    # are unaffected and its stream must not consume the Metropolis uniform
    C, Tc, L, seed = 3, 128, 8, 5
    y, lrv, h0 = _sims(C, Tc, base=300)
    h0[1, 40] = 49.9  # next to the |h| <= 50 boundary: the first kick leaves it
    streams = [O.Stream("sfc64", np.random.SeedSequence([seed, c])) for c in range(C)]
    with P.Ensemble(C, Tc) as ens:
        ens.set_data(y, lrv)
        ens.set_params(THETA)
        ens.set_latent(h0)
        ens.seed(seed)
        acc, dh = ens.hmc_update(0.5, L)
        for c in range(C):
            hc, a, d = O.hmc_update(h0[c], THETA, y[c], lrv[c], 0.5, L, streams[c])
            assert bool(acc[c]) == a
            if np.isinf(d):
                assert np.isinf(dh[c])
            else:
                assert abs(dh[c] - d) <= 1e-9 * max(1.0, abs(d))
        st = ens.streams()
        for c in range(C):
            assert [int(x) for x in st[c]] == streams[c].state_words()[0]
        assert np.isinf(dh[1])


def test_ensemble_rejects_bad_shapes():
    with pytest.raises(ValueError):
        P.Ensemble(2, 100)  # chain length must be a multiple of 8
    with P.Ensemble(2, 64) as ens:
        with pytest.raises(ValueError):
            ens.set_latent(np.zeros((3, 64)))
        with pytest.raises(RuntimeError):
            ens.hmc_update(0.02, 5)  # nothing set yet


def test_paper_protocol_smoke(tmp_path):
    from paper_1603_08114_b200 import bench_protocol as BP
    study = BP.run_scaling_study(BP.BenchConfig(b_values=(2, 4), reps=200, repeats=2), fused=True)
    for name in ("cuda", "cuda_fused"):
        pts = study.timings[name]
        assert [p.b for p in pts] == [2, 4] and all(p.mean_seconds > 0 for p in pts)
    # a fused 100-step segment is one launch: far below 100 streamed launches
    assert study.timings["cuda_fused"][0].mean_seconds < study.timings["cuda"][0].mean_seconds
    paths = BP.emit_report(study, tmp_path)
    lines = paths["fits"].read_text().splitlines()
    assert lines[1] == "backend,intercept_a,slope_c,r_squared" and lines[3].startswith("cuda_fused,")


@pytest.mark.parametrize("T", [2, 1000, 70001])
def test_simulate_on_device_matches_host(T):
    # the same normals bit for bit; the AR(1) path by a parallel scan agrees
    # with the sequential recursion to rounding
    be = P.CudaBackend(0)
    a = P.simulate_rsv(THETA, T, seed=17)
    b = P.simulate_rsv(THETA, T, seed=17, backend=be)
    rel = lambda x, y: float(np.max(np.abs(x - y)) / max(1.0, float(np.max(np.abs(y)))))
    assert rel(b.latent, a.latent) <= 1e-12
    assert rel(b.dataset.log_rv, a.dataset.log_rv) <= 1e-12
    assert float(np.max(np.abs(b.dataset.returns - a.dataset.returns) / np.abs(a.dataset.returns).clip(1e-300))) <= 1e-12
    be.close()
