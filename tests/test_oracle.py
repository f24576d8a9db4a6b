"""The CPU oracle (oracle/, test infrastructure) pinned against the reference.

Golden fixtures in tests/golden/ were produced by running the reference itself
(tests/golden/make_golden.py) and numpy's own bit generators; these tests
check the oracle's restatement against them, plus canonical PRNG KATs."""
import math

import numpy as np
import pytest

import oracle as O
from conftest import TRUE, golden

KINDS = ["philox", "minstd", "pcg32", "sfc64"]


class _P:
    def __init__(self, **kw):
        self.__dict__.update(kw)


THETA = _P(**TRUE)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("seed", [0, 1, 12345])
def test_raw_words_and_normals(kind, seed):
    z = golden("prng.npz")
    assert np.array_equal(O.seed_material(kind, seed), z[f"mat_{kind}_{seed}"])
    assert np.array_equal(O.Stream(kind, seed).raw(64), z[f"raw_{kind}_{seed}"])
    got = O.Stream(kind, seed).normals(4096)
    assert np.array_equal(got.view(np.uint64), z[f"normal_{kind}_{seed}"].view(np.uint64))


def test_numpy_generators_direct():
    z = golden("prng.npz")
    assert np.array_equal(O.Stream("philox", 7).raw(64), z["np_philox_raw_7"])
    assert np.array_equal(O.Stream("sfc64", 7).raw(64), z["np_sfc64_raw_7"])
    assert np.array_equal(O.Stream("philox", 7).normals(8192), z["np_philox_normal_7"])
    assert np.array_equal(O.Stream("sfc64", 7).normals(8192), z["np_sfc64_normal_7"])
    # and against numpy live
    assert np.array_equal(O.Stream("philox", 99).raw(100), np.random.Philox(99).random_raw(100))
    assert np.array_equal(O.Stream("philox", 99).normals(1000),
                          np.random.Generator(np.random.Philox(99)).standard_normal(1000))


def test_tail_draws_exact():
    z = golden("prng.npz")
    assert len(z["tail_word_idx_philox_2024"]) >= 10
    got = O.Stream("philox", 2024).normals(60000)
    assert np.array_equal(got.view(np.uint64), z["normal_philox_2024"].view(np.uint64))


def test_canonical_kats():
    # std::minstd_rand with seed 1: the 10000th output is 399268537 (C++ [rand.predef])
    st = O.Stream("minstd", material=np.array([1, 0, 0, 0], dtype=np.uint64))
    w = st.raw(3334)
    assert int(w[3333]) >> 33 == 399268537
    # pcg32_srandom_r(42, 54) (pcg_basic demo): 0xa15c02b7 0x7b47f409 0xba1d3330 ...
    st = O.Stream("pcg32", material=np.array([42, 54, 0, 0], dtype=np.uint64))
    w = st.raw(2)
    assert int(w[0]) == (0xA15C02B7 << 32) | 0x7B47F409
    assert int(w[1]) >> 32 == 0xBA1D3330


def test_log1p_matches_glibc():
    rng = np.random.default_rng(0)
    xs = np.concatenate([-rng.random(200000), -rng.random(2000) * 1e-9, -1 + rng.random(2000) * 1e-6,
                         -rng.random(2000) * 0.29])
    assert all(O.log1p(float(x)) == math.log1p(float(x)) for x in xs)


def test_generator_consumption_matches_numpy():
    # numpy Generator over the oracle stream consumes exactly the oracle's words
    for kind in KINDS:
        a = O.Stream(kind, 5)
        g = a.generator()
        g.standard_normal(5000)
        b = O.Stream(kind, 5)
        b.normals(5000)
        assert a.state_words() == b.state_words()


def test_model_vs_reference():
    z = golden("model_T2000.npz")
    y, lrv, h, p = z["y"], z["lrv"], z["h_true"], z["p0"]
    lp = O.log_posterior(h, THETA, y, lrv)
    assert abs(lp - float(z["log_post"])) <= 1e-13 * abs(float(z["log_post"]))
    H = O.hamiltonian(h, p, THETA, y, lrv)
    assert abs(H - float(z["ham"])) <= 1e-13 * abs(H)
    g, div = O.gradient(h, THETA, y, lrv)
    assert not div
    assert np.max(np.abs(g - z["grad"])) <= 1e-13 * np.max(np.abs(z["grad"]))


@pytest.mark.parametrize("fuse", [False, True])
def test_trajectory_vs_reference(fuse):
    z = golden("model_T2000.npz")
    hh, pp, div = O.integrate(z["h_true"], z["p0"], THETA, z["y"], z["lrv"], 0.02, 20, fuse=fuse)
    assert not div
    # same arithmetic as the numba kernels; only libm exp could differ
    assert np.max(np.abs(hh - z[f"traj_h_fuse{int(fuse)}"])) <= 1e-13
    assert np.max(np.abs(pp - z[f"traj_p_fuse{int(fuse)}"])) <= 1e-13


def test_multithreaded_oracle_is_bitwise_thread_independent():
    z = golden("model_T2000.npz")
    a = O.integrate(z["h_true"], z["p0"], THETA, z["y"], z["lrv"], 0.02, 20, nthreads=1)
    b = O.integrate(z["h_true"], z["p0"], THETA, z["y"], z["lrv"], 0.02, 20, nthreads=4)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("kind,seed", [("minstd", 1), ("philox", 11)])
def test_hmc_sequence_vs_reference(kind, seed):
    z = golden("model_T2000.npz")
    g = golden(f"hmc_{kind}.npz")
    st = O.Stream(kind, seed)
    h = g["h_start"].copy()
    H = abs(float(z["ham"]))
    for i in range(len(g["accept"])):
        h, acc, dh = O.hmc_update(h, THETA, z["y"], z["lrv"], 0.02, 20, st)
        assert acc == bool(g["accept"][i])
        assert abs(dh - float(g["delta_h"][i])) <= 1e-13 * H
        assert st.pos == int(g["pos"][i])
    assert np.max(np.abs(h - g["h_last"])) <= 1e-12


def test_divergent_sentinel_vs_reference():
    g = golden("hmc_divergent.npz")
    st = O.Stream("pcg32", 9)
    for i in range(3):
        _, acc, dh = O.hmc_update(g["h"], THETA, g["y"], g["lrv"], 0.9, 30, st)
        assert not acc and math.isinf(dh)
    assert st.pos == int(g["pos"])
