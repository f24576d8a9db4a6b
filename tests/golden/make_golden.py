"""Generate the golden fixtures from the REFERENCE itself (build container only).

Runs the unmodified reference package (pkg/src/rsvhmc under /root/reference)
with numpy Generators over the oracle's bit generators (oracle/oracle.py
Stream, a duck-typed numpy BitGenerator), and writes small .npz fixtures
that travel to the GPU box.  Re-run with:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Nothing on the GPU box imports the reference; tests only read these files.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, "/root/reference/pkg/src")

import oracle as O  # noqa: E402
import rsvhmc  # noqa: E402
import rsvhmc.sampler as RS  # noqa: E402

TRUE = rsvhmc.Params(phi=0.97, mu=-9.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)
KINDS = ("philox", "minstd", "pcg32", "sfc64")


def gen(kind, seed):
    st = O.Stream(kind, seed)
    return st, st.generator()


def prng():
    out = {}
    for kind in KINDS:
        for seed in (0, 1, 12345):
            st = O.Stream(kind, seed)
            out[f"raw_{kind}_{seed}"] = st.raw(64)
            out[f"mat_{kind}_{seed}"] = O.seed_material(kind, seed)
            _, g = gen(kind, seed)
            out[f"normal_{kind}_{seed}"] = g.standard_normal(4096)  # numpy's own ziggurat
    # numpy's own generators, no oracle involved
    out["np_philox_raw_7"] = np.random.Philox(7).random_raw(64)
    out["np_sfc64_raw_7"] = np.random.SFC64(7).random_raw(64)
    out["np_philox_normal_7"] = np.random.Generator(np.random.Philox(7)).standard_normal(8192)
    out["np_sfc64_normal_7"] = np.random.Generator(np.random.SFC64(7)).standard_normal(8192)
    # a window with exponential-tail draws (idx == 0 attempts): find words
    st = O.Stream("philox", 2024)
    w = st.raw(62000)
    tail = np.nonzero(((w & 0xFF) == 0) & (((w >> 9) & ((1 << 52) - 1)) >= 0xEF33D8025EF6A))[0]
    out["tail_word_idx_philox_2024"] = tail[:64]
    _, g = gen("philox", 2024)
    out["normal_philox_2024"] = g.standard_normal(60000)
    np.savez_compressed(os.path.join(HERE, "prng.npz"), **out)


def model():
    out = {}
    truth = rsvhmc.simulate_rsv(TRUE, 2000, seed=0)
    out["y"], out["lrv"], out["h_true"] = truth.dataset.returns, truth.dataset.log_rv, truth.latent
    out["theta"] = np.array([TRUE.phi, TRUE.mu, TRUE.xi, TRUE.sigma_eta_sq, TRUE.sigma_u_sq])
    data = truth.dataset
    h = truth.latent
    out["log_post"] = rsvhmc.log_posterior(h, TRUE, data)
    out["grad"] = rsvhmc.grad_neg_log_posterior(h, TRUE, data)
    _, g = gen("minstd", 1)
    p = RS.refresh_momenta(g, 2000)
    out["p0"] = p
    out["ham"] = rsvhmc.hamiltonian(rsvhmc.PhaseState(h.copy(), p.copy()), TRUE, data)
    for fuse in (False, True):
        fin, div = rsvhmc.integrate_trajectory(rsvhmc.PhaseState(h.copy(), p.copy()),
                                               rsvhmc.MDConfig(0.02, 20), TRUE, data, fuse_half_steps=fuse)
        out[f"traj_h_fuse{int(fuse)}"] = fin.h
        out[f"traj_p_fuse{int(fuse)}"] = fin.p
        out[f"traj_div_fuse{int(fuse)}"] = div
        out[f"traj_ham_fuse{int(fuse)}"] = rsvhmc.hamiltonian(fin, TRUE, data)
    st = rsvhmc.PhaseState(h.copy(), p.copy())
    rsvhmc.elementary_step(st, rsvhmc.MDConfig(0.02, 1), TRUE, data)
    out["estep_h"], out["estep_p"] = st.h, st.p
    # divergent trajectory (integrator test analogue: huge momenta)
    _, div = rsvhmc.integrate_trajectory(rsvhmc.PhaseState(h.copy(), np.full(2000, 1e4)),
                                         rsvhmc.MDConfig(0.5, 20), TRUE, data)
    out["div_flag"] = div
    np.savez_compressed(os.path.join(HERE, "model_T2000.npz"), **out)


def hmc_sequence(kind="minstd", seed=1, n=40):
    """Config 1: T=2000, L=20, dt=0.02, minstd; 40 proposals at fixed theta."""
    truth = rsvhmc.simulate_rsv(TRUE, 2000, seed=0)
    data = truth.dataset
    _, h0 = RS.default_init(data)
    # start from the truth-shifted init so proposals are mostly accepted
    h = truth.latent.copy()
    st, g = gen(kind, seed)
    md = rsvhmc.MDConfig(0.02, 20)
    acc, dhs, pos, hs = [], [], [], []
    for i in range(n):
        h, a, dh = rsvhmc.hmc_update_volatility(h, TRUE, data, md, g)
        acc.append(a)
        dhs.append(dh)
        pos.append(st.pos)
        if i in (0, 1, n - 1):
            hs.append(h.copy())
    np.savez_compressed(os.path.join(HERE, f"hmc_{kind}.npz"), accept=np.array(acc), delta_h=np.array(dhs),
                        pos=np.array(pos, dtype=np.uint64), h_first=hs[0], h_second=hs[1], h_last=hs[2],
                        h_start=truth.latent, seed=seed)


def hmc_divergent():
    truth = rsvhmc.simulate_rsv(TRUE, 512, seed=3)
    st, g = gen("pcg32", 9)
    md = rsvhmc.MDConfig(0.9, 30)
    res = [rsvhmc.hmc_update_volatility(truth.latent.copy(), TRUE, truth.dataset, md, g) for _ in range(3)]
    np.savez_compressed(os.path.join(HERE, "hmc_divergent.npz"), accept=np.array([r[1] for r in res]),
                        delta_h=np.array([r[2] for r in res]), pos=np.uint64(st.pos), y=truth.dataset.returns,
                        lrv=truth.dataset.log_rv, h=truth.latent)


def chain(kind="pcg32", seed=3, T=200, n=60):
    truth = rsvhmc.simulate_rsv(rsvhmc.Params(0.95, -1.0, -0.3, 0.05, 0.1), T, seed=24)
    keep = {}

    def mk(s):
        st, g = gen(kind, s)
        keep["st"] = st
        return g

    old = RS.make_rng
    RS.make_rng = mk
    try:
        cfg = rsvhmc.SamplerConfig(seed=seed, md=rsvhmc.MDConfig(0.05, 10), n_burnin=0, n_samples=n, thin=1,
                                   store_latent=True)
        ch = rsvhmc.run_chain(truth.dataset, cfg)
    finally:
        RS.make_rng = old
    np.savez_compressed(os.path.join(HERE, f"chain_{kind}.npz"), y=truth.dataset.returns, lrv=truth.dataset.log_rv,
                        phi=ch.phi, mu=ch.mu, xi=ch.xi, sigma_eta_sq=ch.sigma_eta_sq, sigma_u_sq=ch.sigma_u_sq,
                        accept=ch.accept, delta_h=ch.delta_h, latent_last=ch.latent[-1], seed=seed,
                        pos=np.uint64(keep["st"].pos))


def formats():
    """Files written by the reference's own data.py writers (data.py:154-327)
    and what its readers return, for tests/test_formats.py."""
    import rsvhmc.data as RD
    out_dir = os.path.join(HERE, "formats")
    os.makedirs(out_dir, exist_ok=True)
    truth = RD.simulate_rsv(TRUE, 40, seed=3)
    ds = truth.dataset
    RD.save_dataset(ds, os.path.join(out_dir, "dataset.csv"))
    RD.save_truth(truth, os.path.join(out_dir, "truth.csv"))
    n, T = 6, 40
    r = np.random.default_rng(5)
    ch = RS.Chain(iters=np.arange(100, 100 + 2 * n, 2), phi=r.uniform(0.9, 0.99, n), mu=r.normal(-9, 0.1, n),
                  xi=r.normal(-0.3, 0.01, n), sigma_eta_sq=r.uniform(0.04, 0.06, n),
                  sigma_u_sq=r.uniform(0.09, 0.11, n), accept=r.uniform(size=n) < 0.7,
                  delta_h=np.where(r.uniform(size=n) < 0.2, np.inf, r.normal(0, 1, n)),
                  latent=truth.latent[None, :] + r.normal(0, 0.01, (n, T)))
    RD.save_chain(ch, os.path.join(out_dir, "chain.csv"))
    ch.latent = None
    RD.save_chain(ch, os.path.join(out_dir, "chain_nolatent.csv"))
    # an intraday panel (written by hand: the reference only reads these)
    lines = ["date,time,return"]
    days = ["2000-01-03", "2000-01-04", "2000-01-05"]
    for d in days:
        for k in range(5):
            v = 0.0 if d == "2000-01-05" else float(r.normal(0, 0.001))
            lines.append(f"{d},{9 + k:02d}:30,{RD._fmt(v)}")
    with open(os.path.join(out_dir, "intraday.csv"), "w", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")
    panel = RD.load_intraday(os.path.join(out_dir, "intraday.csv"))
    rv = RD.compute_rv(panel)
    back = RD.load_chain(os.path.join(out_dir, "chain.csv"))
    tp, th = RD.load_truth(os.path.join(out_dir, "truth.csv"))
    np.savez_compressed(os.path.join(HERE, "formats.npz"), returns=ds.returns, rv=ds.rv, log_rv=ds.log_rv,
                        latent=truth.latent, intraday_rv=rv, chain_latent=back.latent, chain_mu=back.mu,
                        chain_dh=back.delta_h, chain_accept=back.accept, truth_h=th,
                        truth_params=np.array([tp.phi, tp.mu, tp.xi, tp.sigma_eta_sq, tp.sigma_u_sq]))


def _batch_se(x, n_batches=40):
    """Monte Carlo standard error of the mean of a correlated series by
    non-overlapping batch means."""
    x = np.asarray(x, dtype=np.float64)
    m = x.size // n_batches
    b = x[: m * n_batches].reshape(n_batches, m).mean(axis=1)
    return float(b.std(ddof=1) / np.sqrt(n_batches))


H_SITES = (0, 250, 500, 999)


def posterior_summary(ch):
    """Posterior means (theta, time-averaged h, h at H_SITES) and their batch-means errors."""
    rows = [getattr(ch, n) for n in ("phi", "mu", "xi", "sigma_eta_sq", "sigma_u_sq")]
    rows.append(ch.latent.mean(axis=1))
    rows += [ch.latent[:, t] for t in H_SITES]
    return np.array([r.mean() for r in rows]), np.array([_batch_se(r) for r in rows])


def posterior(T=1000, seed=7):
    """The reference's own chain on simulated data (T=1000, 2000 burn-in
    sweeps, 2000 samples thinned by 10, latent snapshots kept): posterior
    means of theta and h with their Monte Carlo errors, for the statistical
    parity test (tests/test_gpu_stats.py)."""
    truth = rsvhmc.simulate_rsv(rsvhmc.Params(0.95, -1.0, -0.3, 0.05, 0.1), T, seed=31)
    cfg = rsvhmc.SamplerConfig(seed=seed, md=rsvhmc.MDConfig(0.02, 30), n_burnin=2000, n_samples=2000, thin=10,
                               store_latent=True)
    ch = rsvhmc.run_chain(truth.dataset, cfg)
    mean, se = posterior_summary(ch)
    np.savez_compressed(os.path.join(HERE, "posterior_T1000.npz"), y=truth.dataset.returns,
                        lrv=truth.dataset.log_rv, mean=mean, se=se, accept_rate=float(np.mean(ch.accept)))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "posterior":
        posterior()
        sys.exit(0)
    formats()
    prng()
    model()
    hmc_sequence("minstd", 1)
    hmc_sequence("philox", 11)
    hmc_divergent()
    chain("pcg32", 3)
    chain("philox", 5)
    posterior()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
