"""Momenta / trajectory split of one proposal with and without the L2 flush (dev aid)."""
import sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
be = P.CudaBackend(0)
for T in [2000, 1 << 16, 1 << 20]:
    tr = P.simulate_rsv(theta, T, seed=1)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 5, results=False)
    for fl in (0, 256 << 20):
        ch.set_l2_flush(fl)
        ch.set_timing(2)
        ch.hmc_update_many(0.02, 20, 50, results=False)
        t, m, s = ch.timing()
        ch.set_timing(False)
        print(f"T={T} flush={fl>>20}MiB: momenta {m*1e3:.1f} us traj {t*1e3:.1f} us proposal {s*1e3:.1f} us")
    ch.set_l2_flush(0)
