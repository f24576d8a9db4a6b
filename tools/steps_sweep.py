import sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
for T in [1 << 14, 1 << 20]:
    tr = P.simulate_rsv(theta, T, seed=1)
    be = P.CudaBackend(0)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    for L in [1, 2, 5, 10, 20, 40]:
        ch.hmc_update_many(0.02, L, 3, results=False)
        ch.set_timing(2)
        ch.hmc_update_many(0.02, L, 20, results=False)
        t, m, tot = ch.timing()
        ch.set_timing(False)
        print(f"T={T} L={L:3d} traj {t*1e3:8.2f} us  per-step {t*1e3/L:7.2f} us", flush=True)
    be.close()
