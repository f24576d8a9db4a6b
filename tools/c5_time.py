"""Config 5 run_chain timing vs number of sweeps (fixed-cost check, dev aid)."""
import sys, time
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
T = 1 << 26
be = P.CudaBackend(0)
tr = P.simulate_rsv(theta, T, seed=11, backend=be)
ch = be.chain(tr.dataset, theta)
ch.set_blocked_streams(1, 4096)
cfg = P.SamplerConfig(seed=1, md=P.MDConfig(0.005, 20), n_burnin=0, n_samples=3, prng="sfc64")
P.run_chain(tr.dataset, cfg, backend=be, init_params=theta, init_h=tr.latent)
for n in (1, 20, 20, 100):
    t0 = time.perf_counter()
    ch.run_chain_device(0.005, 20, False, P.PriorSpec(), 0, n, 1)
    el = time.perf_counter() - t0
    print(f"sweeps {n}: {el*1e3:.1f} ms total, {el/n*1e3:.3f} ms/sweep", flush=True)
