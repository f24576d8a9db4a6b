"""run_chain sweeps/s: theta draws on the host vs on the device (dev aid)."""
import sys, time
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
be = P.CudaBackend(0)
for T in [2000, 1 << 14, 1 << 20]:
    tr = P.simulate_rsv(theta, T, seed=0)
    for mode in ("host", "device"):
        n = 400 if T < (1 << 20) else 100
        cfg = P.SamplerConfig(seed=1, md=P.MDConfig(0.02, 20), n_burnin=20, n_samples=20, thin=1, prng="pcg32")
        P.run_chain(tr.dataset, cfg, backend=be, theta_on=mode, init_params=theta, init_h=tr.latent)
        cfg = P.SamplerConfig(seed=1, md=P.MDConfig(0.02, 20), n_burnin=0, n_samples=n, thin=1, prng="pcg32")
        t0 = time.perf_counter()
        ch = P.run_chain(tr.dataset, cfg, backend=be, theta_on=mode, init_params=theta, init_h=tr.latent)
        dt = time.perf_counter() - t0
        print(f"T={T} theta_on={mode}: {n/dt:9.0f} sweeps/s  ({dt/n*1e6:8.1f} us/sweep)  accept {ch.accept.mean():.2f}", flush=True)
