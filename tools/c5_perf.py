import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
T = 1 << 26
t0 = time.perf_counter(); tr = P.simulate_rsv(theta, T, seed=11); print("simulate", time.perf_counter() - t0)
be = P.CudaBackend(0)
ch = be.chain(tr.dataset, theta)
ch.set_latent(tr.latent)
ch.set_stream(P.stream_state(P.make_rng(1, "sfc64")))
t0 = time.perf_counter(); ch.set_blocked_streams(1, 4096); print("seed blocks", time.perf_counter() - t0)
for dt in (0.02, 0.005):
    ch.hmc_update_many(dt, 20, 2, results=False)
    ch.set_timing(1)
    res = ch.hmc_update_many(dt, 20, 5, results=True)
    _, _, tot = ch.timing()
    ch.set_timing(0)
    k = ch.kernel_stamps()
    print(f"dt={dt}: proposal {tot:.3f} ms, traj in-kernel {k['trajectory_us']:.0f} us, accept {np.mean([r.accept for r in res])}")
import ctypes
t0 = time.perf_counter(); ch.refresh_momenta(); print("refresh_momenta (incl D2H 512MB)", time.perf_counter() - t0)
cfg = P.SamplerConfig(seed=2, md=P.MDConfig(0.005, 20), n_burnin=0, n_samples=10, prng="sfc64")
t0 = time.perf_counter(); out = P.run_chain(tr.dataset, cfg, backend=be, init_params=theta, init_h=tr.latent); el = time.perf_counter() - t0
print("run_chain 10 sweeps", el, "accept", out.accept.mean())
