"""Per-proposal time from host wall clock over many graph launches, with and
without the timing event nodes (dev aid)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
be = P.CudaBackend(0)
for T in [2000, 1 << 16, 1 << 20]:
    tr = P.simulate_rsv(theta, T, seed=1)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 5, results=False)
    for timing in (False, True):
        ch.set_timing(timing)
        ch.hmc_update_many(0.02, 20, 5, results=False)
        torch.cuda.synchronize()
        n = 400
        t0 = time.perf_counter()
        ch.hmc_update_many(0.02, 20, n, results=False)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
        extra = ""
        if timing:
            t, m, s = ch.timing()
            extra = f" (events: mom {m*1e3:.1f} traj {t*1e3:.1f} total {s*1e3:.1f})"
        print(f"T={T} timing={timing}: wall {dt*1e6:.1f} us/proposal{extra}")
    ch.set_timing(False)
