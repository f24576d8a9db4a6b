"""Small-T timings: proposals (hmc_update_many) and run_chain sweeps/s,
cluster vs tiled (development aid)."""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402
from paper_1603_08114_b200.integrator import DeviceChain  # noqa: E402

theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
for tiled in (False, True):
    if tiled:
        os.environ["RSV_NO_CLUSTER"] = "1"
    for T in (1024, 2000, 4000):
        tr = P.simulate_rsv(theta, T, seed=1)
        ch = DeviceChain(T, 0)
        ch.set_data(tr.dataset)
        ch.set_params(theta)
        ch.set_latent(tr.latent)
        ch.set_stream(P.stream_state(P.make_rng(1, "minstd")))
        ch.hmc_update_many(0.02, 20, 50, results=False)
        ch.set_timing(1)
        ch.hmc_update_many(0.02, 20, 50, results=False)
        _, _, step = ch.timing()
        ch.set_timing(0)
        n = 2000
        t0 = time.perf_counter()
        ch.hmc_update_many(0.02, 20, n, results=False)
        wall = (time.perf_counter() - t0) / n
        ch.run_chain_device(0.02, 20, False, P.PriorSpec(), 0, 20, 1)
        ns = 3000
        t0 = time.perf_counter()
        ch.run_chain_device(0.02, 20, False, P.PriorSpec(), 0, ns, 1)
        sw = (time.perf_counter() - t0) / ns
        print(f"{'tiled' if tiled else 'cluster'} T={T}: event-timed proposal {step*1e3:.2f} us, "
              f"{n} proposals in one call {wall*1e6:.2f} us each, run_chain {1/sw:.0f} sweeps/s ({sw*1e6:.2f} us)",
              flush=True)
        ch.close()
