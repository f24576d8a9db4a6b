"""Quick device timing of the hot path (development aid, not the bench)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402

theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
for T in [2000, 1 << 14, 1 << 18, 1 << 20, 1 << 22]:
    truth = P.simulate_rsv(theta, T, seed=1)
    be = P.CudaBackend(0)
    ch = be.chain(truth.dataset, theta)
    ch.set_latent(truth.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 5)
    ch.set_timing(2)
    n = 50
    res = ch.hmc_update_many(0.02, 20, n)
    tr, mo, tot = ch.timing()
    ch.set_timing(False)
    import ctypes
    t0 = time.perf_counter()
    ch.hmc_update_many(0.02, 20, n, results=False)
    wall = (time.perf_counter() - t0) / n
    acc = np.mean([r.accept for r in res])
    print(f"T={T:8d} traj {tr*1e3:9.2f} us  momenta {mo*1e3:8.2f} us  total {tot*1e3:9.2f} us  wall/step {wall*1e6:9.2f} us"
          f"  site-upd/s(traj) {T*20/(tr*1e-3):.3e}  acc {acc:.2f}", flush=True)
    be.close()
# streamed elementary step (HBM roofline kernel)
for T in [1 << 24, 1 << 26]:
    truth = P.simulate_rsv(theta, T, seed=2)
    be = P.CudaBackend(0)
    ch = be.chain(truth.dataset, theta)
    h = truth.latent.copy(); p = np.random.default_rng(0).standard_normal(T)
    ch.elementary_step_inplace(h, p, 0.02)
    ms = ctypes.c_float()
    ch._ck(ch._lib.rsv_bench_elementary(ch.ctx, 0.02, 20, ctypes.byref(ms)))
    per = ms.value / 20
    print(f"estep T={T}: {per*1e3:.1f} us/step  {48*T/(per*1e-3)/1e9:.1f} GB/s  {T/(per*1e-3):.3e} site-upd/s", flush=True)
    be.close()
