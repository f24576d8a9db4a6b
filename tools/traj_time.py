"""Trajectory-kernel timing at T (development aid): in-kernel stamps and
event-node breakdown of the proposal graph, plus per-CTA phase stamps."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402

theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
for T in [int(a) for a in sys.argv[1:]] or [1 << 20]:
    tr = P.simulate_rsv(theta, T, seed=1)
    be = P.CudaBackend(0)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 10, results=False)
    ch.set_timing(1)
    ch.hmc_update_many(0.02, 20, 50, results=False)
    _, _, step = ch.timing()
    ch.set_timing(2)
    ch.hmc_update_many(0.02, 20, 50, results=False)
    tq, mq, _ = ch.timing()
    ch.set_timing(0)
    ks = []
    for _ in range(20):
        ch.hmc_update_many(0.02, 20, 1, results=False)
        ks.append(ch.kernel_stamps()["trajectory_us"])
    print(f"T={T}: proposal {step*1e3:.2f} us, traj(event nodes) {tq*1e3:.2f} us, momenta {mq*1e3:.2f} us, "
          f"traj in-kernel median {np.median(ks):.2f} us (min {min(ks):.2f})", flush=True)
    be.close()
