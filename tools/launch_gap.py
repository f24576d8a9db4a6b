"""Where does the proposal's event-timed step go beyond the kernels? (development aid)"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402

theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
tr = P.simulate_rsv(theta, T, seed=1)
be = P.CudaBackend(0)
ch = be.chain(tr.dataset, theta)
ch.set_latent(tr.latent)
ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
ch.hmc_update_many(0.02, 20, 10, results=False)
for flush in (256 << 20, 0):
    ch.set_l2_flush(flush)
    ch.set_timing(1)
    ch.hmc_update_many(0.02, 20, 40, results=False)
    _, _, step = ch.timing()
    ch.set_timing(0)
    ch.set_l2_flush(0)
    print(f"flush={flush>>20} MiB: event-timed proposal {step*1e3:.2f} us", flush=True)
ks = []
for _ in range(20):
    ch.hmc_update_many(0.02, 20, 1, results=False)
    ks.append(ch.kernel_stamps())
print("in-kernel:", {k: round(float(np.median([x[k] for x in ks])), 2) for k in ks[0]})
print(f"trajectory alone (events around 20 launches): {ch.bench_trajectory(0.02, 20, 20)*1e3:.2f} us")
import time
import torch
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
x = torch.zeros(1, device="cuda")
e0.record(); x.add_(1); e1.record(); torch.cuda.synchronize()
for _ in range(5):
    e0.record(); x.add_(1); e1.record(); torch.cuda.synchronize()
print(f"event pair around one tiny kernel: {e0.elapsed_time(e1)*1e3:.2f} us")
be.close()
