import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1603_08114_b200 as P
from paper_1603_08114_b200.rng import stream_state, store_stream_state
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
T = 1 << 20
tr = P.simulate_rsv(theta, T, seed=0)
be = P.CudaBackend(0)
rng = P.make_rng(7, "pcg32")
md = P.MDConfig(0.02, 20)
h = torch.empty(T, dtype=torch.float64, pin_memory=True).numpy(); h[:] = tr.latent
for _ in range(3):
    h, a, d = P.hmc_update_volatility(h, theta, tr.dataset, md, rng, backend=be)
tt = {}
def tic(k, t0):
    tt[k] = tt.get(k, 0) + time.perf_counter() - t0
n = 20
for _ in range(n):
    t0 = time.perf_counter(); ch = be.chain(tr.dataset, theta); tic("chain", t0)
    t0 = time.perf_counter(); ch.set_latent(h); tic("set_latent", t0)
    t0 = time.perf_counter(); ch.set_stream(stream_state(rng)); tic("set_stream", t0)
    t0 = time.perf_counter(); r = ch.hmc_update(0.02, 20, False, stats=False); tic("hmc_update", t0)
    t0 = time.perf_counter(); store_stream_state(rng, ch.get_stream()); tic("store_stream", t0)
    t0 = time.perf_counter(); h2 = ch.get_latent(); tic("get_latent", t0)
print({k: round(v / n * 1e6, 1) for k, v in tt.items()}, "us")
ts = []
acc = 0
for _ in range(20):
    t0 = time.perf_counter()
    h, a, d = P.hmc_update_volatility(h, theta, tr.dataset, md, rng, backend=be)
    ts.append(time.perf_counter() - t0)
    acc += a
print("hmc_update_volatility us:", [round(x * 1e6) for x in ts], "accepted", acc)
