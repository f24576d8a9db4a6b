"""Where the time of one host-buffer proposal goes (development aid):
python wrapper vs C call vs device (kernel %globaltimer stamps)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1603_08114_b200 as P  # noqa: E402
from paper_1603_08114_b200.rng import stream_state  # noqa: E402

theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
tr = P.simulate_rsv(theta, T, seed=0)
be = P.CudaBackend(0)
rng = P.make_rng(7, "pcg32")
md = P.MDConfig(0.02, 20)
h = torch.empty(T, dtype=torch.float64, pin_memory=True).numpy()
h[:] = tr.latent
for _ in range(5):
    h, a, d = P.hmc_update_volatility(h, theta, tr.dataset, md, rng, backend=be)
ch = be.chain(tr.dataset, theta)
n = 20
tc = []
for _ in range(n):
    st = stream_state(rng)
    t0 = time.perf_counter()
    r, out = ch.hmc_update_host(h, st, 0.02, 20)
    tc.append((time.perf_counter() - t0) * 1e6)
    ks = ch.kernel_stamps() if hasattr(ch, "kernel_stamps") else None
    print(f"C call {tc[-1]:.0f} us accept {bool(r.accept)} mode {ch._lib.rsv_last_update_zero_copy(ch.ctx)} "
          f"stamps {ks}", file=sys.stderr)
tw = []
for _ in range(n):
    t0 = time.perf_counter()
    h, a, d = P.hmc_update_volatility(h, theta, tr.dataset, md, rng, backend=be)
    tw.append((time.perf_counter() - t0) * 1e6)
print("wrapper us", [round(x) for x in tw], file=sys.stderr)
