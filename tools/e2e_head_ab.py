"""e2e with the path sent every step (a view of the returned page-locked
path, read in place by the trajectory kernel) at T = 2^20, for the head size
in RSV_ZC_HEAD (sites copied in beside the momenta kernel).  Wall clock per
call, median of 5 blocks of 40 calls.  Development aid (run under gpurun)."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402

T = 1 << 20
theta = P.Params(phi=0.97, mu=-1.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)
truth = P.simulate_rsv(theta, T, seed=0)
data = truth.dataset
md = P.MDConfig(0.02, 20)
be = P.CudaBackend(0)
rng = P.make_rng(7, "pcg32")
h = torch.empty(T, dtype=torch.float64, pin_memory=True).numpy()
h[:] = truth.latent
for _ in range(10):
    h, _, _ = P.hmc_update_volatility(h.view(), theta, data, md, rng, backend=be)
pageable = os.environ.get("E2E_PAGEABLE") == "1"  # the same plain numpy path every step
hp = truth.latent.copy()
blocks, acc = [], 0
for _ in range(5):
    t0 = time.perf_counter()
    for _ in range(40):
        if pageable:
            _, a, _ = P.hmc_update_volatility(hp, theta, data, md, rng, backend=be)
        else:
            h, a, _ = P.hmc_update_volatility(h.view(), theta, data, md, rng, backend=be)
        acc += a
    blocks.append((time.perf_counter() - t0) / 40 * 1e6)
ch = be.chain(data, theta)
print(f"pageable={pageable} RSV_NO_HOST_STAGE={os.environ.get('RSV_NO_HOST_STAGE', '-')} "
      f"RSV_ZC_HEAD={os.environ.get('RSV_ZC_HEAD', 'default')}: {statistics.median(blocks):.1f} us/call "
      f"(blocks {', '.join(f'{b:.1f}' for b in blocks)}), accepts {acc}/200, zero_copy={ch.last_update_zero_copy}")
