"""Config-4 ensemble timing (dev aid): C chains x Tc sites, sfc64 per chain."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1603_08114_b200 as P
C = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
Tc = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
tr = P.simulate_rsv(theta, Tc, seed=0)
ens = P.Ensemble(C, Tc)
ens.set_data(tr.dataset.returns, tr.dataset.log_rv)
ens.set_params(theta)
ens.set_latent(tr.latent)
ens.seed(1)
ens.hmc_update(0.02, 20, rounds=3)
ens.set_timing(1)
ens.hmc_update(0.02, 20, rounds=10)
ms = ens.timing_ms()
ens.set_timing(0)
t0 = time.perf_counter()
for _ in range(3):
    ens.refresh_momenta()
mom = (time.perf_counter() - t0) / 3
a, d = ens.counts()
print(f"C={C} Tc={Tc}: {ms*1e3:.1f} us/round  {C*Tc*20/(ms*1e-3):.3e} site-updates/s  "
      f"{C/(ms*1e-3):.3e} chain-trajectories/s  accept {a.sum()/(13*C):.3f}  (refresh_momenta wall incl. D2H {mom*1e3:.2f} ms)")
import ctypes
st = (ctypes.c_uint64 * 5)()
P._native.check(ens._lib.rsv_kernel_stamps(ens.ctx, st), ens.ctx)
print(f"  trajectory kernel (in-kernel): {(st[3] - st[2]) / 1e3:.1f} us")
