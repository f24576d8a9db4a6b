"""Per-tile phase timestamps of the trajectory kernel (RSV_TRAJ_STAMPS=1)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ["RSV_TRAJ_STAMPS"] = "1"
import paper_1603_08114_b200 as P  # noqa: E402
from paper_1603_08114_b200 import _native as N  # noqa: E402

L = N.lib()
L.rsv_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
for T, Lsteps in [(1 << 14, 20), (1 << 14, 1), (1 << 20, 20)]:
    tr = P.simulate_rsv(theta, T, seed=1)
    be = P.CudaBackend(0)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, Lsteps, 3, results=False)
    st = np.zeros((20000, 8), dtype=np.uint64)
    N.check(L.rsv_debug_stamps(ch.ctx, st.ctypes.data, 20000), ch.ctx)
    st = st[st[:, 0] > 0].astype(np.int64)
    t0 = st[:, 0].min()
    rel = st - t0
    ph = np.diff(st[:, :5], axis=1)
    print(f"T={T} L={Lsteps} tiles={len(st)} kernel span {(st[:, 4].max() - t0)/1e3:.1f} us (+metropolis "
          f"{(st[:,5].max()-st[:,4].max())/1e3 if st[:,5].max() else 0:.1f} us); start spread {(st[:,0].max()-t0)/1e3:.1f} us")
    print("   mean phase us: load %.2f  H_old %.2f  loop %.2f  H_new+write %.2f" % tuple(ph.mean(axis=0) / 1e3))
    print("   max  phase us: load %.2f  H_old %.2f  loop %.2f  H_new+write %.2f" % tuple(ph.max(axis=0) / 1e3))
    be.close()
