import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
os.environ["RSV_TRAJ_STAMPS"] = "1"
import paper_1603_08114_b200 as P
from paper_1603_08114_b200 import _native as N
L = N.lib()
L.rsv_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
tr = P.simulate_rsv(theta, T, seed=1)
be = P.CudaBackend(0)
ch = be.chain(tr.dataset, theta)
ch.set_latent(tr.latent)
ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
for rep in range(3):
    ch.hmc_update_many(0.02, 20, 3, results=False)
    st = np.zeros((400, 8), dtype=np.int64)
    N.check(L.rsv_debug_stamps(ch.ctx, st.ctypes.data, 400), ch.ctx)
    st = st[st[:, 2] > 0]
    tot = st[:, :4].sum(axis=1)
    print("total pct 0/10/50/90/100:", np.percentile(tot, [0, 10, 50, 90, 100]).astype(int),
          " wait:", np.percentile(st[:, 0], [10, 50, 90, 100]).astype(int),
          " loop:", np.percentile(st[:, 2], [10, 50, 90, 100]).astype(int))
    slow = np.argsort(-tot)[:8]
    print("  slowest CTAs:", slow.tolist(), " fastest:", np.argsort(tot)[:8].tolist())
