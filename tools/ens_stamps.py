import ctypes, os, sys
sys.path.insert(0, ".")
os.environ["RSV_ENS_STAMPS"] = "1"
import numpy as np
import paper_1603_08114_b200 as P
from paper_1603_08114_b200 import _native as N
L = N.lib()
L.rsv_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
ens = P.Ensemble(4096, 4096)
ens.seed(1)
ens.refresh_momenta(copy=False)
st = np.zeros((128, 8), dtype=np.int64)
N.check(L.rsv_debug_stamps(ens.ctx, st.ctypes.data, 128), ens.ctx)
r = st[:, 4]
print("rounds %.1f; work cycles per round: generate %.0f, classify %.0f, evaluate %.0f, walk %.0f, emit %.0f" % (
      r.mean(), (st[:, 0] / r).mean(), (st[:, 1] / r).mean(), (st[:, 6] / r).mean(), (st[:, 5] / r).mean(),
      (st[:, 2] / r).mean()))
t0 = st[:, 3].min()
print("us: loop start (mean / max) %.2f / %.2f, exit (mean / max) %.2f / %.2f" % (
      (st[:, 3] - t0).mean() / 1e3, (st[:, 3].max() - t0) / 1e3,
      (st[:, 7] - t0).mean() / 1e3, (st[:, 7].max() - t0) / 1e3))
