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
print("rounds", st[:, 4].mean(), "gen work/round", (st[:, 0] / st[:, 4]).mean(), "gen wait/round", (st[:, 1] / st[:, 4]).mean(),
      "parse work/round", (st[:, 2] / st[:, 4]).mean(), "parse wait/round", (st[:, 3] / st[:, 4]).mean())
