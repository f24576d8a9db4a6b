import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
os.environ["RSV_ZIG_STAMPS"] = "1"
import paper_1603_08114_b200 as P
from paper_1603_08114_b200 import _native as N
L = N.lib()
L.rsv_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
for T in [int(a) for a in sys.argv[1:]] or [2000, 1 << 20]:
    tr = P.simulate_rsv(theta, T, seed=1)
    be = P.CudaBackend(0)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 3, results=False)
    st = np.zeros((2000, 8), dtype=np.int64)
    N.check(L.rsv_debug_stamps(ch.ctx, st.ctypes.data, 2000), ch.ctx)
    st = st[st[:, 0] > 0]
    t0 = st[:, 0].min()
    rel = (st[:, :7] - t0) / 1e3
    print(f"T={T} CTAs={len(st)} span {rel[:,6].max():.1f} us; start spread {rel[:,0].max():.1f}")
    ph = np.diff(st[:, :7], axis=1) / 1e3
    names = ["ticket+tables", "stage", "classify", "walk+scan", "lookback", "write"]
    print("  mean:", "  ".join(f"{n} {v:.2f}" for n, v in zip(names, ph.mean(axis=0))))
    print("  max: ", "  ".join(f"{n} {v:.2f}" for n, v in zip(names, ph.max(axis=0))))
    be.close()
    if T > 1 << 19:
        blk = np.argsort(st[:, 0])
        r4 = rel[:, 4]; r5 = rel[:, 5]
        print("  AGG publish (us) pct 10/50/90/max:", np.percentile(r4, [10, 50, 90, 100]).round(2))
        print("  lookback done    pct 10/50/90/max:", np.percentile(r5, [10, 50, 90, 100]).round(2))
        print("  stage start pct 10/50/90/max:", np.percentile(rel[:, 1], [10, 50, 90, 100]).round(2))
        seen = (st[:, 7] - t0) / 1e3
        print("  count seen (us) pct 0/10/50/90/max:", np.percentile(seen, [0, 10, 50, 90, 100]).round(2))
        ld = rel[:, 5]
        top = np.argsort(-ld)[:5]
        print("  slowest look-back CTAs (index, done us, seen us, publish us):",
              [(int(i), round(float(ld[i]), 2), round(float(seen[i]), 2), round(float(rel[i, 4]), 2)) for i in top])
