import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
os.environ["RSV_TRAJ_STAMPS"] = "1"
import paper_1603_08114_b200 as P
from paper_1603_08114_b200 import _native as N
L = N.lib()
L.rsv_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
for T in [int(a) for a in sys.argv[1:]] or [1 << 20, 1 << 22]:
    tr = P.simulate_rsv(theta, T, seed=1)
    be = P.CudaBackend(0)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 3, results=False)
    st = np.zeros((400, 8), dtype=np.int64)
    N.check(L.rsv_debug_stamps(ch.ctx, st.ctypes.data, 400), ch.ctx)
    st = st[st[:, 2] > 0]
    tot = st[:, :4].sum(axis=1)
    print(f"T={T} CTAs={len(st)} mean cycles: wait {st[:,0].mean():.0f} pre {st[:,1].mean():.0f} loop {st[:,2].mean():.0f} post {st[:,3].mean():.0f}  total {tot.mean():.0f} (max {tot.max()})")
    be.close()
    # per-CTA totals: spread of the finishing times (tail of the persistent grid)
    print("  per-CTA total cycles pct 0/10/50/90/100:", np.percentile(tot, [0, 10, 50, 90, 100]).round(0))
    print("  pre+post share of total: %.3f" % ((st[:, 1] + st[:, 3]).sum() / tot.sum()))
    sm = st[:, 5]
    b = np.arange(len(st))
    print("  total cycles: blockIdx < 148: %.0f, >= 148: %.0f" % (tot[b < 148].mean(), tot[b >= 148].mean()))
    # pairs on the same SM: faster / slower CTA
    fast, slow = [], []
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        if len(idx) == 2:
            a_, c_ = sorted(idx, key=lambda i: tot[i])
            fast.append(tot[a_]); slow.append(tot[c_])
            if len(fast) <= 4:
                print("  SM", s_, "blocks", idx.tolist(), "cycles", tot[idx].tolist())
    print("  SM pairs: fast %.0f slow %.0f" % (np.mean(fast), np.mean(slow)))
    # the grid's tail: last CTA's loop end -> Metropolis start (t_stamp[3])
    import ctypes as _c
    raw = (_c.c_uint64 * 5)()
    ch2 = P.CudaBackend(0).chain(tr.dataset, theta)
    ch2.set_latent(tr.latent)
    ch2.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch2.hmc_update_many(0.02, 20, 3, results=False)
    st2 = np.zeros((400, 8), dtype=np.int64)
    N.check(L.rsv_debug_stamps(ch2.ctx, st2.ctypes.data, 400), ch2.ctx)
    st2 = st2[st2[:, 2] > 0]
    N.check(L.rsv_kernel_stamps(ch2.ctx, raw), ch2.ctx)
    ends = st2[:, 6]
    print("  traj entry -> CTA loop ends (us) pct 0/50/100:", np.percentile((ends - raw[2]) / 1e3, [0, 50, 100]).round(2),
          " metropolis start:", round((raw[3] - raw[2]) / 1e3, 2))
    # entry / end per CTA (globaltimer) and tiles per CTA
    ent = (st2[:, 7] - raw[2]) / 1e3
    endt = (st2[:, 6] - raw[2]) / 1e3
    nt = st2[:, 4]
    b2 = np.arange(len(st2))
    for lo, hi in ((0, 148), (148, 296)):
        m = (b2 >= lo) & (b2 < hi)
        print(f"  CTAs {lo}-{hi}: entry us {ent[m].mean():.2f} (max {ent[m].max():.2f}), end us {endt[m].mean():.2f}"
              f" (max {endt[m].max():.2f}), tiles {np.unique(nt[m]).tolist()}")
    last = int(np.argmax(st2[:, 5] > 10**12)) if (st2[:, 5] > 10**12).any() else None
    if last is not None:
        print("  last CTA", last, ": loop end", round((st2[last, 6] - raw[2]) / 1e3, 2), "count done",
              round((st2[last, 5] - raw[2]) / 1e3, 2), "metropolis start", round((raw[3] - raw[2]) / 1e3, 2))
