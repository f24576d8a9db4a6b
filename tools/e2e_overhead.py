"""Where the host-API proposal's time goes at T = 2^20 (config 3): the public
call with the resident path, the DeviceChain call, the bare C call, and the
device-resident proposal (rsv_hmc_update_many, one per call) -- wall clock
per call, L2 not flushed.  Development aid (run under gpurun)."""
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402
from paper_1603_08114_b200 import _native as N  # noqa: E402
from paper_1603_08114_b200.rng import stream_state, store_stream_state  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = 200
theta = P.Params(phi=0.97, mu=-1.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)
truth = P.simulate_rsv(theta, T, seed=0)
data = truth.dataset
md = P.MDConfig(0.02, 20)
be = P.CudaBackend(0)
rng = P.make_rng(7, "pcg32")
h = truth.latent.copy()
for _ in range(400):
    h, acc, _ = P.hmc_update_volatility(h, theta, data, md, rng, backend=be)
    if not h.flags.writeable:
        break
ch = be.chain(data, theta)


def timed(label, fn):
    for _ in range(5):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    us = (time.perf_counter() - t0) / n * 1e6
    print(f"{label:55s} {us:8.1f} us/call", flush=True)


state = {"h": h}


def api():
    hh, _, _ = P.hmc_update_volatility(state["h"], theta, data, md, rng, backend=be)
    state["h"] = hh


timed("hmc_update_volatility (resident path)", api)
assert ch.last_update_resident


def chain_call():
    st = stream_state(rng)
    r, out = ch.hmc_update_host(state["h"], st, 0.02, 20)
    store_stream_state(rng, st)
    if out is not None:
        state["h"] = out


timed("DeviceChain.hmc_update_host (resident)", chain_call)
lib = ch._lib
out = ch._pinned_out()
r = N.Result()


def bare():
    st = stream_state(rng)
    code = lib.rsv_hmc_update_host(ch.ctx, None, out.ctypes.data, ctypes.byref(st), 0.02, 20, 0, ctypes.byref(r))
    assert code == 0
    store_stream_state(rng, st)


timed("rsv_hmc_update_host(NULL) bare ctypes", bare)
timed("stream_state + store_stream_state", lambda: store_stream_state(rng, stream_state(rng)))
timed("backend.chain(data, params)", lambda: be.chain(data, theta))
timed("rsv_hmc_update_many(n=1) (device-resident graph + result)", lambda: ch.hmc_update_many(0.02, 20, 1))
many = 64
t0 = time.perf_counter()
ch.hmc_update_many(0.02, 20, many)
print(f"{'rsv_hmc_update_many(n=64) per proposal':55s} {(time.perf_counter() - t0) / many * 1e6:8.1f} us/call")
