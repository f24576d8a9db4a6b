"""Per-proposal event-pair time with and without the L2 flush between proposals (dev aid)."""
import sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
T = 1 << 20
tr = P.simulate_rsv(theta, T, seed=0)
be = P.CudaBackend(0)
ch = be.chain(tr.dataset, theta)
ch.set_latent(tr.latent)
ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
ch.hmc_update_many(0.02, 20, 5, results=False)
for flush in (256 << 20, 0, 256 << 20, 0):
    ch.set_l2_flush(flush)
    ch.set_timing(1)
    ch.hmc_update_many(0.02, 20, 20, results=True)
    st = ch.kernel_stamps()
    print("flush", flush >> 20, "MiB: ms/step", round(ch.timing()[2], 4), "in-kernel", st)
