"""Small fixed workload for ncu: T=2^20, L=20, pcg32, a few HMC proposals."""
import sys

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
truth = P.simulate_rsv(theta, T, seed=1)
be = P.CudaBackend(0)
ch = be.chain(truth.dataset, theta)
ch.set_latent(truth.latent)
ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
ch.hmc_update_many(0.02, 20, n)
print("done", ch.launch_count())
