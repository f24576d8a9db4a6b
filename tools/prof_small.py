import sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
T = int(sys.argv[1]); L = int(sys.argv[2])
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
tr = P.simulate_rsv(theta, T, seed=1)
be = P.CudaBackend(0)
ch = be.chain(tr.dataset, theta)
ch.set_latent(tr.latent)
ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
ch.hmc_update_many(0.02, L, 4, results=False)
print("ok")
