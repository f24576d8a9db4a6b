"""A short device run_chain at T (default 2000) for ncu captures (development aid)."""
import sys

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
tr = P.simulate_rsv(theta, T, seed=1)
be = P.CudaBackend(0)
ch = be.chain(tr.dataset, theta)
ch.set_latent(tr.latent)
ch.set_stream(P.stream_state(P.make_rng(1, "minstd")))
ch.run_chain_device(0.02, 20, False, P.PriorSpec(), 0, 40, 1)
print("ok")
