import sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
tr = P.simulate_rsv(theta, 2000, seed=0)
be = P.CudaBackend(0)
cfg = P.SamplerConfig(seed=1, md=P.MDConfig(0.02, 20), n_burnin=0, n_samples=16, prng="minstd")
P.run_chain(tr.dataset, cfg, backend=be, init_params=theta, init_h=tr.latent)
print("ok")
