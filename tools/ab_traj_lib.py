"""A/B of the trajectory kernel launch time (rsv_bench_trajectory, T = 2^20)
between the default library and the one in AB_LIB.  Development aid."""
import sys, os, ctypes, statistics
sys.path.insert(0, ".")
import paper_1603_08114_b200._native as N
if os.environ.get("AB_LIB"):
    N.LIB_PATH = os.environ["AB_LIB"]
import paper_1603_08114_b200 as P
theta = P.Params(phi=0.97, mu=-1.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)
T = 1 << 20
tr = P.simulate_rsv(theta, T, seed=0)
be = P.CudaBackend(0); ch = be.chain(tr.dataset, theta); ch.set_latent(tr.latent)
ch.hmc_update(0.02, 20)
v = [ch.bench_trajectory(0.02, 20, 20) * 1e3 for _ in range(15)]
print(os.path.basename(N.lib()._name), f"median {statistics.median(v):.2f} us min {min(v):.2f}")
