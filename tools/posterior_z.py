import sys, math
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_1603_08114_b200 as P
from conftest import golden
g = golden("posterior_T1000.npz")
data = P.Dataset.from_log_rv(g["y"], g["lrv"])
be = P.CudaBackend(0)
def bse(x, n=40):
    m = x.size // n; b = x[:m*n].reshape(n, m).mean(axis=1); return float(b.std(ddof=1)/math.sqrt(n))
for seed in (1234, 5, 6):
    cfg = P.SamplerConfig(seed=seed, md=P.MDConfig(0.02, 30), n_burnin=2000, n_samples=2000, thin=10, store_latent=True)
    ch = P.run_chain(data, cfg, backend=be)
    rows = [ch.param_series(n) for n in ("phi", "mu", "xi", "sigma_eta_sq", "sigma_u_sq")] + [ch.latent.mean(axis=1)] + [ch.latent[:, t] for t in (0, 250, 500, 999)]
    mean = np.array([r.mean() for r in rows]); se = np.array([bse(r) for r in rows])
    print(seed, np.round((mean - g["mean"]) / np.sqrt(se**2 + g["se"]**2), 2), round(float(np.mean(ch.accept)), 3))
