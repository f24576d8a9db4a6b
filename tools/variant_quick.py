import os, sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
for T in [1 << 20, 1 << 22]:
    tr = P.simulate_rsv(theta, T, seed=1)
    be = P.CudaBackend(0)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 5, results=False)
    r = []
    for k in range(3):
        ch.hmc_update_many(0.02, 20, 10, results=False)
        r.append(ch.kernel_stamps()["trajectory_us"])
    print(os.environ.get("RSV_TRAJ_VARIANT", "auto"), T, r)
    be.close()
