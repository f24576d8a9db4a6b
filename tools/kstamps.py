"""In-kernel %globaltimer split of back-to-back proposals (dev aid)."""
import sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
be = P.CudaBackend(0)
for T in [int(a) for a in sys.argv[1:]] or [2000, 1 << 14, 1 << 18, 1 << 20]:
    tr = P.simulate_rsv(theta, T, seed=1)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 5, results=False)
    for _ in range(3):
        ch.hmc_update_many(0.02, 20, 20, results=False)
        k = ch.kernel_stamps()
        print(f"T={T}: " + "  ".join(f"{a} {b:.2f}" for a, b in k.items()), flush=True)
