import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1603_08114_b200 as P
THETA = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
T, L, n, world = 20000, 12, 14, 2
truth = P.simulate_rsv(THETA, T, seed=19)
data = truth.dataset
be = P.CudaBackend(0)
st0 = P.stream_state(P.make_rng(23, "pcg32"))
single = be.chain(data, THETA); single.set_latent(truth.latent); single.set_stream(st0)
ref = single.hmc_update_many(0.02, L, n)
print("ref ", [int(x.accept) for x in ref], [round(x.delta_h, 6) for x in ref][:5])
for K in (1, 2, 100):
    shards = [P.ShardedChain(data, THETA, r, world, margin=42) for r in range(world)]
    for c in shards:
        c.set_latent_global(truth.latent); c.set_stream(st0)
    res = P.sharded.hmc_update_local_device(shards, 0.02, L, n, halo_every=K)
    print(f"K={K:3d}", [int(x.accept) for x in res], [round(x.delta_h, 6) for x in res][:5])
    for c in shards: c.shard.close()
shards = [P.ShardedChain(data, THETA, r, world, margin=42) for r in range(world)]
for c in shards:
    c.set_latent_global(truth.latent); c.set_stream(st0)
res = [P.hmc_update_local(shards, 0.02, L, stats=False) for _ in range(n)]
print("host ", [int(x.accept) for x in res], [round(x.delta_h, 6) for x in res][:5])
