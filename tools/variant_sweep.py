"""Time the trajectory kernel variants (RSV_TRAJ_VARIANT) across T."""
import os
import subprocess
import sys

code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
theta = P.Params(0.97, -9.0, -0.3, 0.05, 0.1)
out = []
for T in [2000, 1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20]:
    tr = P.simulate_rsv(theta, T, seed=1)
    be = P.CudaBackend(0)
    ch = be.chain(tr.dataset, theta)
    ch.set_latent(tr.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "pcg32")))
    ch.hmc_update_many(0.02, 20, 5, results=False)
    ch.set_timing(2)
    ch.hmc_update_many(0.02, 20, 30, results=False)
    t, m, tot = ch.timing()
    out.append(f"T=2^{T.bit_length()-1}: traj {t*1e3:8.2f}us ({T*20/(t*1e-3):.3e}/s) tot {tot*1e3:8.2f}us")
    be.close()
print(" | ".join(out))
'''
if __name__ == "__main__":
  for v in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    env = dict(os.environ, RSV_TRAJ_VARIANT=str(v))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"variant {v}:", r.stdout.strip() or r.stderr[-500:], flush=True)
