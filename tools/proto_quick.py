"""Elementary-step time vs B, streamed and fused (paper protocol, short reps; dev aid)."""
import sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
from paper_1603_08114_b200 import bench_protocol as BP
for b in (2, 64, 512, 4096):
    data = P.simulate_rsv(BP.BENCH_PARAMS, 512 * b, seed=b).dataset
    s = BP.time_elementary_step(b, None, 2000, BP.BENCH_PARAMS, data, repeats=3)
    f = BP.time_elementary_step(b, None, 2000, BP.BENCH_PARAMS, data, repeats=3, fused=True)
    print(f"B={b}: streamed {s.mean_seconds*1e6:.3f} us, fused {f.mean_seconds*1e6:.3f} us per step", flush=True)
