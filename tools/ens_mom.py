import sys, time
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
for C, Tc in [(32, 4096), (128, 4096), (4096, 4096), (4096, 1024), (32, 1024)]:
    ens = P.Ensemble(C, Tc)
    ens.seed(1)
    ens.refresh_momenta(copy=False)
    t0 = time.perf_counter()
    for _ in range(10):
        ens.refresh_momenta(copy=False)
    dt = (time.perf_counter() - t0) / 10
    print(f"C={C} Tc={Tc}: {dt*1e6:.0f} us per draw (wall, incl. sync)")
    ens.close()
