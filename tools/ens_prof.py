import sys
sys.path.insert(0, ".")
import paper_1603_08114_b200 as P
ens = P.Ensemble(4096, 4096)
ens.seed(1)
for _ in range(3):
    ens.refresh_momenta(copy=False)
print("ok")
