"""Three ensemble momenta draws at 4096 chains x 4096 (config 4) for ncu
captures of zig_ens_kernel (development aid)."""
import sys

sys.path.insert(0, ".")
import paper_1603_08114_b200 as P  # noqa: E402

ens = P.Ensemble(4096, 4096)
ens.seed(1)
for _ in range(3):
    ens.refresh_momenta(copy=False)
print("ok")
