import os, subprocess, sys
sys.path.insert(0, "tools")
from variant_sweep import code  # noqa
for v in [int(x) for x in sys.argv[1].split(",")]:
    env = dict(os.environ, RSV_TRAJ_VARIANT=str(v))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"variant {v}:", r.stdout.strip() or r.stderr[-800:], flush=True)
