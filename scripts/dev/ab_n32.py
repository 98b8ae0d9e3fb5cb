"""N=24 / N=32 RK2 step time per library variant (dev aid): python scripts/dev/ab_n32.py variants/lib_*.so"""
import os, pathlib, subprocess, sys
ROOT = pathlib.Path(__file__).resolve().parents[2]
for lib in sys.argv[1:]:
    env = dict(os.environ, BOLTZ_LIB_VARIANT=str(pathlib.Path(lib).resolve()), BOLTZ_MIRROR="1")
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "kcs_mirror_time.py"), "--child"], env=env,
                       capture_output=True, text=True)
    print(pathlib.Path(lib).name, r.stdout.strip() or r.stderr[-600:], flush=True)
