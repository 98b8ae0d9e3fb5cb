"""e2e (pinned host memory) cfg2 RK2 step for (staging slots, chunk schedule)
pairs (development aid).  python scripts/dev/e2e_grid.py 2:1,3,3,1 3:1,2,4,4,2,1 ...
Each pair runs in its own process (BOLTZ_STAGE_SLOTS, BOLTZ_HOST_CHUNKS)."""
import os, pathlib, subprocess, sys
ROOT = pathlib.Path(__file__).resolve().parents[2]
for arg in sys.argv[1:]:
    slots, sch = arg.split(":")
    env = dict(os.environ, BOLTZ_STAGE_SLOTS=slots, BOLTZ_HOST_CHUNKS=sch)
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "e2e_sched.py"), "--child"], env=env,
                       capture_output=True, text=True)
    print(f"{arg:>28s}", r.stdout.strip() or r.stderr[-600:], flush=True)
