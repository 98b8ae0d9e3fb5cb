"""Build A/B variants of the library into variants/ (development aid)."""
import pathlib, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1301_4195_b200.build import build
V = {
    "base": [],
    "hx": ["BOLTZ_TERM_HX=1"],
    "cpb1": ["BOLTZ_FUSED_BUDGET_KB=100"],
    "cpb1_256": ["BOLTZ_FUSED_BUDGET_KB=100", "BOLTZ_FUSED_THREADS=256"],
}
root = pathlib.Path(__file__).resolve().parent.parent / "variants"
names = sys.argv[1:] or list(V)
with ThreadPoolExecutor(4) as ex:
    list(ex.map(lambda n: build(force=True, out=root / f"lib_{n}.so", defines=V[n]), names))
