"""Build A/B variants of the library into variants/ (development aid)."""
import pathlib, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_1301_4195_b200.build import build
V = {
    "base": [],
    "minb3": ["BOLTZ_CONV_MINB=3"],
    "pref": ["BOLTZ_CONV_PREFETCH=1"],
    "pref_minb3": ["BOLTZ_CONV_PREFETCH=1", "BOLTZ_CONV_MINB=3"],
    "w2_minb6": ["BOLTZ_CONV_WARPS=2", "BOLTZ_CONV_MINB=6", "BOLTZ_CONV_PREFETCH=1"],
    "w8": ["BOLTZ_CONV_WARPS=8", "BOLTZ_CONV_PREFETCH=1"],
}
root = pathlib.Path(__file__).resolve().parent.parent / "variants"
names = sys.argv[1:] or list(V)
with ThreadPoolExecutor(4) as ex:
    list(ex.map(lambda n: build(force=True, out=root / f"lib_{n}.so", defines=V[n]), names))
