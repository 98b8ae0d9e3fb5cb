"""Build A/B variants of the library into variants/ (development aid)."""
import pathlib, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
from paper_1301_4195_b200.build import build
V = {
    "base": [],
    "tma": ["BOLTZ_PIPE_TMA=1"],
    "pipe_m3": ["BOLTZ_PIPE_MINB=3"],
    "pipe_m3_w2": ["BOLTZ_PIPE_MINB=3", "BOLTZ_CONV_WARPS=2"],
    "pipe_m6_w2": ["BOLTZ_PIPE_MINB=6", "BOLTZ_CONV_WARPS=2"],
    "xpf1": ["BOLTZ_XPF=1"],
    "xpf2": ["BOLTZ_XPF=2"],
    "f1t256": ["BOLTZ_FUSED_BUDGET_KB=100", "BOLTZ_FUSED_THREADS=256"],
    "f1t512": ["BOLTZ_FUSED_BUDGET_KB=100", "BOLTZ_FUSED_THREADS=512"],
    "f1t128": ["BOLTZ_FUSED_BUDGET_KB=100", "BOLTZ_FUSED_THREADS=128"],
    "f2t256": ["BOLTZ_FUSED_THREADS=256"],
    "kcs16_m3": ["BOLTZ_CONV_KERNEL=3", "BOLTZ_K0_MINB=3"],
    "kcs16_m2": ["BOLTZ_CONV_KERNEL=3", "BOLTZ_K0_MINB=2"],
    "kcs16_m3w2": ["BOLTZ_CONV_KERNEL=3", "BOLTZ_K0_MINB=3", "BOLTZ_CONV_WARPS=2"],
    "kcsm16": ["BOLTZ_CONV_KERNEL=3"],
    "kcsm16s": ["BOLTZ_CONV_KERNEL=3", "BOLTZ_KCSM_SPLIT=1"],
    "kcsm24s": ["BOLTZ_KCSM_SPLIT=1"],
    "rest3": ["BOLTZ_KCSM_REST_MINB=3"],
    "w2": ["BOLTZ_CONV_WARPS=2"],
    "t24_12": ["BOLTZ_TILE24=12"],
    "w8": ["BOLTZ_CONV_WARPS=8"],
    "ord1": ["BOLTZ_KCSR_ORDER=1"],  # k_conv_kcsr diagonal-major (round-2 order)
    "rest2": ["BOLTZ_KCSM_REST_MINB=2"],  # N <= 16 on k_conv_kcs / the phased k_conv_kcsm mirror
}
root = pathlib.Path(__file__).resolve().parents[2] / "variants"
names = sys.argv[1:] or list(V)
with ThreadPoolExecutor(4) as ex:
    list(ex.map(lambda n: build(force=True, out=root / f"lib_{n}.so", defines=V[n]), names))
