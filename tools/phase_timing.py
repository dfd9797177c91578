"""Per-phase cycle breakdown of the term kernel (needs a POBA_PHASE_TIMING build)."""
import sys
sys.path.insert(0, ".")
import paper_2204_12834_b200 as P
from paper_2204_12834_b200 import configs
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
p = configs.make_config(name, scale)
s = P.assemble(p, lam=1e-4)
dev = s._dp.dev
dev.debug_counters()
ms, msk, _ = dev.time_terms(10)
c = dev.debug_counters()
tiles = c[7]
names = ["wait", "ph1(meta,acc,t,J,w)", "ph2(y,z)", "issue", "ph3(g)", "ph4(seg,RMW)"]
tot = sum(c[:6])
print(f"{name} x{scale}: kernel {msk*1e3:.1f} us; cycles per warp-tile:", {n: round(v / max(tiles,1)) for n, v in zip(names, c[:6])}, "total", round(tot / max(tiles, 1)))
