"""Print the store build's bank-conflict model for the term kernel's apply
(POBA_SLOT_STATS): wavefronts per accumulator access per tile vs the ideal."""
import os
import sys

os.environ["POBA_SLOT_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_12834_b200 import blocks, configs  # noqa: E402

for arg in sys.argv[1:] or ["c5:1.0"]:
    name, scale = (arg.split(":") + ["1.0"])[:2]
    import _cfg
    p = _cfg.load(name, float(scale))
    print(arg, p.n_observations, flush=True)
    blocks.DeviceProblem(p.cam_indices, p.pt_indices, p.pixels, p.n_cameras, p.n_points)
