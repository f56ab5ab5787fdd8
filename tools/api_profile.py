"""Host profile of the drop-in API on the C2 sweep (gvo.rank_sweep), the
bench's e2e_api leg (GPU).  usage: python tools/api_profile.py"""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_01143_b200 import gvo  # noqa: E402

m = gvo.b200_preset()
fam = gvo.KernelFamily("stencil", (640, 640, 640), radius=4)
cfgs = [c for t in (1 << i for i in range(11)) for c in gvo.enumerate_sweep(t)]
rows = gvo.rank_sweep(fam, cfgs, m, skip_invalid=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    rows = gvo.rank_sweep(fam, cfgs, m, skip_invalid=True)
    _ = rows[0].prediction.glups
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
