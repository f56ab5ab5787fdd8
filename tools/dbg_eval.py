import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from golden_util import load
from paper_2107_01143_b200 import gvo
from paper_2107_01143_b200.gvo.machine import machine_from_dict
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
case = load("evaluations")[idx]
k = gvo.kernel_from_dict(case["spec"]); m = machine_from_dict(case["machine"])
b, w, o = case["sampling"]
p = gvo.evaluate_kernel(k, m, block_samples=b, wave_samples=w, override_blocks_per_wave=o)
print("ok", p.glups)
