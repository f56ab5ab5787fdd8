import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from golden_util import load
from paper_2107_01143_b200 import gvo, _native
from paper_2107_01143_b200.gvo.footprint import CollaborativeGroup
cases = load("footprints")
def run(i):
    c = cases[i]
    k = gvo.kernel_from_dict(c["spec"])
    grp = CollaborativeGroup(k.launch, np.asarray(c["blocks"], dtype=np.int64), "L2")
    r = gvo.grid_iteration(k, grp, c["granularity"])
    got = {(f, kd): (x.unique_count, x.total_count) for (f, kd), x in r.per_field.items()}
    want = {(f, kd): (u, t) for f, kd, u, t in c["per_field"]}
    return got == want, got, want
print("fresh 249:", run(249))
bad = [i for i in range(len(cases)) if not run(i)[0]]
print("bad after full pass:", bad[:20], len(bad))
ctx = _native.context()
print("n templates", len(ctx.templates), "max_acc", ctx.max_accesses, "max_fields", ctx.max_fields)
