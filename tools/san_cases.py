"""Bounded parity workload for compute-sanitizer runs (tools/sanitize.sh):
golden footprints (reference tests/golden/footprints.json), full evaluations
with every sampled unit through the set kernel, and a two-phase LBM (C4)
batch through the batched pipeline — each result still compared with the
reference goldens, so a run under a sanitizer is also a parity run.

  python tools/san_cases.py [n_footprints] [n_c4]
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_util import load  # noqa: E402
from paper_2107_01143_b200 import gvo, workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo.footprint import CollaborativeGroup  # noqa: E402
from paper_2107_01143_b200.gvo.machine import machine_from_dict  # noqa: E402


def main():
    n_fp = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    n_c4 = int(sys.argv[2]) if len(sys.argv) > 2 else 48
    bad = 0
    cases = load("footprints")
    for case in cases[:: max(1, len(cases) // n_fp)][:n_fp]:
        k = gvo.kernel_from_dict(case["spec"])
        grp = CollaborativeGroup(k.launch, np.asarray(case["blocks"], dtype=np.int64), "L2")
        r = gvo.grid_iteration(k, grp, case["granularity"])
        got = {(f, kd): (c.unique_count, c.total_count) for (f, kd), c in r.per_field.items()}
        want = {(f, kd): (u, t) for f, kd, u, t in case["per_field"]}
        bad += got != want
    for case in load("evaluations")[:4]:
        k = gvo.kernel_from_dict(case["spec"])
        m = machine_from_dict(case["machine"])
        bsz, wsz, ovr = case["sampling"]
        p = gvo.evaluate_kernel(k, m, block_samples=bsz, wave_samples=wsz, override_blocks_per_wave=ovr)
        bad += float(p.glups).hex() != case["record"]["predictedGLups"]
    g = load("workloads")["rankings"]["C4"]
    ents = [{"template": g["templates"][t], "machine": mm, "block": [bx, by, bz]} for t, mm, bx, by, bz in g["cfg"]]
    pick = np.linspace(0, len(ents) - 1, n_c4).astype(int)
    sp = W.space_from_entries([ents[i] for i in pick], [machine_from_dict(d) for d in load("workloads")["machines"]["C4"]])
    res, _ = W.evaluate_space(sp)
    bad += sum(float(res.records[j, -1]).hex() != g["glups"][i] for j, i in enumerate(pick))
    print(f"san_cases: {n_fp} footprints, 4 evaluations, {n_c4} C4 configs; mismatches: {bad}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
