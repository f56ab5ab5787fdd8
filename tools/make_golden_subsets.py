"""Wide seeded-subset goldens of the two large BASELINE spaces (C3 ~1e5 and
C5 ~1e6 configurations), made by running the UNMODIFIED reference estimator
(kernel-spec dicts, its own interchange format, kernels.py:441-512) on 512
seeded-random configurations of each space (np.random.default_rng(20240811),
BASELINE.md §3: >= 500 configurations for the 1e5 / 1e6 spaces).

Run in the build container (the reference is not on the GPU box):
    python tools/make_golden_subsets.py
writes tests/golden/subsets.json:
  {"columns": [...37 record columns...],
   "spaces": {"C3": {"templates": [...], "cfg": [[tpl, machine, bx, by, bz], ...],
                     "records": [[hex, ...], ...],   # reference record (limiter as its name)
                     "order": [...]},                 # perf.py:131 ranking of the subset
              "C5": {...}}}
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from make_golden_workloads import entry, jobs_of, ref_record  # noqa: E402
from paper_2107_01143_b200 import _native, workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo.machine import b200_preset  # noqa: E402

OUT = ROOT / "tests" / "golden" / "subsets.json"
N_SUBSET = 512
FOLD = {0: "2y", 1: "2z", 2: "none"}


def main():
    m = b200_preset()
    rng = np.random.default_rng(20240811)
    out = {"columns": list(_native.RECORD_COLUMNS), "n": N_SUBSET, "seed": 20240811, "spaces": {}}
    with mp.get_context("spawn").Pool(os.cpu_count(), maxtasksperchild=16) as pool:
        for name in ("C3", "C5"):
            sp = W.space(name, m)
            idx = np.sort(rng.choice(len(sp), size=N_SUBSET, replace=False))
            res = pool.map(ref_record, jobs_of(sp, idx, True), chunksize=1)
            tpls, tix, cfg, recs, keys = [], {}, [], [], []
            for j, (i, r) in enumerate(zip(idx, res)):
                e = entry(sp, int(i))
                tk = json.dumps(e["template"], sort_keys=True)
                if tk not in tix:
                    tix[tk] = len(tpls)
                    tpls.append(e["template"])
                cfg.append([tix[tk], e["machine"], *e["block"]])
                if "error" in r:
                    recs.append({"error": r["error"]})
                    continue
                rec = r["record"]
                recs.append([rec[c] for c in _native.RECORD_COLUMNS])
                keys.append((-float.fromhex(rec["predictedGLups"]), tuple(e["block"]),
                             FOLD[int(sp.fold_rank[int(i)])], j))
            out["spaces"][name] = {"templates": tpls, "cfg": cfg, "records": recs,
                                   "index": [int(i) for i in idx],
                                   "order": [k[-1] for k in sorted(keys)]}
            print(name, "subset", len(res), flush=True)
    OUT.write_text(json.dumps(out, separators=(",", ":")))
    print("written", OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
