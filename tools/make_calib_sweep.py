"""Device side of the calibration golden (GPU): the C3 sweep's ranking CSV
(92k rows, native formatter, ranked) -> gpurun_out/calib_c3_sweep.csv.gz.
tools/make_golden_calib.py then runs the unmodified reference's fit on it.
usage: python tools/make_calib_sweep.py"""
import gzip
import hashlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import calib_util  # noqa: E402

from paper_2107_01143_b200 import _native, workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo import report  # noqa: E402

sp = calib_util.space_c3()
res, order = W.evaluate_space(sp)
body = _native.format_ranking_csv(res.records, calib_util.prefixes(sp), order)
text = ",".join(report.RANKING_CSV_COLUMNS) + "\n" + body
out = ROOT / "gpurun_out" / "calib_c3_sweep.csv.gz"
out.parent.mkdir(exist_ok=True)
out.write_bytes(gzip.compress(text.encode(), mtime=0))
print(len(sp), "rows", hashlib.sha256(text.encode()).hexdigest())
