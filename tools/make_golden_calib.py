"""Reference side of the calibration-at-scale golden (this container, needs
/root/reference): the unmodified reference's read_ranking_csv +
derive_observations + calibrate_all (reference api.py:280-287, fit.py:94-243)
over the C3 device sweep written by tools/make_calib_sweep.py on the GPU box
and the synthetic measurements of tests/calib_util.py.
Writes tests/golden/calib_c3.json (sweep / measurement hashes and the
reference's fit).  usage: python tools/make_golden_calib.py gpurun_out/calib_c3_sweep.csv.gz"""
import gzip
import hashlib
import json
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")
import calib_util  # noqa: E402
from gvo import api as ref_api  # noqa: E402  (the unmodified reference)

sweep = gzip.decompress(Path(sys.argv[1]).read_bytes()).decode()
meas = calib_util.measurement_csv(sweep)
with tempfile.TemporaryDirectory() as d:
    (Path(d) / "s.csv").write_text(sweep)
    (Path(d) / "m.csv").write_text(meas)
    got = ref_api.run_calibrate(str(Path(d) / "m.csv"), str(Path(d) / "s.csv"))
obs = json.dumps(got["observations"], sort_keys=True).encode()
gold = {
    "source": "unmodified reference gvo.api.run_calibrate over the device C3 sweep (tools/make_calib_sweep.py)",
    "rows": sweep.count("\n") - 1,
    "sweep_sha256": hashlib.sha256(sweep.encode()).hexdigest(),
    "measurements_sha256": hashlib.sha256(meas.encode()).hexdigest(),
    "fitParams": got["fitParams"], "residuals": got["residuals"], "observationCounts": got["observationCounts"],
    "observations_sha256": hashlib.sha256(obs).hexdigest(), "skipped": len(got["skipped"]),
    "true": calib_util.TRUE,
}
(ROOT / "tests" / "golden" / "calib_c3.json").write_text(json.dumps(gold, indent=1) + "\n")
print(json.dumps({k: gold[k] for k in ("rows", "fitParams", "observationCounts", "skipped")}))
