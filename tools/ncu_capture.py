"""ncu evidence for bench.py's roofline (run on the GPU box):

  python tools/ncu_capture.py [--workload C5]

1. Launch list of one bench step (`bench.py --steps 1 --warmup 0`) under
   ncu with the issue/DRAM counters of every launch:
   smsp__inst_executed.sum, dram__bytes_read.sum, dram__bytes_write.sum,
   gpu__time_duration.sum, smsp__issue_active.avg.pct_of_peak_sustained_active
   (application replay: the step re-runs once per counter pass, so no device
   memory has to be saved/restored around the persistent set kernel).
2. One `--set full` capture of a representative k_sets launch (the median
   batch of the step) for the hardware breakdown.
Writes profiles/r02_ncu_capture_<workload>.json tagged with the library's
gvo_build_id(); bench.py uses it only when the build id matches the loaded
library.  The CSVs go to gpurun_out/ (scratch).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")
METRICS = ("smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
           "smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg")
FULL_PICK = {
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "local_ld_inst": "smsp__sass_inst_executed_op_local_ld.sum",
    "local_st_inst": "smsp__sass_inst_executed_op_local_st.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "registers": "launch__registers_per_thread",
    "duration": "gpu__time_duration.sum",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "inst": 1, "": 1, "%": 1, "cycle": 1}


def _rows(text):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def _val(r):
    v = float(r["Metric Value"].replace(",", ""))
    return v * SCALE.get(r.get("Metric Unit", ""), 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5")
    args = ap.parse_args()
    from paper_2107_01143_b200 import _native

    bid = _native.build_id()
    out_dir = ROOT / "gpurun_out"
    out_dir.mkdir(exist_ok=True)
    wl = args.workload
    bench = [sys.executable, str(ROOT / "bench.py"), "--workload", wl, "--steps", "1", "--warmup", "0",
             "--no-cpu", "--no-e2e"]
    log = out_dir / f"ncu_launches_{wl.lower()}.csv"
    subprocess.run([NCU, "--metrics", METRICS, "--clock-control", "none", "--replay-mode", "application",
                    "--csv", "--log-file", str(log), *bench], check=True, cwd=ROOT)
    rows = _rows(log.read_text())
    per = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        per.setdefault(key, {})[r["Metric Name"]] = _val(r)
    kernels = {}
    for (lid, name), mv in per.items():
        short = name.split("(")[0].split("::")[-1]
        k = kernels.setdefault(short, {"launches": 0, "inst": 0.0, "dram": 0.0, "time_s": 0.0, "issue_w": 0.0})
        k["launches"] += 1
        k["inst"] += mv.get("smsp__inst_executed.sum", 0.0)
        k["dram"] += mv.get("dram__bytes_read.sum", 0.0) + mv.get("dram__bytes_write.sum", 0.0)
        t = mv.get("gpu__time_duration.sum", 0.0)
        k["time_s"] += t
        k["issue_w"] += t * mv.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0)
    total_t = sum(k["time_s"] for k in kernels.values())
    sets = kernels.get("k_sets")
    if sets is None:
        raise SystemExit(f"no k_sets launch in {log}")
    cap = {"build_id": bid, "workload": wl, "command": " ".join(bench[1:]),
           "ncu": f"--metrics {METRICS} --clock-control none --replay-mode application",
           "kernels": {n: {"launches": k["launches"], "inst_executed": k["inst"], "dram_bytes": k["dram"],
                           "time_ms_ncu": k["time_s"] * 1e3} for n, k in kernels.items()},
           "k_sets": {"launches_per_step": sets["launches"], "inst_executed_per_step": sets["inst"],
                      "dram_bytes_per_step": sets["dram"], "dram_bytes_per_launch": sets["dram"] / sets["launches"],
                      "issue_active_pct": sets["issue_w"] / sets["time_s"] if sets["time_s"] else None,
                      "share_of_step_ncu": sets["time_s"] / total_t if total_t else None}}
    # one full-set capture of the median k_sets launch that does work (a
    # batch queues both residencies of the set kernel when the residency is
    # picked on the device; the other launch exits at once)
    full = out_dir / f"ncu_full_k_sets_{wl.lower()}.csv"
    set_times = [(lid, mv.get("gpu__time_duration.sum", 0.0)) for (lid, name), mv in sorted(per.items(),
                 key=lambda kv: int(kv[0][0])) if name.split("(")[0].split("::")[-1] == "k_sets"]
    real = [i for i, (_, t) in enumerate(set_times) if t > 1e-4]
    by_t = sorted(real, key=lambda i: set_times[i][1])
    skip = by_t[len(by_t) // 2] if by_t else max(0, sets["launches"] // 2)
    cap["k_sets"]["launches_doing_work_per_step"] = len(real)
    if real:
        cap["k_sets"]["dram_bytes_per_launch"] = sets["dram"] / len(real)
    r = subprocess.run([NCU, "--set", "full", "--clock-control", "none", "-k", "regex:k_sets", "--launch-skip",
                        str(skip), "--launch-count", "1", "--import-source", "on",
                        "--export", str(out_dir / f"ncu_k_sets_{wl.lower()}"), "--force-overwrite", *bench], cwd=ROOT)
    if r.returncode == 0:
        raw_txt = subprocess.run([NCU, "-i", str(out_dir / f"ncu_k_sets_{wl.lower()}.ncu-rep"), "--page", "raw",
                                  "--csv"], capture_output=True, text=True).stdout
        full.write_text(raw_txt)
    if r.returncode == 0 and full.exists():
        raw = list(csv.reader(io.StringIO("\n".join(ln for ln in full.read_text().splitlines()
                                                     if ln.startswith('"')))))
        if len(raw) >= 3:
            head, units, vals = raw[0], raw[1], raw[2]
            hw = {}
            for k, metric in FULL_PICK.items():
                if metric in head:
                    j = head.index(metric)
                    try:
                        hw[k] = float(vals[j].replace(",", "")) * SCALE.get(units[j], 1)
                    except ValueError:
                        hw[k] = vals[j]
            hw["launch"] = (f"k_sets launch {skip + 1} of {sets['launches']} in the step (median duration of the "
                            f"{len(real)} launches doing work)")
            cap["k_sets"]["hw"] = hw
    dst = ROOT / "profiles" / f"r02_ncu_capture_{wl.lower()}.json"
    dst.write_text(json.dumps(cap, indent=1) + "\n")
    (out_dir / dst.name).write_text(dst.read_text())
    print(json.dumps(cap["k_sets"], indent=1))


if __name__ == "__main__":
    main()
