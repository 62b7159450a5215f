"""Refresh profiles/ from a tools/gpu_round.sh run in gpurun_out/: raw ncu
pages per workload, traffic.json (what bench.py reports as roofline.traffic;
entries of workloads not captured this time are kept), the launch list and
the bench lines.

    python tools/update_profiles.py r02
"""
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT, PROF = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME = {"ns": 1e-3, "us": 1, "ms": 1e3}

traffic = json.loads((PROF / "traffic.json").read_text()) if (PROF / "traffic.json").exists() else {}


def raw_pages():
    """(workload, raw-page CSV text): exported on the box (prof_<w>_raw.csv),
    else read from a full report (prof_<w>.ncu-rep)."""
    seen = set()
    for csvf in sorted(OUT.glob("prof_*_raw.csv")):
        w = csvf.name[len("prof_"):-len("_raw.csv")]
        seen.add(w)
        yield w, csvf.read_text()
    for rep in sorted(OUT.glob("prof_*.ncu-rep")):
        w = rep.stem[len("prof_"):]
        if w not in seen:
            yield w, subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                                    capture_output=True, text=True).stdout


for w, raw in raw_pages():
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3 or w.startswith("cfg5") or w in ("cfg316",):
        continue
    (PROF / f"{tag}_{w}_kernel_raw.csv").write_text(raw)
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    rd = int(float(d["dram__bytes_read.sum"]) * UNITS[u["dram__bytes_read.sum"]])
    wr = int(float(d["dram__bytes_write.sum"]) * UNITS[u["dram__bytes_write.sum"]])
    traffic[w] = {
        "dram_bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
        "kernel": d["Kernel Name"],
        "duration_us_cold": float(d["gpu__time_duration.sum"]) * TIME[u["gpu__time_duration.sum"]],
        "dram_active_pct": round(float(d["dram__cycles_active.avg.pct_of_peak_sustained_elapsed"]), 1),
        "registers": int(float(d["launch__registers_per_thread"])),
        "grid": int(float(d["launch__grid_size"])),
        "source": f"profiles/{tag}_{w}_kernel_raw.csv (ncu --set full --clock-control none)",
    }
traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu capture "
                    "of the bench's own kernel. Writes still in L2 when a kernel ends are not "
                    "counted (all of cfg1's 16 MiB output stays in L2).")
(PROF / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
if (OUT / "launches_default.csv").exists():
    shutil.copy(OUT / "launches_default.csv", PROF / f"{tag}_default_launches.csv")
with open(PROF / f"{tag}_bench_lines.jsonl", "w") as fh:
    for f in ("bench_default.json", "bench_all.jsonl", "bench_ref.json"):
        if (OUT / f).exists():
            for line in (OUT / f).read_text().splitlines():
                if line.startswith("{"):
                    fh.write(line + "\n")
for w, v in sorted(traffic.items()):
    if not w.startswith("_"):
        print(f"{w:12s} {v['dram_bytes_per_launch'] / 1e9:8.3f} GB {v['duration_us_cold']:9.1f} us "
              f"dram {v['dram_active_pct']}% regs {v['registers']} grid {v['grid']} {v['kernel'][:48]}")
