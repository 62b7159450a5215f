"""Regenerate the number tables in DESIGN.md, README.md and
profiles/r01_summary.md from an evidence pass (tools/gpu_round.sh; run
tools/update_profiles.py first so profiles/traffic.json is current).

    python tools/update_docs.py [gpurun_out]

Reads gpurun_out/bench_cfg2.json, bench_all.jsonl, bench_ref.json and
profiles/r01_size_curve.jsonl.  Each table is replaced between its header row
and the next blank line; surrounding prose is left alone.
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out"
ALG_GB = {"cfg2": 1.074, "cfg3-4": 8.59, "cfg3-8": 17.18, "cfg3-16": 34.36, "cfg4": 4.29,
          "cfg4-fft7": 4.29, "cfg1": 0.034}


def replace_table(text, first_cell, rows):
    i = text.index(first_cell)
    i = text.rindex("\n", 0, i) + 1
    j = text.index("\n\n", i)
    return text[:i] + "\n".join(rows) + text[j:]


def main():
    lines = [json.loads((OUT / "bench_cfg2.json").read_text())]
    lines += [json.loads(x) for x in (OUT / "bench_all.jsonl").read_text().splitlines() if x]
    by = {d["config"]["workload"].split(":")[0]: d for d in lines}
    ref = json.loads((OUT / "bench_ref.json").read_text())

    def design_row(w, label, bold=False):
        d = by[w]
        e, es, cb = d.get("e2e") or {}, d.get("e2e_single_call") or {}, d.get("cpu_baseline") or {}
        v, fr = f"{d['value']:.0f}", f"{d['roofline']['frac']:.3f}"
        if bold:
            v, fr = f"**{v}**", f"**{fr}**"
        e2e = (f"{es.get('value', 0):.1f} (single call)" if w == "cfg4-fft7"
               else f"{e.get('value', 0):.1f}")
        cpu = "n/a (no FFT in the reference)" if w == "cfg4-fft7" else f"{cb.get('value', 0):.1f}"
        if w == "cfg2":
            cpu += f" (ref arm: {ref['value']:.1f})"
        vs = d["roofline"]["frac_of_torch_copy_same_harness"]
        return f"| {label} | {v} | {fr} | {vs:.2f} | {e2e} | {cpu} |"

    design = (ROOT / "DESIGN.md").read_text()
    design = replace_table(design, "| **cfg2 in place, 2^26 f64 (headline)**", [
        design_row("cfg2", "**cfg2 in place, 2^26 f64 (headline)**", True),
        design_row("cfg3-4", "cfg3 oop 2^30 f32"),
        design_row("cfg3-8", "cfg3 oop 2^30 f64"),
        design_row("cfg3-16", "cfg3 oop 2^30 c128"),
        design_row("cfg4", "cfg4 batched 4096 × 2^16 c64"),
        design_row("cfg4-fft7", "cfg4-fft7: cfg4 + 7 fused DIT stages"),
        design_row("cfg1", f"cfg1 oop 2^20 c128 (L2-flushed, "
                           f"~{by['cfg1']['ms_per_step'] * 1e3:.1f} µs step)"),
    ])
    curve = {}
    for x in (ROOT / "profiles" / "r01_size_curve.jsonl").read_text().splitlines():
        r = json.loads(x)
        if r["kind"] == "cell":
            curve[(r["E"], r["inplace"], r["b"])] = r
    bs = [18, 20, 22, 24, 26, 28, 30]
    rows = ["| E, family | " + " | ".join(f"b={b}" for b in bs) + " |", "|---|" + "---|" * len(bs)]
    for E in (4, 8, 16):
        for ip in (False, True):
            cells = [f"{curve[(E, ip, b)]['gbs']:.0f} ({curve[(E, ip, b)]['frac']:.2f}) "
                     f"{curve[(E, ip, b)]['vs_stream']:.2f}" for b in bs]
            rows.append(f"| {E}, {'in place' if ip else 'out of place'} | " + " | ".join(cells) + " |")
    design = replace_table(design, "| E, family | b=18 |", rows)
    (ROOT / "DESIGN.md").write_text(design)

    f = by.__getitem__
    readme = (ROOT / "README.md").read_text()
    readme = replace_table(readme, "| in place 2^26 float64 (headline)", [
        f"| in place 2^26 float64 (headline) | {f('cfg2')['value']:.0f} | "
        f"{f('cfg2')['roofline']['frac']:.3f} |",
        "| out of place 2^30 float32 / float64 / complex128 | "
        + " / ".join(f"{f(w)['value']:.0f}" for w in ("cfg3-4", "cfg3-8", "cfg3-16")) + " | "
        + " / ".join(f"{f(w)['roofline']['frac']:.3f}" for w in ("cfg3-4", "cfg3-8", "cfg3-16"))
        + " |",
        f"| batched 4096 × 2^16 complex64 | {f('cfg4')['value']:.0f} | "
        f"{f('cfg4')['roofline']['frac']:.3f} |",
        f"| same + 7 fused FFT butterfly stages | {f('cfg4-fft7')['value']:.0f} | "
        f"{f('cfg4-fft7')['roofline']['frac']:.3f} |",
        f"| out of place 2^20 complex128 (33 MB, launch/latency bound) | "
        f"{f('cfg1')['value']:.0f} | {f('cfg1')['roofline']['frac']:.3f} |",
    ])
    (ROOT / "README.md").write_text(readme)

    traffic = json.loads((ROOT / "profiles" / "traffic.json").read_text())
    rows = []
    for w in ("cfg2", "cfg3-4", "cfg3-8", "cfg3-16", "cfg4", "cfg4-fft7", "cfg1"):
        t = traffic[w]
        k = t["kernel"].replace("void ", "").replace("bitrev_b200::", "").split("(")[0]
        rows.append(f"| {w} | `{k}` | {t['duration_us_cold']:.1f} | "
                    f"{t['dram_bytes_per_launch'] / 1e9:.3f} / {ALG_GB[w]} | "
                    f"{t['dram_active_pct']} % | {t['registers']} | {t['grid']} |")
    summ = (ROOT / "profiles" / "r01_summary.md").read_text()
    summ = replace_table(summ, "| cfg2 | `", rows)
    (ROOT / "profiles" / "r01_summary.md").write_text(summ)
    c2 = by["cfg2"]
    print(f"cfg2 {c2['value']:.0f} GB/s frac {c2['roofline']['frac']:.3f}; tables updated")


if __name__ == "__main__":
    main()
