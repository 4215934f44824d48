"""Copy the evidence of a scripts/gpu_profiles.sh run (gpurun_out/) into the
tracked profiles/<round>/ directory: ncu summaries, the launch list of one bench
step (+ its per-kernel share table), the bench lines and the per-pass app times.

    python scripts/refresh_profiles.py [r01] [out_dir]

(out_dir defaults to profiles/<round>; the GPU-side script writes to
gpurun_out/prof_<round> so only small summaries travel back.)
"""
import collections
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G = ROOT / "gpurun_out"
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
P = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "profiles" / rnd
P.mkdir(parents=True, exist_ok=True)

reps = [str(G / f"{rnd}_{k}.ncu-rep") for k in ("mb_new", "mb_reduce", "mb_free", "compact", "nbody", "wator")]
reps = [r for r in reps if Path(r).exists()]
if reps:
    txt = subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_summarize.py"), str(P / "ncu_summary.json"), *reps],
                         capture_output=True, text=True).stdout
    (P / "ncu_summary.txt").write_text(txt)

gr = G / f"{rnd}_gol16k.ncu-rep"
if gr.exists():
    txt = subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_summarize.py"), str(P / "ncu_gol16k.json"), str(gr)],
                         capture_output=True, text=True).stdout
    (P / "ncu_gol16k.txt").write_text(txt)

lc = G / f"{rnd}_launches.csv"
if lc.exists():
    shutil.copy(lc, P / "launches_bench_step.csv")
    rows = list(csv.reader(open(lc)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                a = agg[d["Kernel Name"][:100]]
                a[0] += 1
                a[1] += float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    tot = sum(a[1] for a in agg.values()) or 1.0
    lines = [f"# {rnd} launch list: one bench.py step (+ warm-up step; `bench.py --launch-list`), "
             "ncu --metrics gpu__time_duration.sum --clock-control none", "",
             "Cold-cache, serialised launches: compare SHARES, not absolute times.", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {a[0]} | {a[1]:.1f} | {100 * a[1] / tot:.1f}% |")
    (P / "launches_summary.md").write_text("\n".join(lines) + "\n")


def json_lines(path):
    out = []
    if path.exists():
        for l in path.read_text().splitlines():
            l = l.strip()
            if l.startswith("{"):
                try:
                    out.append(json.loads(l))
                except Exception:
                    pass
    return out


b = json_lines(G / "bench.log")
if b:
    (P / "bench_microbench.json").write_text(json.dumps(b[-1]) + "\n")
a = json_lines(G / "bench_apps.log")
if a:
    (P / "bench_apps.jsonl").write_text("".join(json.dumps(x) + "\n" for x in a))
p = json_lines(G / "prof_apps.log")
if p:
    (P / "app_pass_times.jsonl").write_text("".join(json.dumps(x) + "\n" for x in p))
print("refreshed", P, "from", len(reps), "reports")
