"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
by enclosing device function: python scripts/ncu_by_function.py page.csv"""
import csv, re, sys
from pathlib import Path

SRC = Path(__file__).resolve().parents[1] / "paper_1810_11765_b200" / "csrc"


def functions(path):
    out = []
    for i, l in enumerate(path.read_text().split("\n"), 1):
        if re.match(r"^(static )?(__device__|__global__|template|struct|bool|dsr_status|extern)", l) or \
                re.match(r"^\s+static __device__", l):
            m = re.search(r"(\w+)\s*\(", l) if "(" in l else re.search(r"struct (\w+)", l)
            if m:
                out.append((i, m.group(1)))
    return out


fr = {p.name: functions(p) for p in SRC.glob("*.cu*")}


def owner(f, line):
    best = "?"
    for i, n in fr.get(f, []):
        if i <= line:
            best = n
    return f"{f}:{best}"


rows = list(csv.reader(open(sys.argv[1])))
agg, fname, hdr = {}, None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if r and r[0] and r[0].isdigit() and hdr:
        try:
            ex, sm = float(r[7]), float(r[4])
        except ValueError:
            continue
        a = agg.setdefault(owner(fname, int(r[0])), [0.0, 0.0])
        a[0] += ex
        a[1] += sm
tex = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"instructions executed: {tex:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{k:48s} instr {v[0] / tex * 100:5.1f}%   stall samples {v[1] / ts * 100:5.1f}%")
