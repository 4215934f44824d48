"""Registers / spills per kernel from ptxas -v: python scripts/ptxas_regs.py csrc/file.cu [regex]"""
import re, subprocess, sys
src = sys.argv[1]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
extra = ["-ftz=true"] if "nbody" in src else []
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
                      "-Xcompiler", "-fPIC", "-Xptxas", "-v", *extra, "-I", "include", "-c", src, "-o", "/tmp/_x.o"],
                     capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and pat.search(cur):
        print(f"{m.group(1):>4} regs {spill:>4} B spill  {cur[:110]}")
        cur = None
