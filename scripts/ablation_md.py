"""Tables of an ablation run: python scripts/ablation_md.py ablation.jsonl > tables.md"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
mb = [r for r in rows if r["workload"] == "mb"]
wt = [r for r in rows if r["workload"] == "wator"]
ls = [r for r in rows if r["workload"] == "ls"]
print("## Allocator microbenchmark (configs[4], 2^26 + 2^25 objects, one step)\n")
print("| variant | step ms | new1 ms | new4 ms | drain ms | F after new1 | F after new4 |")
print("|---|---|---|---|---|---|---|")
for r in mb:
    if "error" in r:
        print(f"| {r['name']} | {r['error']} | | | | | |")
        continue
    p = r["phase_ms"]
    print(f"| {r['name']} | {r['step_ms']:.2f} | {p['new1']:.2f} | {p['new4']:.2f} | {p['drain6']:.2f} | "
          f"{r['frag_after_new1']:.4f} | {r['frag_after_new4']:.4f} |")
print("\n## Wa-Tor 2048^2 (configs[1])\n")
print("| variant | steps | ms/step | agent F at end | device error | fish | sharks |")
print("|---|---|---|---|---|---|---|")
for r in wt:
    if "error" in r and "ms_per_step" not in r:
        print(f"| {r['name']} | | {r['error']} | | | | |")
        continue
    print(f"| {r['name']} | {r.get('steps', '')} | {r['ms_per_step']:.4f} | {r['agent_frag']:.3f} | "
          f"{r.get('device_error', '')} | {r['fish']} | {r['sharks']} |")
print("\n## Linux Scalability (P:918-923): 16,384 threads x n objects of 64 B, 1 GiB heap\n")
print("| n | alloc ms | free ms | allocated / requested | OOM | heap utilisation |")
print("|---|---|---|---|---|---|")
for r in ls:
    print(f"| {r['n']} | {r['alloc_ms']:.3f} | {r['free_ms']:.3f} | {r['allocated']} / {r['requested']} | {r['oom']} | "
          f"{r['utilisation_of_heap']:.4f} |")
