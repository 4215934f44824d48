"""Summarise gpu_ab_multi.sh logs: python scripts/abm_summary.py gpurun_out/abm_TAG.log"""
import collections, json, sys

cur, res = None, collections.defaultdict(list)
for line in open(sys.argv[1]):
    if line.startswith('LIB'):
        cur = line.split()[1].split('/')[-1]
    elif line.startswith('{'):
        p = json.loads(line)['phase_ms']
        res[cur].append((p['new1'], p['new4'], round(sum(p.values()), 3)))
for k, v in res.items():
    print(f'{k:20s} new1/new4/step', v)
