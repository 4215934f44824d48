"""Stall samples per source line of one kernel in an ncu source-page CSV:
python scripts/ncu_src_stalls.py src.csv.gz kernel_index [top]"""
import collections, csv, gzip, io, sys

txt = gzip.open(sys.argv[1], 'rt').read() if sys.argv[1].endswith('.gz') else open(sys.argv[1]).read()
want = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
rows = list(csv.reader(io.StringIO(txt)))
first = next(r[1] for r in rows if r and r[0] == 'File Path')
kid, sel = -1, []
for r in rows:
    if r and r[0] == 'File Path' and r[1] == first:
        kid += 1
    if kid == want:
        sel.append(r)
fn = next((r[1] for r in sel if r and r[0] == 'Function Name'), '?')
samp, cur, curfile, tot, seen = collections.Counter(), None, None, 0, set()
for r in sel:
    if r and r[0] == 'File Path':
        curfile = r[1].split('/')[-1]
    if len(r) < 8 or r[0] == 'Line No':
        continue
    if r[2] == '-':
        cur = (curfile, r[0], r[1][:80])
        continue
    if r[2].startswith('0x') and r[2] not in seen:
        seen.add(r[2])
        n = int(r[4] or 0)
        samp[cur] += n
        tot += n
print(fn[:100], 'samples', tot)
for l, n in samp.most_common(top):
    print(f'{n / max(tot, 1):.3f}', l)
