"""Dynamic SASS mix of an ncu source-page CSV (--print-source cuda,sass):
python scripts/ncu_src_summary.py src.csv.gz [top_lines] [kernel index, 0-based, in capture order]"""
import collections, csv, gzip, io, sys

txt = gzip.open(sys.argv[1], 'rt').read() if sys.argv[1].endswith('.gz') else open(sys.argv[1]).read()
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = list(csv.reader(io.StringIO(txt)))
# kernels follow one another; each starts again with the first source file
first = next(r[1] for r in rows if r and r[0] == 'File Path')
kid, sel = -1, []
for r in rows:
    if r and r[0] == 'File Path' and r[1] == first:
        kid += 1
    if kid == want:
        sel.append(r)
rows = sel
ops, lines, seen, cur, curfile, tot = collections.Counter(), collections.Counter(), set(), None, None, 0
thr = 0
for r in rows:
    if r and r[0] == 'File Path':
        curfile = r[1].split('/')[-1]
    if len(r) < 9 or r[0] == 'Line No':
        continue
    if r[2] == '-':
        cur = (curfile, r[0], r[1][:80])
        continue
    if r[2].startswith('0x') and r[2] not in seen:
        seen.add(r[2])
        n = int(r[7] or 0)
        tot += n
        thr += int(r[8] or 0)
        op = r[3].split()[0]
        if op.startswith('@'):
            op = r[3].split()[1]
        ops[op.split('.')[0]] += n
        lines[cur] += n
print(f'warp instructions {tot / 1e6:.1f} M, active threads per instruction {thr / max(tot, 1):.1f}')
print(' '.join(f'{o}:{n / tot:.3f}' for o, n in ops.most_common(16)))
for l, n in lines.most_common(top):
    print(f'{n / 1e6:8.1f} {n / tot:.3f}', l)
