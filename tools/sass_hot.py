"""Aggregate an ncu source-page SASS csv: instructions executed by opcode and hottest ranges."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iS, iE, iW = hdr.index('Address'), hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
ops = collections.Counter(); tot = 0; recs = []
for r in rows[2:]:
    try:
        n = int(r[iE] or 0); w = int(r[iW] or 0)
    except (ValueError, IndexError):
        continue
    op = r[iS].split()[0] if r[iS].split() else ''
    if op.startswith('@'):
        op = r[iS].split()[1]
    ops[op.split('.')[0]] += n; tot += n
    recs.append((r[iA], r[iS], n, w))
print('total warp-instr', tot)
for op, n in ops.most_common(25):
    print(f'  {op:12s} {n:14d} {100*n/tot:5.1f}%')
# hottest windows of 32 instructions
K = int(sys.argv[2]) if len(sys.argv) > 2 else 12
win = []
for s in range(0, len(recs), 16):
    seg = recs[s:s + 16]
    win.append((sum(x[2] for x in seg), sum(x[3] for x in seg), s))
win.sort(reverse=True)
for n, w, s in win[:K]:
    print(f'--- block @{recs[s][0]} instr={n} stall_samples={w}')
    for a, src, c, ww in recs[s:s + 16]:
        print(f'    {a} {c:12d} {ww:6d}  {src[:90]}')
