"""Per-CUDA-line instruction counts from `ncu --page source --print-source cuda,sass --csv`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
for hi, r in enumerate(rows):
    if r and r[0] == 'Line No':
        break
hdr = rows[hi]
iE = hdr.index('Instructions Executed'); iW = hdr.index('Warp Stall Sampling (All Samples)')
per = collections.OrderedDict(); cur = None; fname = ''
for r in rows:
    if r and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if len(r) <= iE or (r and r[0] in ('Line No', 'Function Name')):
        continue
    if r[0]:
        cur = (fname + ':' + r[0], r[1][:100]); per.setdefault(cur, [0, 0])
        continue
    try:
        per[cur][0] += int(r[iE] or 0); per[cur][1] += int(r[iW] or 0)
    except (ValueError, KeyError):
        pass
tot = sum(v[0] for v in per.values()); totw = sum(v[1] for v in per.values())
print('total instr', tot, 'stall samples', totw)
K = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for (ln, src), (n, w) in sorted(per.items(), key=lambda kv: -kv[1][0])[:K]:
    print(f'{n:12d} {100*n/tot:5.1f}%  stall {100*w/max(totw,1):5.1f}%  {ln:<22s} {src}')
