import csv, collections, io, json, sys
def launches(path):
    txt=open(path).read(); txt=txt[txt.index('"ID"'):]
    agg=collections.defaultdict(list)
    for r in csv.DictReader(io.StringIO(txt)):
        if r.get('Metric Name')=='gpu__time_duration.sum':
            agg[r['Kernel Name'].split('(')[0][:50]].append(float(r['Metric Value']))
    for k,v in agg.items():
        print(f"  {k:50s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.1f} us  min={min(v)/1e3:9.1f}")
def bench(path):
    d=json.loads(open(path).read().strip().splitlines()[-1])
    e=d['extract']; s=d['smooth']
    print(f"  step {d['ms_per_step']:.3f} ms | ext {e['ms']:.3f} ms {e['voxels_per_s']/1e9:.1f} Gvox/s {e['gbs']:.0f} GB/s frac {e['frac']:.2f} | smooth {s['ms']:.3f} ms {s['pt_iters_per_s']/1e9:.1f} Gpt-it/s {s['gbs']:.0f} GB/s frac {s['frac']:.2f} | clocks {d['clocks']}")
for p in sys.argv[1:]:
    print(p); (launches if p.endswith('.csv') else bench)(p)
