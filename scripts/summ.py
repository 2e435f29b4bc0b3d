"""Summarise a gpurun job's bench lines and ncu launch list (scratch helper)."""
import csv, collections, json, sys, glob
tag = sys.argv[1]
for f in sorted(glob.glob(f'gpurun_out/{tag}_bench_*.json')):
    try:
        d = json.load(open(f))
        print(f.split('_bench_')[1][:-5], round(d['ms_per_step'], 3), round(d['e2e']['ms_per_step'], 3),
              {k: round(v, 3) for k, v in (d.get('stage_ms') or {}).items()})
    except Exception as e:
        print(f, 'ERR', e)
for f in sorted(glob.glob(f'gpurun_out/{tag}_launches_*.csv')):
    rows = list(csv.reader(open(f)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]; ki = h.index('Kernel Name'); mi = h.index('Metric Name'); vi = h.index('Metric Value'); ii = h.index('ID')
    per = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi: continue
        key = (r[ii], r[ki].split('(')[0].split('<')[0].replace('void ', ''))
        per.setdefault(key, {})[r[mi]] = float(r[vi].replace(',', ''))
    agg = collections.OrderedDict()
    for (i, n), m in per.items():
        a = agg.setdefault(n, [0, 0, 0, 0])
        a[0] += 1; a[1] += m.get('gpu__time_duration.sum', 0); a[2] += m.get('dram__bytes_read.sum', 0); a[3] += m.get('dram__bytes_write.sum', 0)
    print('==', f, 'total %.3f ms' % (sum(a[1] for a in agg.values()) / 1e6))
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
        print(f"  {n:32s} x{a[0]:4d} {a[1]/1e3:9.1f} us  rd {a[2]/1e6:8.1f} MB wr {a[3]/1e6:8.1f} MB")
