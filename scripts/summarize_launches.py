"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections, csv, io, sys
txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    name = r['Kernel Name'].split('(')[0]
    us = float(r['Metric Value'].replace(',', '')) * scale[r['Metric Unit']]
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(a[1] for a in agg.values())
print(f"{'share':>7} {'launches':>8} {'total_ms':>10}  kernel")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us / tot * 100:6.2f}% {n:8d} {us / 1000:10.3f}  {k[:120]}")
print(f"total {tot / 1000:.3f} ms over {sum(a[0] for a in agg.values())} launches "
      "(ncu: serialized, cold-cache per launch; compare shares, not absolutes)")
