"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, d, order = None, collections.defaultdict(list), []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    rec = dict(zip(hdr, r))
    if rec.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    name = rec['Kernel Name']
    for pre in ('void ', 'npcg::', '<unnamed>::', 'npcg::<unnamed>::'):
        name = name.replace(pre, '')
    name = name.split('(')[0][:48]
    v = float(rec['Metric Value'].replace(',', ''))
    unit = rec.get('Metric Unit', 'nsecond')
    us = v / 1e3 if unit.startswith('n') else (v if unit.startswith('u') else v * 1e3)
    d[name].append(us)
tot = sum(sum(v) for v in d.values())
print("%-48s %5s %10s %10s %6s" % ("kernel", "n", "mean_us", "total_us", "share"))
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print("%-48s %5d %10.1f %10.1f %5.1f%%" % (k, len(v), sum(v) / len(v), sum(v), 100 * sum(v) / tot))
print("total %.1f us over %d launches" % (tot, sum(len(v) for v in d.values())))
