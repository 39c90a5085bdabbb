"""Summarise an ncu gpu__time_duration launch list per kernel.  python tools/launch_summary.py launches.csv"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
agg = collections.OrderedDict()
for r in rows:
    name = r[4].split('(')[0].replace('<unnamed>::', '').replace('void ', '')
    a = agg.setdefault(name, [0, 0.0, []]); a[0] += 1; a[1] += float(r[-1]); a[2].append(float(r[-1]) / 1e3)
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    per = "" if v[0] == 1 else " [" + ", ".join(f"{x:.0f}" for x in v[2][:16]) + "]"
    print(f"{k:28s} n={v[0]:3d} {v[1] / 1e6:7.3f} ms{per}")
print(f"{'total':28s}       {tot / 1e6:7.3f} ms")
