"""Per-family DRAM traffic of ONE step from an ncu launch list with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (the last step of the capture).
python tools/ncu_traffic.py launches.csv out.json [launches_per_step]"""
import collections, csv, json, sys

FAM = [("k_aca", "aca"), ("k_leaf_chol", "leaf_chol"), ("k_leaf_zsyrk", "leaf_factor"), ("k_leaf_factor", "leaf_factor"),
       ("k_tree_factor", "coupling_tree"), ("k_logdet", "coupling_tree"), ("k_solve", "solve"),
       ("k_make_keys", "sort"), ("k_hist", "sort"), ("k_scan", "sort"), ("k_scatter", "sort"), ("k_finish", "sort")]


def family(name):
    for pre, f in FAM:
        if pre in name:
            return f
    return "other"


rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
per = collections.OrderedDict()
for r in rows:
    per.setdefault(int(r[0]), {"name": r[4].split("(")[0].replace("<unnamed>::", "").replace("void ", "")})[r[12]] = \
        float(r[14].replace(",", ""))
launches = list(per.values())
# one step = the launches after the last k_make_keys (the sort is the first kernel of a build)
starts = [i for i, l in enumerate(launches) if "k_make_keys" in l["name"]]
step = launches[starts[-1]:] if starts else launches
fam = collections.OrderedDict()
for l in step:
    f = fam.setdefault(family(l["name"]), {"launches": 0, "ms": 0.0, "dram_bytes": 0.0, "kernels": {}})
    b = l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    f["launches"] += 1; f["ms"] += l.get("gpu__time_duration.sum", 0.0) / 1e6; f["dram_bytes"] += b
    k = f["kernels"].setdefault(l["name"], {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    k["launches"] += 1; k["ms"] += l.get("gpu__time_duration.sum", 0.0) / 1e6; k["dram_bytes"] += b
tot = sum(f["ms"] for f in fam.values())
for f in fam.values():
    f["share_of_step"] = f["ms"] / tot if tot else None
json.dump({"source": sys.argv[1], "note": "ncu --clock-control none, serialized cold-cache launches of one step",
           "step_launches": len(step), "serialized_ms": tot, "families": fam}, open(sys.argv[2], "w"), indent=1)
for k, f in fam.items():
    print(f"{k:14s} n={f['launches']:3d} {f['ms']:7.3f} ms  {f['dram_bytes'] / 1e9:7.3f} GB  share {f['share_of_step']:.2f}")
