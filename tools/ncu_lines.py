"""Aggregate ncu warp-stall samples per CUDA source line from a report (cuda,sass view).
python tools/ncu_lines.py <report.ncu-rep> [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = {}; fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]
    if len(r) > 6 and r[0] not in ("", "Line No") and r[4].isdigit():
        agg[(fname, int(r[0]))] = (int(r[4]), r[1][:100])
tot = sum(v[0] for v in agg.values()) or 1
for (f, l), (v, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v / tot * 100:5.1f}% {f}:{l:<5d} {s}")
