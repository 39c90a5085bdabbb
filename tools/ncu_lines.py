"""Aggregate ncu warp-stall samples and executed instructions per CUDA source line (cuda,sass view).
python tools/ncu_lines.py <report.ncu-rep> [top] [--inst]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
by_inst = "--inst" in sys.argv
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = {}; fname = ""; hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]
    if len(r) > 6 and r[0] == "Line No": hdr = r
    if hdr and len(r) > 6 and r[0] not in ("", "Line No") and r[4].isdigit():
        ie = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else 7
        agg[(fname, int(r[0]))] = (int(r[4]), int(r[ie] or 0), r[1][:100])
k = 1 if by_inst else 0
tot = sum(v[k] for v in agg.values()) or 1
print(f"total {'instructions' if by_inst else 'stall samples'}: {tot}")
for (f, l), v in sorted(agg.items(), key=lambda kv: -kv[1][k])[:top]:
    print(f"{v[k] / tot * 100:5.1f}% {f}:{l:<5d} {v[2]}")
