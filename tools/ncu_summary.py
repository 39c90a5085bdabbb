"""Summarise the ncu --set full captures of tools/round_profile.sh into profiles/rNN_ncu_summary.json
(per kernel: duration, DRAM bytes, throughputs, registers, FP64 pipe use, grid) and copy the per-line stall
tables.  python tools/ncu_summary.py gpurun_out/<tag> <round> "<note on the capture>" """
import csv, glob, json, os, subprocess, sys

src, rnd = sys.argv[1], int(sys.argv[2])
note = sys.argv[3] if len(sys.argv) > 3 else ""
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = {
    "duration_s": ("gpu__time_duration.sum", 1e-9),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "mem_throughput_pct": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fp64_tensor_pct": ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", 1.0),
    "grid": ("launch__grid_size", 1.0),
}
UNIT = {"msecond": 1e6, "usecond": 1e3, "nsecond": 1.0, "second": 1e9, "ms": 1e6, "us": 1e3, "ns": 1.0, "s": 1e9,
        "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def val(row, units, key, scale):
    if key not in row or row[key] in ("", "n/a"):
        return None
    v = float(row[key].replace(",", ""))
    u = units.get(key, "")
    if key == "gpu__time_duration.sum":
        return v * UNIT.get(u, 1.0) * scale
    if key.startswith("dram__bytes"):
        return v * UNIT.get(u, 1.0)
    return v * scale


out = {"round": rnd, "source": note, "kernels": {}}
for f in sorted(glob.glob(os.path.join(src, "*.raw.csv"))):
    name = os.path.basename(f)[:-len(".raw.csv")]
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    hdr, units, row = rows[0], dict(zip(rows[0], rows[1])), dict(zip(rows[0], rows[2]))
    k = {fld: val(row, units, key, sc) for fld, (key, sc) in FIELDS.items()}
    if k["dram_read_bytes"] is not None and k["dram_write_bytes"] is not None:
        k["dram_bytes"] = k["dram_read_bytes"] + k["dram_write_bytes"]
    out["kernels"][name] = k
    rep = f[:-len(".raw.csv")] + ".ncu-rep"
    if os.path.exists(rep):
        txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep],
                             capture_output=True, text=True).stdout
        with open(os.path.join(ROOT, "profiles", f"r{rnd:02d}_{name}_source_stalls.txt"), "w") as g:
            g.write(txt)
path = os.path.join(ROOT, "profiles", f"r{rnd:02d}_ncu_summary.json")
with open(path, "w") as g:
    json.dump(out, g, indent=1)
print(path, {n: round(v["duration_s"] * 1e6, 1) for n, v in out["kernels"].items() if v.get("duration_s")})
