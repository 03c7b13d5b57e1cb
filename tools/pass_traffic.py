"""Summarise an ncu --set full capture of the fused pass into profiles/ncu_pass_traffic.json."""
import csv, io, json, subprocess, sys
rep, n, p_bar, q = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
def num(k):
    v = float(d[k].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}.get(u[k], 1)
    return v * scale
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
w = n - p_bar
res = {"kernel": d.get("Kernel Name", "").split("(")[0], "lag": q, "n": n, "p_bar": p_bar,
       "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch_avg": rd + wr,
       "algorithmic_bytes_per_launch": 24.0 * w, "moved_bytes_model": 40.0 * w,
       "duration_s_under_ncu": num("gpu__time_duration.sum"),
       "note": "one ncu --set full capture of the launch at this lag inside a C2 LSAR sweep (clock-control none); algorithmic = 24 B/row (y, s in, s out); "
               "the kernel also reads and writes r (40 B/row moved)"}
json.dump(res, open("profiles/ncu_pass_traffic.json", "w"), indent=1)
print(json.dumps(res))
