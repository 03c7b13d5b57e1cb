"""Summarise the round's two ncu --set full captures (k_lsar_pass_fft, k_fft_fold at C4; tools/r02_profile.sh)
into profiles/r02_ncu_fft_pass_c4.txt and the FFT entry of profiles/r02_pass_traffic.json.

  python tools/r02_ncu_report.py gpurun_out/ncu_fft_c4.ncu-rep gpurun_out/ncu_fold_c4.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W = 999_999_500
SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis", "Occupancy",
            "Launch Statistics", "Scheduler Statistics", "Warp State Statistics")
NAMES = ("Duration", "SM Frequency", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
         "L2 Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
         "Registers Per Thread", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block",
         "Shared Memory Configuration Size", "Grid Size", "Block Size", "Theoretical Occupancy", "Achieved Occupancy",
         "Warp Cycles Per Issued Instruction", "No Eligible", "Executed Ipc Active")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def ncu(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "raw"))))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (x, y) for k, x, y in zip(h, u, v)}


def num(d, k):
    u, v = d[k]
    return float(v.replace(",", "")) * SCALE.get(u, 1)


def report(rep):
    d = raw(rep)
    name = d["Kernel Name"][1].split("(")[0].replace("void ", "")
    rd, wr, t = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum"), num(d, "gpu__time_duration.sum")
    lines = [f"== {name}: one launch at lag ~ 260 of the C4 sweep (w = {W} rows)",
             f"dram__bytes_read.sum {rd / 1e9:.3f} GB, dram__bytes_write.sum {wr / 1e9:.3f} GB -> {(rd + wr) / 1e9:.2f} GB "
             f"per launch ({(rd + wr) / W:.1f} B/row)",
             f"gpu__time_duration  {t * 1e3:.3f} ms -> {(rd + wr) / t / 1e12:.2f} TB/s of DRAM traffic",
             f"fp64 pipe {num(d, 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f} % of active cycles, "
             f"LSU data-pipe wavefronts {num(d, 'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed'):.1f} % "
             f"(shared-memory wavefronts {num(d, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'):.3g})"]
    st = sorted(((num(d, k), k) for k in d if "issue_stalled" in k and k.endswith("_per_issue_active.ratio")
                 and "not_issued" not in k), reverse=True)[:6]
    lines.append("warp stall cycles per issued instruction: " + ", ".join(
        f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {x:.2f}" for x, k in st))
    lines.append("")
    for r in csv.reader(io.StringIO(ncu(rep, "details"))):
        if len(r) > 14 and r[11] in SECTIONS and r[12] in NAMES:
            lines.append(f"{r[11]} | {r[12]} | {r[13]} | {r[14]}")
    return name, rd, wr, t, "\n".join(lines)


def main():
    reps = sys.argv[1:3]
    out, tot = [], {}
    for rep in reps:
        name, rd, wr, t, text = report(rep)
        out.append(text)
        tot[name] = dict(dram_bytes_read=rd, dram_bytes_write=wr, duration_s_under_ncu=t)
    rd = sum(v["dram_bytes_read"] for v in tot.values())
    wr = sum(v["dram_bytes_write"] for v in tot.values())
    t = sum(v["duration_s_under_ncu"] for v in tot.values())
    head = ("FFT lags of the C4 sweep (n = 1e9, p = 1..500, s = 2e5) after the split: k_lsar_pass_fft (transform -> r_q, chunk\n"
            "sums of r_q^2) and k_fft_fold (the deferred score update; beside the solve in the timed sweeps, alone here).\n"
            "ncu --set full --clock-control none --import-source on -k regex:<kernel> --launch-skip 200 --launch-count 1\n"
            "  python bench.py --steps 1 --warmup 3 --no-cpu      (reports: gpurun_out/ncu_fft_c4.ncu-rep, ncu_fold_c4.ncu-rep)\n\n"
            f"per lag, both kernels: {(rd + wr) / 1e9:.2f} GB of DRAM traffic ({(rd + wr) / W:.1f} B/row; algorithmic 24 B/row -> "
            f"{(rd + wr) / (24.0 * W):.2f}x) in {t * 1e3:.2f} ms back to back = {24.0 * W / t / 1e12:.2f} TB/s on the algorithmic "
            f"bytes = {24.0 * W / t / 6546.9e9:.2f} of the 6547 GB/s copy peak\n\n")
    open(os.path.join(ROOT, "profiles", "r02_ncu_fft_pass_c4.txt"), "w").write(head + "\n\n".join(out) + "\n")
    pj = os.path.join(ROOT, "profiles", "r02_pass_traffic.json")
    j = json.load(open(pj))
    j["k_lsar_pass_fft"] = {
        "w": W, "dram_bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
        "algorithmic_bytes_per_launch": 24.0 * W, "traffic_over_algorithmic": (rd + wr) / (24.0 * W),
        "kernels": tot,
        "source": "ncu --set full --clock-control none at C4 (bench.py), one launch each of k_lsar_pass_fft (split) and "
                  "k_fft_fold at lag ~260 -- profiles/r02_ncu_fft_pass_c4.txt",
        "note": "30.7 B/row by design: the series spectrum 10.7 + r_q out 8 (the pass) + the deferred score update "
                "(8 + 4*8 + 8)/4 = 12 (the fold), plus the L2 prefetches' overfetch"}
    json.dump(j, open(pj, "w"), indent=1)
    print(head)


if __name__ == "__main__":
    main()
