"""Summarise an ncu --set full report (one kernel launch) for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_k2.ncu-rep [algorithmic_bytes] > profiles/xxx.md

Prints the metrics the roofline line is built from (duration, dram bytes,
dram / tensor-pipe utilisation), occupancy facts, the top warp-stall reasons
and the SASS evidence (UTC*MMA / LDTM / LDGSTS counts).
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__cluster_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block",
    "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers",
]


def ncu(path: str, *args: str) -> str:
    return subprocess.run(["ncu", "-i", path, *args], capture_output=True, text=True).stdout


def main():
    path = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = list(csv.reader(io.StringIO(ncu(path, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    print(f"# ncu summary: `{path.split('/')[-1]}`\n")
    print(f"kernel: `{m.get('Kernel Name', ('', '?'))[1]}`\n")
    print("| metric | unit | value |\n|---|---|---|")
    for k in KEYS:
        if k in m:
            print(f"| {k} | {m[k][0]} | {m[k][1]} |")
    stalls = []
    for h, (u, v) in m.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print("\ntop warp stalls (warps per issue-active cycle): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
    if alg is not None and "gpu__time_duration.sum" in m:
        u, v = m["gpu__time_duration.sum"]
        t = float(v) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(u, 1e-9)
        rd = m["dram__bytes_read.sum"]
        wr = m["dram__bytes_write.sum"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic = float(rd[1]) * scale.get(rd[0], 1) + float(wr[1]) * scale.get(wr[0], 1)
        print(f"\nalgorithmic bytes {alg:.4g}; dram traffic {traffic:.4g} ({traffic / alg:.3f}x algorithmic); "
              f"algorithmic GB/s at the ncu (cold, serialised) duration: {alg / t / 1e9:.1f}")
    src = ncu(path, "--page", "source", "--csv", "--print-source", "sass")
    counts = {}
    for line in csv.reader(io.StringIO(src)):
        if len(line) < 2:
            continue
        ins = line[1].strip()
        if ins.startswith("@"):
            ins = ins.split(None, 1)[1] if " " in ins else ins
        op = ins.split(" ")[0]
        for key in ("UTCHMMA", "UTCQMMA", "LDTM", "STTM", "UTCBAR", "LDGSTS", "UBLKCP", "UTMALDG", "HMMA", "REDG"):
            if op.startswith(key):
                counts[key] = counts.get(key, 0) + 1
    print("\nSASS evidence (static instruction counts): " + ", ".join(f"{k} {v}" for k, v in sorted(counts.items())))


if __name__ == "__main__":
    main()
