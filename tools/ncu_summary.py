"""Summarise an ncu report (.ncu-rep) into a short text file for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_name.txt
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
]


def run(args):
    return subprocess.check_output(["ncu", "-i", *args], stderr=subprocess.DEVNULL).decode()


def main(rep):
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print(f"# ncu summary of {rep}")
    print(f"kernel: {d.get('Kernel Name')}")
    for k in KEYS:
        if k in d:
            print(f"  {k:62s} {d[k]:>22s} {u.get(k, '')}")
    st = []
    for k in hdr:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(d[k].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1.0
    print("warp stall samples (share):")
    for v, k in sorted(st, reverse=True)[:10]:
        print(f"  {k:30s} {100 * v / tot:6.1f}%")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = src[1]
    I = h.index
    c, e = Counter(), Counter()
    for r in src[2:]:
        op = re.sub(r"^@!?U?P\w+\s+", "", r[I("Source")].strip()).split(" ")[0].split(".")[0]
        c[op] += int(r[I("Warp Stall Sampling (All Samples)")] or 0)
        e[op] += int(r[I("Instructions Executed")] or 0)
    ts, te = sum(c.values()) or 1, sum(e.values()) or 1
    print("by SASS opcode: stall-sample share / executed-instruction share:")
    for op, v in c.most_common(15):
        print(f"  {op:10s} {100 * v / ts:6.1f}%  {100 * e[op] / te:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
