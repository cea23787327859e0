"""Per-opcode share of warp-stall samples and of executed warp instructions for one kernel
capture (ncu --set full --import-source on), plus the headline pipe metrics:
    python tools/ncu_ops.py gpurun_out/x.ncu-rep [more.ncu-rep ...]"""
import collections
import csv
import io
import subprocess
import sys

HEAD = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, v = raw[0], raw[2]
    print(rep, v[h.index("Kernel Name")][:60])
    for n in HEAD:
        if n in h:
            print(f"  {n} = {v[h.index(n)]}")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source",
                                           "sass"))))
    hh, data = rows[1], rows[2:]
    i_s, i_i = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    ts = sum(float(r[i_s] or 0) for r in data)
    ti = sum(float(r[i_i] or 0) for r in data)
    st, ins = collections.Counter(), collections.Counter()
    for r in data:
        t = r[1].split()
        o = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
        st[o] += float(r[i_s] or 0)
        ins[o] += float(r[i_i] or 0)
    print(f"  warp instructions {ti:.3g}; opcode: stall share / instruction share")
    print("  " + "  ".join(f"{o} {100 * s / ts:.0f}/{100 * ins[o] / ti:.0f}"
                           for o, s in st.most_common(16)))
