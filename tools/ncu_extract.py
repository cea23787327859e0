"""Summarise `ncu --set full` reports into profiles/: per-kernel key metrics (CSV) and the DRAM
traffic per X pass that bench.py reports as roofline.traffic (profiles/ncu_traffic.json).

usage: python tools/ncu_extract.py gpurun_out/prof_tc.ncu-rep [more.ncu-rep ...] --round r01
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return [{h: (v, u) for h, u, v in zip(hdr, units, r)} for r in data]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    recs = []
    for rep in a.reports:
        for k in raw(rep):
            rec = {"report": os.path.basename(rep), "kernel": k["Kernel Name"][0]}
            for key in KEYS:
                if key in k:
                    rec[key] = k[key][0]
                    rec[key + " [unit]"] = k[key][1]
            recs.append(rec)
    cols = ["report", "kernel"] + [c for key in KEYS for c in (key, key + " [unit]")]
    path = os.path.join(root, "profiles", f"{a.round}_ncu_full_metrics.csv")
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=cols, extrasaction="ignore")
        w.writeheader()
        for r in recs:
            w.writerow(r)
    print("wrote", path)

    def gb(v, u):
        f = float(v.replace(",", ""))
        return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)

    p1 = [r for r in recs if "tc_i8_kernel<3>" in r["kernel"] or "tc_i8_kernel<(int)3>" in r["kernel"]]
    p2 = [r for r in recs if "tc_i8_kernel<4>" in r["kernel"] or "tc_i8_kernel<(int)4>" in r["kernel"]]
    if p1 and p2:
        def tb(r):
            return gb(r["dram__bytes_read.sum"], r["dram__bytes_read.sum [unit]"]) + \
                gb(r["dram__bytes_write.sum"], r["dram__bytes_write.sum [unit]"])
        b1, b2 = tb(p1[0]), tb(p2[0])
        tj = {"tc-i8x4-exact": {"bytes_per_pass": (b1 + b2) / 2, "pass1_bytes": b1,
                                "pass2_bytes": b2,
                                "source": f"profiles/{a.round}_ncu_full_metrics.csv (ncu --set full, "
                                          "dram__bytes_read.sum + dram__bytes_write.sum)"}}
        with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as fh:
            json.dump(tj, fh, indent=1)
        print("traffic per pass", tj)


if __name__ == "__main__":
    main()
