"""Summarise the raw-page CSVs of tools/round_measure.sh into
profiles/ncu_summary.json (per bench kernel name; bench.py reads
dram_bytes_per_launch as roofline.traffic) and a text table.

    python tools/ncu_raw_summary.py <tag> [config]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
SC = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
TS = {"ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}


def rows_of(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        d = {"kernel": r[ix["Kernel Name"]]}
        for k in KEYS:
            if k in ix:
                d[k] = r[ix[k]]
        rb = float(r[ix["dram__bytes_read.sum"]]) * SC[units[ix["dram__bytes_read.sum"]]]
        wb = float(r[ix["dram__bytes_write.sum"]]) * SC[units[ix["dram__bytes_write.sum"]]]
        t = float(r[ix["gpu__time_duration.sum"]]) * TS[units[ix["gpu__time_duration.sum"]]]
        d["dram_bytes_per_launch"] = rb + wb
        d["time_s"] = t
        d["dram_GBps"] = (rb + wb) / t / 1e9
        yield d


def main():
    tag = sys.argv[1]
    cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg5"
    out = {}
    e = list(rows_of(os.path.join(ROOT, "gpurun_out", f"{tag}_e_raw.csv")))
    s = list(rows_of(os.path.join(ROOT, "gpurun_out", f"{tag}_s_raw.csv")))
    for i, d in enumerate(e):
        out[f"explicit_stage{i}"] = d
    for i, d in enumerate(s):
        out[f"solve_stage{i}"] = d
    summ = {cfg: out}
    cpath = os.path.join(ROOT, "gpurun_out", f"{tag}_c_raw.csv")
    if os.path.exists(cpath):   # set2c: explicit stage 1 (k_ecolc M_S2)
        summ[cfg + ":set2c"] = {"explicit_stage1": list(rows_of(cpath))[0]}
    summ["source"] = (f"tools/round_measure.sh {tag}: ncu --set full --clock-control none, "
                      "first timed step of bench.py --steps 1 --warmup 3 [--set set2c]")
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    rows = list(out.items()) + [("set2c " + k, d) for k, d in summ.get(cfg + ":set2c", {}).items()]
    for k, d in rows:
        print(f"{k:16s} {d['time_s'] * 1e3:7.3f} ms  dram {d['dram_bytes_per_launch'] / 1e9:6.3f} GB "
              f"({d['dram_GBps']:7.1f} GB/s)  issue {float(d[KEYS[3]]):5.1f}%  warps "
              f"{float(d[KEYS[5]]):5.1f}%  regs {d[KEYS[6]]}  inst {float(d[KEYS[4]]):.3e}  "
              f"fp64 {float(d[KEYS[7]]):5.1f}%  bank-conflict wavefronts "
              f"{float(d[KEYS[8]]) / max(float(d[KEYS[9]]), 1):.3f}")
        print("    stalls/issue: long_sb %.2f barrier %.2f short_sb %.2f wait %.2f mio %.2f"
              % tuple(float(d.get(k, "nan")) for k in KEYS[11:16]))


if __name__ == "__main__":
    main()
