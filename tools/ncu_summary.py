"""Summarise ncu --set full reports (raw page) into one line per kernel."""
import csv, subprocess, sys, json
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
TSCALE = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1.0, "second": 1.0}
def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[ix["Kernel Name"]]}
        for k in KEYS:
            if k in ix:
                d[k] = r[ix[k]]
        rb = float(r[ix["dram__bytes_read.sum"]]) * SCALE[units[ix["dram__bytes_read.sum"]]]
        wb = float(r[ix["dram__bytes_write.sum"]]) * SCALE[units[ix["dram__bytes_write.sum"]]]
        t = float(r[ix["gpu__time_duration.sum"]]) * TSCALE[units[ix["gpu__time_duration.sum"]]]
        d["dram_bytes_per_launch"] = rb + wb
        d["time_s"] = t
        d["dram_GBps"] = (rb + wb) / t / 1e9
        res.append(d)
    return res
if __name__ == "__main__":
    for rep in sys.argv[1:]:
        for d in summarise(rep):
            short = {k.split("__")[-1].replace(".avg.pct_of_peak_sustained_active", "%").replace("average_warps_issue_stalled_", "stall_").replace("_per_issue_active.ratio", ""): v for k, v in d.items() if k != "kernel"}
            print(d["kernel"][:60])
            print("   ", json.dumps({k: (round(float(v), 3) if isinstance(v, (int, float)) or v.replace('.', '', 1).replace('e', '', 1).replace('-', '', 1).replace('+','',1).isdigit() else v) for k, v in short.items()}))
