"""Per-source-line instruction / stall breakdown from an ncu report."""
import csv, subprocess, sys
rep, kfilter = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = cur_fn = None
hdr = None
acc = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        cur_fn = r[1]; continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in reversed(list(enumerate(r)))}; continue
    if hdr is None or r[0] == "" or kfilter not in (cur_fn or ""):
        continue
    try:
        ins = int(float(r[hdr["Instructions Executed"]] or 0))
        smp = int(float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0))
    except (ValueError, KeyError):
        continue
    key = (cur_file, r[0])
    a = acc.setdefault(key, [0, 0, r[1][:90]])
    a[0] += ins; a[1] += smp
tot = sum(v[0] for v in acc.values()); ts = sum(v[1] for v in acc.values())
print("total warp-inst", tot, "samples", ts)
for (f, ln), (ins, smp, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 35]:
    print(f"{f}:{ln:>5} inst {ins/tot*100:5.1f}% stall {smp/ts*100:5.1f}%  {src}")
