"""Per-instruction SASS execution counts / stall samples from an ncu source-page CSV.
    python tools/sass_hot.py <src.csv> <points>  -> opcode mix per point + top stalls"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
pts = float(sys.argv[2]) if len(sys.argv) > 2 else 20378025.0
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
warps = pts / 32
ops, stalls, lines = collections.Counter(), collections.Counter(), []
for r in rows[2:]:
    try:
        n = int(r[ix["Instructions Executed"]]); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError, IndexError):
        continue
    src = r[ix["Source"]].strip()
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)', src)
    op = m.group(2) if m else "?"
    ops[op] += n
    stalls[op] += s
    reasons = {h.replace("stall_", ""): int(v) for h, v in zip(hdr, r)
               if h.startswith("stall_") and "Not Issued" not in h and v not in ("", "0", "-")}
    lines.append((s, n / warps, r[ix["Address"]][-5:], src, reasons))
tot = sum(ops.values()); stot = sum(stalls.values())
print(f"warp instructions per point-warp: {tot / warps:.1f}; stall samples {stot}")
for k, v in ops.most_common(24):
    print(f"  {k:10s} {v / warps:7.1f}  stall {100 * stalls[k] / max(stot, 1):5.1f}%")
print("top stall instructions:")
for s, n, a, src, rs in sorted(lines, key=lambda x: -x[0])[:25]:
    top = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
    print(f"  {100 * s / max(stot, 1):5.1f}% x{n:5.2f} {a} {src[:60]:60s} {top}")
