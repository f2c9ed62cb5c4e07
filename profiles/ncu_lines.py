"""Per-CUDA-line executed warp instructions and stall samples of one launch in an ncu report.

    python profiles/ncu_lines.py REPORT [top] [launch_index(1-based)]

Reads `ncu -i REPORT --page source --csv --print-source cuda,sass` (no GPU needed): every CUDA line
is followed by its SASS rows; inlined code is attributed to the line of the inlined function."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
which = int(sys.argv[3]) if len(sys.argv) > 3 else 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, launch, seen_files = "", None, 0, set()
agg = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        if r[1] in seen_files:
            launch += 1
            seen_files = set()
        seen_files.add(r[1])
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ci = hdr.index("Instructions Executed")
        cs = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or launch + 1 != which:
        continue
    if r[0]:  # a CUDA line
        cur = (fname, r[0], r[1].strip()[:100])
        agg.setdefault(cur, [0.0, 0.0])
        continue
    try:
        agg[cur][0] += float(r[ci] or 0)
        agg[cur][1] += float(r[cs] or 0)
    except (ValueError, IndexError):
        pass
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"warp instructions {tot:.4g}, stall samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% inst {100 * v[1] / ts:5.1f}% stall | {k[0]}:{k[1]} {k[2]}")
