"""Per-source-line global-memory sectors and stall samples from an ncu report's source page.

    python profiles/ncu_source_sectors.py REPORT [top]

Reads `ncu -i REPORT --page source --csv --print-source cuda,sass` (no GPU needed) and prints the
CUDA lines with the most L2 theoretical sectors (with ideal / excessive) and the most stall samples.
With several launches in the report the page aggregates the first one."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows_all = []
fname = ""
hdr = None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Function Name":
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None:
        continue
    rows_all.append((fname, rec))
col = {}
for i, h in enumerate(hdr):
    col.setdefault(h, i)


def num(r, k):
    try:
        return float(r[col[k]])
    except (KeyError, ValueError, IndexError):
        return 0.0


tot_s = sum(num(r, "L2 Theoretical Sectors Global") for _, r in rows_all)
tot_i = sum(num(r, "L2 Theoretical Sectors Global Ideal") for _, r in rows_all)
tot_samp = sum(num(r, "Warp Stall Sampling (All Samples)") for _, r in rows_all)
tot_w = sum(num(r, "L1 Wavefronts Shared") for _, r in rows_all)
tot_wi = sum(num(r, "L1 Wavefronts Shared Ideal") for _, r in rows_all)
print(f"L2 theoretical sectors {tot_s * 32 / 1e6:.1f} MB (ideal {tot_i * 32 / 1e6:.1f} MB); shared wavefronts "
      f"{tot_w:.3g} (ideal {tot_wi:.3g}); stall samples {tot_samp:.0f}")
print("lines by L2 sectors:")
for f, r in sorted(rows_all, key=lambda x: -num(x[1], "L2 Theoretical Sectors Global"))[:top]:
    s = num(r, "L2 Theoretical Sectors Global")
    if s <= 0:
        break
    print(f"  {s * 32 / 1e6:8.1f} MB ideal {num(r, 'L2 Theoretical Sectors Global Ideal') * 32 / 1e6:8.1f} "
          f"| {f}:{r[0]} {r[1].strip()[:90]}")
print("lines by shared wavefronts:")
for f, r in sorted(rows_all, key=lambda x: -num(x[1], "L1 Wavefronts Shared"))[:6]:
    print(f"  {num(r, 'L1 Wavefronts Shared'):10.3g} ideal {num(r, 'L1 Wavefronts Shared Ideal'):10.3g} "
          f"| {f}:{r[0]} {r[1].strip()[:90]}")
print("lines by stall samples:")
for f, r in sorted(rows_all, key=lambda x: -num(x[1], "Warp Stall Sampling (All Samples)"))[:top]:
    print(f"  {num(r, 'Warp Stall Sampling (All Samples)') / max(tot_samp, 1) * 100:5.1f}% | {f}:{r[0]} "
          f"{r[1].strip()[:100]}")
