"""Per-opcode executed warp instructions and stall totals of the first kernel in an ncu report.

    python profiles/ncu_sass_opcodes.py REPORT [top] [kernel_index]

Reads `ncu -i REPORT --page source --csv --print-source sass` (no GPU needed)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
which = int(sys.argv[3]) if len(sys.argv) > 3 else 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
col = {h: i for i, h in reversed(list(enumerate(hdr)))}
ops = collections.Counter()
stalls = collections.Counter()
total = 0
kernels = 0
for r in rows:
    if not r:
        continue
    if r[0] == "Kernel Name":
        kernels += 1
        continue
    if kernels != which or r[0] == "Address" or len(r) < len(hdr) - 2:
        continue
    src = r[col["Source"]].strip()
    tok = src.split()
    if tok and tok[0].startswith("@"):
        tok = tok[1:]
    op = tok[0].rstrip(";") if tok else "?"
    base = op.split(".")[0]
    if base in ("LDS", "LDG", "STS", "STG", "ATOMG", "ATOM", "RED", "LD", "ST"):
        base = ".".join(op.split(".")[:3])
    n = float(r[col["Instructions Executed"]] or 0)
    ops[base] += n
    total += n
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stalls[h] += float(r[col[h]] or 0)
            except ValueError:
                pass
print(f"total warp instructions {total:.4g}")
for op, n in ops.most_common(top):
    print(f"  {op:28s} {n:12.4g} {100 * n / total:5.1f}%")
ts = sum(stalls.values())
print("stall samples:")
for k, v in stalls.most_common(10):
    print(f"  {k:24s} {v:9.0f} {100 * v / ts:5.1f}%")
