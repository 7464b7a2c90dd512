"""Per-kernel hot SASS regions (runs of equal execution count) of an ncu report.

    python tools/ncu_regions2.py REP.ncu-rep KERNEL_REGEX [min_frac] [launch_skip]
Prints the region's share of executed warp instructions and stall samples, and the
opcode histogram of each hot region.
"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
minf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
lines = []
base = None
for r in rows[hi + 1:]:
    try:
        a = int(r[0], 16)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    lines.append((a - base, int(r[ix["Instructions Executed"]] or 0), int(r[ix["# Samples"]] or 0), r[1].strip()))
tot = sum(l[1] for l in lines)
S = sum(l[2] for l in lines) or 1
print(f"{rows[0][1][:90]}\ntotal warp inst {tot}  samples {S}")
runs = []
for a, n, s, t in lines:
    if runs and runs[-1][2] == n:
        runs[-1][1] = a
        runs[-1][3] += 1
        runs[-1][4] += s
        runs[-1][6].append(t)
    else:
        runs.append([a, a, n, 1, s, t, [t]])
for st, la, n, c, s, t, ops in runs:
    if n * c > tot * minf or s > S * minf * 2:
        hist = collections.Counter(o.split()[0].lstrip("@!P0123456789UPT ").split(".")[0] if not o.startswith("@")
                                   else o.split()[1].split(".")[0] for o in ops)
        top = " ".join(f"{k}:{v}" for k, v in hist.most_common(9))
        print(f"{st:#07x}-{la:#07x} n={n:10d} x{c:4d} = {100 * n * c / tot:5.1f}% inst {100 * s / S:5.1f}% samp | {top}")
