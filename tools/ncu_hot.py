"""Hot SASS regions of one kernel in an ncu report: runs of equal execution count.

    python tools/ncu_hot.py REP.ncu-rep [min_frac] [KERNEL_REGEX]

Without KERNEL_REGEX the rows of every kernel in the report are merged (addresses restart per
kernel); give one (e.g. cols2, stream_rows) for a report that holds several kernels.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
minf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
kfilter = ["-k", f"regex:{sys.argv[3]}"] if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, *kfilter, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
lines = []
base = None
for r in rows[2:]:
    try:
        a = int(r[0], 16)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    lines.append((a - base, int(r[ix['Instructions Executed']] or 0), int(r[ix['# Samples']] or 0), r[1].strip()))
tot = sum(l[1] for l in lines)
S = sum(l[2] for l in lines)
print(f"total warp inst {tot}  samples {S}")
runs = []
for a, n, s, t in lines:
    if runs and runs[-1][2] == n:
        runs[-1][1] = a
        runs[-1][3] += 1
        runs[-1][4] += s
    else:
        runs.append([a, a, n, 1, s, t])
for st, la, n, c, s, t in runs:
    if n * c > tot * minf or s > S * minf * 2:
        print(f"{st:#07x}-{la:#07x} n={n:10d} x{c:4d} = {100 * n * c / tot:5.1f}% inst  {100 * s / S:5.1f}% samp  {t[:50]}")
