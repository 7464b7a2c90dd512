"""Stall reasons summed over SASS address ranges of one kernel in an ncu report.

    python tools/ncu_stalls.py REP.ncu-rep KERNEL_REGEX START-END [START-END ...]   (hex offsets from the first instruction)
"""
import csv
import io
import subprocess
import sys

rep, k = sys.argv[1], sys.argv[2]
ranges = [tuple(int(x, 16) for x in r.split("-")) for r in sys.argv[3:]]
txt = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{k}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
base = None
acc = [dict.fromkeys(cols, 0) for _ in ranges]
for r in rows[2:]:
    try:
        a = int(r[0], 16)
    except (ValueError, IndexError):
        if base is not None:
            break
        continue
    base = a if base is None else base
    off = a - base
    for j, (lo, hi) in enumerate(ranges):
        if lo <= off <= hi:
            for c in cols:
                acc[j][c] += int(r[ix[c]] or 0)
for (lo, hi), d in zip(ranges, acc):
    tot = sum(d.values()) or 1
    top = sorted(d.items(), key=lambda kv: -kv[1])[:6]
    print(f"{lo:#07x}-{hi:#07x} samples {tot:7d}: " + ", ".join(f"{c[6:]} {100 * v / tot:.0f}%" for c, v in top))
