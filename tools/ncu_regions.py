"""Stall breakdown per SASS address region of one kernel in an ncu report.

    ncu -i REP --page source --csv --print-source sass > src.csv
    python tools/ncu_regions.py src.csv 0x52e0:0x5340:spin 0xa240:0xb240:rows ...
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
base = int(data[0][0], 16)
regions = []
for spec in sys.argv[2:]:
    lo, hi, name = spec.split(':')
    regions.append((int(lo, 16), int(hi, 16), name))
tot = {}
for r in data:
    try:
        a = int(r[0], 16) - base
    except ValueError:
        continue
    reg = 'other'
    for lo, hi, n in regions:
        if lo <= a < hi:
            reg = n
    d = tot.setdefault(reg, {k: 0.0 for k in stalls + ['samples', 'inst']})
    for k in stalls:
        d[k] += float(r[ix[k]] or 0)
    d['samples'] += float(r[ix['# Samples']] or 0)
    d['inst'] += float(r[ix['Instructions Executed']] or 0)
S = sum(d['samples'] for d in tot.values())
I = sum(d['inst'] for d in tot.values())
for reg, d in sorted(tot.items(), key=lambda x: -x[1]['samples']):
    top = sorted(((d[k], k) for k in stalls), reverse=True)[:6]
    print(f"{reg:12s} samples {100 * d['samples'] / S:5.1f}% inst {100 * d['inst'] / I:5.1f}% ",
          ' '.join(f"{k[6:]}={100 * v / S:.1f}" for v, k in top))
