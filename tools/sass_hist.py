"""Per-kernel SASS dump (exec counts, stall samples) and opcode histogram from an ncu report.

    python tools/sass_hist.py REP.ncu-rep KERNEL_REGEX [OUT.txt]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def dump(rep, k):
    txt = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{k}", "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    ix = {n: i for i, n in enumerate(h)}
    out = []
    for r in rows[2:]:
        try:
            a = int(r[0], 16)
        except (ValueError, IndexError):
            if out:
                break
            continue
        out.append((a, int(r[ix['Instructions Executed']] or 0), int(r[ix['# Samples']] or 0), r[1].strip()))
    return out


def main():
    rep, k = sys.argv[1], sys.argv[2]
    out = dump(rep, k)
    base = out[0][0]
    tot = sum(o[1] for o in out)
    S = sum(o[2] for o in out)
    if len(sys.argv) > 3:
        with open(sys.argv[3], "w") as f:
            f.write(f"total {tot} samples {S}\n")
            for a, n, s, t in out:
                f.write(f"{a - base:#07x} {n:10d} {s:6d} {t}\n")
    c = collections.Counter()
    sm = collections.Counter()
    for a, n, s, t in out:
        ins = re.sub(r'^@!?U?P\w+\s+', '', t)
        op = (ins.split()[0] if ins else '?').split('.')[0]
        c[op] += n
        sm[op] += s
    print(f"total warp inst {tot}  samples {S}")
    for op, n in c.most_common(25):
        print(f"  {op:10s} {100 * n / tot:5.1f}%  samp {100 * sm[op] / max(S, 1):5.1f}%")


if __name__ == "__main__":
    main()
