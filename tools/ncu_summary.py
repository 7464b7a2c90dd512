"""Summarise an ncu report: headline metrics, stall reasons, hot SASS regions.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--px N] [--regions]
"""
import argparse
import collections
import csv
import io
import subprocess

WANT = ['Duration', 'DRAM Throughput', 'Executed Ipc Active', 'Issue Slots Busy', 'Executed Instructions',
        'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy', 'No Eligible', 'Grid Size',
        'Block Limit Shared Mem', 'Block Limit Registers', 'Dynamic Shared Memory Per Block', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'SM Frequency', 'Memory Throughput']


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--px", type=float, default=0)
    ap.add_argument("--regions", action="store_true")
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "details", "--csv"))))
    hdr = rows[0]
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in WANT:
            print(f"{d['Metric Name']:<40} {d['Metric Unit']:<14} {d['Metric Value']}")
    raw = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "raw", "--csv"))))
    hdr, vals = raw[0], raw[2] if len(raw) > 2 else raw[1]
    stalls = []
    for h, v in zip(hdr, vals):
        if h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size"):
            print(f"{h:<40} {v}")
        if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("_not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    print("stalls:", ", ".join(f"{n} {s / tot * 100:.0f}%" for s, n in sorted(stalls, reverse=True)[:8]))
    if not a.regions:
        return
    src = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "source", "--csv", "--print-source=sass"))))
    hdr = src[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = []
    for r in src[2:]:
        if len(r) < len(hdr):
            continue
        data.append((int(r[idx["Address"]], 16), r[idx["Source"]].strip(), int(r[idx["Instructions Executed"]] or 0),
                     int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)))
    base = data[0][0]
    total = sum(d[2] for d in data)
    stt = sum(d[3] for d in data) or 1
    regions, cur, start, cnt, acc, sacc, ops = [], None, None, 0, 0, 0, collections.Counter()
    for adr, s, n, st in data:
        if cur is None or abs(n - cur) > cur * 0.05 + 10:
            if cur is not None:
                regions.append((start, adr - base, cur, cnt, acc, sacc, ops))
            cur, start, cnt, acc, sacc, ops = n, adr - base, 0, 0, 0, collections.Counter()
        cnt += 1
        acc += n
        sacc += st
        op = s.split()[1] if s.startswith("@") else s.split()[0]
        ops[op.split(".")[0]] += 1
    regions.append((start, 0, cur, cnt, acc, sacc, ops))
    for st, en, n, c, acc, sa, ops in sorted(regions, key=lambda x: -x[4])[:12]:
        per_px = f" thr-instr/px={acc * 32 / a.px:6.2f}" if a.px else ""
        print(f"{hex(st):>8}-{hex(en):>8} execs={n:>9} ninstr={c:4d} share={acc / total * 100:5.1f}%{per_px} "
              f"stall={sa / stt * 100:4.1f}% top={ops.most_common(6)}")


if __name__ == "__main__":
    main()
