"""Copy a refresh run (tools/refresh_profiles.sh) from gpurun_out/ into profiles/.

    python tools/collect_profiles.py r01

Writes profiles/<round>_ncu_<cfg>.txt (ncu_summary of the --set full capture),
profiles/<round>_launches_c3.csv, the bench / pytest logs, and profiles/traffic.json
(dram__bytes_read.sum + dram__bytes_write.sum of one step's launches per config).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
LAUNCHES_PER_STEP = {"c3": 1, "c4": 2, "c5": 2}  # fused sweep / rows + cols
ALG_BYTES = {"c3": 256 * 1024 * 1024 * 5, "c4": 8192 * 8192 * 3 * 8, "c5": 32768 * 32768 * 8}  # read in + write out


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    traffic = {}
    report = []
    for cfg, nl in LAUNCHES_PER_STEP.items():
        rep = os.path.join(OUT, f"{rnd}_prof_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                              text=True).stdout
        rows, units = raw(rep)
        total = 0.0
        lines = []
        for r in rows[:nl]:
            rd = to_bytes(r["dram__bytes_read.sum"], units["dram__bytes_read.sum"])
            wr = to_bytes(r["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
            total += rd + wr
            lines.append(f"{r['Kernel Name'][:60]}: duration {r.get('gpu__time_duration.sum', '?')} "
                         f"{units.get('gpu__time_duration.sum', '')}, dram read {rd / 1e9:.3f} GB, write {wr / 1e9:.3f} GB")
        traffic[cfg] = int(total)
        report += [f"{cfg}: {ln}" for ln in lines]
        report.append(f"{cfg}: total dram traffic {total / 1e9:.3f} GB vs algorithmic {ALG_BYTES[cfg] / 1e9:.3f} GB "
                      f"(x{total / ALG_BYTES[cfg]:.2f})")
        with open(os.path.join(PROF, f"{rnd}_ncu_{cfg}.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none, {cfg} (tools/prof_run.py), one step = {nl} launch(es)\n")
            f.write("\n".join(lines) + "\n\n" + summ)
    traffic["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per step (all launches of the step), from the "
                        f"ncu --set full captures summarised in profiles/{rnd}_ncu_<cfg>.txt")
    with open(os.path.join(PROF, f"{rnd}_dram_traffic.txt"), "w") as f:
        f.write("# per-kernel DRAM bytes of one step (ncu --set full, cold L2, serialised launches)\n")
        f.write("\n".join(report) + "\n")
    with open(os.path.join(PROF, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    for name in [f"{rnd}_launches_c3.csv", f"{rnd}_pytest_gpu.log"] + [f"{rnd}_bench_{c}.jsonl" for c in
                                                                        ("c3", "c4", "c5", "reference_c3")]:
        src = os.path.join(OUT, name)
        if os.path.exists(src):
            shutil.copy(src, os.path.join(PROF, name))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
