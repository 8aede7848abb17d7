"""Writes profiles/ncu_summary.json (bench.py's roofline `traffic`) from the ncu --set full
captures of the dominant kernel of each workload: dram read + write bytes per launch.
usage: python profiles/make_ncu_summary.py <dir with prof_*.ncu-rep> [label]"""
import csv
import io
import json
import os
import subprocess
import sys

CAPTURES = {"morlet_direct": "prof_morlet_direct", "morlet_multiply_batch": "prof_batch",
            "scalogram": "prof_scalogram"}


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))

        def num(k, scale_units=True):
            x = float(d[k].replace(",", ""))
            unit = u.get(k, "")
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
                   "ms": 1e3, "msecond": 1e3}.get(unit, 1) if scale_units else 1
            return x * mul
        res.append({"kernel": d["Kernel Name"], "dram_read": num("dram__bytes_read.sum"),
                    "dram_write": num("dram__bytes_write.sum"),
                    "duration_us": num("gpu__time_duration.sum"),
                    "regs": float(d["launch__registers_per_thread"]),
                    "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
                    "dram_pct": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"])})
    return res


def main(src, label):
    summary = {}
    for w, f in CAPTURES.items():
        rep = os.path.join(src, f + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        launches = metrics(rep)
        summary[w] = {"dram_bytes_per_launch": sum(x["dram_read"] + x["dram_write"] for x in launches) / len(launches),
                      "launches": launches,
                      "source": f"{rep} (ncu --set full --clock-control none), {label}; digest profiles/r2_ncu_digest_*.txt"}
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_summary.json")
    with open(out, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({k: v["dram_bytes_per_launch"] for k, v in summary.items()}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "round 2")
