"""Digest of an ncu --set full report: headline metrics, stall reasons, SASS opcode mix.
usage: python profiles/ncu_digest.py <report.ncu-rep>"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "smsp__inst_issued.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct")


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(hdr, zip(units, v)))
        print("kernel:", d["Kernel Name"][1][:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:60s} {d[k][1]} {d[k][0]}")
        stalls = {h.split("stalled_")[1]: float(d[h][1].replace(",", "")) for h in hdr
                  if "pcsamp_warps_issue_stalled" in h and "not_issued" not in h and d[h][1] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1
        print("  stall samples:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]))
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2:
        h = src[1]
        ie, sc = h.index("Instructions Executed"), h.index("Source")
        ops, tot = collections.Counter(), 0
        for row in src[2:]:
            try:
                n = int(row[ie])
            except (ValueError, IndexError):
                continue
            toks = row[sc].split()
            op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
            ops[op] += n
            tot += n
        print("  SASS mix:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in ops.most_common(12)))


if __name__ == "__main__":
    main(sys.argv[1])
