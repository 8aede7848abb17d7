"""Per-source-line digest of an ncu --set full report captured with -lineinfo and
--import-source on: instructions executed and warp-stall samples per CUDA line.
usage: python profiles/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
    hdr = rows[hi]
    nm = len(hdr) - 4
    names = hdr[4:]
    i_samp, i_inst = names.index("Warp Stall Sampling (All Samples)"), names.index("Instructions Executed")
    stall_cols = [j for j, h in enumerate(names) if h.startswith("stall_") and "Not Issued" not in h]
    lines = []
    for r in rows[hi + 1:]:
        if not r or not r[0].isdigit():
            continue
        m = r[-nm:]
        src = ",".join(r[1:len(r) - nm - 2]).strip()[:70]
        num = lambda v: float(v) if v not in ("", "-") else 0.0
        st = sorted(((num(m[j]), names[j][6:]) for j in stall_cols), reverse=True)[:3]
        lines.append((num(m[i_samp]), num(m[i_inst]), int(r[0]), src, st))
    tot_s = sum(l[0] for l in lines) or 1
    tot_i = sum(l[1] for l in lines) or 1
    print(f"{'line':>5} {'samp%':>6} {'inst%':>6}  top stalls / source")
    for s, i, ln, src, st in sorted(lines, reverse=True)[:top]:
        stalls = " ".join(f"{n}:{v / tot_s * 100:.1f}" for v, n in st if v)
        print(f"{ln:5d} {s / tot_s * 100:6.1f} {i / tot_i * 100:6.1f}  {src}   [{stalls}]")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
