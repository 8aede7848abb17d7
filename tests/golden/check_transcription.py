"""Re-reads the reference sources (when /root/reference is present, i.e. in the build
container, never on the GPU box) and confirms every number in reference_values.json
appears verbatim in the cited file. Run: python tests/golden/check_transcription.py"""
import json
import os
import re
import sys

REF = "/root/reference/proj"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> int:
    if not os.path.isdir(REF):
        print("reference tree absent; nothing to check")
        return 0
    vals = json.load(open(os.path.join(HERE, "reference_values.json")))
    out = open(os.path.join(REF, "test_output.txt")).read()
    kern = open(os.path.join(REF, "tests", "test_kernels.cpp")).read()
    missing = []
    for tok in ("7.405e-03", "3.851e-04", "228.5", "6554", "rounds=6", "total_adds=7744", "0.60179204665006281",
                "0.39072104685894421", "0.64590375981497894", "0.4613%", "5.96e-12", "16.499", "4930.027"):
        if tok not in out:
            missing.append(tok)
    for tok in ("0.064758797832945863807", "0.011502947198904352644", "0.084719231205723545531",
                "0.012076433354503311808", "0.3989422804014327"):
        if tok not in kern:
            missing.append(tok)
    for var, rows in vals["table1"].items():
        if var.startswith("_"):
            continue
        for P, (s, g, gd, gdd) in rows.items():
            pat = rf"{var}\s+P={P}\s+sigma\*=\s*{s}\s+e\(G\)={g}\s+e\(GD\)={gd}\s+e\(GDD\)={gdd}"
            if not re.search(pat, out):
                missing.append(f"table1 {var} P={P}")
    print("missing:", missing or "none")
    return 1 if missing else 0


if __name__ == "__main__":
    sys.exit(main())
