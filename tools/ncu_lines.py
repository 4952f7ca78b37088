"""Aggregate ncu warp-stall samples by CUDA source line for one kernel.
Usage: python tools/ncu_lines.py rep.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys
from collections import defaultdict


def main(rep, kernel, top=40):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kernel, "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = defaultdict(lambda: [0, 0, ""])
    fname = "?"
    hdr = None
    last_line = None
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 6:
            continue
        if r[0].strip():
            last_line = (fname, int(r[0]), r[1][:90])
        if last_line is None:
            continue
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        a = agg[last_line[:2]]
        a[0] += s
        a[2] = last_line[2]
    tot = sum(v[0] for v in agg.values()) or 1
    for (f, ln), (s, _, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * s / tot:5.1f}% {f}:{ln}  {src.strip()}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
