"""Summarise an ncu report's per-CUDA-line warp-stall samples and executed
instructions (needs -lineinfo builds and --import-source on captures).

    python tools/ncu_hotspots.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys


def hotspots(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    lines = []
    hdr = None
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            i_st = hdr.index("Warp Stall Sampling (All Samples)")
            i_ie = hdr.index("Instructions Executed")
            continue
        if hdr is None or not r or not r[0]:
            continue
        try:
            lines.append((float(r[i_st] or 0), float(r[i_ie] or 0), r[0], r[1].strip()))
        except (ValueError, IndexError):
            continue
    tot = sum(x[0] for x in lines) or 1.0
    res = []
    for st, ie, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
        res.append(f"{100 * st / tot:6.1f}% {ie:12.0f}  L{ln}: {src[:100]}")
    return res


if __name__ == "__main__":
    print("\n".join(hotspots(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)))
