"""Per-CUDA-line warp-stall samples for one launch of an ncu report.

    python tools/ncu_lines.py report.ncu-rep <launch-skip> [top]
"""
import collections
import csv
import subprocess
import sys


def main(rep, skip, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    fn = next((r[1] for r in rows if r and r[0] == "Function Name"), "?")
    i_st = hdr.index("Warp Stall Sampling (All Samples)")
    stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.OrderedDict()
    src = {}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= i_st or not r[0].isdigit():
            continue
        ln = int(r[0])
        src.setdefault(ln, r[1].strip())
        a = agg.setdefault(ln, collections.Counter())
        try:
            a["_all"] += float(r[i_st] or 0)
            for i in stalls:
                a[hdr[i]] += float(r[i] or 0)
        except ValueError:
            pass
    tot = sum(a["_all"] for a in agg.values()) or 1.0
    print(fn, f"samples={tot:.0f}")
    for ln, a in sorted(agg.items(), key=lambda kv: -kv[1]["_all"])[:top]:
        top_st = ", ".join(f"{k[6:]}={100 * v / a['_all']:.0f}%" for k, v in a.most_common(4)
                           if k != "_all" and v > 0)
        print(f"{100 * a['_all'] / tot:5.1f}% L{ln}: {src[ln][:80]}  [{top_st}]")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 25)
