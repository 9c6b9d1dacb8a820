"""Summarise an ncu --csv launch list (per-kernel time share, DRAM bytes,
tensor-pipe %) for profiles/. Usage: summarize_launches.py launches.csv [forwards]"""
import collections
import csv
import json
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    recs = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        key = d["ID"]
        rec = recs.setdefault(key, {"name": d["Kernel Name"].split("(")[0].replace("void ", "")
                                    .replace("ds::<unnamed>::", "").replace("unnamed>::", "")})
        try:
            rec[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
        rec[d["Metric Name"] + "_unit"] = d["Metric Unit"]
    return list(recs.values())


def main(path, forwards=1):
    recs = load(path)
    agg = collections.OrderedDict()
    for r in recs:
        a = agg.setdefault(r["name"], {"n": 0, "ns": 0.0, "bytes": 0.0, "tensor_pct_x_ns": 0.0})
        ns = r.get("gpu__time_duration.sum", 0.0)
        unit = r.get("gpu__time_duration.sum_unit", "ns")
        ns *= {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6}.get(unit, 1)
        a["n"] += 1
        a["ns"] += ns
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = r.get(k, 0.0)
            u = r.get(k + "_unit", "byte")
            a["bytes"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        # (tools/gpu_round.sh captures the _elapsed form; older captures _active)
        tp = r.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                   r.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0))
        a["tensor_pct_x_ns"] += tp * ns
    tot = sum(a["ns"] for a in agg.values())
    out = {}
    print(f"{'kernel':40s} {'launches':>8s} {'share':>7s} {'us/fwd':>9s} {'DRAM MB/fwd':>12s} {'GB/s':>7s} {'tensor%':>8s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        us = a["ns"] / 1e3 / forwards
        mb = a["bytes"] / 1e6 / forwards
        gbs = a["bytes"] / a["ns"] if a["ns"] else 0
        tp = a["tensor_pct_x_ns"] / a["ns"] if a["ns"] else 0
        print(f"{k:40s} {a['n']:8d} {a['ns']/tot:7.3f} {us:9.1f} {mb:12.1f} {gbs:7.0f} {tp:8.1f}")
        out[k] = {"launches": a["n"], "share": a["ns"] / tot, "us_per_forward": us,
                  "dram_mb_per_forward": mb, "dram_gbs": gbs, "tensor_pipe_pct": tp}
    return out


if __name__ == "__main__":
    res = main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    if len(sys.argv) > 3:
        json.dump(res, open(sys.argv[3], "w"), indent=1)
