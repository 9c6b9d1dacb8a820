"""DRAM traffic per forward from an ncu launch list (dram__bytes_read/write.sum
per launch), for bench.py's roofline.traffic. Only complete forwards (first
kernel .. softmax) are counted.

    python tools/make_traffic.py launches.csv mobilenet_v1:bs128 [profiles/ncu_traffic.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_launches import load  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def forwards(recs):
    cur, out = [], []
    for r in recs:
        if r["name"].startswith(("stage_input_kernel", "stem_")) and cur:
            cur = []
        cur.append(r)
        if r["name"].startswith("softmax_kernel"):
            out.append(cur)
            cur = []
    return out


def dram(r):
    return sum(r.get(k, 0.0) * UNIT.get(r.get(k + "_unit", "byte"), 1)
               for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))


def main(path, key, dst):
    fw = forwards(load(path))
    if not fw:
        raise SystemExit("no complete forward in " + path)
    conv = [sum(dram(r) for r in f if r["name"].startswith("conv_gemm")) for f in fw]
    tot = [sum(dram(r) for r in f) for f in fw]
    data = json.load(open(dst)) if os.path.exists(dst) else {}
    data[key] = {"conv_gemm_dram_bytes_per_forward": sum(conv) / len(conv),
                 "forward_dram_bytes": sum(tot) / len(tot), "forwards": len(fw),
                 "source": os.path.basename(path)}
    json.dump(data, open(dst, "w"), indent=1)
    print(json.dumps(data[key]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json")
