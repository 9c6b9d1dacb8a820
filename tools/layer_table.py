"""Per-layer table from an ncu launch list of tools/fwd_loop.py: launch i of
each forward joined with kernel_costs()[i] (kind, flops, bytes), reporting
us, achieved GB/s and TFLOP/s, roofline time and the ratio.

    python tools/layer_table.py launches.csv fwd_loop.json
"""
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
from summarize_launches import load  # noqa: E402

recs = load(sys.argv[1])
meta = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
costs, bs = meta["costs"], meta["bs"]
k = meta["kernels_per_forward"]
peaks = json.load(open(__import__("os").path.join(
    __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(
        __file__))), "MEASURED_PEAKS.json"))) if len(sys.argv) < 4 else {}
hbm = peaks.get("hbm_gbs", 6550.0)
tfl = peaks.get("bf16_tflops", 1650.0)


def ns(r):
    v = r.get("gpu__time_duration.sum", 0.0)
    return v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6}.get(
        r.get("gpu__time_duration.sum_unit", "ns"), 1)


n_fwd = len(recs) // k
tot = 0.0
tot_rl = 0.0
print(f"{'#':>3s} {'kind':10s} {'kernel':28s} {'us':>8s} {'GB/s':>7s} {'TF/s':>7s} {'roof us':>8s} {'x roof':>6s} {'tensor%':>7s}")
for i in range(k):
    t = sum(ns(recs[f * k + i]) for f in range(n_fwd)) / n_fwd / 1e3
    c = costs[i]
    by = bs * c["bytes_per_image"] + c["fixed_bytes"]
    fl = bs * c["flops_per_image"]
    rl = max(by / hbm / 1e3, fl / tfl / 1e6)
    tp = recs[i].get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
    tot += t
    tot_rl += rl
    print(f"{i:3d} {c['kind']:10s} {recs[i]['name'][:28]:28s} {t:8.2f} {by / t / 1e3:7.0f} "
          f"{fl / t / 1e6:7.1f} {rl:8.2f} {t / rl:6.1f} {tp:7.1f}")
print(f"total {tot:.1f} us per forward (roofline {tot_rl:.1f} us, {tot_rl / tot:.3f}); {n_fwd} forwards")
