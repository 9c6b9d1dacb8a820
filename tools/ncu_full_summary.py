"""Key counters of every kernel in an `ncu --set full` report, as JSON for
profiles/ (time, DRAM bytes and throughput, tensor-pipe and SM utilisation,
L2 reads, launch shape).

    python tools/ncu_full_summary.py report.ncu-rep out.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {}
        for k in KEYS:
            if k in d:
                u = units[hdr.index(k)]
                e[k] = d[k] + (f" {u}" if u and k != "Kernel Name" else "")
        res.append(e)
    return res


if __name__ == "__main__":
    s = summary(sys.argv[1])
    json.dump(s, open(sys.argv[2], "w"), indent=1)
    for e in s:
        print(e.get("Kernel Name", "")[:60], e.get("gpu__time_duration.sum"),
              e.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
              e.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"))
