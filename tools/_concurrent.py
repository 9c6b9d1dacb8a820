"""Bring-up experiment: two backends (own streams) running batches concurrently."""
import sys, threading, time
sys.path.insert(0, '.')
from paper_2308_13803_b200 import Config, GpuBackend
bs = int(sys.argv[1]); n = int(sys.argv[2]); k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
bes = [GpuBackend("mobilenet_v1", Config(abs_max_bs=bs, max_mtl=1)) for _ in range(k)]
for be in bes:
    be.run_batches(bs, 5)
def work(be):
    be.run_batches(bs, n)
for rep in range(2):
    ts = [threading.Thread(target=work, args=(be,)) for be in bes]
    t0 = time.perf_counter()
    for t in ts: t.start()
    for t in ts: t.join()
    dt = time.perf_counter() - t0
    print(f"{k} backends x bs {bs} x {n} batches: {k*bs*n/dt:.0f} img/s (wall)")
t0 = time.perf_counter(); bes[0].run_batches(bs, n); dt = time.perf_counter() - t0
print(f"1 backend x bs {bs}: {bs*n/dt:.0f} img/s (wall)")
