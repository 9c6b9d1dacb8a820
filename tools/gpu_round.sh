#!/bin/bash
# One gpurun call: GPU tests, the headline bench, a launch list and one full
# ncu capture of the top kernels. Outputs land in gpurun_out/<tag>/.
# Usage (from the repo root, under gpurun): tools/gpu_round.sh <tag> [tests|notests]
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
if [ "${2:-tests}" = "tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -q --timeout=300 --timeout-method=thread > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.log"
fi
timeout 900 python bench.py --kernel-table > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" >> "$OUT/bench.err"
# launch list of a static-knob run (one forward = 1 graph; skip the set-up)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --nvtx --nvtx-include "timed/" -c 300 --csv --log-file "$OUT/launches.csv" \
  python bench.py --knob batching:128 --steps 3 --warmup 3 --no-cpu-baseline --max-converge 1 > "$OUT/launches_bench.log" 2>&1
echo "ncu launches exit $?" >> "$OUT/launches_bench.log"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'conv_gemm|dw_tma' --nvtx --nvtx-include "timed/" -c 8 \
  -o "$OUT/prof" python bench.py --knob batching:128 --steps 3 --warmup 3 --no-cpu-baseline --max-converge 1 > "$OUT/prof_bench.log" 2>&1
echo "ncu full exit $?" >> "$OUT/prof_bench.log"
