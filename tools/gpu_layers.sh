#!/bin/bash
# Per-layer launch lists (ncu: time, DRAM bytes, tensor pipe) of R forwards of
# one model at one batch, joined to the layer costs by tools/layer_table.py.
# Usage (under gpurun): tools/gpu_layers.sh <tag> <model> <bs> [reps]
set -u
TAG=$1; MODEL=$2; BS=$3; REPS=${4:-3}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
F="$OUT/${MODEL}_bs${BS}"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file "$F.csv" \
  python tools/fwd_loop.py "$MODEL" "$BS" "$REPS" > "$F.json" 2> "$F.err"
echo "ncu exit $?" >> "$F.err"
python tools/layer_table.py "$F.csv" "$F.json" > "$F.table.txt" 2>&1
