#!/bin/bash
# ncu --set full of the first N conv_gemm/dw launches inside the timed region of a
# static-knob bench run. Usage: tools/gpu_ncu.sh <tag> <count> [kernel regex] [bench args]
set -u
TAG=$1; N=$2; RE=${3:-conv_gemm|dw_tma}; shift 3 || shift $#
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RE" --nvtx --nvtx-include "timed/" -c "$N" \
  -o "$OUT/prof" python bench.py --knob batching:128 --steps 3 --warmup 3 --no-cpu-baseline --max-converge 1 "$@" > "$OUT/prof_bench.log" 2>&1
echo "ncu full exit $?" >> "$OUT/prof_bench.log"
