#!/bin/bash
# Quick GPU iteration: selected GPU tests + a bench line with the per-kernel table.
# Usage: tools/gpu_quick.sh <tag> "<pytest -k expr or empty>" [bench args...]
set -u
TAG=$1; K=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
if [ -n "$K" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q --timeout=150 --timeout-method=thread -k "$K" > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
fi
timeout 300 python bench.py --kernel-table --no-cpu-baseline "$@" > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" >> "$OUT/bench.err"
