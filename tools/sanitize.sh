#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over one forward of each
# network (every default conv mode: kS2D, kS2DWide, kStemU8, kTmaA, kPairTmaA,
# kWindow, kIm2col, kGather16, the TMA depthwise, pools, GAP, softmax) plus
# the MT green-context path. Logs land in gpurun_out/<tag>/.
# Usage (under gpurun): tools/sanitize.sh <tag>
set -u
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for tool in memcheck synccheck racecheck; do
  for model in synthetic_cnn mobilenet_v1 resnet50_v1 inception_v3; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/fwd_loop.py $model 2 1 > "$OUT/${tool}_${model}.log" 2>&1
    echo "exit $?" >> "$OUT/${tool}_${model}.log"
  done
done
for f in "$OUT"/*.log; do echo "$(basename $f): $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $f | tail -1) $(tail -1 $f)"; done > "$OUT/summary.txt"
cat "$OUT/summary.txt"
