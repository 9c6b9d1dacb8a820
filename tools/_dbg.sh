mkdir -p gpurun_out/dbg15
for f in 0 1 16 17; do
  DS_CONV_DEBUG=3:$f timeout 300 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/dbg15/g$f.json 2>/dev/null
  DS_CONV_WINDOW=1 DS_CONV_DEBUG=3:$f timeout 300 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/dbg15/w$f.json 2>/dev/null
done
