mkdir -p gpurun_out/dbg12
for f in 0 1 16 17; do
  DS_CONV_DEBUG=0:$f timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/dbg12/b$f.json 2>/dev/null
done
