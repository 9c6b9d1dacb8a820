mkdir -p gpurun_out/dbg4
for f in 9; do
  DS_CONV_DEBUG=0:$f timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/dbg4/b$f.json 2>gpurun_out/dbg4/b$f.err
done
