mkdir -p gpurun_out/dw14
for r in 14 7 4; do
  DS_DW14_ROWS=$r timeout 300 python bench.py --no-cpu-baseline --kernel-table --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/dw14/r$r.json 2>/dev/null
done
