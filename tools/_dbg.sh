mkdir -p gpurun_out/pool
for c in 1 2 4; do
  DS_POOL_COLS=$c timeout 600 python bench.py --model inception_v3 --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/pool/i$c.json 2>gpurun_out/pool/i$c.err
done
DS_POOL_LEGACY=1 timeout 600 python bench.py --model inception_v3 --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/pool/ileg.json 2>gpurun_out/pool/ileg.err
