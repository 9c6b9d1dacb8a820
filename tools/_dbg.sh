mkdir -p gpurun_out/fc
for b in 64 32 16; do
DS_FC_BN=$b timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/fc/b$b.json 2>gpurun_out/fc/b$b.err
done
