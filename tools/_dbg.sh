mkdir -p gpurun_out/rstem
for r in 64 32; do
DS_S2D_ROWS=$r timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/rstem/r$r.json 2>gpurun_out/rstem/r$r.err
done
