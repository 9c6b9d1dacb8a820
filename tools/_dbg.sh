mkdir -p gpurun_out/res3
for v in 0 1 2; do
DS_RES_PREFETCH=$v timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/res3/r$v.json 2>gpurun_out/res3/r$v.err
done
