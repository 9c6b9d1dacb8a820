mkdir -p gpurun_out/st
for mode in tap box; do
for m in resnet50_v1 inception_v3 mobilenet_v1; do
DS_STEM_S2D_MODE=$mode timeout 300 python bench.py --model $m --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/st/${m}_$mode.json 2>/dev/null
done; done
