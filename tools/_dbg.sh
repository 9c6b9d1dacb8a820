mkdir -p gpurun_out/w5
for m in resnet50_v1 inception_v3; do
timeout 300 python bench.py --model $m --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/w5/${m}.json 2>/dev/null
done
timeout 600 python -m pytest tests -m gpu -q --timeout=300 --timeout-method=thread > gpurun_out/w5/pt.txt 2>&1
