mkdir -p gpurun_out/fu3
DS_DW_FUSION=1 timeout 300 python bench.py --no-cpu-baseline --kernel-table --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/fu3/f.json 2>gpurun_out/fu3/f.err
DS_DW_FUSION=1 timeout 300 python -m pytest tests -m gpu -q -k "depthwise_fusion" --timeout=150 --timeout-method=thread > gpurun_out/fu3/pt.txt 2>&1
