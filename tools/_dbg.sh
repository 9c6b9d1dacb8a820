mkdir -p gpurun_out/epi1
timeout 600 python -m pytest tests -m gpu -x -q --timeout=150 --timeout-method=thread -k "logits or pair or s2d" > gpurun_out/epi1/pytest.log 2>&1; echo "exit $?" >> gpurun_out/epi1/pytest.log
timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/epi1/mb.json 2>gpurun_out/epi1/mb.err
timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/epi1/r.json 2>gpurun_out/epi1/r.err
