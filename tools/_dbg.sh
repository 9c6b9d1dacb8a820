mkdir -p gpurun_out/pool2
timeout 600 python -m pytest tests -m gpu -x -q --timeout=150 --timeout-method=thread -k "pool or logits" > gpurun_out/pool2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pool2/pytest.log
timeout 600 python bench.py --model inception_v3 --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/pool2/i.json 2>gpurun_out/pool2/i.err
timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/pool2/r.json 2>gpurun_out/pool2/r.err
