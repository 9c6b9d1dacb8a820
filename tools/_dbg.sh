mkdir -p gpurun_out/g0
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread > gpurun_out/g0/pytest.log 2>&1; echo "exit $?" >> gpurun_out/g0/pytest.log
timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/g0/r.json 2>gpurun_out/g0/r.err
timeout 600 python bench.py --model inception_v3 --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/g0/i.json 2>gpurun_out/g0/i.err
timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/g0/mb.json 2>gpurun_out/g0/mb.err
