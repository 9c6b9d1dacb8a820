mkdir -p gpurun_out/res2x
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread > gpurun_out/res2x/pytest.log 2>&1; echo "exit $?" >> gpurun_out/res2x/pytest.log
timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/res2x/r.json 2>gpurun_out/res2x/r.err
timeout 600 python bench.py --model inception_v3 --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/res2x/i.json 2>gpurun_out/res2x/i.err
timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/res2x/mb.json 2>gpurun_out/res2x/mb.err
