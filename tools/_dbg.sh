mkdir -p gpurun_out/dw3
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread -k "depthwise" > gpurun_out/dw3/pytest.log 2>&1; echo "exit $?" >> gpurun_out/dw3/pytest.log
timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/dw3/mb.json 2>gpurun_out/dw3/mb.err
