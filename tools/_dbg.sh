mkdir -p gpurun_out/pool4
DS_POOL_ROWS=4 timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread -k "pool" > gpurun_out/pool4/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pool4/pytest.log
DS_POOL_ROWS=4 timeout 600 python bench.py --model inception_v3 --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/pool4/i4.json 2>gpurun_out/pool4/i4.err
DS_POOL_ROWS=4 timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/pool4/r4.json 2>gpurun_out/pool4/r4.err
