mkdir -p gpurun_out/pool3
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread -k "pool or logits" > gpurun_out/pool3/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pool3/pytest.log
for r in 2 1; do
DS_POOL_ROWS=$r timeout 600 python bench.py --model inception_v3 --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/pool3/i$r.json 2>gpurun_out/pool3/i$r.err
done
timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/pool3/r.json 2>gpurun_out/pool3/r.err
