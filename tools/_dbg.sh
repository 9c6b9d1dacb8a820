mkdir -p gpurun_out/wint
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread -k "window or logits" > gpurun_out/wint/pytest.log 2>&1; echo "exit $?" >> gpurun_out/wint/pytest.log
timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/wint/r.json 2>gpurun_out/wint/r.err
