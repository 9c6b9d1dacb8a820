mkdir -p gpurun_out/st1
timeout 600 python -m pytest tests -m gpu -x -q --timeout=150 --timeout-method=thread -k "s2d or logits or stem" > gpurun_out/st1/pytest.log 2>&1; echo "exit $?" >> gpurun_out/st1/pytest.log
timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/st1/b.json 2>gpurun_out/st1/b.err
