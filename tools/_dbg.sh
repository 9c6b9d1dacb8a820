mkdir -p gpurun_out/dwopt
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread -k "depthwise or logits or pwdw" > gpurun_out/dwopt/pytest.log 2>&1; echo "exit $?" >> gpurun_out/dwopt/pytest.log
timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/dwopt/mb.json 2>gpurun_out/dwopt/mb.err
