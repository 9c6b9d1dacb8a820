mkdir -p gpurun_out/narrow
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread -k "narrow or logits or s2d or stem" > gpurun_out/narrow/pytest.log 2>&1; echo "exit $?" >> gpurun_out/narrow/pytest.log
timeout 600 python bench.py --model inception_v3 --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/narrow/i.json 2>gpurun_out/narrow/i.err
timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/narrow/mb.json 2>gpurun_out/narrow/mb.err
