mkdir -p gpurun_out/pd5
timeout 600 python -m pytest tests -m gpu -x -q --timeout=150 --timeout-method=thread -k "pwdw or logits" > gpurun_out/pd5/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pd5/pytest.log
timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/pd5/mb.json 2>gpurun_out/pd5/mb.err
DS_PWDW=0 timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/pd5/mb0.json 2>gpurun_out/pd5/mb0.err
