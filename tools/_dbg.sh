mkdir -p gpurun_out/g4
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread -k "depthwise or logits" > gpurun_out/g4/pytest.log 2>&1; echo "exit $?" >> gpurun_out/g4/pytest.log
for v in 1 0; do
DS_DW_G4=$v timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/g4/mb$v.json 2>gpurun_out/g4/mb$v.err
done
