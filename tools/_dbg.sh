mkdir -p gpurun_out/s2d64
timeout 600 python -m pytest tests -m gpu -x -q --timeout=150 --timeout-method=thread -k "s2d or stem or logits" > gpurun_out/s2d64/pytest.log 2>&1; echo "exit $?" >> gpurun_out/s2d64/pytest.log
for r in 64 32; do
DS_S2D_ROWS=$r timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/s2d64/r$r.json 2>gpurun_out/s2d64/r$r.err
done
