mkdir -p gpurun_out/rtma
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread > gpurun_out/rtma/pytest.log 2>&1; echo "exit $?" >> gpurun_out/rtma/pytest.log
for v in 1 0; do
DS_RES_TMA=$v timeout 600 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline --knob batching:193 --max-converge 1 > gpurun_out/rtma/r$v.json 2>gpurun_out/rtma/r$v.err
done
