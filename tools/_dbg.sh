mkdir -p gpurun_out/e2e
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread > gpurun_out/e2e/pytest.log 2>&1; echo "exit $?" >> gpurun_out/e2e/pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/e2e/mb.json 2>gpurun_out/e2e/mb.err
timeout 600 python bench.py --model resnet50_v1 --no-cpu-baseline > gpurun_out/e2e/r.json 2>gpurun_out/e2e/r.err
