mkdir -p gpurun_out/rtma2
timeout 900 python -m pytest tests -m gpu -q --timeout=200 --timeout-method=thread -k "residual or pair" > gpurun_out/rtma2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/rtma2/pytest.log
timeout 900 python bench.py --model resnet50_v1 --kernel-table --no-cpu-baseline > gpurun_out/rtma2/r.json 2>gpurun_out/rtma2/r.err
