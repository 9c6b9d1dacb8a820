mkdir -p gpurun_out/pair4
timeout 600 python -m pytest tests -m gpu -x -q --timeout=150 --timeout-method=thread -k "pair or logits or cluster" -s > gpurun_out/pair4/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pair4/pytest.log
for cfg in "1 1" "0 1" "1 0" "0 0"; do set -- $cfg
DS_CONV_PAIR=$1 DS_CONV_TPA=$2 timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --max-converge 1 > gpurun_out/pair4/b_$1$2.json 2>gpurun_out/pair4/b_$1$2.err
done
