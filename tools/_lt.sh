set -u
mkdir -p gpurun_out/lt
for cfg in "mobilenet_v1 1" "resnet50_v1 1" "inception_v3 1" "mobilenet_v1 128"; do
  set -- $cfg
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/lt/$1_$2.csv python tools/fwd_loop.py $1 $2 3 > gpurun_out/lt/$1_$2.json 2> gpurun_out/lt/$1_$2.err
done
ls -la gpurun_out/lt
