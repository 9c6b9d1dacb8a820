mkdir -p gpurun_out/models5
for m in resnet50_v1 inception_v3; do
  timeout 600 python bench.py --model $m --kernel-table --no-cpu-baseline > gpurun_out/models5/$m.json 2>gpurun_out/models5/$m.err
done
