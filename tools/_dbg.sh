mkdir -p gpurun_out/dbg13
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/dbg13/$tag.json 2>gpurun_out/dbg13/$tag.err; }
run cl
run nocl DS_CONV_CLUSTER=0
