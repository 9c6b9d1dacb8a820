mkdir -p gpurun_out/models3
run() { tag=$1; m=$2; shift 2; env "$@" timeout 600 python bench.py --model $m --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/models3/$tag.json 2>gpurun_out/models3/$tag.err; }
run r_base resnet50_v1
run r_win resnet50_v1 DS_STEM_S2D_MODE=window
run r_win2 resnet50_v1 DS_STEM_S2D_MODE=window DS_CONV_WINDOW=1
run i_base inception_v3
run i_win inception_v3 DS_CONV_WINDOW=1
run i_win2 inception_v3 DS_CONV_WINDOW=1 DS_STEM_S2D_MODE=window
