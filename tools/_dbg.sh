mkdir -p gpurun_out/dbg7
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --kernel-table --no-cpu-baseline --knob batching:128 --steps 3 --warmup 3 --max-converge 1 > gpurun_out/dbg7/$tag.json 2>/dev/null; }
run base
run tma2t4 DS_CONV_MT_TMA=2
run tma2t2 DS_CONV_MT_TMA=2 DS_CONV_TEAMS_TMA=2
run stem2 DS_CONV_MT=2
run stem1 DS_CONV_MT=1
