set -u
mkdir -p gpurun_out/n2
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:conv_gemm_kernel --launch-skip 7 -c 1 -o gpurun_out/n2/pair14 python tools/fwd_loop.py mobilenet_v1 128 3 > gpurun_out/n2/a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:dw_tma_kernel --launch-skip 6 -c 1 -o gpurun_out/n2/dw14 python tools/fwd_loop.py mobilenet_v1 128 3 > gpurun_out/n2/b.log 2>&1
ls -la gpurun_out/n2
