mkdir -p gpurun_out/pw1
timeout 120 ./tools/test_conv_gemm "mbv1 pw" > gpurun_out/pw1/base.txt 2>&1
