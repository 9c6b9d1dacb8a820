// Launchers for the HBM-bound layers of the forward pass (K3/K4/K5b/K6 in
// DESIGN.md). All tensors are NHWC bf16; every kernel moves 16 B (8 channels)
// per thread per access, fp32 math inside, bf16 rounding on store.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace ds {

// Space-to-depth staging for stride-2 stems: u8 [n][h][w][3] -> bf16
// [n][hs][ws][16], channel (a*2+b)*4+c = normalised x(2Y+a-pad, 2X+b-pad, c),
// x = (p - 127.5) / 63.75 (zero outside the image and for c == 3).
cudaError_t launch_stage_s2d(const uint8_t* img, __nv_bfloat16* out, int n, int h, int w, int hs,
                             int ws, int pad, cudaStream_t stream);

// Depthwise 3x3, pad 1, stride 1|2, + bias, ReLU, w: [9][C] bf16 (tap-major),
// streamed by TMA halo boxes (dwconv_tma.cu); C must be a
// power of two >= 8. The input map comes from dwconv_tma_input_map over the
// (max-batch) input buffer.
bool dwconv_tma_supported(int c);
bool dwconv_tma_plan_ok(int h, int w, int c, int stride);
bool dwconv_tma_input_map(CUtensorMap* map, const void* x, int max_n, int h, int w, int c,
                          int stride);
cudaError_t launch_dwconv3x3_tma(const CUtensorMap& in_map, const __nv_bfloat16* w,
                                 const float* bias, __nv_bfloat16* y, int n, int h, int wd, int c,
                                 int stride, cudaStream_t stream);

// 3x3 max pool (stride, pad) or 3x3 average pool (count_include_pad, /9).
// Output may be a channel slice of a wider buffer (ldo channels, c_off).
cudaError_t launch_pool3x3(const __nv_bfloat16* x, __nv_bfloat16* y, int n, int h, int w, int c,
                           int stride, int pad, bool is_max, int ldo, int c_off,
                           cudaStream_t stream);

// The same pooling streamed through TMA halo boxes (pool_tma.cu), bit-identical
// to launch_pool3x3 for average pools and for max pools whose edge taps are
// zeros-equivalent (pad 0, or inputs >= 0). The input map comes from
// pool_tma_input_map over the (max-batch) input buffer.
bool pool_tma_plan_ok(int h, int w, int c, int stride, int pad);
bool pool_tma_input_map(CUtensorMap* map, const void* x, int max_n, int h, int w, int c,
                        int stride, int pad);
cudaError_t launch_pool3x3_tma(const CUtensorMap& in_map, __nv_bfloat16* y, int n, int h, int w,
                               int c, int stride, int pad, bool is_max, int ldo, int c_off,
                               cudaStream_t stream, const float* post_bias = nullptr,
                               bool post_relu = false);

// Mean over all pixels: [n][hw][c] -> [n][c] bf16.
cudaError_t launch_global_avgpool(const __nv_bfloat16* x, __nv_bfloat16* y, int n, int hw, int c,
                                  cudaStream_t stream);

// Row softmax over fp32 logits [n][classes] (one warp per row).
cudaError_t launch_softmax(const float* logits, float* probs, int n, int classes,
                           cudaStream_t stream);

}  // namespace ds
