// Depthwise 3x3 (+bias, ReLU) streamed through TMA (K3 in DESIGN.md).
//
// A persistent CTA walks output tiles of 8 rows x 16 (stride 1) or 8 x 8
// (stride 2) pixels x 64 channels. Each tile's input halo is one 4-D TMA box
// {64 ch, IW, IH, 1 image} landing in shared memory; boxes that hang over the
// image edge read zeros, which is exactly the convolution's padding. Two
// stages double-buffer the boxes (mbarrier transaction counts), so the
// next tile's halo streams in while the current one is computed; every input
// byte crosses HBM once (plus the halo), and the 9 taps of every output come
// from smem. Output: 16 B stores, 8 consecutive threads per pixel's 64
// channels, consecutive pixels along the row.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "conv_gemm.cuh"
#include "sm100_ptx.cuh"
#include "stream_ops.cuh"

namespace ds {

namespace {

constexpr int kDwThreads = 256;

template <int S>
struct DwGeom {
  static constexpr int TH = S == 1 ? 16 : 8;
  static constexpr int TW = S == 1 ? 16 : 8;
  static constexpr int IH = (TH - 1) * S + 3;
  static constexpr int IW = (TW - 1) * S + 3;
};

__device__ __forceinline__ void unpack8f(const uint4& u, float (&f)[8]) {
  const uint32_t v[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(v[e] << 16);
    f[2 * e + 1] = __uint_as_float(v[e] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint32_t pack2f(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int S>
__global__ void __launch_bounds__(kDwThreads) dw_tma_kernel(
    const __grid_constant__ CUtensorMap in_map, const __nv_bfloat16* __restrict__ w,
    const float* __restrict__ bias, uint4* __restrict__ y, int c, int ho, int wo, int cb_log2,
    int tiles_x, int tiles_y, int cblocks, int tiles) {
  using G = DwGeom<S>;
  const int cb = 1 << cb_log2;          // channels per tile (<= 64)
  const int groups_log2 = cb_log2 - 3;  // 8-channel groups per pixel
  const uint32_t box_bytes = static_cast<uint32_t>(G::IH * G::IW) << (cb_log2 + 1);
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * box_bytes);

  auto coords = [&](int t, int& cbk, int& tx, int& ty, int& img) {
    cbk = t % cblocks;
    t /= cblocks;
    tx = t % tiles_x;
    t /= tiles_x;
    ty = t % tiles_y;
    img = t / tiles_y;
  };
  auto issue = [&](int t, int stage) {
    int cbk, tx, ty, img;
    coords(t, cbk, tx, ty, img);
    ptx::mbar_arrive_expect_tx(&full[stage], box_bytes);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(ptx::smem_u32(smem + stage * box_bytes)),
        "l"(&in_map), "r"(ptx::smem_u32(&full[stage])), "r"(cbk << cb_log2),
        "r"(tx * G::TW * S - 1), "r"(ty * G::TH * S - 1), "r"(img)
        : "memory");
  };

  if (threadIdx.x == 0) {
    ptx::mbar_init(&full[0], 1);
    ptx::mbar_init(&full[1], 1);
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&in_map);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (blockIdx.x < tiles) issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < tiles) issue(blockIdx.x + gridDim.x, 1);
  }

  const int g = threadIdx.x & ((1 << groups_log2) - 1);  // fixed channel group per thread
  const int cg_all = c >> 3;
  const int items = (G::TH * G::TW) << groups_log2;
  uint32_t j = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
    const int stage = j & 1;
    int cbk, tx, ty, img;
    coords(t, cbk, tx, ty, img);
    const int gg = (cbk << (cb_log2 - 3)) + g;  // global channel group
    uint4 wraw[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) wraw[k] = __ldg(reinterpret_cast<const uint4*>(w) + k * cg_all + gg);
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias) + 2 * gg);
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias) + 2 * gg + 1);
    float wf[9][8];
#pragma unroll
    for (int k = 0; k < 9; ++k) unpack8f(wraw[k], wf[k]);

    ptx::mbar_wait(&full[stage], (j >> 1) & 1);
    const uint4* tile = reinterpret_cast<const uint4*>(smem + stage * box_bytes);
    for (int it = threadIdx.x; it < items; it += kDwThreads) {
      const int p = it >> groups_log2;
      const int oyl = p / G::TW, oxl = p % G::TW;
      const int oy = ty * G::TH + oyl, ox = tx * G::TW + oxl;
      if (oy >= ho || ox >= wo) continue;
      float acc[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          float xf[8];
          unpack8f(tile[(((oyl * S + r) * G::IW + oxl * S + s) << groups_log2) + g], xf);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = fmaf(xf[e], wf[r * 3 + s][e], acc[e]);
        }
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaxf(acc[e], 0.0f);
      y[((static_cast<long long>(img) * ho + oy) * wo + ox) * cg_all + gg] =
          make_uint4(pack2f(acc[0], acc[1]), pack2f(acc[2], acc[3]), pack2f(acc[4], acc[5]),
                     pack2f(acc[6], acc[7]));
    }
    __syncthreads();  // every thread is done with this stage's box
    if (threadIdx.x == 0 && t + 2 * static_cast<int>(gridDim.x) < tiles)
      issue(t + 2 * gridDim.x, stage);
  }
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

bool dwconv_tma_supported(int c) {
  return c >= 8 && (c & (c - 1)) == 0;  // power-of-two channel count (>= one 16 B group)
}

cudaError_t launch_dwconv3x3_tma(const CUtensorMap& in_map, const __nv_bfloat16* w,
                                 const float* bias, __nv_bfloat16* y, int n, int h, int wd, int c,
                                 int stride, cudaStream_t stream) {
  if (!dwconv_tma_supported(c) || (stride != 1 && stride != 2)) return cudaErrorInvalidValue;
  const int ho = (h + 2 - 3) / stride + 1, wo = (wd + 2 - 3) / stride + 1;
  const int cb = std::min(c, 64);
  int cb_log2 = 0;
  while ((1 << cb_log2) < cb) ++cb_log2;
  const int cblocks = c / cb;
  auto launch = [&](auto geom, auto kernel) -> cudaError_t {
    using Gm = decltype(geom);
    const int tiles_x = (wo + Gm::TW - 1) / Gm::TW, tiles_y = (ho + Gm::TH - 1) / Gm::TH;
    const int tiles = n * tiles_x * tiles_y * cblocks;
    const size_t box = static_cast<size_t>(Gm::IH) * Gm::IW * cb * 2;
    const size_t smem = 2 * box + 64;
    static bool configured = false;
    if (!configured) {
      cudaError_t e =
          cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    const int per_sm = std::max(1, static_cast<int>((227 * 1024) / smem));
    const int grid = std::min(tiles, sm_count() * std::min(per_sm, 4));
    kernel<<<grid, kDwThreads, smem, stream>>>(in_map, w, bias, reinterpret_cast<uint4*>(y), c,
                                               ho, wo, cb_log2, tiles_x, tiles_y, cblocks, tiles);
    return cudaGetLastError();
  };
  if (stride == 1) return launch(DwGeom<1>{}, dw_tma_kernel<1>);
  return launch(DwGeom<2>{}, dw_tma_kernel<2>);
}

bool dwconv_tma_input_map(CUtensorMap* map, const void* x, int max_n, int h, int w, int c,
                          int stride) {
  const int cb = std::min(c, 64);
  if (stride == 1)
    return encode_tmap_nhwc(map, x, max_n, h, w, c, cb, DwGeom<1>::IW, DwGeom<1>::IH);
  return encode_tmap_nhwc(map, x, max_n, h, w, c, cb, DwGeom<2>::IW, DwGeom<2>::IH);
}

}  // namespace ds
