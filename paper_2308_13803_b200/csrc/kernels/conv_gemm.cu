// Implicit-GEMM convolution on the sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// This is the device compute that replaces the analytic stand-in
// `mean_batch_latency` / `mean_mt_latency` (reference perf_model.cpp:70-78)
// behind GpuSim::run_batch / run_mt_request (reference gpu_sim.cpp:13-24):
// every dense conv, 1x1 conv and FC layer of the served networks runs here.
//
// Persistent CTA (one per SM) walking 128 x BN output tiles (or 128-row
// sub-tile groups / pixel blocks per mode), N-tile fastest so the CTAs sharing
// an A row-block run together and A is read from DRAM once. Eighteen warps,
// three pipelines (operand ring, up to eight TMEM accumulators, tile loop):
//   warps 0-7  epilogue teams of four (one warp per TMEM lane quarter):
//              TMEM -> registers (tcgen05.ld), + bias (+ residual), ReLU,
//              packed into swizzled smem staging and written by TMA bulk
//              tensor stores into the (possibly channel-sliced, or per fused
//              sibling) NHWC output; each releases its accumulator to the MMA
//              warp, so tile i's epilogue overlaps tile i+1's main loop.
//   warps 8-15 A producers in the gather modes: the im2col rows of each tile
//              straight from the NHWC input with zero-filling cp.async
//              (padding, K tail and M tail become zeros), in the 128 B-swizzled
//              K-major layout of the UMMA descriptor; completion reaches the
//              stage's full barrier via cp.async.mbarrier.arrive.noinc. In the
//              TMA-A / im2col modes (A loaded by the TMA warp) they are
//              epilogue teams 2-3.
//   warp 16    TMA producer for the weight tiles (and A / halo boxes); owns TMEM.
//   warp 17    issues tcgen05.mma (M = 128, or M = 256 cta_group::2 on CTA
//              pairs, N = BN, K = 16) into the current fp32 TMEM accumulator
//              and commits stage releases; on a pair's peer CTA it forwards
//              the gather completion to the leader (kPairGather).
#include "conv_gemm.cuh"
#include "pdl.cuh"
#include "sm100_ptx.cuh"

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstdio>
#include <mutex>

namespace ds {

namespace {

constexpr int kABytes = kConvBM * kConvBK * 2;  // 16 KiB per stage

// Output staging for the TMA-store epilogue: per epilogue warp two buffers
// of 32 rows x 128 B (64 bf16 or 32 fp32 columns, 128 B-swizzled).
constexpr int kYStageBytes = 32 * 128;
// Staging buffers per epilogue warp: two (the next group fills while the
// last one's TMA store reads), one when sixteen warps drain (smem for the ring).
__host__ __device__ constexpr int y_bufs(int epi_warps) { return epi_warps > 8 ? 1 : 2; }
// Staging bytes per epilogue warp: narrow (32-column slices, two 2 KiB 64 B-
// swizzled buffers) or wide (64-column groups, y_bufs 4 KiB buffers).
__host__ __device__ constexpr int y_warp_bytes(int epi_warps, bool narrow) {
  return narrow ? kYStageBytes : y_bufs(epi_warps) * kYStageBytes;
}

// Warp roles (kConvThreads = 18 warps).
constexpr int kEpiWarps = 8;      // warps 0-7: epilogue (two teams of four)
// (TMA-A modes: the idle gather warps 8-15 join as epilogue teams 2-3)
constexpr int kMaxAcc = 8;        // TMEM accumulators (tmem_full/tmem_empty barrier pairs)
constexpr int kGatherWarp0 = 8;   // warps 8-15: A gather
constexpr int kGatherWarps = 8;
constexpr int kTmaWarp = 16;      // weight (and A) TMA producer, TMEM owner
// warp 17: tcgen05.mma issuer (the role branch's final else)

struct SmemLayout {
  uint32_t a_off, b_off, win_off, y_off, bar_off, bias_off, total;
};

// b_res_blocks > 0: the layer's whole weight matrix (num_kb blocks of
// BN x 64) stays resident in shared memory for all tiles (one N tile, small
// K); otherwise each ring stage carries its own B block.
__host__ __device__ inline SmemLayout smem_layout(int BN, int stages, int cout, int epi_warps,
                                                  int b_res_blocks = 0, int mt = 1, int win_bytes = 0,
                                                  bool narrow = false) {
  SmemLayout L;
  L.a_off = 0;
  L.b_off = static_cast<uint32_t>(stages) * mt * kABytes;  // stage = mt A sub-tiles
  const int b_blocks = b_res_blocks > 0 ? b_res_blocks : stages;
  L.y_off = L.b_off + static_cast<uint32_t>(b_blocks) * BN * 128;
  // kWindow: raw[2] + chunk-major[2] halo boxes
  L.win_off = L.y_off;
  L.y_off += 4 * static_cast<uint32_t>((win_bytes + 1023) / 1024 * 1024);
  L.bar_off = L.y_off + epi_warps * y_warp_bytes(epi_warps, narrow);
  // full[stages], empty[stages], tmem_full[kMaxAcc], tmem_empty[kMaxAcc], b_full,
  // win barriers[8], tmem slot, residual-staging barriers[2 x 16 warps]
  L.bias_off = L.bar_off + ((2 * stages + 2 * kMaxAcc + 2 + 8 + 32) * 8 + 15) / 16 * 16;
  // bias padded so a 32-column epilogue slice never reads past it
  L.total = L.bias_off + static_cast<uint32_t>((cout + 63) / 64 * 64 + 64) * 4;
  return L;
}

// Bring-up timeline stamps (args.ts, tools/test_conv_gemm TS=1): slot k of
// this CTA's 64 = %globaltimer (ns). Slots: 0 and 1 pdl_wait done, 2 MMA loop
// done, 3 exit, 4 entry, 5 prologue done (before pdl_wait); per tile j < 8:
// 8+j first A/B stage landed (MMA), 16+j tile committed (MMA), 24+j epilogue
// got the accumulator, 32+j epilogue stores issued, 40+j TMA first load issued.
__device__ __forceinline__ void ts_mark(unsigned long long* ts, int k, long long = 0) {
  if (ts) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ts[blockIdx.x * 64 + k] = t;
  }
}

// floor(a / d) for a < 2^24 through a float reciprocal computed once per
// kernel, corrected to exact (the per-tile pixel-block decode would otherwise
// run two ~40-instruction integer divisions on every tile).
struct SmallDiv {
  int d;
  float rcp;
  __device__ __forceinline__ explicit SmallDiv(int dv) : d(dv), rcp(1.0f / static_cast<float>(dv)) {}
  __device__ __forceinline__ int div(int a) const {
    int q = __float2int_rz(__int2float_rz(a) * rcp);
    if (q * d > a) --q;
    if ((q + 1) * d <= a) ++q;
    return q;
  }
};

// In-order position on the operand ring (iteration it = lap * stages + slot),
// advanced incrementally: the single-thread MMA/TMA loops are latency-bound,
// so no integer division sits on their per-tile path.
struct RingPos {
  uint32_t slot = 0, lap = 0;
  __device__ __forceinline__ void next(int stages) {
    if (++slot == static_cast<uint32_t>(stages)) {
      slot = 0;
      ++lap;
    }
  }
};

// This CTA's tiles (tile = blockIdx.x + j * gridDim.x) as (M block, N block),
// N block fastest, walked without divisions.
// With clusters of 2 (multicast weights), the unit is an (M-block pair, N
// block): cluster c walks units c, c + C, ... (C clusters) and its CTA of rank
// r takes M block 2 * pair + r, so both CTAs share every B block.
struct TileWalk {
  int mb, nb, step_m, step_n, n_tiles, pair, rank, cl;
  __device__ __forceinline__ explicit TileWalk(int n, int cluster = 1) : n_tiles(n), cl(cluster) {
    const int first = blockIdx.x / cluster, stride = gridDim.x / cluster;
    rank = cluster > 1 ? static_cast<int>(ptx::cluster_ctarank()) : 0;
    pair = first / n;
    nb = first - pair * n;
    step_m = stride / n;
    step_n = stride - step_m * n;
    mb = pair * cluster + rank;
  }
  __device__ __forceinline__ void next() {
    pair += step_m;
    nb += step_n;
    if (nb >= n_tiles) {
      nb -= n_tiles;
      ++pair;
    }
    mb = pair * cl + rank;
  }
};

// kStemU8: the eight gather warps form 8/mt groups of mt warps; a group
// produces whole tiles on its own (tile j -> group j % groups, warp q of the
// group fills sub-tile q) and owns ring slot j % groups (stages == groups),
// so its waits on that slot stay in order (a shared ring would let one group
// wait on a slot two phases ahead, which a parity wait cannot tell apart).
// `use` counts earlier uses of the slot.
__device__ __forceinline__ void stem_slot(uint32_t j, int kb, int num_kb, int groups,
                                          uint32_t& slot, uint32_t& use) {
  slot = j % static_cast<uint32_t>(groups);
  use = (j / static_cast<uint32_t>(groups)) * static_cast<uint32_t>(num_kb) + static_cast<uint32_t>(kb);
}

// Gathers the A tiles of one output tile (128 im2col rows) for every K
// block into the stage ring. `it` is the CTA-wide pipeline iteration counter
// (continues across tiles), so stage/phase follow the global sequence.
template <int G>
__device__ __forceinline__ void gather_a_tile(const ConvGemmArgs& a, uint8_t* smem,
                                              uint64_t* full, uint64_t* empty, int m0,
                                              RingPos& rp) {
  constexpr int GPR = 64 / G;                   // granules per 128 B row
  constexpr int RPP = kGatherWarps * 32 / GPR;  // rows covered per pass of the gather warps
  constexpr int PASSES = kConvBM / RPP;         // passes per tile
  constexpr int GB = G * 2;          // granule bytes
  const int t = threadIdx.x - kGatherWarp0 * 32;
  const int gi = t % GPR;
  const int r0 = t / GPR;

  // Output coordinates of this thread's rows m0+r0+p*RPP, by one division
  // for the first row and carries after that (rows are consecutive pixels):
  // per row the element offset of its window origin (may lie in the padding)
  // and the origin itself for the bounds checks.
  int base[PASSES], hi0[PASSES], wi0[PASSES];
  {
    const int HoWo = a.Ho * a.Wo;
    const int m_first = m0 + r0;
    int n = m_first / HoWo;
    const int rem = m_first - n * HoWo;
    int ho = rem / a.Wo;
    int wo = rem - ho * a.Wo;
#pragma unroll
    for (int p = 0; p < PASSES; ++p) {
      const bool live = m_first + p * RPP < a.M;
      hi0[p] = live ? ho * a.stride_h - a.pad_h : -(1 << 28);  // dead rows read zeros
      wi0[p] = wo * a.stride_w - a.pad_w;
      base[p] = live ? ((n * a.H + hi0[p]) * a.W + wi0[p]) * a.C : 0;
      wo += RPP;
      while (wo >= a.Wo) {
        wo -= a.Wo;
        if (++ho == a.Ho) {
          ho = 0;
          ++n;
        }
      }
    }
  }

  const uint32_t smem_base = ptx::smem_u32(smem);
  const int col_bytes = gi * GB;
  // Rows of one thread differ by multiples of 8, so the 128 B swizzle phase
  // (row & 7) is fixed per thread.
  const uint32_t lane_off = static_cast<uint32_t>(r0) * 128 +
                            ((((col_bytes >> 4) ^ (r0 & 7)) << 4) | (col_bytes & 15));
  // This thread's K position k = kb * 64 + gi * G as (kernel row r, kernel
  // column sx, channel c), divided once and then advanced by 64 per K block
  // with carries (the per-K-block integer divisions were the gather warps'
  // critical path: ~190 instructions per K block, now ~40).
  int c = gi * G, r = 0, sx = 0;
  {
    const int tap = c / a.C;
    c -= tap * a.C;
    r = tap / a.S;
    sx = tap - r * a.S;
  }
  for (int kb = 0; kb < a.num_kb; ++kb, rp.next(a.stages)) {
    const uint32_t s = rp.slot;
    if (rp.lap > 0) ptx::mbar_wait(&empty[s], (rp.lap - 1) & 1);
    const bool kvalid = r < a.R;  // (K padding past the last tap reads zeros)
    const int delta = (r * a.W + sx) * a.C + c;
    const uint32_t sbase = smem_base + s * kABytes + lane_off;
#pragma unroll
    for (int p = 0; p < PASSES; ++p) {
      const int hi = hi0[p] + r;
      const int wi = wi0[p] + sx;
      const bool v = kvalid && static_cast<unsigned>(hi) < static_cast<unsigned>(a.H) &&
                     static_cast<unsigned>(wi) < static_cast<unsigned>(a.W);
      const __nv_bfloat16* src = v ? a.x + (base[p] + delta) : a.x;
      const uint32_t off = static_cast<uint32_t>(p * RPP * 128);
      if constexpr (GB == 16) {
        ptx::cp_async_16(sbase + off, src, v ? 16u : 0u);
      } else {
        ptx::cp_async_8(sbase + off, src, v ? 8u : 0u);
      }
    }
    ptx::cp_async_mbar_arrive_noinc(&full[s]);
    c += kConvBK;
    while (c >= a.C) {
      c -= a.C;
      if (++sx == a.S) {
        sx = 0;
        ++r;
      }
    }
  }
}

__device__ __forceinline__ uint32_t pack2_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Stem producer (kStemU8): the stem conv reads the u8 images [n][H][W][3]
// directly, so the staged bf16 input tensor is never materialised. Each of
// the eight gather warps owns whole tiles (tile j of this CTA -> warp j % 8),
// so eight tiles' loads are in flight and no block-level barrier is needed.
// Lane l owns tile rows l, l+32, l+64, l+96 (consecutive output pixels across
// lanes, so a warp's byte loads of one tap fall in one or two 128 B lines):
// for each tap it loads the pixel's 3 bytes, normalises them and writes the
// row's 16 B granules (two taps x 4 channels, the 4th zero) into the
// 128 B-swizzled A stage; padding and the K tail become zeros.
//
// Normalisation: the staging kernel stores bf16_rn((p - 127.5f) / 63.75f).
// Here it is bf16_rn((p - 127.5f) * (1 / 63.75f)): the fp32 values differ for
// some p, but after bf16 rounding the two agree for all 256 byte values
// (checked exhaustively, tests/test_oracle.py::test_stem_normalisation_exact).

// u8 -> fp32 without the conversion pipe: the float with bits 0x4B000000 | p
// is 2^23 + p exactly, so subtracting 2^23 gives p exactly.
__device__ __forceinline__ float u8_to_f32(uint32_t p) {
  return __fsub_rn(__uint_as_float(0x4B000000u | p), 8388608.0f);
}

__device__ __forceinline__ uint32_t stem_norm2(uint32_t p0, uint32_t p1) {
  const float r = 1.0f / 63.75f;
  const float v0 = __fmul_rn(__fsub_rn(u8_to_f32(p0), 127.5f), r);
  const float v1 = __fmul_rn(__fsub_rn(u8_to_f32(p1), 127.5f), r);
  return pack2_bf16(v0, v1);
}

// L2 prefetch of the image rows a stem tile reads (one contiguous byte range:
// NHWC rows of consecutive images are contiguous), issued ahead because every
// tile of a persistent CTA touches rows no other tile of it did.
__device__ __forceinline__ void stem_prefetch(const ConvGemmArgs& a, int m0) {
  if (m0 >= a.M) return;
  const int HoWo = a.Ho * a.Wo;
  const int m1 = min(m0 + kConvBM, a.M) - 1;
  const int n0 = m0 / HoWo, n1 = m1 / HoWo;
  const int g_lo = n0 * a.H + max(0, ((m0 - n0 * HoWo) / a.Wo) * a.stride_h - a.pad_h);
  const int g_hi = n1 * a.H + min(a.H, ((m1 - n1 * HoWo) / a.Wo) * a.stride_h - a.pad_h + a.R);
  const size_t lo = static_cast<size_t>(g_lo) * a.W * 3, hi = static_cast<size_t>(g_hi) * a.W * 3;
  if (hi <= lo) return;
  const size_t lo16 = lo & ~static_cast<size_t>(15);
  const size_t bytes = min(static_cast<size_t>(1 << 16), (hi - lo16 + 15) & ~static_cast<size_t>(15));
  ptx::bulk_prefetch_l2(a.img + lo16, static_cast<uint32_t>(bytes));
}

// Bits [lo, hi) of a mask (empty when hi <= lo); lo, hi in [0, 16].
__device__ __forceinline__ uint32_t bit_range(int lo, int hi) {
  return hi > lo ? ((1u << hi) - 1u) & ~((1u << lo) - 1u) : 0u;
}

__device__ __forceinline__ void stem_a_tile(const ConvGemmArgs& a, uint32_t smem_a, uint64_t* full,
                                            uint64_t* empty, int m0, uint32_t j, int lane, int q,
                                            int groups) {
  // sub-tile q of the tile at m0 (rows m0 + 128 q ..)
  const uint32_t a_stage = static_cast<uint32_t>(a.mt) * kABytes;
  m0 += q * kConvBM;
  smem_a += q * kABytes;
  const int HoWo = a.Ho * a.Wo;
  for (int kb = 0; kb < a.num_kb; ++kb) {
    uint32_t s, use;
    stem_slot(j, kb, a.num_kb, groups, s, use);
    if (use > 0) ptx::mbar_wait(&empty[s], (use - 1) & 1);
    const int ntaps = min(16, a.taps - kb * 16);  // real taps in this K block (uniform)
    // lane l: tile rows l, l+32, l+64, l+96 (kept rolled: the body is large)
    int m = m0 + lane;
    int n = m / HoWo;
    const int rem = m - n * HoWo;
    int ho = rem / a.Wo;
    int wo = rem - ho * a.Wo;
#pragma unroll 1
    for (int r = lane; r < (a.debug_flags & 8 ? 0 : kConvBM); r += 32, m += 32) {  // (flag 8: bring-up)
      const int hi0 = ho * a.stride_h - a.pad_h;
      const int wi0 = wo * a.stride_w - a.pad_w;
      // kernel rows / columns that fall inside the image (none for rows >= M)
      const uint32_t rmask = m < a.M ? bit_range(max(0, -hi0), min(a.R, a.H - hi0)) : 0u;
      const uint32_t cmask = bit_range(max(0, -wi0), min(a.S, a.W - wi0));
      const uint8_t* base = a.img + (static_cast<long long>(n * a.H + hi0) * a.W + wi0) * 3;
      const uint32_t rowa = smem_a + s * a_stage + r * 128;
      const int sw = r & 7;
      uint32_t px[16][3];
      bool ok[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int info = a.tap_info[(kb * 16 + e) & 63];
        ok[e] = e < ntaps && ((rmask >> ((info >> 24) & 15)) & (cmask >> ((info >> 28) & 15)) & 1u);
        const uint8_t* src = base + (ok[e] ? (info & 0xFFFFFF) : 0);
        src = ok[e] ? src : a.img;
        px[e][0] = __ldg(src);
        px[e][1] = __ldg(src + 1);
        px[e][2] = __ldg(src + 2);
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        uint32_t wv[4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int e = 2 * g + u;
          wv[2 * u] = ok[e] ? stem_norm2(px[e][0], px[e][1]) : 0u;
          wv[2 * u + 1] = ok[e] ? stem_norm2(px[e][2], 0u) & 0xFFFFu : 0u;
        }
        ptx::sts128(rowa + ((g ^ sw) << 4), make_uint4(wv[0], wv[1], wv[2], wv[3]));
      }
      wo += 32;
      while (wo >= a.Wo) {
        wo -= a.Wo;
        if (++ho == a.Ho) {
          ho = 0;
          ++n;
        }
      }
    }
    ptx::fence_proxy_async_smem();  // generic smem writes -> tensor-core (async proxy) reads
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&full[s]);
  }
}

__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// pack to bf16 pairs, then max with `floor` (0: ReLU; bf16 -inf pair: none).
// ReLU after rounding equals rounding after ReLU (rounding is monotonic and
// maps 0 to 0).
__device__ __forceinline__ uint32_t relu_pack_bf16(float lo, float hi, uint32_t floor) {
  uint32_t d;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(pack_bf16(lo, hi)), "r"(floor));
  return d;
}

// bias_s: the layer's bias staged in shared memory (indexed by channel).
template <bool RES>
__device__ __forceinline__ void epilogue_chunk(const ConvGemmArgs& a, const float* bias_s, int m,
                                               int n, const uint32_t (&raw)[16]) {
  float v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(raw[j]);
  if (n + 16 <= a.Cout) {
    const float4* b4 = reinterpret_cast<const float4*>(bias_s + n);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 b = b4[q];
      v[4 * q + 0] += b.x;
      v[4 * q + 1] += b.y;
      v[4 * q + 2] += b.z;
      v[4 * q + 3] += b.w;
    }
    if (RES && a.residual) {
      const uint4* rp =
          reinterpret_cast<const uint4*>(a.residual + static_cast<size_t>(m) * a.ld_res + n);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint4 rr = __ldg(rp + q);
        const uint32_t w[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[8 * q + 2 * e] += bf16_lo(w[e]);
          v[8 * q + 2 * e + 1] += bf16_hi(w[e]);
        }
      }
    }
    if (a.relu) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.0f);
    }
    if (a.out_f32) {
      float4* yp = reinterpret_cast<float4*>(static_cast<float*>(a.y) +
                                             static_cast<size_t>(m) * a.ldy + a.c_off + n);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        yp[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
      uint4* yp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.y) +
                                           static_cast<size_t>(m) * a.ldy + a.c_off + n);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        yp[q] = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                           pack_bf16(v[8 * q + 4], v[8 * q + 5]),
                           pack_bf16(v[8 * q + 6], v[8 * q + 7]));
      }
    }
  } else {
    for (int j = 0; j < 16 && n + j < a.Cout; ++j) {
      float x = v[j] + bias_s[n + j];
      if (RES && a.residual) x += __bfloat162float(a.residual[static_cast<size_t>(m) * a.ld_res + n + j]);
      if (a.relu) x = fmaxf(x, 0.0f);
      const size_t o = static_cast<size_t>(m) * a.ldy + a.c_off + n + j;
      if (a.out_f32)
        static_cast<float*>(a.y)[o] = x;
      else
        static_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(x);
    }
  }
}

// TMA-store epilogue for one 32-column slice of the warp's 32 rows: TMEM ->
// registers, + bias (+ residual), ReLU, packed into the 128 B-swizzled
// staging rows (lane = row, conflict-free 16 B stores). `col` is the slice's
// offset inside its staging group.
template <bool RES>
__device__ __forceinline__ void epilogue_slice_tma(const ConvGemmArgs& a, const float* bias_s, int m,
                                                   int n, const uint32_t (&raw)[32], uint8_t* group,
                                                   int col, int lane, const uint4 (&res)[4],
                                                   bool narrow, bool relu) {
  float v[32];
  const float4* b4 = reinterpret_cast<const float4*>(bias_s + n);  // n % 32 == 0
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 b = b4[q];
    v[4 * q + 0] = __uint_as_float(raw[4 * q + 0]) + b.x;
    v[4 * q + 1] = __uint_as_float(raw[4 * q + 1]) + b.y;
    v[4 * q + 2] = __uint_as_float(raw[4 * q + 2]) + b.z;
    v[4 * q + 3] = __uint_as_float(raw[4 * q + 3]) + b.w;
  }
  if (RES && a.residual && m < a.M) {
    const __nv_bfloat16* rrow = a.residual + static_cast<size_t>(m) * a.ld_res + n;
    if (n + 32 <= a.Cout) {  // (loaded by the caller before the TMEM load)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 rr = res[q];
        const uint32_t w[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[8 * q + 2 * e] += bf16_lo(w[e]);
          v[8 * q + 2 * e + 1] += bf16_hi(w[e]);
        }
      }
    } else {
      for (int j = 0; j < 32 && n + j < a.Cout; ++j) v[j] += __bfloat162float(rrow[j]);
    }
  }
  // (bf16 outputs: the ReLU runs on the packed pairs, after rounding — the
  // same values, one max.bf16x2 per pair instead of two FMNMX)
  if (relu && a.out_f32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
  }
  const uint32_t relu_floor = relu ? 0u : 0xFF80FF80u;  // max with 0, or with -inf (identity)
  if (narrow) {  // 64 B rows, 64 B swizzle: 16 B chunk c of row r at c ^ ((r >> 1) & 3)
    uint8_t* row64 = group + lane * 64;
    const int sw64 = (lane >> 1) & 3;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<uint4*>(row64 + ((q ^ sw64) << 4)) =
          make_uint4(relu_pack_bf16(v[8 * q], v[8 * q + 1], relu_floor),
                     relu_pack_bf16(v[8 * q + 2], v[8 * q + 3], relu_floor),
                     relu_pack_bf16(v[8 * q + 4], v[8 * q + 5], relu_floor),
                     relu_pack_bf16(v[8 * q + 6], v[8 * q + 7], relu_floor));
    return;
  }
  uint8_t* row = group + lane * 128;
  const int sw = lane & 7;  // 128 B swizzle: 16 B chunk c lives at c ^ (row & 7)
  if (a.out_f32) {
#pragma unroll
    for (int q = 0; q < 8; ++q)  // 32 fp32 = the whole 128 B row
      *reinterpret_cast<float4*>(row + ((q ^ sw) << 4)) =
          make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
    const int c16 = col >> 3;  // 8 bf16 per 16 B chunk
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<uint4*>(row + (((c16 + q) ^ sw) << 4)) =
          make_uint4(relu_pack_bf16(v[8 * q], v[8 * q + 1], relu_floor),
                     relu_pack_bf16(v[8 * q + 2], v[8 * q + 3], relu_floor),
                     relu_pack_bf16(v[8 * q + 4], v[8 * q + 5], relu_floor),
                     relu_pack_bf16(v[8 * q + 6], v[8 * q + 7], relu_floor));
  }
}

// Before griddepcontrol.wait (the weights do not depend on earlier layers):
// land resident weights in shared memory, or pull the first tile's streamed
// weight blocks into L2, off the post-wait critical path. Out of line: one
// thread runs it once, and inlined it cost the epilogue registers.
template <bool kWin, bool kPair>
__device__ __noinline__ void prewait_weights(const ConvGemmArgs& args, uint32_t b_smem, uint64_t* b_full,
                                             int n_tiles, int cl, int walk_first, int walk_count) {
  const uint32_t bb = static_cast<uint32_t>(kPair ? args.BN / 2 : args.BN) * 128;
  if (kWin) {
    const int ntap = args.R * args.S, ncb = (args.C + 63) / 64;
    if (args.b_res > 0) {  // every (K block, tap) weight tile, once
      ptx::mbar_arrive_expect_tx(b_full, static_cast<uint32_t>(ncb * ntap) * bb);
      for (int kb = 0; kb < ncb; ++kb)
        for (int t = 0; t < ntap; ++t)
          ptx::tma_load_2d(b_smem + (kb * ntap + t) * bb, &args.tmap_b, b_full, t * args.C + kb * 64, 0);
    } else if (walk_first < walk_count) {
      const int n0 = TileWalk(n_tiles).nb * args.BN;
      for (int kb = 0; kb < ncb; ++kb)
        for (int t = 0; t < ntap; ++t) ptx::tma_prefetch_2d(&args.tmap_b, t * args.C + kb * 64, n0);
    }
  } else if (args.b_res > 0) {  // the whole weight matrix, once
    ptx::mbar_arrive_expect_tx(b_full, static_cast<uint32_t>(args.num_kb) * bb);
    for (int kb = 0; kb < args.num_kb; ++kb)
      ptx::tma_load_2d(b_smem + kb * bb, &args.tmap_b, b_full, kb * kConvBK, 0);
  } else if (walk_first < walk_count) {
    const TileWalk t0(n_tiles, cl);
    const int n0 = t0.nb * args.BN + (kPair ? t0.rank * (args.BN / 2) : 0);
    for (int kb = 0; kb < args.num_kb; ++kb) ptx::tma_prefetch_2d(&args.tmap_b, kb * kConvBK, n0);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kConvThreads, 1)
    conv_gemm_kernel(const __grid_constant__ ConvGemmArgs args) {
  // kPairTmaA: a TMA-A conv on CTA pairs, one M = 256 pair MMA per K step
  // (cta_group::2 throughout), each CTA holding half of every B block
  // (kPairIm2col: the same over TMA im2col A loads)
  // (kPairGather: over the cp.async im2col gather; the peer CTA's idle MMA
  // warp forwards its gather completion to the leader's full barrier)
  constexpr bool kPairG = MODE == static_cast<int>(ConvLoadMode::kPairGather);
  constexpr bool kPair = MODE == static_cast<int>(ConvLoadMode::kPairTmaA) ||
                         MODE == static_cast<int>(ConvLoadMode::kPairIm2col) || kPairG;
  // kIm2col: R x S / strided convs whose A blocks are TMA im2col loads (one per
  // (tap, 64-channel block)); otherwise the TMA-A machinery
  constexpr bool kI2C = MODE == static_cast<int>(ConvLoadMode::kIm2col) ||
                        MODE == static_cast<int>(ConvLoadMode::kPairIm2col);
  constexpr bool kTmaA = MODE == static_cast<int>(ConvLoadMode::kTmaA) || (kPair && !kPairG) || kI2C;
  // residual adds are compiled into the 1x1 modes only (the runtime routes
  // every residual conv there); the other modes carry none of that state
  constexpr bool kRes = kTmaA;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 128 B swizzle atoms must sit on 1 KiB boundaries.
  // (offsetting smem_raw, rather than masking the generic address, keeps the
  // pointer in the shared window so accesses through it compile to LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  if (threadIdx.x == 0) ts_mark(args.ts, 4);
  constexpr long long ts0 = 0;
  const int epi_warps = 4 * args.teams;
  // kWindowT: kWindow with the transposed (C % 64 != 0) halo boxes, its own
  // instantiation so the default in-place mode carries none of that code
  constexpr bool kWinT = MODE == static_cast<int>(ConvLoadMode::kWindowT);
  constexpr bool kWin = MODE == static_cast<int>(ConvLoadMode::kWindow) || kWinT;
  const bool win_direct = kWin && !kWinT;
  // kS2DWide: kS2D over 16 or 32 channels (C / 16 boxes per block); its own
  // instantiation keeps the single-box stem kernel's registers lean
  constexpr bool kS2W = MODE == static_cast<int>(ConvLoadMode::kS2DWide);
  constexpr bool kS2 = MODE == static_cast<int>(ConvLoadMode::kS2D) || kS2W;
  constexpr bool kBlk = kWin || kS2;  // 2-D pixel-block tiles, 4-D TMA-store epilogue
  // (kWindow's A operands live in the halo boxes: its ring stages carry B only)
  // (kS2D ring stages are sized for two sub-tiles: a halo box of a 64-row
  // block is still under 32 KiB)
  const SmemLayout L = smem_layout(kPair ? args.BN / 2 : args.BN, args.stages, args.Cout, epi_warps, args.b_res,
                                   kWin ? 0 : kS2 ? 2 : args.mt,
                                   kWin ? static_cast<int>(args.win_box_bytes) : 0, !kBlk && args.y_narrow != 0);
  const uint32_t win_stride = (args.win_box_bytes + 1023) / 1024 * 1024;
  const int mt = args.mt;  // 128-row sub-tiles per tile (one accumulator: mt x BN columns)
  const uint32_t a_stage = static_cast<uint32_t>(kS2 ? 2 : mt) * kABytes;
  // kS2D: per 16-channel block one halo box, 1 KiB apart in the stage
  const uint32_t s2_box_stride = (args.win_box_bytes + 1023) / 1024 * 1024;
  float* bias_s = reinterpret_cast<float*>(smem + L.bias_off);
  const int cout_pad = (args.Cout + 63) / 64 * 64 + 64;
  if (args.y_tma && threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&args.tmap_y);
    if constexpr (!kBlk)
      for (int sg = 0; sg < args.nseg; ++sg) ptx::tma_prefetch_desc(&args.tmap_seg[sg]);
  }
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + args.stages;
  uint64_t* tmem_full = empty + args.stages;  // [n_acc]
  uint64_t* tmem_empty = tmem_full + kMaxAcc;  // [n_acc]
  uint64_t* b_full = tmem_empty + kMaxAcc;    // resident B landed (b_res)
  // kWindow barriers [8]: transposing mode raw_full[2] raw_free[2] cm_full[2]
  // cm_empty[2]; direct mode (128 B-swizzled box read in place) slot_full[4]
  // slot_free[4]
  uint64_t* raw_full = b_full + 1;              // [2] kWindow: pixel-major box landed
  uint64_t* raw_free = raw_full + 2;            // [2] ... transposed (gather warps)
  uint64_t* cm_full = raw_free + 2;             // [2] chunk-major box ready
  uint64_t* cm_empty = cm_full + 2;             // [2] all taps of its K block consumed
  uint64_t* slot_full = raw_full;               // [4] direct mode: box landed
  uint64_t* slot_free = raw_full + 4;           // [4] direct mode: all taps consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cm_empty + 2);
  uint64_t* res_bar = cm_empty + 3;  // [2 per epilogue warp] residual slice landed (res_tma)

  // warp index via a shuffle: provably warp-uniform, so role branches are
  // uniform and the MMA-issue loops keep their operands in uniform registers
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int n_tiles = (args.Cout + args.BN - 1) / args.BN;
  const int tile_rows = kConvBM * mt;
  // kDwFused: M blocks are TH x TW pixel blocks of one image
  const int dw_blocks_per_img = args.dw_tiles_y * args.dw_tiles_x;
  const int m_blocks = kBlk ? (args.M / (args.Ho * args.Wo)) * dw_blocks_per_img
                            : (args.M + tile_rows - 1) / tile_rows;
  const int win_cblocks = (args.C + 63) / 64;  // kWindow: 64-channel K blocks
  const int win_taps = args.R * args.S;
  const int tiles = n_tiles * m_blocks;
  // (cluster mode: the loops below walk units = (M-block pair, N block))
  const int cl = args.cluster > 1 ? args.cluster : 1;
  const int walk_first = blockIdx.x / cl, walk_stride = gridDim.x / cl;
  const int walk_count = cl == 1 ? tiles : n_tiles * ((m_blocks + cl - 1) / cl);
  const int n_acc = args.n_acc;  // power of two
  const int acc_log2 = __ffs(n_acc) - 1;
  const uint32_t acc_stride = args.tmem_cols / n_acc;
  constexpr bool kStem = MODE == static_cast<int>(ConvLoadMode::kStemU8);

  if (warp == kTmaWarp) {
    if (lane == 0) {
      for (int s = 0; s < args.stages; ++s) {
        const uint32_t producers = kTmaA || kWin || kS2 ? 0u
                                   : MODE == static_cast<int>(ConvLoadMode::kStemU8)
                                       ? static_cast<uint32_t>(mt)  // lane 0 of each warp of the group
                                       : kGatherWarps * 32u;
        if constexpr (kPairG)  // leader: gather + its expect_tx + the peer's forward; peer: gather
          ptx::mbar_init(&full[s], producers + (ptx::cluster_ctarank() == 0 ? 2u : 0u));
        else
          ptx::mbar_init(&full[s], producers + (kTmaA || kS2 || args.b_res == 0 ? 1u : 0u));
        // (cluster multicast: both CTAs' MMAs consume a B slot; pairs: the
        // leader's commit arrives in both CTAs once)
        ptx::mbar_init(&empty[s], 1);
      }
      ptx::mbar_init(b_full, 1);
      for (int b = 0; b < 2; ++b) {
        ptx::mbar_init(&raw_full[b], 1);
        ptx::mbar_init(&raw_free[b], win_direct ? 1 : kGatherWarps);
        ptx::mbar_init(&cm_full[b], win_direct ? 1 : kGatherWarps);
        ptx::mbar_init(&cm_empty[b], 1);
      }
      for (int b = 0; b < n_acc; ++b) {
        ptx::mbar_init(&tmem_full[b], 1);
        // one arrival per warp of the owning teams (pairs: of both CTAs' teams)
        ptx::mbar_init(&tmem_empty[b], 4 * args.tpa * (kPair ? 2 : 1));
      }
      if (kRes && args.res_tma)
        for (int b = 0; b < 2 * epi_warps; ++b) ptx::mbar_init(&res_bar[b], 1);
      ptx::fence_barrier_init();
      ptx::tma_prefetch_desc(&args.tmap_b);
      if (kTmaA || kBlk) ptx::tma_prefetch_desc(&args.tmap_a);  // (A / halo / tap boxes)
    }
    __syncwarp();
    if constexpr (kPair) {
      ptx::tmem_alloc_pair(tmem_slot, args.tmem_cols);
      ptx::tmem_relinquish_pair();
    } else {
      ptx::tmem_alloc(tmem_slot, args.tmem_cols);
      ptx::tmem_relinquish();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (cl > 1) ptx::cluster_sync();  // peers' barriers exist before any multicast lands
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) ts_mark(args.ts, 5);
  pdl_trigger();
  // The weights do not depend on earlier layers: before waiting for the
  // previous grid, land resident weights in shared memory, or pull the first
  // tile's streamed weight blocks into L2 (off the post-wait critical path).
  if (!kS2 && warp == kTmaWarp && lane == 0)  // (the stems load theirs after the wait: registers)
    prewait_weights<kWin, kPair>(args, ptx::smem_u32(smem + L.b_off), b_full, n_tiles, cl, walk_first, walk_count);
  pdl_wait();  // activations (and the residual) come from earlier layers
  span_mark(args.span);
  if (args.ts && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    args.ts[blockIdx.x * 64] = gt;
    ts_mark(args.ts, 1, ts0);
  }

  if (warp < epi_warps) {
    // Epilogue: warp w reads TMEM lane quarter w%4 (tile rows 32*(w%4)..+31);
    // team w/4 takes every teams-th tile of this CTA, all its column groups,
    // so up to `teams` tiles drain concurrently.
    // The epilogue warps stage the bias themselves (named barrier 1), off the
    // critical path of the first tile's loads and MMAs.
    for (int i = threadIdx.x; i < cout_pad; i += epi_warps * 32)
      bias_s[i] = i < args.Cout ? __ldg(args.bias + i) : 0.0f;
    asm volatile("bar.sync 1, %0;" ::"r"(epi_warps * 32) : "memory");
    const int quarter = warp & 3;
    // teams per accumulator: with more teams than accumulators, tpa teams
    // share each tile, team t taking column part t % tpa
    const int tpa = args.tpa;
    const int team = (warp >> 2) / tpa;
    const int part = (warp >> 2) % tpa;
    const int tile_teams = args.teams / tpa;
    const int part_cols = args.BN / tpa;
    const int ybufs = y_bufs(epi_warps);
    const int sub_rows = kBlk ? kConvBM / args.dw_tw : 0;  // block rows per 128-row sub-tile
    uint8_t* ystage = smem + L.y_off + warp * y_warp_bytes(epi_warps, !kBlk && args.y_narrow != 0);
    // store groups: one 128 B swizzle row per lane (64 bf16 / 32 fp32), or
    // with y_narrow (sixteen epilogue warps) 32 bf16 in two 2 KiB 64 B-swizzled
    // buffers, so the next slice fills while the last one's TMA store reads
    const bool narrow = !kBlk && args.y_narrow != 0;
    const int group_cols = narrow || args.out_f32 ? 32 : 64;
    const int nbufs = narrow ? 2 : ybufs;
    const uint32_t buf_bytes = narrow ? kYStageBytes / 2 : kYStageBytes;
    uint32_t j = 0, groups = 0;
    TileWalk tw(n_tiles, cl);
    for (int tile = walk_first; tile < walk_count; tile += walk_stride, ++j, tw.next()) {
      if (static_cast<int>(j & (tile_teams - 1)) != team) continue;  // teams: power of two
      const int n0 = tw.nb * args.BN;
      const uint32_t acc = j & (n_acc - 1);
      // residual-staging mode: this tile's first residual slice is TMA-loaded
      // into the staging buffer it will be added in, before the accumulator
      // wait (each later slice is loaded one slice ahead)
      const bool rtma = kRes && narrow && args.res_tma != 0;
      if (rtma && lane == 0) {
        ptx::bulk_wait_read<0>();  // (the buffer's last store has read it)
        const uint32_t b = groups & 1;
        ptx::mbar_arrive_expect_tx(&res_bar[2 * warp + b], 2048);
        ptx::tma_load_2d(ptx::smem_u32(ystage + b * buf_bytes), &args.tmap_r, &res_bar[2 * warp + b],
                         n0 + part * part_cols, tw.mb * tile_rows + quarter * 32);
      }
      if (kRes && args.residual) {
        // pull this lane's residual rows (its column part) into L2 a tile
        // ahead — this team's next tile (and, the first time, this one) — so
        // the epilogue's loads do not each wait on HBM
        auto prefetch_res = [&](const TileWalk& w) {
          for (int q = 0; q < mt; ++q) {
            const int m = w.mb * tile_rows + q * kConvBM + quarter * 32 + lane;
            const int c0 = w.nb * args.BN + part * part_cols;
            if (m >= args.M || c0 >= args.Cout) break;
            const char* rrow =
                reinterpret_cast<const char*>(args.residual + static_cast<size_t>(m) * args.ld_res + c0);
            const int bytes = min(part_cols, args.Cout - c0) * 2;
            for (int c = 0; c < bytes; c += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rrow + c));
          }
        };
        if (args.res_prefetch == 1 || (args.res_prefetch == 2 && j < static_cast<uint32_t>(tile_teams)))
          prefetch_res(tw);
        if (args.res_prefetch == 2 && tile + tile_teams * walk_stride < walk_count) {
          TileWalk ahead = tw;
          for (int k = 0; k < tile_teams; ++k) ahead.next();
          prefetch_res(ahead);
        }
      }
      ptx::mbar_wait(&tmem_full[acc], (j >> acc_log2) & 1);
      ptx::tc_fence_after();
      if (args.ts && quarter == 0 && lane == 0 && j < 8) ts_mark(args.ts, 24 + j, ts0);
      // pixel block of this tile (kBlk): image, block row / column
      int b_img = 0, b_y = 0, b_x = 0;
      if constexpr (kBlk) {
        b_img = SmallDiv(dw_blocks_per_img).div(tw.mb);
        const int blk = tw.mb - b_img * dw_blocks_per_img;
        b_y = SmallDiv(args.dw_tiles_x).div(blk);
        b_x = blk - b_y * args.dw_tiles_x;
      }
      for (int q = 0; q < mt; ++q) {  // sub-tile q: rows m0 .. m0+127, columns q*BN ..
        const int m0 = tw.mb * tile_rows + q * kConvBM;
        if (!kBlk && m0 >= args.M) break;
        int m = m0 + quarter * 32 + lane;
        if (kBlk && (args.residual || !args.y_tma)) {  // A row -> pixel (args.M = not stored)
          const int r = q * kConvBM + quarter * 32 + lane;
          const int oy = b_y * args.dw_th + r / args.dw_tw;
          const int ox = b_x * args.dw_tw + r % args.dw_tw;
          m = r < args.dw_th * args.dw_tw && oy < args.Ho && ox < args.Wo
                  ? (b_img * args.Ho + oy) * args.Wo + ox
                  : args.M;
        }
        const uint32_t t_row = tmem_base + acc * acc_stride + q * args.BN +
                               (static_cast<uint32_t>(quarter * 32) << 16);
        if (args.debug_flags & 1) {
          // release only
        } else if (args.y_tma) {
          const int g_end = (part + 1) * part_cols;
          for (int g0 = part * part_cols; g0 < g_end && n0 + g0 < args.Cout; g0 += group_cols) {
            uint8_t* group = ystage + (nbufs == 2 ? (groups & 1) * buf_bytes : 0);
            // (fused siblings: a segment without ReLU, e.g. ResNet's projection)
            const bool relu_g = args.relu != 0 && (kBlk || !((args.norelu_g >> ((n0 + g0) >> 6)) & 1));
            if (rtma) {
              // next slice's residual into the other buffer once its store has read it
              if (lane == 0 && g0 + group_cols < g_end && n0 + g0 + group_cols < args.Cout) {
                ptx::bulk_wait_read<0>();
                const uint32_t b = (groups + 1) & 1;
                ptx::mbar_arrive_expect_tx(&res_bar[2 * warp + b], 2048);
                ptx::tma_load_2d(ptx::smem_u32(ystage + b * buf_bytes), &args.tmap_r,
                                 &res_bar[2 * warp + b], n0 + g0 + group_cols, m0 + quarter * 32);
              }
              __syncwarp();
            } else if (groups >= static_cast<uint32_t>(nbufs)) {  // the store that used `group` has read it
              if (lane == 0) {
                if (nbufs == 2)
                  ptx::bulk_wait_read<1>();
                else
                  ptx::bulk_wait_read<0>();
              }
              __syncwarp();
            }
            for (int c = 0; c < group_cols && g0 + c < g_end; c += 32) {
              // residual slice first: its global load overlaps the TMEM load
              uint4 res[4];
              if (rtma) {
                ptx::mbar_wait(&res_bar[2 * warp + (groups & 1)], (groups >> 1) & 1);
                const uint32_t row64 = ptx::smem_u32(group) + lane * 64;
                const int sw64 = (lane >> 1) & 3;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                               : "=r"(res[q].x), "=r"(res[q].y), "=r"(res[q].z), "=r"(res[q].w)
                               : "r"(row64 + ((q ^ sw64) << 4)));
              } else if (kRes && args.residual && m < args.M && n0 + g0 + c + 32 <= args.Cout) {
                const uint4* rp = reinterpret_cast<const uint4*>(
                    args.residual + static_cast<size_t>(m) * args.ld_res + n0 + g0 + c);
#pragma unroll
                for (int q = 0; q < 4; ++q) res[q] = __ldg(rp + q);
              }
              uint32_t raw[32];
              ptx::tmem_ld_32x32b_x32(t_row + g0 + c, raw);
              ptx::tmem_ld_wait();
              epilogue_slice_tma<kRes>(args, bias_s, m, n0 + g0 + c, raw, group, c, lane, res, narrow,
                                       relu_g);
            }
            ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> TMA engine
            __syncwarp();
            if (lane == 0) {
              if constexpr (kBlk) {  // this warp's rw pixel rows of the TH x TW block
                const int yq = q * sub_rows + quarter * args.dw_rw;  // in-block row
                if (yq < args.dw_th)
                  ptx::tma_store_4d(&args.tmap_y, ptx::smem_u32(group), n0 + g0, b_x * args.dw_tw,
                                    b_y * args.dw_th + yq, b_img);
              } else {
                if (args.nseg > 0) {  // a fused sibling's columns go to its own buffer
                  const int sg = args.seg_g[(n0 + g0) >> 6];
                  ptx::tma_store_2d(&args.tmap_seg[sg], ptx::smem_u32(group), n0 + g0 - args.seg_col[sg],
                                    m0 + quarter * 32);
                } else {
                  ptx::tma_store_2d(&args.tmap_y, ptx::smem_u32(group), n0 + g0, m0 + quarter * 32);
                }
              }
              ptx::bulk_commit();
            }
            ++groups;
          }
        } else {
          for (int c0 = part * part_cols; c0 < (part + 1) * part_cols && n0 + c0 < args.Cout; c0 += 16) {
            uint32_t raw[16];
            ptx::tmem_ld_32x32b_x16(t_row + c0, raw);
            ptx::tmem_ld_wait();
            if (m < args.M) epilogue_chunk<kRes>(args, bias_s, m, n0 + c0, raw);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kPair && tw.rank != 0)
          ptx::mbar_arrive_cluster(&tmem_empty[acc], 0);  // the leader's MMA reuses it
        else
          ptx::mbar_arrive(&tmem_empty[acc]);
      }
      if (args.ts && quarter == 0 && lane == 0 && j < 8) ts_mark(args.ts, 32 + j, ts0);
    }
    if (lane == 0) ptx::bulk_wait<0>();
  } else if (warp < kGatherWarp0) {
    // (with a single epilogue team, warps 4-7 have no role)
  } else if (warp < kGatherWarp0 + kGatherWarps) {
    if constexpr (MODE == static_cast<int>(ConvLoadMode::kStemU8)) {
      // one producer warp per tile (tile j -> gather warp j % 8); tile j's
      // K blocks are pipeline iterations j*num_kb ..
      // (the stem conv has one N tile: tile index == M block)
      const int pw = warp - kGatherWarp0;
      const int groups = kGatherWarps / mt;
      const int grp = pw / mt, q = pw % mt;
      uint32_t j = 0;
      if (lane == 0) {  // warm up: this group's first two tiles
        stem_prefetch(args, (blockIdx.x + grp * gridDim.x) * tile_rows + q * kConvBM);
        stem_prefetch(args, (blockIdx.x + (grp + groups) * gridDim.x) * tile_rows + q * kConvBM);
      }
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++j) {
        if (static_cast<int>(j % groups) != grp) continue;
        if (lane == 0)  // two of this group's tiles ahead
          stem_prefetch(args, (tile + 2 * groups * gridDim.x) * tile_rows + q * kConvBM);
        stem_a_tile(args, ptx::smem_u32(smem + L.a_off), full, empty, tile * tile_rows, j, lane, q,
                    groups);
      }
    } else if constexpr (kWin) {
      // transpose each K block's halo box: raw [pixel][cb] -> chunk-major
      // [chunk][pixel] 16 B pieces (the no-swizzle K-major operand layout)
      const int tid = threadIdx.x - kGatherWarp0 * 32;
      const int npix = args.win_iw * args.win_ih;
      const int cb = args.C < 64 ? args.C : 64;
      const int raw_chunks = cb / 8;  // 16 B chunks per raw pixel row
      uint32_t u = 0;                  // box uses so far (slot u & 1, phase u >> 1)
      // (direct mode: the MMA reads the TMA's 128 B-swizzled box itself)
      for (int tile = blockIdx.x; tile < (win_direct ? 0 : tiles); tile += gridDim.x) {
        for (int kb = 0; kb < win_cblocks; ++kb, ++u) {
          const uint32_t b = u & 1, ph = (u >> 1) & 1;
          ptx::mbar_wait(&raw_full[b], ph);
          if (u >= 2) ptx::mbar_wait(&cm_empty[b], ph ^ 1);
          const uint32_t raw = ptx::smem_u32(smem + L.win_off + b * win_stride);
          const uint32_t cm = ptx::smem_u32(smem + L.win_off + (2 + b) * win_stride);
          const int kch = min(8, (args.C - kb * 64) / 8);  // real chunks of this K block
          for (int i = tid; i < npix * kch; i += kGatherWarps * 32) {
            const int p = i / kch, k = i - p * kch;
            uint4 v;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(raw + (p * raw_chunks + k) * 16));
            ptx::sts128(cm + (k * npix + p) * 16, v);
          }
          ptx::fence_proxy_async_smem();  // generic smem writes -> tensor-core reads
          __syncwarp();
          if (lane == 0) {
            ptx::mbar_arrive(&raw_free[b]);
            ptx::mbar_arrive(&cm_full[b]);
          }
        }
      }
    } else if constexpr (!kTmaA) {  // (in TMA-A mode these warps are epilogue teams 2-3)
      RingPos rp;
      TileWalk tw(n_tiles, cl);
      for (int tile = walk_first; tile < walk_count; tile += walk_stride, tw.next()) {
        const int m0 = tw.mb * kConvBM;
        gather_a_tile<8>(args, smem + L.a_off, full, empty, m0, rp);
      }
    }
  } else if (warp == kTmaWarp && kS2) {
    if (lane == 0) {
      const uint32_t b_bytes = static_cast<uint32_t>(args.BN) * 128;
      ptx::mbar_arrive_expect_tx(b_full, static_cast<uint32_t>(args.num_kb) * b_bytes);
      for (int kb = 0; kb < args.num_kb; ++kb)
        ptx::tma_load_2d(ptx::smem_u32(smem + L.b_off + kb * b_bytes), &args.tmap_b, b_full,
                         kb * kConvBK, 0);
      RingPos rp;
      TileWalk tw(n_tiles);
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, tw.next()) {
        const int img = SmallDiv(dw_blocks_per_img).div(tw.mb);
        const int blk = tw.mb - img * dw_blocks_per_img;
        const int by = SmallDiv(args.dw_tiles_x).div(blk);
        const int bx = blk - by * args.dw_tiles_x;
        {  // one halo box per block holds every tap's window
          const uint32_t s = rp.slot;
          if (rp.lap > 0) ptx::mbar_wait(&empty[s], (rp.lap - 1) & 1);
          // one box per 16-channel block (C = 16 or 32), origin shifted by the
          // padding (negative coordinates read zeros)
          const int nc = kS2W ? args.C >> 4 : 1;
          ptx::mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nc) * args.win_box_bytes);
          for (int cb = 0; cb < nc; ++cb)
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
                    ptx::smem_u32(smem + L.a_off + s * a_stage + cb * s2_box_stride)),
                "l"(&args.tmap_a), "r"(ptx::smem_u32(&full[s])), "r"(cb * 16),
                "r"(bx * args.dw_tw - args.pad_w), "r"(by * args.dw_th - args.pad_h), "r"(img)
                : "memory");
          rp.next(args.stages);
        }
      }
    }
  } else if (warp == kTmaWarp && kWin) {
    if (lane == 0) {
      const uint32_t b_bytes = static_cast<uint32_t>(args.BN) * 128;
      const bool b_res = args.b_res > 0;  // (resident weights issued before pdl_wait)
      RingPos rp;
      TileWalk tw(n_tiles);
      uint32_t u = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, tw.next()) {
        const int n0 = tw.nb * args.BN;
        const int img = SmallDiv(dw_blocks_per_img).div(tw.mb);
        const int blk = tw.mb - img * dw_blocks_per_img;
        const int by = SmallDiv(args.dw_tiles_x).div(blk);
        const int bx = blk - by * args.dw_tiles_x;
        for (int kb = 0; kb < win_cblocks; ++kb, ++u) {
          // (direct mode: 4 box slots, the MMA frees them; else 2 + 2 transposed)
          const uint32_t nb_slots = win_direct ? 4u : 2u;
          const uint32_t b = u % nb_slots, ph = (u / nb_slots) & 1;
          if (u >= nb_slots) ptx::mbar_wait(win_direct ? &slot_free[b] : &raw_free[b], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&raw_full[b], args.win_box_bytes);  // (== slot_full[b])
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
                  ptx::smem_u32(smem + L.win_off + b * win_stride)),
              "l"(&args.tmap_a), "r"(ptx::smem_u32(&raw_full[b])), "r"(kb * 64),
              "r"(bx * args.dw_tw - args.pad_w), "r"(by * args.dw_th - args.pad_h), "r"(img)
              : "memory");
          if (b_res) continue;
          for (int t = 0; t < win_taps; ++t, rp.next(args.stages)) {
            const uint32_t s = rp.slot;
            if (rp.lap > 0) ptx::mbar_wait(&empty[s], (rp.lap - 1) & 1);
            ptx::mbar_arrive_expect_tx(&full[s], b_bytes);
            ptx::tma_load_2d(ptx::smem_u32(smem + L.b_off + s * b_bytes), &args.tmap_b, &full[s],
                             t * args.C + kb * 64, n0);
          }
        }
      }
    }
  } else if (warp == kTmaWarp) {
    if (lane == 0) {
      const uint32_t b_bytes = static_cast<uint32_t>(kPair ? args.BN / 2 : args.BN) * 128;
      const bool b_res = args.b_res > 0;  // (resident weights issued before pdl_wait)
      const uint32_t tx = (b_res ? 0u : b_bytes) + (kTmaA ? a_stage : 0);
      uint32_t j = 0;
      RingPos rp;
      TileWalk tw(n_tiles, cl);
      for (int tile = walk_first; tile < (tx ? walk_count : 0); tile += walk_stride, ++j, tw.next()) {
        const int m0 = tw.mb * tile_rows;
        const int n0 = tw.nb * args.BN;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          uint32_t s, use;
          if constexpr (kStem) {
            stem_slot(j, kb, args.num_kb, kGatherWarps / mt, s, use);
          } else {
            s = rp.slot;
            use = rp.lap;
            rp.next(args.stages);
          }
          if (use > 0) ptx::mbar_wait(&empty[s], (use - 1) & 1);
          if (args.ts && kb == 0 && j < 8) ts_mark(args.ts, 40 + j, ts0);
          if constexpr (kPair) {
            // both CTAs' bytes count on the leader's full barrier
            if (tw.rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * tx);
            ptx::tma_load_2d_pair(ptx::smem_u32(smem + L.b_off + s * b_bytes), &args.tmap_b, &full[s],
                                  kb * kConvBK, n0 + tw.rank * (args.BN / 2));
            if constexpr (kI2C) {  // this CTA's 128 output pixels' windows (mt == 1)
              const int cbs = args.C >> 6;
              const int t = kb / cbs, cb = kb - t * cbs;
              const int tr = t / args.S, tc = t - tr * args.S;
              const int hw_o = args.Ho * args.Wo;
              const int n = m0 / hw_o, rem = m0 - n * hw_o;
              const int ho = rem / args.Wo, wo = rem - ho * args.Wo;
              ptx::tma_load_im2col_pair(ptx::smem_u32(smem + L.a_off + s * a_stage), &args.tmap_a, &full[s],
                                        cb * 64, wo * args.stride_w - args.pad_w,
                                        ho * args.stride_h - args.pad_h, n, tc, tr);
            } else if constexpr (kTmaA) {
              for (int q = 0; q < mt; ++q)
                ptx::tma_load_2d_pair(ptx::smem_u32(smem + L.a_off + s * a_stage + q * kABytes), &args.tmap_a,
                                      &full[s], kb * kConvBK, m0 + q * kConvBM);
            }
            continue;
          }
          ptx::mbar_arrive_expect_tx(&full[s], tx);
          if (!b_res) {
            ptx::tma_load_2d(ptx::smem_u32(smem + L.b_off + s * b_bytes), &args.tmap_b, &full[s],
                             kb * kConvBK, n0);
          }
          if constexpr (kI2C) {
            // K block kb = (tap t, channel block cb); sub-tile q starts at output
            // pixel m0 + 128 q, whose input window origin is (wo*sw - pw, ho*sh - ph)
            const int cbs = args.C >> 6;
            const int t = kb / cbs, cb = kb - t * cbs;
            const int tr = t / args.S, tc = t - tr * args.S;
            const int hw_o = args.Ho * args.Wo;
            for (int q = 0; q < mt; ++q) {
              const int mq = m0 + q * kConvBM;
              const int n = mq / hw_o, rem = mq - n * hw_o;
              const int ho = rem / args.Wo, wo = rem - ho * args.Wo;
              asm volatile(
                  "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(
                      ptx::smem_u32(smem + L.a_off + s * a_stage + q * kABytes)),
                  "l"(&args.tmap_a), "r"(cb * 64), "r"(wo * args.stride_w - args.pad_w),
                  "r"(ho * args.stride_h - args.pad_h), "r"(n), "r"(ptx::smem_u32(&full[s])),
                  "h"(static_cast<uint16_t>(tc)), "h"(static_cast<uint16_t>(tr))
                  : "memory");
            }
          } else if constexpr (kTmaA)
            for (int q = 0; q < mt; ++q)  // (rows past M arrive as zeros)
              ptx::tma_load_2d(ptx::smem_u32(smem + L.a_off + s * a_stage + q * kABytes),
                               &args.tmap_a, &full[s], kb * kConvBK, m0 + q * kConvBM);
        }
      }
    }
  } else if (kS2) {  // kMmaWarp: per tap, sub-tile q reads its 128 rows of the tap box
    {  // (whole warp: uniform descriptors, elected issue)
      const uint32_t idesc = ptx::umma_idesc_bf16_f32(kConvBM, args.BN);
      const uint32_t b_bytes = static_cast<uint32_t>(args.BN) * 128;
      ptx::mbar_wait(b_full, 0);
      const int taps = args.R * args.S;
      uint32_t j = 0;
      RingPos rp;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++j) {
        const uint32_t acc = j & (n_acc - 1);
        if (j >= static_cast<uint32_t>(n_acc))
          ptx::mbar_wait(&tmem_empty[acc], ((j >> acc_log2) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + acc * acc_stride;
        {  // windows of the block's halo box: tap (dr, dc) starts at
           // pixel (16 q + dr) * IW + dc, pixel rows sbo = IW * 32 B apart
          const uint32_t s = rp.slot;
          ptx::mbar_wait(&full[s], rp.lap & 1);
          ptx::tc_fence_after();
          const uint32_t box = ptx::smem_u32(smem + L.a_off + s * a_stage);
          const uint32_t sbo = static_cast<uint32_t>(args.win_iw) * 32;
          const uint32_t b_base = ptx::smem_u32(smem + L.b_off);
          // 2x2 / 4x4 taps (3x3 / 7x7 stems) with two or four sub-tiles:
          // fully unrolled, every descriptor a compile-time offset (uniform issue)
          // (NC 16-channel boxes: K step of (tap t, block cb) = t * NC + cb)
          auto unrolled = [&](auto dr_c, auto ds_c, auto mt_c, auto nc_c) {
            constexpr int DR = decltype(dr_c)::value, DS = decltype(ds_c)::value;
            constexpr int MT = decltype(mt_c)::value, NC = decltype(nc_c)::value;
            constexpr int IW = 8 + DS - 1;
            const uint64_t da0 = ptx::umma_desc_sw32_kmajor_sbo(box, IW * 32);
            const uint64_t db0 = ptx::umma_desc_sw128_kmajor(b_base);
            const uint64_t bstep = b_bytes >> 4;
            const uint64_t cstep = s2_box_stride >> 4;
#pragma unroll
            for (int t = 0; t < DR * DS; ++t)
#pragma unroll
              for (int cb = 0; cb < NC; ++cb)
#pragma unroll
                for (int q = 0; q < MT; ++q) {
                  const int k = t * NC + cb;
                  ptx::umma_bf16_warp(d + q * args.BN,
                                      da0 + cb * cstep +
                                          static_cast<uint64_t>(((16 * q + t / DS) * IW + t % DS) * 2),
                                      db0 + static_cast<uint64_t>(k >> 2) * bstep + 2 * (k & 3), idesc,
                                      k != 0);
                }
          };
          const bool fast = mt == 2 || mt == 4;
          using I1 = std::integral_constant<int, 1>;
          using I2 = std::integral_constant<int, 2>;
          using I3 = std::integral_constant<int, 3>;
          using I4 = std::integral_constant<int, 4>;
          bool done = false;
          if constexpr (kS2W) {
            if (fast && mt == 2 && args.R == 3 && args.S == 3 && (args.C == 16 || args.C == 32)) {
              if (args.C == 16) unrolled(I3{}, I3{}, I2{}, I1{});
              else unrolled(I3{}, I3{}, I2{}, I2{});
              done = true;
            }
          } else {
            if (fast && args.R == 2 && args.S == 2) {
              if (mt == 2) unrolled(I2{}, I2{}, I2{}, I1{});
              else unrolled(I2{}, I2{}, I4{}, I1{});
              done = true;
            } else if (fast && args.R == 4 && args.S == 4) {
              if (mt == 2) unrolled(I4{}, I4{}, I2{}, I1{});
              else unrolled(I4{}, I4{}, I4{}, I1{});
              done = true;
            }
          }
          const int ncb = kS2W ? args.C >> 4 : 1;
          for (int t = 0, dr = 0, dc = 0; t < (done ? 0 : taps);
               ++t, dc = dc + 1 == args.S ? 0 : dc + 1, dr = dc == 0 ? dr + 1 : dr) {
            for (int cb = 0; cb < ncb; ++cb) {
              const int k = t * ncb + cb;
              const uint64_t db = ptx::umma_desc_sw128_kmajor(
                  ptx::smem_u32(smem + L.b_off + (k >> 2) * b_bytes));
              for (int q = 0; q < mt; ++q) {
                const uint64_t da = ptx::umma_desc_sw32_kmajor_sbo(
                    box + cb * s2_box_stride + static_cast<uint32_t>((16 * q + dr) * args.win_iw + dc) * 32,
                    sbo);
                ptx::umma_bf16_warp(d + q * args.BN, da, db + 2 * (k & 3), idesc, k != 0);
              }
            }
          }
          ptx::umma_commit_warp(&empty[s]);
          rp.next(args.stages);
          ptx::umma_commit_warp(&tmem_full[acc]);
        }
      }
    }
    __syncwarp();
  } else if (kWin) {  // kMmaWarp, shifted-window MMAs (whole warp, elected issue)
    {
      const uint32_t idesc = ptx::umma_idesc_bf16_f32(kConvBM, args.BN);
      const uint32_t b_bytes = static_cast<uint32_t>(args.BN) * 128;
      const bool b_res = args.b_res > 0;
      if (b_res) ptx::mbar_wait(b_full, 0);
      const uint32_t npix = static_cast<uint32_t>(args.win_iw * args.win_ih);
      const uint32_t lbo = npix * 16, sbo = static_cast<uint32_t>(args.win_iw) * 16;
      uint32_t j = 0, u = 0;
      RingPos rp;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++j) {
        const uint32_t acc = j & (n_acc - 1);
        if (j >= static_cast<uint32_t>(n_acc))
          ptx::mbar_wait(&tmem_empty[acc], ((j >> acc_log2) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + acc * acc_stride;
        bool first = true;
        for (int kb = 0; kb < win_cblocks; ++kb, ++u) {
          const bool direct = win_direct;
          const uint32_t b = direct ? u & 3 : u & 1;
          if (direct) {
            ptx::mbar_wait(&slot_full[b], (u >> 2) & 1);
          } else {
            ptx::mbar_wait(&cm_full[b], (u >> 1) & 1);
          }
          ptx::tc_fence_after();
          const uint32_t cm =
              ptx::smem_u32(smem + L.win_off + (direct ? b : 2 + b) * win_stride);
          const int ksteps = min(8, (args.C - kb * 64) / 8) / 2;
          if (direct && ksteps == 4 && mt == 1 && args.R == 3 && args.S == 3) {
            // 3x3: the nine taps fully unrolled, every A descriptor a
            // compile-time offset from the K block's box (uniform issue)
            const uint64_t da0 = ptx::umma_desc_sw128_kmajor_sbo(cm, 10 * 128);  // IW = 10
            const uint32_t b_base = ptx::smem_u32(smem + L.b_off);
#pragma unroll
            for (int t = 0; t < 9; ++t) {
              uint32_t s = 0;
              if (!b_res) {  // weights stream through the ring, one tap per slot
                s = rp.slot;
                ptx::mbar_wait(&full[s], rp.lap & 1);
                ptx::tc_fence_after();
              }
              const uint64_t db = ptx::umma_desc_sw128_kmajor(
                  b_base + (b_res ? static_cast<uint32_t>(kb * 9 + t) : s) * b_bytes);
              ptx::umma_bf16_warp_k64(d, da0 + static_cast<uint64_t>(((t / 3) * 10 + t % 3) * 8),
                                      db, idesc, first && t == 0 ? 0u : 1u);
              if (!b_res) {
                ptx::umma_commit_warp(&empty[s]);
                rp.next(args.stages);
              }
            }
            first = false;
            ptx::umma_commit_warp(&slot_free[b]);
            continue;
          }
          int tap_r = 0, tap_c = 0;
          for (int t = 0; t < win_taps; ++t) {
            uint32_t s = 0;
            if (!b_res) {
              s = rp.slot;
              ptx::mbar_wait(&full[s], rp.lap & 1);
              ptx::tc_fence_after();
            }
            const int dr = tap_r, dc = tap_c;  // (tap t = dr * S + dc, advanced below)
            if (++tap_c == args.S) {
              tap_c = 0;
              ++tap_r;
            }
            const uint64_t db = ptx::umma_desc_sw128_kmajor(ptx::smem_u32(
                smem + L.b_off + (b_res ? kb * win_taps + t : static_cast<int>(s)) * b_bytes));
            for (int q = 0; q < mt; ++q) {  // sub-tile q: pixel rows 16q .. 16q+15 of the block
              const uint32_t pix = static_cast<uint32_t>((16 * q + dr) * args.win_iw + dc);
              if (direct) {  // 128 B-swizzled pixel rows; K=16 steps are +32 B in the row
                const uint64_t da = ptx::umma_desc_sw128_kmajor_sbo(
                    cm + pix * 128, static_cast<uint32_t>(args.win_iw) * 128);
                if (ksteps == 4) {
                  ptx::umma_bf16_warp_k64(d + q * args.BN, da, db, idesc, first ? 0u : 1u);
                } else {
                  for (int k = 0; k < ksteps; ++k)
                    ptx::umma_bf16_warp(d + q * args.BN, da + 2 * k, db + 2 * k, idesc,
                                        first && k == 0 ? 0u : 1u);
                }
              } else {
                const uint64_t da = ptx::umma_desc_none_kmajor(cm + pix * 16, lbo, sbo);
                for (int k = 0; k < ksteps; ++k)  // next K=16 step: two chunk planes further
                  ptx::umma_bf16_warp(d + q * args.BN, da + static_cast<uint64_t>(2 * k) * (lbo >> 4),
                                 db + 2 * k, idesc, first && k == 0 ? 0u : 1u);
              }
            }
            first = false;
            if (!b_res) {
              ptx::umma_commit_warp(&empty[s]);
              rp.next(args.stages);
            }
          }
          ptx::umma_commit_warp(direct ? &slot_free[b] : &cm_empty[b]);
        }
        ptx::umma_commit_warp(&tmem_full[acc]);
      }
    }
    __syncwarp();
  } else {  // kMmaWarp: MMA issuer (whole warp: uniform descriptors, elected issue)
    // (pairs: the leader CTA's MMA warp issues for both; the peer's idles)
    if (!kPair || ptx::cluster_ctarank() == 0) {
      const uint32_t idesc = ptx::umma_idesc_bf16_f32(kPair ? 2 * kConvBM : kConvBM, args.BN);
      const uint32_t b_bytes = static_cast<uint32_t>(kPair ? args.BN / 2 : args.BN) * 128;
      if (args.b_res > 0) ptx::mbar_wait(b_full, 0);
      // operand descriptors = per-CTA bases + slot / sub-tile offsets in the
      // 16 B start-address units (addresses stay below 2^18, so the 14-bit
      // start field never carries)
      const uint64_t da_base = ptx::umma_desc_sw128_kmajor(ptx::smem_u32(smem + L.a_off));
      const uint64_t db_base = ptx::umma_desc_sw128_kmajor(ptx::smem_u32(smem + L.b_off));
      const uint64_t a_step = a_stage >> 4, b_step = b_bytes >> 4;
      uint32_t j = 0;
      RingPos rp;
      for (int tile = walk_first; tile < walk_count; tile += walk_stride, ++j) {
        const uint32_t acc = j & (n_acc - 1);
        if (j >= static_cast<uint32_t>(n_acc))
          ptx::mbar_wait(&tmem_empty[acc], ((j >> acc_log2) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem_base + acc * acc_stride;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          uint32_t s, use;
          if constexpr (kStem) {
            stem_slot(j, kb, args.num_kb, kGatherWarps / mt, s, use);
          } else {
            s = rp.slot;
            use = rp.lap;
            rp.next(args.stages);
          }
          ptx::mbar_wait(&full[s], use & 1);
          ptx::tc_fence_after();
          if (args.ts && kb == 0 && lane == 0 && j < 8) ts_mark(args.ts, 8 + j, ts0);
          const uint64_t db =
              db_base + static_cast<uint64_t>(args.b_res > 0 ? static_cast<uint32_t>(kb) : s) * b_step;
          const uint64_t da = da_base + static_cast<uint64_t>(s) * a_step;
          // the K block's four K=16 steps (+32 B in the swizzle row each), per sub-tile
          if constexpr (kPair) {
            ptx::umma_bf16_pair_k64(d, da, db, idesc, kb != 0);
            ptx::umma_commit_pair_warp(&empty[s], 3);  // both CTAs' slots
            continue;
          }
          if (mt == 2) {
            ptx::umma_bf16_warp_k64(d, da, db, idesc, kb != 0);
            ptx::umma_bf16_warp_k64(d + args.BN, da + (kABytes >> 4), db, idesc, kb != 0);
          } else {
            for (int q = 0; q < mt; ++q)
              ptx::umma_bf16_warp_k64(d + q * args.BN, da + static_cast<uint64_t>(q) * (kABytes >> 4),
                                      db, idesc, kb != 0);
          }
          ptx::umma_commit_warp(&empty[s]);
        }
        if constexpr (kPair)
          ptx::umma_commit_pair_warp(&tmem_full[acc], 3);
        else
          ptx::umma_commit_warp(&tmem_full[acc]);
        if (args.ts && lane == 0 && j < 8) ts_mark(args.ts, 16 + j, ts0);
      }
      if (args.ts && lane == 0) ts_mark(args.ts, 2, ts0);
    } else if constexpr (kPairG) {
      // peer CTA: forward each ring slot's gather completion (its 128 A rows
      // landed in this CTA's smem) to the leader's full barrier
      if (lane == 0) {
        RingPos rp;
        for (int tile = walk_first; tile < walk_count; tile += walk_stride)
          for (int kb = 0; kb < args.num_kb; ++kb, rp.next(args.stages)) {
            ptx::mbar_wait(&full[rp.slot], rp.lap & 1);
            ptx::fence_proxy_async_smem();  // (cp.async writes -> the leader's tensor-core reads)
            ptx::mbar_arrive_cluster(&full[rp.slot], 0);
          }
      }
    }
    __syncwarp();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (args.ts && threadIdx.x == 0) ts_mark(args.ts, 3, ts0);
  if (cl > 1) ptx::cluster_sync();  // no CTA leaves while its peer may still signal it
  if (warp == kTmaWarp) {
    ptx::tc_fence_after();
    if constexpr (kPair)
      ptx::tmem_dealloc_pair(tmem_base, args.tmem_cols);
    else
      ptx::tmem_dealloc(tmem_base, args.tmem_cols);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

EncodeIm2colFn get_encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
}

}  // namespace

bool encode_tmap_im2col(CUtensorMap* map, const void* base, int n, int h, int w, int c, int r, int s,
                        int stride_h, int stride_w, int pad_h, int pad_w) {
  EncodeIm2colFn fn = get_encode_im2col_fn();
  if (!fn || c % 64 != 0 || pad_h > 127 || pad_w > 127 || stride_h > 8 || stride_w > 8) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                              static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 2,
                                 static_cast<cuuint64_t>(c) * 2 * w,
                                 static_cast<cuuint64_t>(c) * 2 * w * h};
  // the window origins walk [-pad, extent + pad - filter] (W first, then H)
  const int lower[2] = {-pad_w, -pad_h};
  const int upper[2] = {pad_w - (s - 1), pad_h - (r - 1)};
  const cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(stride_w), static_cast<cuuint32_t>(stride_h), 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, lower,
            upper, 64u, static_cast<cuuint32_t>(kConvBM), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint64_t row_stride_elems, uint32_t box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_stride_elems * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kConvBK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tmap_out(CUtensorMap* map, void* base, uint64_t rows, uint64_t cols,
                     uint64_t row_stride_elems, bool f32) {
  EncodeTiledFn fn = get_encode_fn();
  const uint64_t esz = f32 ? 4 : 2;
  if (!fn || (row_stride_elems * esz) % 16 != 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0)
    return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_stride_elems * esz};
  const cuuint32_t box[2] = {f32 ? 32u : 64u, 32};  // one 128 B row per output row
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base,
            dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tmap_out_narrow(CUtensorMap* map, void* base, uint64_t rows, uint64_t cols,
                            uint64_t row_stride_elems) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn || (row_stride_elems * 2) % 16 != 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0)
    return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_stride_elems * 2};
  const cuuint32_t box[2] = {32u, 32u};  // one 64 B row per output row
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tmap_nhwc_sw32(CUtensorMap* map, const void* base, int n, int h, int w, int c,
                           int box_w, int box_h) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn || c % 16 != 0) return false;  // (boxes of 16 channels = one 32 B swizzle row)
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                              static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 2,
                                 static_cast<cuuint64_t>(c) * 2 * w,
                                 static_cast<cuuint64_t>(c) * 2 * w * h};
  const cuuint32_t box[4] = {16u, static_cast<cuuint32_t>(box_w),
                             static_cast<cuuint32_t>(box_h), 1u};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tmap_out4d(CUtensorMap* map, void* base, int n, int h, int w, int cols, int ld,
                       int box_w, int box_h) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn || (static_cast<uint64_t>(ld) * 2) % 16 != 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0)
    return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(w),
                              static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 2,
                                 static_cast<cuuint64_t>(ld) * 2 * w,
                                 static_cast<cuuint64_t>(ld) * 2 * w * h};
  const cuuint32_t box[4] = {64u, static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1u};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tmap_nhwc(CUtensorMap* map, const void* base, int n, int h, int w, int c, int box_c,
                      int box_w, int box_h, int box_n, bool sw128) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn || (static_cast<uint64_t>(c) * 2) % 16 != 0) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                              static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 2,
                                 static_cast<cuuint64_t>(c) * 2 * w,
                                 static_cast<cuuint64_t>(c) * 2 * w * h};
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(box_c), static_cast<cuuint32_t>(box_w),
                             static_cast<cuuint32_t>(box_h), static_cast<cuuint32_t>(box_n)};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

uint32_t conv_gemm_tmem_cols(int BN) {
  uint32_t c = 32;
  while (static_cast<int>(c) < 2 * BN) c <<= 1;  // two fp32 accumulators
  return c;
}

namespace {
uint32_t pow2_at_least(int x) {
  uint32_t c = 32;
  while (static_cast<int>(c) < x) c <<= 1;
  return c;
}
}  // namespace

int conv_gemm_stages(int BN, int cout, int epi_warps, int b_res_blocks, int mt, bool narrow) {
  const int ctas = 1;  // 18 warps: one CTA per SM
  const int per_stage = mt * kABytes + (b_res_blocks > 0 ? 0 : BN * kConvBK * 2);
  const int fixed =
      static_cast<int>(smem_layout(BN, 0, cout, epi_warps, b_res_blocks, mt, 0, narrow).total) + 64 * 8 + 1024;
  const int budget = (227 * 1024) / ctas - fixed;
  return std::max(1, std::min(kConvMaxStages, budget / per_stage));
}

size_t conv_gemm_smem_bytes(int BN, int stages, int cout, int epi_warps, int b_res_blocks, int mt,
                            bool narrow) {
  return smem_layout(BN, stages, cout, epi_warps, b_res_blocks, mt, 0, narrow).total + 1024;  // + alignment slack
}

// kWindow ring sizing (shared by the launcher and conv_gemm_window_ok).
bool window_rings(int R, int S, int C, int cout, int BN, int box_bytes, int& b_res, int& teams,
                  int& stages) {
  const int taps = R * S, cblocks = (C + 63) / 64;
  const int win = 4 * ((box_bytes + 1023) / 1024 * 1024);
  const int res_bytes = cblocks * taps * BN * 128;
  const int n_tiles = (cout + BN - 1) / BN;
  auto fits = [&](int res_blocks, int tm, int st) {
    const int total = static_cast<int>(smem_layout(BN, st, cout, 4 * tm, res_blocks, 0, box_bytes).total);
    (void)win;
    return total + 1024 <= 227 * 1024;
  };
  for (int tm = 2; tm >= 1; --tm) {
    if (n_tiles == 1 && fits(cblocks * taps, tm, 1)) {
      b_res = cblocks * taps, teams = tm, stages = 1;
      (void)res_bytes;
      return true;
    }
  }
  // (window ring stages carry one tap's weight tile only — no A sub-tile —
  // so the freed space buys ring depth: 28^2 3x3 128->128 at bs 256 95.7 ->
  // 66.8 us, 35^2 3x3 64->96 41.2 -> 28.2 us going from 2 to 6+ stages)
  for (int tm = 2; tm >= 1; --tm)
    for (int st = 8; st >= 2; --st)
      if (fits(0, tm, st)) {
        b_res = 0, teams = tm, stages = st;
        return true;
      }
  return false;
}

bool conv_gemm_window_ok(int r, int s, int c, int cout) {
  if (r * s < 2 || c % 16 != 0 || r > 9 || s > 9) return false;
  const int bn = cout <= 256 ? (cout + 15) / 16 * 16 : ((cout + (cout + 255) / 256 - 1) / ((cout + 255) / 256) + 63) / 64 * 64;
  const int cb = std::min(c, 64);
  const int box = (8 + s - 1) * (16 + r - 1) * cb * 2;
  int b_res, teams, stages;
  return window_rings(r, s, c, cout, bn, box, b_res, teams, stages);
}

bool conv_gemm_stem_fits(int R, int S, int cout) {
  // kernel-row / kernel-column masks are 16-bit fields; eight ring slots
  // (one per producer warp) with one epilogue team must fit in shared memory
  if (R > 15 || S > 15 || R * S > 64) return false;
  int bn = cout <= 256 ? (cout + 15) / 16 * 16 : 256;
  return conv_gemm_stages(bn, cout, 4, 0) >= kGatherWarps;
}

cudaError_t conv_gemm_init() {
  // Opt every instantiation into the full 227 KiB of dynamic shared memory
  // once, outside any stream capture.
  static cudaError_t status = [] {
    const int cap = 227 * 1024;
    cudaError_t e = cudaSuccess;
    for (auto* k : {conv_gemm_kernel<0>, conv_gemm_kernel<2>, conv_gemm_kernel<4>, conv_gemm_kernel<5>,
                    conv_gemm_kernel<6>, conv_gemm_kernel<7>, conv_gemm_kernel<10>, conv_gemm_kernel<11>,
                    conv_gemm_kernel<12>, conv_gemm_kernel<13>,
                    conv_gemm_kernel<14>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    return e;
  }();
  return status;
}

int conv_gemm_sm_count() {
  static int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return budgeted_sms(sms);
}

cudaError_t launch_conv_gemm(const ConvGemmArgs& in_args, ConvLoadMode mode, cudaStream_t stream) {
  // A store group (64 bf16 / 32 fp32 columns) must not straddle two N tiles.
  ConvGemmArgs args = in_args;
  args.span = launch_span();
  const bool pair = mode == ConvLoadMode::kPairTmaA || mode == ConvLoadMode::kPairIm2col ||
                    mode == ConvLoadMode::kPairGather;
  if (pair) {
    // CTA pairs: each CTA's B half is BN / 2 rows of 128 B swizzle atoms
    if (args.BN % 16 != 0 || args.BN > 256) return cudaErrorInvalidValue;
    args.cluster = 2;
  } else {
    args.cluster = 1;
  }
  const int group_cols = args.out_f32 ? 32 : 64;
  if (args.y_tma && args.Cout > args.BN && args.BN % group_cols != 0) args.y_tma = 0;
  if (args.nseg > 0 && (!args.y_tma || args.nseg > 4 || args.Cout > 64 * 64))
    return cudaErrorInvalidValue;  // (segments store by TMA, 64-column group tables)
  args.norelu_g = 0;
  for (int sg = 0; sg < args.nseg; ++sg)
    for (int g = args.seg_col[sg] / 64; g < args.seg_col[sg + 1] / 64; ++g) {
      args.seg_g[g] = static_cast<uint8_t>(sg);
      if ((args.seg_norelu >> sg) & 1) args.norelu_g |= 1ull << g;
    }
  // Sub-tiles per tile (TMA-A and stem modes): mt 128-row sub-tiles share
  // one ring stage, one accumulator (mt x BN columns) and one trip through
  // the barriers, amortising the per-tile MMA-issue / barrier latency that
  // bounds small-N layers.
  const int mt_stem = 4, mt_tma = 2, teams_tma = 4;
  const int mt_cap = mode == ConvLoadMode::kWindow ? std::max(1, in_args.mt)
                     : (mode == ConvLoadMode::kS2D || mode == ConvLoadMode::kS2DWide)
                         ? std::max(2, in_args.dw_th / 16)
                     : mode == ConvLoadMode::kStemU8 ? mt_stem
                     : (mode == ConvLoadMode::kTmaA || mode == ConvLoadMode::kIm2col) ? mt_tma
                                                   : 1;
  args.mt = 1;
  while (args.mt * 2 <= mt_cap && args.mt * 2 * static_cast<int>(pow2_at_least(args.BN)) <= 256)
    args.mt *= 2;
  // TMEM: as many accumulators as 512 columns hold (2..kMaxAcc), so the MMA
  // runs ahead of the epilogue; epilogue teams: 2, or 4 when the gather warps
  // are idle (TMA-A) and tiles are single small ones, never more than the
  // accumulators.
  const uint32_t acc_cols = pow2_at_least(args.mt * args.BN);
  args.n_acc = std::max(2, std::min(kMaxAcc, static_cast<int>(512 / acc_cols)));
  args.tmem_cols = pow2_at_least(args.n_acc * static_cast<int>(acc_cols));
  const bool tmaa = mode == ConvLoadMode::kTmaA || mode == ConvLoadMode::kIm2col;
  // (the gather modes' warps 8-15 produce A: at most two epilogue teams)
  const bool gather = mode == ConvLoadMode::kGather16 || mode == ConvLoadMode::kPairGather;
  const bool pair_t = pair && !gather;
  args.teams = std::min((tmaa || pair_t) && args.BN <= 64 ? teams_tma : kEpiWarps / 4,
                        args.n_acc);
  if (args.teams == 3) args.teams = 2;  // a power of two
  // wide TMA-A tiles with two accumulators: the idle gather warps join and
  // two teams split each tile's columns (DS_CONV_TPA=0: off)
  args.res_prefetch = 1;  // (epilogue L2 prefetch of this tile's residual rows)
  const bool tpa_on = [] {
    const char* e = std::getenv("DS_CONV_TPA");
    return !(e && e[0] == '0');
  }();
  if (tpa_on && (tmaa || pair_t) && args.BN >= 128 && args.n_acc == 2 &&
      args.BN % (2 * group_cols) == 0)
    args.teams = 4;
  args.tpa = (tmaa || pair_t) && args.teams > args.n_acc ? args.teams / args.n_acc : 1;
  // all four teams on one tile (tpa 4: each warp drains a quarter of the
  // tile's columns, half the per-warp slices of tpa 2); the other accumulator
  // keeps the MMA busy meanwhile. The epilogue's per-slice chain (TMEM load,
  // math, staging, fence, store: ~1300 cycles) is latency-bound, so more
  // warps per tile shorten it — but the sixteen warps' TMA stores then queue
  // behind each other (pw 28^2 -4 %, 56^2 +3 %): opt-in, DS_CONV_TPA4=1.
  {
    const char* e = std::getenv("DS_CONV_TPA4");
    if (e && e[0] == '1' && args.tpa == 2 && args.teams == 4 && args.BN % (4 * 32) == 0)
      args.tpa = 4;
  }
  // sixteen epilogue warps (one staging buffer each at 64-column groups):
  // store 32-column slices through a 64 B-swizzled map instead, two buffers
  // per warp (DS_Y_NARROW=0: off)
  args.y_narrow = 0;
  {
    // default: only residual layers (they stage their residual slices in the
    // narrow buffers); elsewhere the 64-column groups through one 4 KiB
    // buffer per warp issue half the TMA stores and measured 2-5 % faster
    // on MobileNet's 1x1s (DS_Y_NARROW=1: every sixteen-warp epilogue, 0: none)
    const char* e = std::getenv("DS_Y_NARROW");
    const bool on = e ? e[0] == '1' : args.residual != nullptr;
    const bool blk_mode = mode == ConvLoadMode::kWindow || mode == ConvLoadMode::kS2D ||
                          mode == ConvLoadMode::kS2DWide;
    if (on && args.y_tma && !args.out_f32 && !blk_mode && 4 * args.teams > 8) {
      CUtensorMap ty, tseg[4];
      bool ok = encode_tmap_out_narrow(&ty, static_cast<__nv_bfloat16*>(args.y) + args.c_off,
                                       static_cast<uint64_t>(args.M), static_cast<uint64_t>(args.Cout),
                                       static_cast<uint64_t>(args.ldy));
      for (int sg = 0; sg < args.nseg && ok; ++sg)
        ok = encode_tmap_out_narrow(&tseg[sg], args.seg_y[sg], static_cast<uint64_t>(args.M),
                                    static_cast<uint64_t>(args.seg_w[sg]), static_cast<uint64_t>(args.seg_ld[sg]));
      if (ok) {
        args.tmap_y = ty;
        for (int sg = 0; sg < args.nseg; ++sg) args.tmap_seg[sg] = tseg[sg];
        args.y_narrow = 1;
      }
    }
  }
  // ... and residual layers stage each residual slice into that buffer by TMA
  // (DS_RES_TMA=0: off)
  args.res_tma = 0;
  {
    const char* e = std::getenv("DS_RES_TMA");
    const bool on = !(e && e[0] == '0');
    if (on && args.y_narrow && args.residual && args.mt == 1 &&
        encode_tmap_out_narrow(&args.tmap_r, const_cast<__nv_bfloat16*>(args.residual),
                               static_cast<uint64_t>(args.M), static_cast<uint64_t>(args.Cout),
                               static_cast<uint64_t>(args.ld_res)))
      args.res_tma = 1;
  }
  // B resident in smem when the layer has one N tile and a small K: no
  // per-tile weight loads (and no TMA hop on the operand ring's critical path)
  const int n_tiles = (args.Cout + args.BN - 1) / args.BN;
  args.b_res = !pair && n_tiles == 1 && args.num_kb * args.BN * 128 <= 64 * 1024 ? args.num_kb : 0;
  args.stages = conv_gemm_stages(pair ? args.BN / 2 : args.BN, args.Cout, 4 * args.teams, args.b_res, args.mt,
                                 args.y_narrow != 0);
  if (mode == ConvLoadMode::kStemU8) {
    // one private slot per producer group (stem_slot); drop to one epilogue
    // team if that is what makes the slots fit
    const int groups = kGatherWarps / args.mt;
    if (args.stages < groups) {
      args.teams = 1;
      args.stages = conv_gemm_stages(args.BN, args.Cout, 4, args.b_res, args.mt);
    }
    if (args.stages < groups) return cudaErrorInvalidValue;
    args.stages = groups;
    if (args.taps > 64 || args.R > 15 || args.S > 15) return cudaErrorInvalidValue;
    for (int t = 0; t < 64; ++t) {
      const int r = t < args.taps ? t / args.S : 0, c = t < args.taps ? t % args.S : 0;
      args.tap_info[t] = ((r * args.W + c) * 3) | (r << 24) | (c << 28);
    }
  }
  const bool s2 = mode == ConvLoadMode::kS2D || mode == ConvLoadMode::kS2DWide;
  if (s2) {
    // pixel blocks of dw_th x 8 (one halo box each) = dw_th / 16 128-row
    // sub-tiles; all weights resident
    args.mt = args.dw_th / 16;
    if (args.mt != 2 && args.mt != 4) return cudaErrorInvalidValue;
    if (!args.y_tma || n_tiles != 1 || args.num_kb * args.BN * 128 > 64 * 1024)
      return cudaErrorInvalidValue;
    args.b_res = args.num_kb;
    // no producer warps: all sixteen non-TMA/MMA warps drain accumulators
    // (four epilogue teams) when their staging still leaves a 2-deep ring
    if (args.n_acc >= 4 && conv_gemm_stages(args.BN, args.Cout, 16, args.b_res, 2) >= 2) args.teams = 4;
    // (ring stage = 2 sub-tiles: C / 16 boxes, 1 KiB apart)
    if ((args.C != 16 && args.C != 32) ||
        static_cast<uint32_t>(args.C / 16) * ((args.win_box_bytes + 1023) / 1024 * 1024) > 2u * kABytes)
      return cudaErrorInvalidValue;
    args.stages = std::min(6, conv_gemm_stages(args.BN, args.Cout, 4 * args.teams, args.b_res, 2));
    if (args.stages < 2) return cudaErrorInvalidValue;
  }
  const bool win = mode == ConvLoadMode::kWindow;
  if (win) {
    // rings: 2 pixel-major + 2 chunk-major halo boxes; weights resident when
    // every (K block, tap) tile fits, else streamed per tap; staging for the
    // 4-D TMA-store epilogue
    if (!args.y_tma) return cudaErrorInvalidValue;
    if (!window_rings(args.R, args.S, args.C, args.Cout, args.BN, static_cast<int>(args.win_box_bytes),
                      args.b_res, args.teams, args.stages))
      return cudaErrorInvalidValue;
  }
  const size_t smem =
      win ? smem_layout(args.BN, args.stages, args.Cout, 4 * args.teams, args.b_res, 0,
                        static_cast<int>(args.win_box_bytes)).total + 1024
          : conv_gemm_smem_bytes(pair ? args.BN / 2 : args.BN, args.stages, args.Cout, 4 * args.teams,
                                 args.b_res, s2 ? 2 : args.mt, args.y_narrow != 0);
  const int tiles = win || s2 ? n_tiles * (args.M / (args.Ho * args.Wo)) * args.dw_tiles_y * args.dw_tiles_x
                              : n_tiles * ((args.M + kConvBM * args.mt - 1) / (kConvBM * args.mt));
  // Resident CTAs per SM: shared memory and TMEM columns (512 per SM) decide.
  const int by_smem = static_cast<int>((227 * 1024) / smem);
  const int by_tmem = static_cast<int>(512 / args.tmem_cols);
  const int per_sm = std::max(1, std::min(by_smem, by_tmem));
  if (std::getenv("DS_CONV_DEBUG"))  // bring-up: the launch's derived configuration
    std::fprintf(stderr,
                 "conv_gemm mode %d: BN %d mt %d stages %d b_res %d teams %d tpa %d n_acc %d smem %zu "
                 "per_sm %d tiles %d\n",
                 static_cast<int>(mode), args.BN, args.mt, args.stages, args.b_res, args.teams, args.tpa,
                 args.n_acc, smem, per_sm, tiles);
  if (pair) {  // CTA pairs over (M-block pair, N block) units
    if (args.mt != 1) return cudaErrorInvalidValue;
    const int m_blocks = (args.M + kConvBM - 1) / kConvBM;
    const int units = n_tiles * ((m_blocks + 1) / 2);
    const int ctas = std::min(2 * units, conv_gemm_sm_count() * per_sm) / 2 * 2;
    auto* k = mode == ConvLoadMode::kPairIm2col   ? conv_gemm_kernel<13>
              : mode == ConvLoadMode::kPairGather ? conv_gemm_kernel<14>
                                                  : conv_gemm_kernel<7>;
    return launch_pdl_cluster(k, dim3(ctas), dim3(kConvThreads), smem, stream, 2, args);
  }
  const dim3 grid(std::min(tiles, conv_gemm_sm_count() * per_sm));
  switch (mode) {
    case ConvLoadMode::kGather16:
      return launch_pdl(conv_gemm_kernel<0>, grid, dim3(kConvThreads), smem, stream, args);
    case ConvLoadMode::kTmaA:
      return launch_pdl(conv_gemm_kernel<2>, grid, dim3(kConvThreads), smem, stream, args);
    case ConvLoadMode::kStemU8:
      return launch_pdl(conv_gemm_kernel<4>, grid, dim3(kConvThreads), smem, stream, args);
    case ConvLoadMode::kWindow:
      if (!args.win_direct)
        return launch_pdl(conv_gemm_kernel<11>, grid, dim3(kConvThreads), smem, stream, args);
      return launch_pdl(conv_gemm_kernel<5>, grid, dim3(kConvThreads), smem, stream, args);
    case ConvLoadMode::kS2D:
      return launch_pdl(conv_gemm_kernel<6>, grid, dim3(kConvThreads), smem, stream, args);
    case ConvLoadMode::kS2DWide:
      return launch_pdl(conv_gemm_kernel<10>, grid, dim3(kConvThreads), smem, stream, args);
    case ConvLoadMode::kIm2col:
      return launch_pdl(conv_gemm_kernel<12>, grid, dim3(kConvThreads), smem, stream, args);
    default:
      return cudaErrorInvalidValue;  // (kWindowT is selected through kWindow + win_direct = 0)
  }
}

}  // namespace ds
