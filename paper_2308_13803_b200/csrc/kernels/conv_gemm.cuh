// Host-facing description of one implicit-GEMM convolution launch (K1/K2/K5
// in DESIGN.md). Shared by the runtime (which plans launches per layer and
// batch size) and the kernel translation unit.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace ds {

constexpr int kConvBM = 128;       // UMMA M: output pixels per tile
constexpr int kConvBK = 64;        // K elements per pipeline stage (one 128 B swizzle row)
// Persistent CTA (one per SM): 8 epilogue warps, 8 gather warps, 1 TMA
// warp, 1 MMA warp.
constexpr int kConvThreads = 576;
constexpr int kConvMaxStages = 8;
constexpr int kConvSmemBudget = 200 * 1024;  // operand ring budget per CTA (1 CTA / SM)

// One conv (or FC, as a 1x1 conv over a 1x1 image) as a GEMM
//   Y[m, n] = act( sum_k A[m, k] * Wt[n, k] + bias[n] (+ R[m, n]) )
// with m = (image, ho, wo), k = (r, s, c) flattened in that order (KRSC
// weights), A gathered from the NHWC input on the fly.
struct ConvGemmArgs {
  // Scalars first, the ones every tile / epilogue slice reads at the front:
  // kernel parameters live in the constant bank, and with the tensor maps
  // (1 KB+) between them the hot fields spread over many constant-cache lines
  // and missed on every epilogue slice.
  int M;       // images * Ho * Wo
  int Cout, BN;
  int mt;      // 128-row sub-tiles per tile (TMA-A / stem modes; launch_conv_gemm sets it)
  // Epilogue teams (4 warps each, one per TMEM lane quarter) and TMEM
  // accumulators: tile j goes to accumulator j % n_acc and team j % teams
  // (n_acc a multiple of teams, so each accumulator has one team). Set by
  // launch_conv_gemm from the mode and BN.
  int teams, n_acc;
  int tpa;     // teams per tile (sharing its columns); teams / tpa tiles drain at once
  int y_tma;           // epilogue stores through smem + TMA (else direct stores)
  int y_narrow;        // tmap_y has 32 x 32 boxes, 64 B swizzle (launch_conv_gemm sets it)
  int res_tma;         // epilogue stages residual slices by TMA (launch_conv_gemm sets it)
  int out_f32, relu;
  int ldy, c_off;  // output row stride (channels) and channel offset (concat slices)
  int ld_res;
  int nseg;        // fused sibling segments (below; 0: none)
  int debug_flags;  // bring-up experiments only (tools/test_conv_gemm): 1 = no epilogue
  unsigned long long norelu_g;  // bit g: no ReLU on 64-column group g (from seg_norelu)
  const float* bias;
  const __nv_bfloat16* residual;
  void* y;
  // bring-up timeline (tools/test_conv_gemm TS=1): per CTA 64 clock64 stamps
  // relative to kernel entry, see conv_gemm.cu ts_mark(); nullptr in the runtime
  unsigned long long* ts;
  int res_prefetch;  // epilogue L2 prefetch of residual rows (launch_conv_gemm sets it)
  int num_kb;  // ceil(R*S*C / 64)
  int stages;
  uint32_t tmem_cols;
  int b_res;  // > 0: all num_kb weight blocks resident in smem (one N tile)
  int cluster;  // 2 = CTA pairs (kPairTmaA; launch_conv_gemm sets it): tmap_b box rows
                // are then BN / 2 (each CTA loads its half of every weight block)
  const __nv_bfloat16* x;
  int H, W, C;  // input spatial dims; C = channels per pixel (row stride)
  int R, S, stride_h, stride_w, pad_h, pad_w;
  int Ho, Wo;
  int taps;    // R*S
  // Fused sibling 1x1 convs (model.hpp fuse_sibling_1x1): nseg > 0 splits
  // the N columns into segments [seg_col[s], seg_col[s + 1]) (multiples of
  // 64), each stored through tmap_seg[s] into its own buffer / channel slice
  // (clipped at its real width seg_w[s]); bit s of seg_norelu: no ReLU.
  int seg_col[5];
  int seg_norelu;
  uint8_t seg_g[64];            // segment of 64-column group g
  void* seg_y[4];  // (host: segment bases, widths and row strides for re-encoding)
  int seg_w[4], seg_ld[4];
  unsigned long long* span;  // live per-kernel timing slot (pdl.cuh span_mark), or nullptr
  // Pixel-block tiles (kWindow, kS2D, kS2DWide): dw_th x dw_tw output pixels
  // of one image, dw_tiles_y x dw_tiles_x blocks per image; epilogue warp q
  // stores pixel rows q*dw_rw .. (TMEM lane l <-> pixel (q*rw + l/tw, l%tw)).
  int dw_th, dw_tw, dw_tiles_y, dw_tiles_x;
  int dw_rw;
  // kWindow (stride-1 R x S conv, no im2col): tiles are 16 x 8 output-pixel
  // blocks; per 64-channel K block
  // the TMA lands the halo box {min(64, C), win_iw, win_ih} (pixel-major), the
  // gather warps transpose it to chunk-major (16 B channel chunks x pixels),
  // and every tap (r, s) is one MMA operand read straight out of that box
  // at pixel offset r*win_iw + s (K-major, no swizzle).
  int win_iw, win_ih;
  uint32_t win_box_bytes;
  int win_direct;  // 1: C % 64 == 0, the 128 B-swizzled pixel-major box is read in place
                   // (4 box slots, no transpose); 0: transposed to chunk-major
  // kStemU8: A gathered straight from the u8 images [n][H][W][3]; the
  // staging normalisation x = bf16((p - 127.5) / 63.75) happens in the
  // producer (C = 4 logical channels, the 4th zero, as in the staged layout).
  const uint8_t* img;
  // Tensor maps (64 B aligned, read by the TMA unit through their addresses)
  CUtensorMap tmap_b;  // weights [Cout][Kpad] bf16, box {64, BN}, 128 B swizzle
  CUtensorMap tmap_a;  // input viewed as [rows][C] (1x1 stride-1 convs only)
  CUtensorMap tmap_y;  // output slice [rows][Cout] at y + c_off, 128 B x 32-row boxes (y_tma)
  CUtensorMap tmap_r;  // residual with the same 32 x 32 boxes (res_tma)
  CUtensorMap tmap_seg[4];
  // kStemU8 tap table (launch_conv_gemm fills it): tap t = r*S + s ->
  // byte offset (r*W + s)*3 | r << 24 | s << 28
  int tap_info[64];
};

enum class ConvLoadMode : int {
  kGather16 = 0,  // cp.async gather, 8 channels (16 B) per granule, C % 8 == 0
  kTmaA = 2,      // 1x1 stride-1 conv: A is a plain 2D tile, loaded by TMA
  kStemU8 = 4,    // stem conv over the u8 images, input staging fused into the producer
  kWindow = 5,    // stride-1 R x S conv as shifted-window MMAs over a per-K-block halo box
  kS2D = 6,       // stride-2 stem over its space-to-depth input: one 32 B-swizzled halo box
                  // per pixel block, every tap an MMA window of it; no producer warps
  kPairTmaA = 7,  // kTmaA on CTA pairs: one M = 256 cta_group::2 MMA per K step, each CTA
                  // loading its 128 A rows and half of the B block (tmap_b box rows BN / 2)
  kS2DWide = 10,  // kS2D window MMAs for 16 / 32-channel stride-1 3x3 convs (one halo box
                  // per 16-channel block, padding as negative box coordinates)
  kWindowT = 11,  // (internal) kWindow with transposed boxes: launch as kWindow, win_direct 0
  kIm2col = 12,   // R x S / strided convs with C % 64 == 0: A blocks by TMA im2col loads
                  // (tmap_a from encode_tmap_im2col), then the TMA-A pipeline
  kPairGather = 14,  // kGather16 on CTA pairs (the peer's gather completion is forwarded to
                     // the leader's full barrier by its otherwise idle MMA warp)
  kPairIm2col = 13,  // kIm2col on CTA pairs (cta_group::2 M = 256 MMAs, each CTA loading
                     // its 128 output pixels' im2col A block and half of the B block)
};

// Im2col map over an NHWC bf16 activation for an R x S conv (stride, padding):
// 64-channel x 128-output-pixel blocks, 128 B swizzle.
bool encode_tmap_im2col(CUtensorMap* map, const void* base, int n, int h, int w, int c, int r, int s,
                        int stride_h, int stride_w, int pad_h, int pad_w);

// Encodes a 2D bf16 tensor map [rows][cols] (cols contiguous, row stride in
// elements) with a {64, box_rows} box and 128 B swizzle.
bool encode_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                         uint64_t row_stride_elems, uint32_t box_rows);

// Output map for the TMA-store epilogue: [rows][cols] bf16 or fp32 starting
// at `base` (the channel slice), row stride in elements, boxes of 32 rows x
// 128 B (64 bf16 / 32 fp32 columns) with 128 B swizzle. False when TMA
// cannot address it (row stride or base not 16 B aligned).
bool encode_tmap_out(CUtensorMap* map, void* base, uint64_t rows, uint64_t cols,
                     uint64_t row_stride_elems, bool f32);

// The same for bf16 with 32-column x 32-row boxes and 64 B swizzle (the
// double-buffered 2 KiB staging of sixteen-warp epilogues).
bool encode_tmap_out_narrow(CUtensorMap* map, void* base, uint64_t rows, uint64_t cols,
                            uint64_t row_stride_elems);

// NHWC bf16 activation as a 4-D map {C, W, H, N} with a {box_c, box_w,
// box_h, 1} box, no swizzle (used by the depthwise halo loads). Negative or
// past-the-edge box coordinates read zeros (the convolution's padding).
bool encode_tmap_nhwc(CUtensorMap* map, const void* base, int n, int h, int w, int c, int box_c,
                      int box_w, int box_h, int box_n = 1, bool sw128 = false);

size_t conv_gemm_smem_bytes(int BN, int stages, int cout, int epi_warps = 8, int b_res_blocks = 0,
                            int mt = 1, bool narrow = false);

// kStemU8 needs eight operand-ring slots (one per producer warp) next to one
// epilogue team; false when this stem cannot have them (the runtime then
// stages the input).
bool conv_gemm_stem_fits(int R, int S, int cout);

// Operand-ring depth for an N tile: as deep as kConvMaxStages allows within
// the per-CTA budget, where two CTAs share an SM whenever their TMEM
// (2 x BN accumulator columns each) fits.
int conv_gemm_stages(int BN, int cout, int epi_warps = 8, int b_res_blocks = 0, int mt = 1,
                     bool narrow = false);
uint32_t conv_gemm_tmem_cols(int BN);

// Whether a conv runs as kWindow: stride 1, R*S > 1, C % 16 == 0, and the
// operand rings fit in shared memory next to the epilogue staging.
bool conv_gemm_window_ok(int r, int s, int c, int cout);

// 4-D NHWC bf16 map (c a multiple of 16) with a {16, box_w, box_h, 1} box and
// 32 B swizzle: the kS2D A boxes (one per 16-channel block).
bool encode_tmap_nhwc_sw32(CUtensorMap* map, const void* base, int n, int h, int w, int c,
                           int box_w, int box_h);

// 4-D output map {C, W, H, N} over an NHWC activation (channel slice at
// `base`, row stride ld channels) with a {64, box_w, box_h, 1} box and 128 B
// swizzle: the pixel-block epilogues store each warp's pixel rows with it.
bool encode_tmap_out4d(CUtensorMap* map, void* base, int n, int h, int w, int cols, int ld,
                       int box_w, int box_h);

// Must run once per device before the first launch (and before any capture).
cudaError_t conv_gemm_init();

cudaError_t launch_conv_gemm(const ConvGemmArgs& args, ConvLoadMode mode, cudaStream_t stream);

}  // namespace ds
