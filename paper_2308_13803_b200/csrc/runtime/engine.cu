#include "engine.hpp"

#include <cstdio>
#include <string>
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "../kernels/pdl.cuh"
#include "../kernels/stream_ops.cuh"

namespace ds {

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int round_up(int x, int a) { return (x + a - 1) / a * a; }

// N tile: one tile when Cout fits in 256 (UMMA N <= 256, multiple of 16),
// otherwise the smallest even split in multiples of 64, so the epilogue's
// 64-column TMA store boxes never cross into the neighbouring N tile.
int choose_bn(int cout) {
  if (cout <= 256) return round_up(cout, 16);
  const int n = (cout + 255) / 256;
  return round_up((cout + n - 1) / n, 64);
}

// The operand ring spans tiles (persistent kernel), so it is sized by the
// shared-memory budget, not by the layer's K.
int choose_stages(int bn, int cout) { return conv_gemm_stages(bn, cout); }

uint32_t tmem_cols_for(int bn) { return conv_gemm_tmem_cols(bn); }

// DS_CONV_PAIR: TMA-A layers whose weights stream (not resident) run on CTA
// pairs with M = 256 cta_group::2 MMAs, each CTA staging half of every B
// block (a third less shared-memory traffic per MMA at 128 x 256 tiles).
// 1 (default): BN >= 128; 0: off.
bool pair_on(int bn) {
  const int m = [] {
    const char* e = std::getenv("DS_CONV_PAIR");
    return e ? std::atoi(e) : 1;
  }();
  return m == 1 && bn >= 128;
}

// 1x1s with K <= 64 and several N tiles are bound by their output stores,
// not by weight traffic: single-CTA 128-column tiles (two 128-row sub-tiles
// per tile, all sixteen epilogue warps) beat CTA-pair 192-column tiles —
// ResNet's fused 56^2 64 -> 64 + 256 at bs 256: 152 -> 116 us
// (tools/test_conv_gemm). DS_CONV_K64_BN128=0: off (A/B).
bool k64_bn128_on(int num_kb, int cout) {
  const char* e = std::getenv("DS_CONV_K64_BN128");
  return !(e && e[0] == '0') && num_kb == 1 && cout > 256;
}

// Gather (and opt-in TMA im2col) convs on CTA pairs: M = 256 pair MMAs, each
// CTA gathering its own 128 A rows and staging half of every weight block
// (kPairGather; the peer's gather completion is forwarded to the leader).
// Half the weight traffic and shared-memory writes per MMA: ResNet-50's
// 3x3s at bs 256 77 -> 68 us (28^2), 51 -> 45 (14^2), 62 -> 54 (7^2).
// Off with DS_CONV_PAIR=0 (all pairs) or DS_CONV_PAIR_GATHER=0.
bool pair_gather_on(int bn) {
  const char* p = std::getenv("DS_CONV_PAIR");
  const char* e = std::getenv("DS_CONV_PAIR_GATHER");
  return !(p && p[0] == '0') && !(e && e[0] == '0') && bn >= 64 && bn <= 256 && bn % 16 == 0;
}

// Stride-1 R x S convs as kWindow (shifted-window MMAs, no im2col). Default:
// only where the halo box is read in place (C % 64 == 0) and the map is at
// least 56 x 56: ResNet's 56^2 3x3s run in half the pair gather's time; at
// 28^2 / 35^2 the window ties or wins per layer (64.2 vs 64.5 us, 26.6 vs
// 32.2 us) but the power-capped networks do not move, and below that the
// 16 x 8 tiles waste too many rows; with the transposed (C % 64 != 0) boxes
// the gather is always faster.
// DS_CONV_WINDOW_MIN overrides the map side.
// DS_CONV_WINDOW=1: every eligible conv; DS_CONV_WINDOW=0: none (A/B).
int window_mode() {
  const int m = [] {
    const char* e = std::getenv("DS_CONV_WINDOW");
    return e ? (e[0] == '1' ? 1 : 0) : 2;
  }();
  return m;
}

// DS_CONV_NARROW=0: 16/32-channel stride-1 3x3 convs back on the im2col
// gather (A/B); default: as kS2D window MMAs.
bool narrow_window_on() {
  const char* e = std::getenv("DS_CONV_NARROW");
  return !(e && e[0] == '0');
}

// TMA im2col A loads for convs with C % 64 == 0 on maps of at least 28 x 28
// (opt-in, DS_CONV_IM2COL=1): since the gather's per-K-block address math
// went incremental and the gather runs on CTA pairs, the cp.async gather is
// faster on every map size (ResNet 28^2 3x3 at bs 256: 68 vs 88 us; the TMA
// unit's per-pixel im2col walk bounds the im2col mode).
bool im2col_on() {
  const char* e = std::getenv("DS_CONV_IM2COL");
  return e && e[0] == '1';
}

bool window_on(int c, int ho, int wo) {
  const int m = window_mode();
  const char* e = std::getenv("DS_CONV_WINDOW_MIN");  // smallest map side (A/B)
  const int min_side = e ? std::atoi(e) : 56;
  return m == 1 || (m == 2 && c % 64 == 0 && ho >= min_side && wo >= min_side);
}

}  // namespace

// ------------------------------------------------------------------ Instance

Instance::Instance(const ModelSpec& m, int max_bs, int device)
    : m_(m), max_bs_(max_bs), device_(device) {
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  check_cuda(conv_gemm_init(), "conv_gemm_init");
  check_cuda(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  cur_stream_ = stream_;
  const HostParams& hp = params_for(m);

  size_t off = 0;
  auto take = [&off](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t w_off = take(hp.w.size() * sizeof(uint16_t));
  const size_t b_off = take(hp.b.size() * sizeof(float));
  const size_t img_off = take(static_cast<size_t>(max_bs) * m.in_h * m.in_w * 3);
  const size_t img2_off = take(static_cast<size_t>(max_bs) * m.in_h * m.in_w * 3);
  std::vector<size_t> buf_off;
  for (const auto& b : m.buffers)
    buf_off.push_back(
        take(static_cast<size_t>(max_bs) * b.h * b.w * b.c * (b.f32 ? sizeof(float) : 2)));
  const size_t probs_off = take(static_cast<size_t>(max_bs) * m.classes * sizeof(float));
  // fused sibling 1x1 convs: concatenated weights / biases, each sibling's
  // rows padded to a multiple of 64 (its store group never straddles two)
  auto seg_rows = [&](int param) { return round_up(m.params.at(param).cout, 64); };
  std::vector<size_t> fw_off(m.ops.size(), 0), fb_off(m.ops.size(), 0);
  // zeros for bias-free convs (swap_avgpool_1x1: their bias is added after the pool)
  const size_t zero_bias_off = take(4096 * sizeof(float));
  for (size_t i = 0; i < m.ops.size(); ++i) {
    const OpSpec& op = m.ops[i];
    if (op.fused.empty()) continue;
    int rows = seg_rows(op.param);
    for (const auto& f : op.fused) rows += seg_rows(f.param);
    fw_off[i] = take(static_cast<size_t>(rows) * hp.kpad.at(op.param) * 2);
    fb_off[i] = take(static_cast<size_t>(rows) * sizeof(float));
  }
  s2d_ = stem_s2d(m);
  size_t s2d_off = 0, stem_w_off = 0;
  if (s2d_.op >= 0) {
    s2d_off = take(static_cast<size_t>(max_bs) * s2d_.hs * s2d_.ws * 16 * 2);
    stem_w_off = take(static_cast<size_t>(m.params[m.ops[s2d_.op].param].cout) * s2d_.kpad * 2);
  }
  device_bytes_ = off;
  check_cuda(cudaMalloc(&d_arena_, off), "cudaMalloc(instance arena)");
  uint8_t* base = static_cast<uint8_t*>(d_arena_);
  check_cuda(cudaMemsetAsync(d_arena_, 0, off, stream_), "cudaMemset");
  d_w_ = reinterpret_cast<uint16_t*>(base + w_off);
  d_b_ = reinterpret_cast<float*>(base + b_off);
  d_images_[0] = base + img_off;
  d_images_[1] = base + img2_off;
  if (s2d_.op >= 0) {
    // stem weights for the s2d taps: W'[co][(dr*ds + dc)*16 + (a*2 + b)*4 + c] =
    // W[co][(2dr+a)*S + (2dc+b)][c] (zero where 2dr+a >= R or 2dc+b >= S)
    d_s2d_ = reinterpret_cast<__nv_bfloat16*>(base + s2d_off);
    d_stem_w_ = reinterpret_cast<__nv_bfloat16*>(base + stem_w_off);
    const OpSpec& op = m.ops[s2d_.op];
    const ParamSpec& p = m.params[op.param];
    const int kpad0 = hp.kpad.at(op.param);
    std::vector<uint16_t> w2(static_cast<size_t>(p.cout) * s2d_.kpad, 0);
    for (int co = 0; co < p.cout; ++co)
      for (int r = 0; r < op.r; ++r)
        for (int q = 0; q < op.s; ++q)
          for (int c = 0; c < 4; ++c) {
            const int k0 = (r * op.s + q) * 4 + c;
            const int k1 = ((r / 2) * s2d_.ds + q / 2) * 16 + ((r % 2) * 2 + q % 2) * 4 + c;
            w2[static_cast<size_t>(co) * s2d_.kpad + k1] =
                hp.w[hp.w_off.at(op.param) + static_cast<size_t>(co) * kpad0 + k0];
          }
    // (on stream_, after the arena memset; synchronised before w2 goes away)
    check_cuda(cudaMemcpyAsync(d_stem_w_, w2.data(), w2.size() * 2, cudaMemcpyHostToDevice, stream_),
               "upload s2d stem weights");
    check_cuda(cudaStreamSynchronize(stream_), "upload s2d stem weights");
  }
  check_cuda(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  check_cuda(cudaStreamCreateWithFlags(&out_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  for (int s = 0; s < 2; ++s) {
    check_cuda(cudaEventCreateWithFlags(&slot_free_[s], cudaEventDisableTiming), "event");
    check_cuda(cudaEventCreateWithFlags(&h2d_done_[s], cudaEventDisableTiming), "event");
    check_cuda(cudaEventCreateWithFlags(&out_ready_[s], cudaEventDisableTiming), "event");
    check_cuda(cudaEventCreateWithFlags(&out_read_[s], cudaEventDisableTiming), "event");
    check_cuda(cudaMalloc(&d_out_[s], static_cast<size_t>(max_bs) * m.classes * sizeof(float)),
               "cudaMalloc logits slot");
  }
  for (size_t o : buf_off) bufs_.push_back(base + o);
  d_probs_ = reinterpret_cast<float*>(base + probs_off);
  d_logits_ = static_cast<float*>(bufs_.at(m.logits));
  check_cuda(cudaMemcpyAsync(d_w_, hp.w.data(), hp.w.size() * sizeof(uint16_t),
                             cudaMemcpyHostToDevice, stream_),
             "upload weights");
  check_cuda(cudaMemcpyAsync(d_b_, hp.b.data(), hp.b.size() * sizeof(float),
                             cudaMemcpyHostToDevice, stream_),
             "upload biases");

  for (size_t i = 0; i < m.ops.size(); ++i) {
    const OpSpec& op = m.ops[i];
    if (op.fused.empty()) continue;
    const int kpad = hp.kpad.at(op.param);
    std::vector<int> params{op.param};
    std::vector<char> nob{op.no_bias};
    for (const auto& f : op.fused) {
      params.push_back(f.param);
      nob.push_back(f.no_bias);
    }
    int rows = 0;
    for (int p : params) rows += seg_rows(p);
    std::vector<uint16_t> w(static_cast<size_t>(rows) * kpad, 0);
    std::vector<float> b(rows, 0.0f);
    int r0 = 0;
    for (size_t k = 0; k < params.size(); ++k) {
      const int p = params[k];
      if (hp.kpad.at(p) != kpad) throw std::logic_error("fused 1x1 siblings with different K");
      const int co = m.params[p].cout;
      std::copy(hp.w.begin() + hp.w_off.at(p), hp.w.begin() + hp.w_off.at(p) + static_cast<size_t>(co) * kpad,
                w.begin() + static_cast<size_t>(r0) * kpad);
      if (!nob[k])  // (bias-free segments keep zeros)
        std::copy(hp.b.begin() + hp.b_off.at(p), hp.b.begin() + hp.b_off.at(p) + co, b.begin() + r0);
      r0 += seg_rows(p);
    }
    check_cuda(cudaMemcpyAsync(base + fw_off[i], w.data(), w.size() * 2, cudaMemcpyHostToDevice, stream_),
               "upload fused weights");
    check_cuda(cudaMemcpyAsync(base + fb_off[i], b.data(), b.size() * 4, cudaMemcpyHostToDevice, stream_),
               "upload fused biases");
    check_cuda(cudaStreamSynchronize(stream_), "upload fused weights");
  }
  plans_.resize(m.ops.size());
  stem_ = fused_stem(m);
  if (stem_ < 0 && s2d_.op < 0)
    throw std::logic_error("stem conv neither stride-2 (space-to-depth) nor a fused u8 stem");
  kernels_per_forward_ = stem_ >= 0 ? 1 : 2;  // (s2d staging +) softmax
  for (size_t i = 0; i < m.ops.size(); ++i) {
    const OpSpec& op = m.ops[i];
    ++kernels_per_forward_;
    if (op.kind == OpKind::kDwConv) {
      const BufferSpec& din = m.buffers.at(op.in);
      dw_maps_.resize(m.ops.size());
      if (!dwconv_tma_plan_ok(din.h, din.w, din.c, op.sh) ||
          !dwconv_tma_input_map(&dw_maps_[i], bufs_[op.in], max_bs, din.h, din.w, din.c, op.sh))
        throw CudaError("depthwise layer without a TMA plan (dwconv_tma.cu)");
    }
    if (op.kind == OpKind::kMaxPool || op.kind == OpKind::kAvgPool) {
      // TMA halo-box pooling (pool_tma.cu). A padded max pool reads its edge
      // taps as zeros there, so it qualifies only when its input is a ReLU
      // output (every input >= 0): the producer of op.in must apply ReLU.
      const BufferSpec& pin = m.buffers.at(op.in);
      bool relu_input = false;
      for (size_t j = 0; j < i; ++j) {
        if (m.ops[j].out == op.in) relu_input = m.ops[j].relu;
        for (const auto& f : m.ops[j].fused)
          if (f.out == op.in) relu_input = f.relu;
      }
      const char* legacy = std::getenv("DS_POOL_TMA");
      const bool allow = !(legacy && legacy[0] == '0');
      pool_maps_.resize(m.ops.size());
      pool_tma_.resize(m.ops.size(), false);
      pool_tma_[i] = allow && (op.kind == OpKind::kAvgPool || op.ph == 0 || relu_input) &&
                     pool_tma_input_map(&pool_maps_[i], bufs_[op.in], max_bs, pin.h, pin.w, pin.c,
                                        op.sh, op.ph);
    }
    if (op.kind != OpKind::kConv && op.kind != OpKind::kFc) continue;
    const ParamSpec& p = m.params.at(op.param);
    const BufferSpec& in = m.buffers.at(op.in);
    const BufferSpec& out = m.buffers.at(op.out);
    ConvPlan& pl = plans_[i];
    ConvGemmArgs& a = pl.args;
    std::memset(&a, 0, sizeof(a));
    a.x = static_cast<const __nv_bfloat16*>(bufs_[op.in]);
    a.H = in.h;
    a.W = in.w;
    a.C = in.c;
    a.R = op.r;
    a.S = op.s;
    a.stride_h = op.sh;
    a.stride_w = op.sw;
    a.pad_h = op.ph;
    a.pad_w = op.pw;
    pl.ho = a.Ho = out.h;
    pl.wo = a.Wo = out.w;
    if (op.kind == OpKind::kFc) {
      a.H = a.W = 1;
      a.Ho = a.Wo = pl.ho = pl.wo = 1;
    }
    const int kpad = hp.kpad.at(op.param);
    a.num_kb = kpad / kConvBK;
    a.taps = op.r * op.s;
    a.Cout = p.cout;
    // FC heads have one or two M tiles at serving batch sizes: narrow N tiles
    // spread their long K loop over 63 SMs (N = 16: MobileNet's FC 8.9 -> 7.9
    // us at bs 128 against N = 64; DS_FC_BN = 16 / 32 / 64 / 128)
    const int fc_bn = [] {
      const char* e = std::getenv("DS_FC_BN");
      const int v = e ? std::atoi(e) : 16;
      return (v == 16 || v == 32 || v == 64 || v == 128) ? v : 16;
    }();
    a.BN = op.kind == OpKind::kFc ? fc_bn : choose_bn(p.cout);
    a.stages = choose_stages(a.BN, p.cout);
    a.tmem_cols = tmem_cols_for(a.BN);
    a.bias = op.no_bias ? reinterpret_cast<const float*>(base + zero_bias_off) : d_b_ + hp.b_off.at(op.param);
    if (op.no_bias && p.cout > 4096) throw std::logic_error("bias-free conv wider than the zero bias");
    if (op.residual >= 0) {
      a.residual = static_cast<const __nv_bfloat16*>(bufs_[op.residual]);
      a.ld_res = m.buffers.at(op.residual).c;
    }
    a.y = bufs_[op.out];
    a.ldy = out.c;
    a.c_off = op.c_off;
    a.out_f32 = out.f32 ? 1 : 0;
    a.relu = op.relu ? 1 : 0;
    if (static_cast<int>(i) == s2d_.op) {
      // stride-2 stem as a stride-1 dr x ds conv over the 16-channel s2d input
      // (padding already inside it), one halo box per dw_th x 8 block: every
      // tap is a window of it (8-pixel rows = the MMA's 8-row groups, SBO =
      // box row pitch); 64-row blocks (four sub-tiles per tile) for the narrow
      // stems, whose epilogue is bound by per-tile work
      pl.mode = ConvLoadMode::kS2D;
      a.R = s2d_.dr;
      a.S = s2d_.ds;
      a.C = 16;
      a.pad_h = a.pad_w = 0;  // (the s2d buffer holds the stem's padding)
      a.taps = s2d_.dr * s2d_.ds;
      a.num_kb = s2d_.kpad / kConvBK;
      a.dw_th = p.cout <= 32 ? 64 : 32;
      a.dw_tw = 8;
      a.dw_rw = 4;
      a.dw_tiles_y = (out.h + a.dw_th - 1) / a.dw_th;
      a.dw_tiles_x = (out.w + 7) / 8;
      a.win_iw = 8 + a.S - 1;
      a.win_ih = a.dw_th + a.R - 1;
      a.win_box_bytes = static_cast<uint32_t>(a.win_iw * a.win_ih * 32);
      if (!encode_tmap_nhwc_sw32(&a.tmap_a, d_s2d_, max_bs, s2d_.hs, s2d_.ws, 16, a.win_iw,
                                 a.win_ih))
        throw CudaError("cuTensorMapEncodeTiled failed (s2d stem halo boxes)");
    } else if (static_cast<int>(i) == stem_) {
      pl.mode = ConvLoadMode::kStemU8;  // a.img is bound per launch (input slot)
    } else if (in.c % 8 != 0) {
      throw std::logic_error("conv input channels must be a multiple of 8");
    } else if (narrow_window_on() && op.kind == OpKind::kConv && op.sh == 1 && op.sw == 1 &&
               op.r == 3 && op.s == 3 && (in.c == 16 || in.c == 32) && op.residual < 0 && !out.f32 &&
               p.cout <= 256 && out.h >= 28 && out.w >= 28 &&
               kpad / kConvBK * ((p.cout + 15) / 16 * 16) * 128 <= 64 * 1024) {
      // 3x3 stride-1 conv over 16 / 32 channels (Inception's 147^2 stem convs):
      // kS2D's window MMAs over one 32 B-swizzled halo box per 16-channel block
      // and 32 x 8 pixel block, instead of a 16 B-granule im2col gather
      pl.mode = ConvLoadMode::kS2DWide;
      a.dw_th = 32;
      a.dw_tw = 8;
      a.dw_rw = 4;
      a.dw_tiles_y = (out.h + 31) / 32;
      a.dw_tiles_x = (out.w + 7) / 8;
      a.win_iw = 8 + op.s - 1;
      a.win_ih = 32 + op.r - 1;
      a.win_box_bytes = static_cast<uint32_t>(a.win_iw * a.win_ih * 32);
      if (!encode_tmap_nhwc_sw32(&a.tmap_a, bufs_[op.in], max_bs, in.h, in.w, in.c, a.win_iw,
                                 a.win_ih))
        throw CudaError("cuTensorMapEncodeTiled failed (narrow window boxes)");
    } else if (window_on(in.c, out.h, out.w) && op.kind == OpKind::kConv && op.sh == 1 &&
               op.sw == 1 &&
               op.residual < 0 && !out.f32 && conv_gemm_window_ok(op.r, op.s, in.c, p.cout)) {
      // stride-1 R x S conv: shifted-window MMAs over per-K-block halo boxes
      pl.mode = ConvLoadMode::kWindow;
      a.dw_th = 16;
      a.dw_tw = 8;
      a.dw_rw = 4;
      a.dw_tiles_y = (out.h + 15) / 16;
      a.dw_tiles_x = (out.w + 7) / 8;
      a.win_iw = 8 + op.s - 1;
      a.win_ih = 16 + op.r - 1;
      const int cb = in.c < 64 ? in.c : 64;
      a.win_box_bytes = static_cast<uint32_t>(a.win_iw * a.win_ih * cb * 2);
      a.win_direct = in.c % 64 == 0 ? 1 : 0;  // 128 B pixel rows: windows read in place
      if (!encode_tmap_nhwc(&a.tmap_a, bufs_[op.in], max_bs, in.h, in.w, in.c, cb, a.win_iw,
                            a.win_ih, 1, a.win_direct != 0))
        throw CudaError("cuTensorMapEncodeTiled failed (window halo boxes)");
    } else if (op.r == 1 && op.s == 1 && op.sh == 1 && op.sw == 1 && op.ph == 0 && op.pw == 0) {
      // A is a plain [pixels][C] matrix; for C < 64 the TMA box runs past
      // the row and the out-of-bounds columns arrive as zeros.
      pl.mode = ConvLoadMode::kTmaA;
    } else if (im2col_on() && in.c % 64 == 0 && op.kind == OpKind::kConv && !out.f32 &&
               out.h >= 28 && out.w >= 28 &&
               encode_tmap_im2col(&a.tmap_a, bufs_[op.in], max_bs, in.h, in.w, in.c, op.r, op.s,
                                  op.sh, op.sw, op.ph, op.pw)) {
      // R x S / strided conv over 64-channel blocks: each K block's A tile is one
      // TMA im2col load (the hardware walks the 128 output pixels' windows)
      pl.mode = ConvLoadMode::kIm2col;
    } else {
      pl.mode = ConvLoadMode::kGather16;
    }
    if (op.residual >= 0 && pl.mode != ConvLoadMode::kTmaA)
      throw std::logic_error("residual adds are supported on 1x1 stride-1 convs only");
    const bool k64 = pl.mode == ConvLoadMode::kTmaA && op.kind == OpKind::kConv &&
                     k64_bn128_on(a.num_kb, p.cout);
    if (k64) {
      a.BN = 128;
      a.stages = choose_stages(a.BN, p.cout);
      a.tmem_cols = tmem_cols_for(a.BN);
    }
    // streamed-weight TMA-A layers run on CTA pairs
    const bool b_resident = (p.cout + a.BN - 1) / a.BN == 1 && a.num_kb * a.BN * 128 <= 64 * 1024;
    a.cluster = 1;
    if (pl.mode == ConvLoadMode::kTmaA && !b_resident && !k64 && pair_on(a.BN)) {
      pl.mode = ConvLoadMode::kPairTmaA;
      a.cluster = 2;  // (tmap_b boxes of BN / 2 rows: each CTA's half)
    } else if (pl.mode == ConvLoadMode::kIm2col && pair_gather_on(a.BN)) {
      pl.mode = ConvLoadMode::kPairIm2col;
      a.cluster = 2;
    } else if (pl.mode == ConvLoadMode::kGather16 && pair_gather_on(a.BN)) {
      pl.mode = ConvLoadMode::kPairGather;
      a.cluster = 2;
    }
    if (static_cast<int>(i) == s2d_.op) {
      if (!encode_tmap_2d_bf16(&a.tmap_b, d_stem_w_, p.cout, s2d_.kpad, s2d_.kpad, a.BN))
        throw CudaError("cuTensorMapEncodeTiled failed (s2d stem weights)");
    } else if (!encode_tmap_2d_bf16(&a.tmap_b, d_w_ + hp.w_off.at(op.param), p.cout, kpad, kpad,
                                    a.BN / a.cluster)) {
      throw CudaError("cuTensorMapEncodeTiled failed (weights)");
    }
    if (pl.mode == ConvLoadMode::kTmaA || pl.mode == ConvLoadMode::kPairTmaA) {
      const uint64_t rows = static_cast<uint64_t>(max_bs) * a.H * a.W;
      if (!encode_tmap_2d_bf16(&a.tmap_a, bufs_[op.in], rows, in.c, in.c, kConvBM))
        throw CudaError("cuTensorMapEncodeTiled failed (activations)");
    }
    // TMA-store epilogue over the output channel slice (falls back to direct
    // stores when TMA cannot address it, e.g. a 10-class fp32 head).
    {
      const uint64_t rows = static_cast<uint64_t>(max_bs) * pl.ho * pl.wo;
      const size_t esz = out.f32 ? 4 : 2;
      void* base = static_cast<uint8_t*>(bufs_[op.out]) + static_cast<size_t>(op.c_off) * esz;
      if (pl.mode == ConvLoadMode::kWindow || pl.mode == ConvLoadMode::kS2D ||
          pl.mode == ConvLoadMode::kS2DWide)  // pixel-row boxes
        a.y_tma = !out.f32 && encode_tmap_out4d(&a.tmap_y, base, max_bs, pl.ho, pl.wo, p.cout, out.c,
                                                a.dw_tw, a.dw_rw)
                      ? 1
                      : 0;
      else
        a.y_tma = encode_tmap_out(&a.tmap_y, base, rows, p.cout, out.c, out.f32) ? 1 : 0;
    }
    if (!op.fused.empty()) {
      // one launch over the concatenated weights; segment s's columns are
      // stored into its own buffer / channel slice
      if (pl.mode != ConvLoadMode::kTmaA && pl.mode != ConvLoadMode::kPairTmaA &&
          pl.mode != ConvLoadMode::kGather16 && pl.mode != ConvLoadMode::kPairGather &&
          pl.mode != ConvLoadMode::kIm2col && pl.mode != ConvLoadMode::kPairIm2col)
        throw std::logic_error("fused 1x1 siblings need a TMA-A, im2col or gather conv");
      std::vector<ConvSeg> segs{ConvSeg{op.param, op.out, op.c_off, op.relu, op.no_bias}};
      segs.insert(segs.end(), op.fused.begin(), op.fused.end());
      const uint64_t rows = static_cast<uint64_t>(max_bs) * pl.ho * pl.wo;
      int col = 0;
      a.nseg = static_cast<int>(segs.size());
      a.seg_norelu = 0;
      for (int sg = 0; sg < a.nseg; ++sg) {
        const ConvSeg& f = segs[sg];
        const int co = m.params[f.param].cout;
        const BufferSpec& ob = m.buffers.at(f.out);
        if (ob.h != out.h || ob.w != out.w || ob.f32) throw std::logic_error("fused sibling output shape");
        a.seg_col[sg] = col;
        a.seg_y[sg] = static_cast<uint8_t*>(bufs_[f.out]) + static_cast<size_t>(f.c_off) * 2;
        a.seg_w[sg] = co;
        a.seg_ld[sg] = ob.c;
        if (!f.relu) a.seg_norelu |= 1 << sg;
        if (!encode_tmap_out(&a.tmap_seg[sg], a.seg_y[sg], rows, co, ob.c, false))
          throw CudaError("cuTensorMapEncodeTiled failed (fused sibling output)");
        col += round_up(co, 64);
      }
      a.seg_col[a.nseg] = col;
      a.relu = 1;  // (per segment through seg_norelu)
      a.Cout = col;
      const bool k64 = (pl.mode == ConvLoadMode::kTmaA || pl.mode == ConvLoadMode::kPairTmaA) &&
                       k64_bn128_on(a.num_kb, col);
      a.BN = k64 ? 128 : choose_bn(col);
      a.stages = choose_stages(a.BN, col);
      a.tmem_cols = tmem_cols_for(a.BN);
      a.bias = reinterpret_cast<const float*>(base + fb_off[i]);
      a.cluster = 1;
      if (pl.mode == ConvLoadMode::kPairTmaA) pl.mode = ConvLoadMode::kTmaA;
      if (pl.mode == ConvLoadMode::kPairGather) pl.mode = ConvLoadMode::kGather16;
      if (pl.mode == ConvLoadMode::kPairIm2col) pl.mode = ConvLoadMode::kIm2col;
      const bool b_res = (col + a.BN - 1) / a.BN == 1 && a.num_kb * a.BN * 128 <= 64 * 1024;
      if (pl.mode == ConvLoadMode::kTmaA && !b_res && !k64 && pair_on(a.BN)) {
        pl.mode = ConvLoadMode::kPairTmaA;
        a.cluster = 2;
      } else if (pl.mode == ConvLoadMode::kGather16 && pair_gather_on(a.BN)) {
        pl.mode = ConvLoadMode::kPairGather;
        a.cluster = 2;
      } else if (pl.mode == ConvLoadMode::kIm2col && pair_gather_on(a.BN)) {
        pl.mode = ConvLoadMode::kPairIm2col;
        a.cluster = 2;
      }
      if (!encode_tmap_2d_bf16(&a.tmap_b, base + fw_off[i], col, kpad, kpad, a.BN / a.cluster))
        throw CudaError("cuTensorMapEncodeTiled failed (fused weights)");
      if (!a.y_tma) throw CudaError("fused sibling 1x1 without a TMA-store epilogue");
    }
  }
  spans_bytes_ = sizeof(unsigned long long) * 2 * (kernels_per_forward_ + 1);
  check_cuda(cudaMalloc(&d_spans_, spans_bytes_), "cudaMalloc spans");
  check_cuda(cudaMemsetAsync(d_spans_, 0, spans_bytes_, stream_), "zero spans");
  check_cuda(cudaStreamSynchronize(stream_), "instance setup");
}

void Instance::reset_spans() {
  check_cuda(cudaMemset(d_spans_, 0, spans_bytes_), "reset spans");
}

int64_t Instance::read_spans(std::vector<double>* ms) const {
  std::vector<unsigned long long> h(spans_bytes_ / sizeof(unsigned long long));
  check_cuda(cudaMemcpy(h.data(), d_spans_, spans_bytes_, cudaMemcpyDeviceToHost), "read spans");
  const int k = kernels_per_forward_;
  const unsigned long long n = h[1];
  ms->assign(k, 0.0);
  for (int i = 0; i <= k; ++i)
    if (h[2 * i + 1] != n) return -1;  // a kernel without a live-timing slot, or in flight
  if (n == 0) return 0;
  for (int i = 0; i < k; ++i)
    (*ms)[i] = static_cast<double>(h[2 * (i + 1)] - h[2 * i]) / static_cast<double>(n) / 1e6;
  return static_cast<int64_t>(n);
}

Instance::~Instance() {
  cudaSetDevice(device_);
  if (d_spans_) cudaFree(d_spans_);
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
  if (copy_stream_) cudaStreamSynchronize(copy_stream_);
  if (out_stream_) cudaStreamSynchronize(out_stream_);
  if (d_arena_) cudaFree(d_arena_);
  for (int s = 0; s < 2; ++s) {
    if (slot_free_[s]) cudaEventDestroy(slot_free_[s]);
    if (h2d_done_[s]) cudaEventDestroy(h2d_done_[s]);
    if (out_ready_[s]) cudaEventDestroy(out_ready_[s]);
    if (out_read_[s]) cudaEventDestroy(out_read_[s]);
    if (d_out_[s]) cudaFree(d_out_[s]);
  }
  if (copy_stream_) cudaStreamDestroy(copy_stream_);
  if (out_stream_) cudaStreamDestroy(out_stream_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Instance::enqueue_layers(int bs, const std::vector<cudaEvent_t>* marks, int slot) {
  const ModelSpec& m = m_;
  const HostParams& hp = params_for(m);
  size_t mark = 0;
  int launch = 0;  // kernel index in the forward: its live-timing slot
  launch_span() = d_spans_;
  auto record_mark = [&] {
    ++launch;
    launch_span() = d_spans_ + 2 * launch;
    if (marks)
      check_cuda(cudaEventRecordWithFlags((*marks)[mark++], cur_stream_, cudaEventRecordExternal),
                 "mark");
  };
  struct SpanReset {
    ~SpanReset() { launch_span() = nullptr; }
  } span_reset;
  if (marks)
    check_cuda(cudaEventRecordWithFlags((*marks)[mark++], cur_stream_, cudaEventRecordExternal),
               "mark");
  if (s2d_.op >= 0) {
    check_cuda(launch_stage_s2d(d_images_[slot], d_s2d_, bs, m.in_h, m.in_w, s2d_.hs, s2d_.ws,
                                s2d_.pad, cur_stream_),
               "stage_s2d");
    record_mark();
  }
  for (size_t i = 0; i < m.ops.size(); ++i) {
    const OpSpec& op = m.ops[i];
    const BufferSpec& in = m.buffers[op.in];
    const BufferSpec& out = m.buffers[op.out];
    const auto* x = static_cast<const __nv_bfloat16*>(bufs_[op.in]);
    auto* y = static_cast<__nv_bfloat16*>(bufs_[op.out]);
    cudaError_t e = cudaSuccess;
    switch (op.kind) {
      case OpKind::kConv:
      case OpKind::kFc: {
        ConvGemmArgs a = plans_[i].args;
        a.M = bs * plans_[i].ho * plans_[i].wo;
        if (static_cast<int>(i) == stem_) a.img = d_images_[slot];
        e = launch_conv_gemm(a, plans_[i].mode, cur_stream_);
        break;
      }
      case OpKind::kDwConv: {
        const auto* w = reinterpret_cast<const __nv_bfloat16*>(d_w_ + hp.w_off[op.param]);
        e = launch_dwconv3x3_tma(dw_maps_[i], w, d_b_ + hp.b_off[op.param], y, bs, in.h, in.w, in.c,
                                 op.sh, cur_stream_);
        break;
      }
      case OpKind::kMaxPool:
      case OpKind::kAvgPool:
        if (i < pool_tma_.size() && pool_tma_[i]) {
          e = launch_pool3x3_tma(pool_maps_[i], y, bs, in.h, in.w, in.c, op.sh, op.ph,
                                 op.kind == OpKind::kMaxPool, out.c, op.c_off, cur_stream_,
                                 op.post_bias >= 0 ? d_b_ + hp.b_off[op.post_bias] : nullptr, op.relu);
          break;
        }
        if (op.post_bias >= 0)  // (swap_avgpool_1x1 pools run on the TMA kernel only)
          throw std::logic_error("average pool with a post-bias needs the TMA pool (DS_POOL_SWAP=0)");
        e = launch_pool3x3(x, y, bs, in.h, in.w, in.c, op.sh, op.ph, op.kind == OpKind::kMaxPool,
                           out.c, op.c_off, cur_stream_);
        break;
      case OpKind::kGlobalAvgPool:
        e = launch_global_avgpool(x, y, bs, in.h * in.w, in.c, cur_stream_);
        break;
    }
    check_cuda(e, "layer launch");
    record_mark();
  }
  check_cuda(launch_softmax(d_logits_, d_probs_, bs, m.classes, cur_stream_), "softmax");
  record_mark();
}

std::vector<double> Instance::profile_kernels(int bs, int reps) {
  if (bs < 1 || bs > max_bs_) throw std::invalid_argument("invalid batch size");
  const int nk = kernels_per_forward_;
  std::vector<cudaEvent_t> marks(nk + 1);
  for (auto& e : marks) check_cuda(cudaEventCreate(&e), "cudaEventCreate");
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<double> acc(nk, 0.0);
  try {
    check_cuda(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
    try {
      enqueue_layers(bs, &marks);
    } catch (...) {
      cudaStreamEndCapture(stream_, &g);
      throw;
    }
    check_cuda(cudaStreamEndCapture(stream_, &g), "capture end");
    check_cuda(cudaGraphInstantiate(&exec, g, 0), "instantiate");
    for (int r = 0; r < reps + 1; ++r) {  // first launch is a warm-up
      check_cuda(cudaGraphLaunch(exec, stream_), "launch");
      check_cuda(cudaStreamSynchronize(stream_), "profile");
      if (r == 0) continue;
      for (int k = 0; k < nk; ++k) {
        float ms = 0.0f;
        check_cuda(cudaEventElapsedTime(&ms, marks[k], marks[k + 1]), "elapsed");
        acc[k] += ms;
      }
    }
  } catch (...) {
    if (exec) cudaGraphExecDestroy(exec);
    if (g) cudaGraphDestroy(g);
    for (auto& e : marks) cudaEventDestroy(e);
    throw;
  }
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(g);
  for (auto& e : marks) cudaEventDestroy(e);
  for (auto& v : acc) v /= reps;
  return acc;
}

void Instance::read_buffer(int id, int bs, void* host) const {
  const BufferSpec& b = m_.buffers.at(id);
  const size_t bytes = static_cast<size_t>(bs) * b.h * b.w * b.c * (b.f32 ? 4 : 2);
  check_cuda(cudaStreamSynchronize(stream_), "read_buffer");
  check_cuda(cudaMemcpy(host, bufs_.at(id), bytes, cudaMemcpyDeviceToHost), "read_buffer");
}

void Instance::enqueue_forward(int bs, int slot) { enqueue_forward_on(bs, slot, stream_, 0, 0); }

void Instance::enqueue_forward_on(int bs, int slot, cudaStream_t s, int sms, int lane_key) {
  if (bs < 1 || bs > max_bs_) throw std::invalid_argument("invalid batch size");
  const int64_t key = (static_cast<int64_t>(lane_key) * 4096 + bs) * 2 + slot;
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    // Capture on the lane's stream with the persistent kernels' grids sized
    // to its SM budget (green-context partitions; 0 = whole device).
    struct Budget {
      int saved;
      explicit Budget(int v) : saved(launch_sm_budget()) { launch_sm_budget() = v; }
      ~Budget() { launch_sm_budget() = saved; }
    } budget(sms);
    cur_stream_ = s;
    cudaGraph_t g = nullptr;
    check_cuda(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture begin");
    try {
      enqueue_layers(bs, nullptr, slot);
    } catch (...) {
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      cur_stream_ = stream_;
      throw;
    }
    cur_stream_ = stream_;
    check_cuda(cudaStreamEndCapture(s, &g), "capture end");
    cudaGraphExec_t exec = nullptr;
    check_cuda(cudaGraphInstantiate(&exec, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    it = graphs_.emplace(key, exec).first;
  }
  check_cuda(cudaGraphLaunch(it->second, s), "graph launch");
}

// ------------------------------------------------------------------ Backend

Backend::Backend(const std::string& model_id, BackendConfig cfg, uint64_t seed, int device)
    : model_(build_model(model_id)), cfg_(cfg), seed_(seed), device_(device) {
  if (cfg_.abs_max_bs < 1 || cfg_.max_mtl < 1)
    throw std::invalid_argument("invalid device limits");  // reference gpu_sim.cpp:9-10
  check_cuda(cudaSetDevice(device_), "cudaSetDevice");
  params_for(model_);
  pool_images_ = std::max(cfg_.abs_max_bs, cfg_.max_mtl);
  const size_t img_bytes = static_cast<size_t>(model_.in_h) * model_.in_w * 3;
  host_images_.resize(img_bytes * pool_images_);
  generate_images(model_.in_h, model_.in_w, seed_, 0, pool_images_, host_images_.data());
  // instances [0, max_mtl): the batching instance and the MT (bs = 1)
  // instances; [max_mtl, 2 max_mtl - 1): full-size instances 1.. of the
  // B x MT combination (combo instance 0 is the batching instance)
  inst_.resize(2 * cfg_.max_mtl);
  inflight_.resize(2 * cfg_.max_mtl);
  io_cursor_.assign(2 * cfg_.max_mtl, 0);
  io_seq_.assign(2 * cfg_.max_mtl, 0);
  pinned_logits_.assign(2 * cfg_.max_mtl, nullptr);
  last_first_.assign(2 * cfg_.max_mtl, -1);
  last_bs_.assign(2 * cfg_.max_mtl, 0);
  instance(0);
}

Backend::~Backend() {
  cudaSetDevice(device_);
  try {
    drain();
  } catch (...) {
  }
  inst_.clear();
  green_.reset();
  for (cudaEvent_t e : all_events_) cudaEventDestroy(e);
  for (cudaEvent_t e : timer_)
    if (e) cudaEventDestroy(e);
  if (pinned_images_) cudaFreeHost(pinned_images_);
  for (float* p : pinned_logits_)
    if (p) cudaFreeHost(p);
}

Instance& Backend::instance(int i) {
  if (!inst_.at(i)) {
    const bool full = i == 0 || i >= cfg_.max_mtl;
    const int max_bs = full ? cfg_.abs_max_bs : 1;
    inst_[i] = std::make_unique<Instance>(model_, max_bs, device_);
    const size_t img_bytes = static_cast<size_t>(model_.in_h) * model_.in_w * 3;
    const int first = full ? 0 : (i % pool_images_);
    check_cuda(cudaMemcpy(inst_[i]->images(), host_images_.data() + img_bytes * first,
                          img_bytes * max_bs, cudaMemcpyHostToDevice),
               "upload images");
  }
  return *inst_[i];
}

int Backend::instances_created() const {
  int n = 0;
  for (const auto& p : inst_) n += p ? 1 : 0;
  return n;
}

size_t Backend::device_bytes() const {
  size_t n = 0;
  for (const auto& p : inst_)
    if (p) n += p->device_bytes();
  return n;
}

cudaStream_t Backend::batch_stream() const { return inst_[0]->stream(); }

cudaEvent_t Backend::take_event() {
  if (free_events_.empty()) {
    cudaEvent_t e;
    check_cuda(cudaEventCreate(&e), "cudaEventCreate");
    all_events_.push_back(e);
    return e;
  }
  cudaEvent_t e = free_events_.back();
  free_events_.pop_back();
  return e;
}

void Backend::enqueue_request(int i, int bs) {
  Instance& I = instance(i);
  Inflight f{take_event(), take_event(), bs};
  // MT requests in green-context mode run on instance i's SM partition lane
  const GreenLane* lane = nullptr;
  if (mt_mode_ == 1 && mt_active_ && bs == 1 && i < cfg_.max_mtl) {
    const auto& lanes = green_->level(mtl_);
    lane = &lanes[i % lanes.size()];
  }
  cudaStream_t s = lane ? lane->stream : I.stream();
  auto forward = [&](int slot) {
    if (lane)
      I.enqueue_forward_on(bs, slot, lane->stream, lane->sms, mtl_);
    else
      I.enqueue_forward(bs, slot);
  };
  const size_t img_bytes = static_cast<size_t>(model_.in_h) * model_.in_w * 3;
  last_bs_[i] = bs;
  if (!host_io_) {
    last_first_[i] = (i == 0 || i >= cfg_.max_mtl) ? 0 : i % pool_images_;
    check_cuda(cudaEventRecord(f.start, s), "event record");
    forward(0);
  } else {
    // End to end: the request's images cross PCIe on the instance's copy
    // stream into one of two input slots (so the next request's copy runs
    // under this forward); the timed span starts before the copy and ends
    // after the logits are back in pinned host memory.
    const int slot = static_cast<int>(io_seq_[i]++ & 1);
    int64_t& cur = io_cursor_[i];
    if (cur + bs > pool_images_) cur = 0;
    const uint8_t* src = pinned_images_ + img_bytes * static_cast<size_t>(cur);
    last_first_[i] = cur;
    const bool full = i == 0 || i >= cfg_.max_mtl;
    cur = full ? cur + bs : (cur + cfg_.max_mtl) % pool_images_;
    if (!pinned_logits_[i])
      check_cuda(cudaMallocHost(&pinned_logits_[i], static_cast<size_t>(I.max_bs()) *
                                                        model_.classes * sizeof(float)),
                 "cudaMallocHost");
    cudaStream_t cs = I.copy_stream();
    check_cuda(cudaStreamWaitEvent(cs, I.slot_free(slot), 0), "wait slot");
    check_cuda(cudaEventRecord(f.start, cs), "event record");
    check_cuda(cudaMemcpyAsync(I.images(slot), src, img_bytes * bs, cudaMemcpyHostToDevice, cs),
               "H2D images");
    check_cuda(cudaEventRecord(I.h2d_done(slot), cs), "event record");
    h2d_bytes_ += static_cast<int64_t>(img_bytes) * bs;
    check_cuda(cudaStreamWaitEvent(s, I.h2d_done(slot), 0), "wait h2d");
    forward(slot);
    check_cuda(cudaEventRecord(I.slot_free(slot), s), "event record");
    // logits -> this slot's buffer (on the compute stream, once the D2H that
    // last read it is done), then D2H on the instance's output stream, so
    // the next request's forward does not queue behind the PCIe read
    const size_t lb = static_cast<size_t>(bs) * model_.classes * sizeof(float);
    check_cuda(cudaStreamWaitEvent(s, I.out_read(slot), 0), "wait out slot");
    check_cuda(cudaMemcpyAsync(I.out(slot), I.logits(), lb, cudaMemcpyDeviceToDevice, s),
               "logits to slot");
    check_cuda(cudaEventRecord(I.out_ready(slot), s), "event record");
    cudaStream_t os = I.out_stream();
    check_cuda(cudaStreamWaitEvent(os, I.out_ready(slot), 0), "wait logits");
    check_cuda(cudaMemcpyAsync(pinned_logits_[i], I.out(slot), lb, cudaMemcpyDeviceToHost, os),
               "D2H logits");
    check_cuda(cudaEventRecord(I.out_read(slot), os), "event record");
    d2h_bytes_ += static_cast<int64_t>(lb);
    s = os;  // (the request ends when its logits are in host memory)
  }
  kernel_launches_ += I.kernels_per_forward();
  check_cuda(cudaEventRecord(f.end, s), "event record");
  inflight_[i].push_back(f);
}

double Backend::complete_oldest(int i) {
  Inflight f = inflight_[i].front();
  inflight_[i].pop_front();
  check_cuda(cudaEventSynchronize(f.end), "request");
  float ms = 0.0f;
  check_cuda(cudaEventElapsedTime(&ms, f.start, f.end), "cudaEventElapsedTime");
  free_events_.push_back(f.start);
  free_events_.push_back(f.end);
  return static_cast<double>(ms);
}

void Backend::drain() {
  for (size_t i = 0; i < inflight_.size(); ++i)
    while (!inflight_[i].empty()) complete_oldest(static_cast<int>(i));
  batch_bs_ = 0;
  mt_active_ = false;
  rr_ = 0;
}

void Backend::run_batches(int bs, int count, double* lat_out) {
  if (bs < 1 || bs > cfg_.abs_max_bs) throw std::invalid_argument("invalid batch size");
  if (mt_active_ || (batch_bs_ != 0 && batch_bs_ != bs)) drain();
  batch_bs_ = bs;
  for (int j = 0; j < count; ++j) {
    while (static_cast<int>(inflight_[0].size()) < kDepth) enqueue_request(0, bs);
    const double lat = complete_oldest(0);
    clock_ms_ += lat;  // reference gpu_sim.cpp:16
    lat_out[j] = lat;
  }
}

void Backend::run_combo_requests(int bs, int mtl, int count, double* lat_out) {
  // B x MT combination (reference combination_sweep, harness.cpp:356-386, on
  // the analytic model): mtl full-size instances, each on its own stream,
  // each keeping kDepth batches of bs in flight; latencies of completed
  // batches round robin over the instances; clock += latency / mtl as for MT.
  if (bs < 1 || bs > cfg_.abs_max_bs) throw std::invalid_argument("invalid batch size");
  if (mtl < 1 || mtl > cfg_.max_mtl) throw std::invalid_argument("invalid instance count");
  drain();
  auto idx = [&](int k) { return k == 0 ? 0 : cfg_.max_mtl + k - 1; };
  for (int k = 0; k < mtl; ++k) instance(idx(k));  // (created outside the timed calls)
  // exactly `count` batches are issued (request j on instance j % mtl), so
  // every batch run between the drains is one of the returned latencies
  int issued = 0;
  for (int j = 0; j < count; ++j) {
    while (issued < count && static_cast<int>(inflight_[idx(issued % mtl)].size()) < kDepth) {
      enqueue_request(idx(issued % mtl), bs);
      ++issued;
    }
    const double lat = complete_oldest(idx(j % mtl));
    clock_ms_ += lat / static_cast<double>(mtl);
    lat_out[j] = lat;
  }
  drain();
}

void Backend::run_mt_requests(int count, double* lat_out) {
  if (batch_bs_ != 0) drain();
  mt_active_ = true;
  for (int j = 0; j < count; ++j) {
    for (int i = 0; i < mtl_; ++i)
      while (static_cast<int>(inflight_[i].size()) < kDepth) enqueue_request(i, 1);
    const double lat = complete_oldest(rr_);
    rr_ = (rr_ + 1) % mtl_;
    clock_ms_ += lat / static_cast<double>(mtl_);  // reference gpu_sim.cpp:22
    lat_out[j] = lat;
  }
}

double Backend::run_batch(int bs) {
  double lat = 0.0;
  run_batches(bs, 1, &lat);
  return lat;
}

double Backend::run_mt_request() {
  double lat = 0.0;
  run_mt_requests(1, &lat);
  return lat;
}

double Backend::apply_instance_change(int delta) {
  // Validation and messages follow reference gpu_sim.cpp:26-37.
  if (delta == 0) return 0.0;
  if (delta != 1 && delta != -1) throw std::invalid_argument("instance changes are single steps");
  const int target = mtl_ + delta;
  if (target < 1) throw std::invalid_argument("cannot terminate last instance");
  if (target > cfg_.max_mtl) throw std::invalid_argument("instance limit exceeded");
  drain();
  const auto t0 = std::chrono::steady_clock::now();
  if (delta > 0) {
    // Launch: weights, workspace and stream (first time), then one warm-up
    // request, which also captures the instance's bs=1 graph.
    Instance& I = instance(target - 1);
    I.enqueue_forward(1);
    check_cuda(cudaStreamSynchronize(I.stream()), "instance warm-up");
  }
  mtl_ = target;
  if (mt_mode_ == 1) {
    // green mode: the new level's partitions (created once per level) and
    // every active instance's lane graph, so requests never capture
    const auto& lanes = green_->level(mtl_);
    for (int i = 0; i < mtl_; ++i) {
      const GreenLane& l = lanes[i % lanes.size()];
      instance(i).enqueue_forward_on(1, 0, l.stream, l.sms, mtl_);
    }
    for (const auto& l : lanes) check_cuda(cudaStreamSynchronize(l.stream), "lane warm-up");
  }
  const double delay =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  clock_ms_ += delay;
  return delay;
}

double Backend::set_mtl(int target) {
  // reference gpu_sim.cpp:39-46
  if (target < 1) throw std::invalid_argument("cannot terminate last instance");
  if (target > cfg_.max_mtl) throw std::invalid_argument("instance limit exceeded");
  double total = 0.0;
  while (mtl_ < target) total += apply_instance_change(1);
  while (mtl_ > target) total += apply_instance_change(-1);
  return total;
}

void Backend::forward(const uint8_t* host_images, int bs, float* host_logits, float* host_probs) {
  if (bs < 1 || bs > cfg_.abs_max_bs) throw std::invalid_argument("invalid batch size");
  drain();
  Instance& I = instance(0);
  cudaStream_t s = I.stream();
  const size_t img_bytes = static_cast<size_t>(model_.in_h) * model_.in_w * 3;
  check_cuda(cudaMemcpyAsync(I.images(), host_images, img_bytes * bs, cudaMemcpyHostToDevice, s),
             "H2D images");
  I.enqueue_forward(bs);
  kernel_launches_ += I.kernels_per_forward();
  const size_t lb = static_cast<size_t>(bs) * model_.classes * sizeof(float);
  if (host_logits)
    check_cuda(cudaMemcpyAsync(host_logits, I.logits(), lb, cudaMemcpyDeviceToHost, s), "D2H");
  if (host_probs)
    check_cuda(cudaMemcpyAsync(host_probs, I.probs(), lb, cudaMemcpyDeviceToHost, s), "D2H");
  // Put the resident synthetic batch back for the serving paths.
  check_cuda(cudaMemcpyAsync(I.images(), host_images_.data(), img_bytes * I.max_bs(),
                             cudaMemcpyHostToDevice, s),
             "restore images");
  check_cuda(cudaStreamSynchronize(s), "forward");
}

void Backend::timer_start() {
  drain();
  for (auto& e : timer_)
    if (!e) check_cuda(cudaEventCreate(&e), "cudaEventCreate");
  check_cuda(cudaDeviceSynchronize(), "timer sync");
  check_cuda(cudaEventRecord(timer_[0], inst_[0]->stream()), "timer start");
}

double Backend::timer_stop() {
  drain();
  check_cuda(cudaDeviceSynchronize(), "timer sync");
  check_cuda(cudaEventRecord(timer_[1], inst_[0]->stream()), "timer stop");
  check_cuda(cudaEventSynchronize(timer_[1]), "timer stop");
  float ms = 0.0f;
  check_cuda(cudaEventElapsedTime(&ms, timer_[0], timer_[1]), "timer elapsed");
  return static_cast<double>(ms);
}

void Backend::set_host_io(bool enabled) {
  drain();
  if (enabled && !pinned_images_) {
    check_cuda(cudaMallocHost(&pinned_images_, host_images_.size()), "cudaMallocHost");
    std::memcpy(pinned_images_, host_images_.data(), host_images_.size());
  }
  host_io_ = enabled;
}

void Backend::set_mt_mode(int mode) {
  if (mode != 0 && mode != 1) throw std::invalid_argument("invalid multi-tenancy mode");
  drain();
  if (mode == 1 && !green_) {
    check_cuda(cudaSetDevice(device_), "cudaSetDevice");
    green_ = std::make_unique<GreenPartitions>(device_);
  }
  mt_mode_ = mode;
  if (mode == 1) {  // current level's lanes and graphs
    const auto& lanes = green_->level(mtl_);
    for (int i = 0; i < mtl_; ++i) {
      const GreenLane& l = lanes[i % lanes.size()];
      instance(i).enqueue_forward_on(1, 0, l.stream, l.sms, mtl_);
    }
    for (const auto& l : lanes) check_cuda(cudaStreamSynchronize(l.stream), "lane warm-up");
  }
}

int Backend::last_output(int i, float* host_logits, int64_t* first_image) {
  if (i < 0 || i >= static_cast<int>(inst_.size()) || !inst_[i] || last_bs_[i] == 0)
    throw std::invalid_argument("instance has served no request");
  drain();
  const int bs = last_bs_[i];
  const size_t lb = static_cast<size_t>(bs) * model_.classes * sizeof(float);
  if (host_logits) {
    // host-I/O requests: the logits the request itself read back to pinned
    // memory; device-resident requests: the instance's logits buffer
    if (host_io_ && pinned_logits_[i])
      std::memcpy(host_logits, pinned_logits_[i], lb);
    else
      check_cuda(cudaMemcpy(host_logits, inst_[i]->logits(), lb, cudaMemcpyDeviceToHost),
                 "read logits");
  }
  if (first_image) *first_image = last_first_[i];
  return bs;
}

}  // namespace ds
