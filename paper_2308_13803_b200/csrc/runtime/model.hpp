// Network IR for the served models. The reference has no model code at all
// (its "forward pass" is the analytic latency of perf_model.cpp:70-86); these
// are the canonical architectures named by BASELINE.json's configs, laid out
// for the B200 kernels: NHWC bf16 activations, KRSC bf16 weights with folded
// batch-norm (bias only), fp32 logits.
#pragma once

#include <string>
#include <vector>

namespace ds {

enum class OpKind { kConv, kDwConv, kMaxPool, kAvgPool, kGlobalAvgPool, kFc };

// Per-image activation buffer shape (NHWC). Buffer 0 is always the staged
// input (C = 4: RGB + one zero channel).
struct BufferSpec {
  int h = 1, w = 1, c = 1;
  bool f32 = false;
};

// A parameterised layer, in canonical generation order.
struct ParamSpec {
  OpKind kind = OpKind::kConv;
  int cout = 0, r = 1, s = 1;
  int cin = 0;         // real input channels (3 for stems)
  int cin_stored = 0;  // channels in the device layout (4 for stems)
  float gain = 1.0f;   // multiplies the He std (residual-branch ends use 0.5)
  bool fc = false;     // FC: std sqrt(1/fan_in), zero bias
};

// A sibling 1x1 conv fused into an op (same input, same stride): its weights
// are concatenated after the op's own along N and its outputs go to its own
// buffer / channel slice (fuse_sibling_1x1 below).
struct ConvSeg {
  int param = -1;
  int out = 0;
  int c_off = 0;
  bool relu = true;
  bool no_bias = false;
};

struct OpSpec {
  OpKind kind = OpKind::kConv;
  int in = 0;
  int out = 0;
  int c_off = 0;      // channel offset inside `out` (concat slices)
  int residual = -1;  // buffer added in the epilogue before ReLU
  int r = 1, s = 1, sh = 1, sw = 1, ph = 0, pw = 0;
  bool relu = true;
  int param = -1;
  std::vector<ConvSeg> fused;  // siblings computed by this op's launch (after its own columns)
  // conv: skip the bias (it is added after a following average pool);
  // average pool: add param's bias (then ReLU if relu) to the pooled values
  bool no_bias = false;
  int post_bias = -1;
};

struct ModelSpec {
  std::string id;
  int in_h = 0, in_w = 0;
  int classes = 0;
  std::vector<BufferSpec> buffers;
  std::vector<ParamSpec> params;
  std::vector<OpSpec> ops;
  int logits = -1;  // fp32 [classes] buffer
  double macs_per_image = 0.0;  // algorithmic multiply-accumulates (real channels)
};

// "synthetic_cnn", "mobilenet_v1", "resnet50_v1", "inception_v3". Sibling
// 1x1 convs are fused (fuse_sibling_1x1) unless DS_FUSE_1X1=0.
ModelSpec build_model(const std::string& id);

// Merges 1x1 convs that read the same buffer with the same stride (Inception's
// branch heads, ResNet's first conv + projection shortcut) into the first of
// them: one launch over the concatenated weights, each sibling's columns
// stored to its own buffer. Same products in the same K order per output, so
// bit-identical to the separate launches. At most 4 segments per op.
void fuse_sibling_1x1(ModelSpec& m);

// avgpool3x3(s1, p1, count_include_pad) followed by a 1x1 conv (bias b,
// ReLU) equals ReLU(avgpool3x3(W x) + b): both are linear, the padding taps
// are zeros either way. Rewrites such pairs to a bias-free 1x1 over the pool's
// input (which then fuses with its siblings) and a pool over the conv's
// Cout channels (Inception: 32-192 instead of 192-2048) that adds b and
// applies the ReLU. Not bit-identical (bf16 rounding moves from the pooled
// input to the conv output); within the oracle tolerance. DS_POOL_SWAP=0: off.
void swap_avgpool_1x1(ModelSpec& m);

// Algorithmic cost of every kernel of one forward, in launch order:
// input staging, one entry per op, softmax. Bytes are the minimum DRAM
// traffic (each input, output, residual and weight tensor moved once, bf16
// activations, fp32 logits); FLOPs are 2 x real multiply-accumulates.
enum class KernelKind { kStage = 0, kConvGemm = 1, kDwConv = 2, kPool = 3, kGap = 4, kSoftmax = 5 };
struct KernelCost {
  KernelKind kind;
  double flops_per_image = 0.0;
  double bytes_per_image = 0.0;
  double fixed_bytes = 0.0;  // weights + bias, once per launch
};
std::vector<KernelCost> kernel_costs(const ModelSpec& m);

// Index of the stem conv when it reads the u8 images directly (ConvLoadMode
// kStemU8: staging fused into its producer), -1 when it is not a stride-1
// conv that alone reads buffer 0 (or a stride-2 stem runs on the s2d input).
int fused_stem(const ModelSpec& m);

// Stride-2 stem over a space-to-depth input (ConvLoadMode kS2D): a staging
// kernel writes S[n][hs][ws][16] (2 x 2 pixel blocks of the normalised image)
// and the stem becomes a stride-1 dr x ds conv over it. Returns the stem op
// index (and the geometry) or -1 (not a stride-2 stem).
struct S2dPlan {
  int op = -1;
  int hs = 0, ws = 0, dr = 0, ds = 0, pad = 0, kpad = 0;
};
S2dPlan stem_s2d(const ModelSpec& m);
std::vector<std::string> model_ids();

}  // namespace ds
