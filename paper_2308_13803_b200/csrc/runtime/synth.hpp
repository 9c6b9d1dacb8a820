// Seeded synthetic weights and images. The generator is the reference's own
// RandomStream / mix_seed (reference random.hpp:10-47): std::mt19937_64, a
// 53-bit uniform and the pinned Box-Muller, so a weight tensor is a pure
// function of (seed, layer index) on every host.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "model.hpp"

namespace ds {

// splitmix64 finaliser (reference random.hpp:10-15).
inline uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Same draws as reference random.hpp:17-47.
class RandomStream {
 public:
  explicit RandomStream(uint64_t seed = 0) : eng_(seed) {}
  double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double gaussian() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
    spare_ = rad * std::sin(kTwoPi * u2);
    has_spare_ = true;
    return rad * std::cos(kTwoPi * u2);
  }
  uint64_t next_u64() { return eng_(); }

 private:
  std::mt19937_64 eng_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// Device-layout parameters of one model, generated on the host.
//   conv: bf16 [cout][kpad], k = (r*S + s)*cin_stored + c (KRSC), zero-padded
//   dw:   bf16 [9][C] (tap-major)
//   fc:   bf16 [classes][kpad]
// Offsets are in elements and keep every layer 128 B aligned.
// Calibrated classifier head (paper_2308_13803_b200/data/heads/<model>.head,
// written by tools/calibrate_heads.py from the device's own pooled features
// over a calibration image set): feature mean mu[C], the top-k principal
// directions v[k][C] and per-direction scales. The FC becomes
// W = bf16(R diag(scale) V) with R ~ N(0,1) [classes][k] from the FC layer's
// stream and b = -W mu, so the logits respond to the input-dependent part of
// the features instead of being dominated by their common mean (random-init
// CNNs map every input to nearly the same pooled feature vector).
// File: "DSHEAD1\0", int32 C, int32 k, f64 mu[C], f64 scale[k], f64 v[k][C].
struct HeadCalib {
  int c = 0, k = 0;  // k == 0: no file, plain random head
  std::vector<double> mu, scale, v;
};
std::string head_dir();  // $DS_HEAD_DIR, else <library dir>/data/heads
HeadCalib load_head(const std::string& model_id);

struct HostParams {
  HeadCalib head;
  std::vector<uint16_t> w;
  std::vector<float> b;
  std::vector<size_t> w_off, b_off;
  std::vector<int> kpad;
};

constexpr uint64_t kWeightSeed = 42;        // scenario default seed (reference scenario.hpp:20)
constexpr uint64_t kWeightSalt = 1000;      // layer l uses mix_seed(seed, 1000 + l)
constexpr uint64_t kImageSalt = 1000000;    // image i uses mix_seed(seed, 1000000 + i)

const HostParams& params_for(const ModelSpec& m);  // cached per model id
HostParams generate_params(const ModelSpec& m, uint64_t seed = kWeightSeed);

uint16_t f32_to_bf16_rne(float f);

// u8 NHWC images [count][h][w][3], image index first..first+count-1:
// textured (base colour + three triangle gratings + per-pixel noise).
void generate_images(int h, int w, uint64_t seed, int64_t first, int count, uint8_t* out);

}  // namespace ds
