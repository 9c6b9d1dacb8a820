// Domain statistics, noise stream, analytic model and the non-device seams.
// Restated from reference domain.cpp, random.hpp, perf_model.cpp and
// gpu_sim.cpp with the same operation order (file:line per function).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "../../../include/dnnscaler_b200/control.hpp"

namespace ds {

const char* knob_kind_name(KnobKind kind) {  // domain.cpp:10-12
  return kind == KnobKind::kBatching ? "batching" : "multi-tenancy";
}

double percentile(const std::vector<double>& samples, double q) {  // domain.cpp:14-24
  if (samples.empty()) throw std::invalid_argument("no samples");
  if (!(q > 0.0) || q > 1.0) throw std::invalid_argument("quantile out of range");
  const size_t n = samples.size();
  // Nearest rank ceil(q*n); the 1e-9 keeps an exact integer rank from rounding up.
  size_t rank = static_cast<size_t>(std::ceil(q * static_cast<double>(n) - 1e-9));
  rank = std::clamp<size_t>(rank, 1, n);
  std::vector<double> work(samples);
  std::nth_element(work.begin(), work.begin() + static_cast<std::ptrdiff_t>(rank - 1), work.end());
  return work[rank - 1];
}

double throughput_improvement(double tput_new, double tput_base) {  // domain.cpp:26-29
  if (!(tput_base > 0.0)) throw std::invalid_argument("invalid baseline");
  return (tput_new - tput_base) / tput_base * 100.0;
}

LatencyWindow::LatencyWindow(size_t capacity) : capacity_(capacity) {  // domain.cpp:31-33
  if (capacity_ == 0) throw std::invalid_argument("window capacity must be positive");
}

void LatencyWindow::push(double latency_ms) {  // domain.cpp:35-38
  if (samples_.size() == capacity_) samples_.pop_front();
  samples_.push_back(latency_ms);
}

void LatencyWindow::clear() { samples_.clear(); }

std::vector<double> LatencyWindow::to_vector() const {
  return std::vector<double>(samples_.begin(), samples_.end());
}

double LatencyWindow::p95() const { return percentile(to_vector(), 0.95); }

double LatencyWindow::mean() const {  // domain.cpp:48-52
  if (samples_.empty()) throw std::invalid_argument("no samples");
  return std::accumulate(samples_.begin(), samples_.end(), 0.0) /
         static_cast<double>(samples_.size());
}

// ------------------------------------------------------------------ random
uint64_t mix_seed_u64(uint64_t seed, uint64_t salt) {  // random.hpp:10-15
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double NoiseStream::uniform() {  // random.hpp:22
  return static_cast<double>(eng_() >> 11) * 0x1.0p-53;
}

double NoiseStream::gaussian() {  // random.hpp:26-38
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  double u1 = uniform();
  while (u1 <= 0.0) u1 = uniform();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  constexpr double kPi = 3.14159265358979323846;
  spare_ = r * std::sin(2.0 * kPi * u2);
  have_spare_ = true;
  return r * std::cos(2.0 * kPi * u2);
}

// ------------------------------------------------------------------ perf model
namespace {

double point_latency(const std::pair<int, double>& p) {  // perf_model.cpp:11-15
  if (p.first < 1) throw std::invalid_argument("invalid batch size");
  if (!(p.second > 0.0)) throw std::invalid_argument("invalid throughput");
  return 1000.0 * static_cast<double>(p.first) / p.second;
}

double noise(double sigma, NoiseStream& rng) {  // perf_model.cpp:17-20
  if (sigma <= 0.0) return 1.0;
  return std::exp(sigma * rng.gaussian());
}

}  // namespace

BatchingModel calibrate_batching(const std::vector<std::pair<int, double>>& points,
                                 double sigma) {  // perf_model.cpp:24-46
  if (points.size() < 2) throw std::invalid_argument("need at least two batching points");
  double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
  for (const auto& p : points) {
    const double x = static_cast<double>(p.first);
    const double y = point_latency(p);
    sx += x;
    sy += y;
    sxx += x * x;
    sxy += x * y;
  }
  const double n = static_cast<double>(points.size());
  const double det = n * sxx - sx * sx;
  if (std::abs(det) < 1e-12 * n * sxx) throw std::invalid_argument("singular calibration system");
  const double b = (n * sxy - sx * sy) / det;
  double a = (sy - b * sx) / n;
  if (a < 0.0 && a > -1e-9) a = 0.0;
  if (a < 0.0) throw std::invalid_argument("calibration gives negative base cost");
  if (!(b > 0.0)) throw std::invalid_argument("calibration gives non-increasing batch cost");
  return BatchingModel{a, b, sigma};
}

MtModel calibrate_mt(const std::vector<std::pair<int, double>>& points,
                     double sigma) {  // perf_model.cpp:48-68
  double tput1 = 0.0, tput_hi = 0.0;
  int hi = 0;
  for (const auto& p : points) {
    if (p.first < 1) throw std::invalid_argument("invalid instance count");
    if (!(p.second > 0.0)) throw std::invalid_argument("invalid throughput");
    if (p.first == 1) tput1 = p.second;
    if (p.first > hi) {
      hi = p.first;
      tput_hi = p.second;
    }
  }
  if (tput1 <= 0.0) throw std::invalid_argument("missing single-instance point");
  if (hi < 2) throw std::invalid_argument("missing multi-instance point");
  MtModel m;
  m.l1_ms = 1000.0 / tput1;
  m.capacity = std::clamp(tput_hi / tput1, 1.0, static_cast<double>(hi));
  m.sigma = sigma;
  return m;
}

double mean_batch_latency(const BatchingModel& m, int bs) {  // perf_model.cpp:70-73
  if (bs < 1) throw std::invalid_argument("invalid batch size");
  return m.a_ms + m.b_ms * static_cast<double>(bs);
}

double mean_mt_latency(const MtModel& m, int mtl) {  // perf_model.cpp:75-78
  if (mtl < 1) throw std::invalid_argument("invalid instance count");
  return m.l1_ms * std::max(1.0, static_cast<double>(mtl) / m.capacity);
}

double batch_latency(const BatchingModel& m, int bs, NoiseStream& rng) {
  return mean_batch_latency(m, bs) * noise(m.sigma, rng);
}

double mt_latency(const MtModel& m, int mtl, NoiseStream& rng) {
  return mean_mt_latency(m, mtl) * noise(m.sigma, rng);
}

double utilization(const PowerModel& pm, const Knob& knob,
                   const BatchingModel& bm) {  // perf_model.cpp:88-96
  if (knob.value < 1) throw std::invalid_argument("invalid knob value");
  if (knob.kind == KnobKind::kMultiTenancy)
    return std::min(1.0, pm.u1 * static_cast<double>(knob.value));
  const double total = bm.a_ms + bm.b_ms * static_cast<double>(knob.value);
  const double busy = total > 0.0 ? bm.b_ms * static_cast<double>(knob.value) / total : 1.0;
  return std::min(1.0, pm.u1 * busy * pm.s_bs);
}

double power_draw(const PowerModel& pm, double u) {  // perf_model.cpp:98-101
  const double c = std::clamp(u, 0.0, 1.0);
  return pm.p_idle_w + (pm.p_max_w - pm.p_idle_w) * c;
}

// ------------------------------------------------------------------ seams
double Seam::set_mtl(int target) {  // gpu_sim.cpp:39-46
  if (target < 1) throw std::invalid_argument("cannot terminate last instance");
  if (target > config().max_mtl) throw std::invalid_argument("instance limit exceeded");
  double total = 0.0;
  while (mtl() < target) total += apply_instance_change(1);
  while (mtl() > target) total += apply_instance_change(-1);
  return total;
}

void Seam::run_batches(int bs, int count, double* out) {
  for (int i = 0; i < count; ++i) out[i] = run_batch(bs);
}

void Seam::run_mt_requests(int count, double* out) {
  for (int i = 0; i < count; ++i) out[i] = run_mt_request();
}

namespace {

void check_instance_change(int delta, int mtl, int max_mtl) {  // gpu_sim.cpp:28-32
  if (delta != 1 && delta != -1) throw std::invalid_argument("instance changes are single steps");
  const int target = mtl + delta;
  if (target < 1) throw std::invalid_argument("cannot terminate last instance");
  if (target > max_mtl) throw std::invalid_argument("instance limit exceeded");
}

}  // namespace

AnalyticSeam::AnalyticSeam(BatchingModel bm, MtModel mm, Config config, uint64_t seed)
    : bm_(bm), mm_(mm), config_(config), rng_(seed) {
  if (config_.abs_max_bs < 1 || config_.max_mtl < 1)
    throw std::invalid_argument("invalid device limits");
}

double AnalyticSeam::run_batch(int bs) {  // gpu_sim.cpp:13-18
  if (bs < 1 || bs > config_.abs_max_bs) throw std::invalid_argument("invalid batch size");
  const double lat = batch_latency(bm_, bs, rng_);
  clock_ms_ += lat;
  return lat;
}

double AnalyticSeam::run_mt_request() {  // gpu_sim.cpp:20-24
  const double lat = mt_latency(mm_, mtl_, rng_);
  clock_ms_ += lat / static_cast<double>(mtl_);
  return lat;
}

double AnalyticSeam::apply_instance_change(int delta) {  // gpu_sim.cpp:26-37
  if (delta == 0) return 0.0;
  check_instance_change(delta, mtl_, config_.max_mtl);
  const double delay = delta > 0 ? mm_.launch_delay_ms : mm_.terminate_delay_ms;
  clock_ms_ += delay;
  mtl_ += delta;
  return delay;
}

ReplaySeam::ReplaySeam(std::vector<double> tape, Config config)
    : tape_(std::move(tape)), config_(config) {
  if (config_.abs_max_bs < 1 || config_.max_mtl < 1)
    throw std::invalid_argument("invalid device limits");
}

double ReplaySeam::next() {
  if (pos_ >= tape_.size()) throw std::runtime_error("replay tape exhausted");
  return tape_[pos_++];
}

double ReplaySeam::run_batch(int bs) {
  if (bs < 1 || bs > config_.abs_max_bs) throw std::invalid_argument("invalid batch size");
  const double lat = next();
  clock_ms_ += lat;
  return lat;
}

double ReplaySeam::run_mt_request() {
  const double lat = next();
  clock_ms_ += lat / static_cast<double>(mtl_);
  return lat;
}

double ReplaySeam::apply_instance_change(int delta) {
  if (delta == 0) return 0.0;
  check_instance_change(delta, mtl_, config_.max_mtl);
  const double delay = next();
  clock_ms_ += delay;
  mtl_ += delta;
  return delay;
}

bool ReplaySeam::energy_reading(double* mj, double* wall_ms, double* power_w) {
  if (energy_.empty()) return false;
  if (epos_ + 3 > energy_.size()) throw std::runtime_error("energy tape exhausted");
  *mj = energy_[epos_++];
  *wall_ms = energy_[epos_++];
  *power_w = energy_[epos_++];
  return true;
}

bool RecordingSeam::energy_reading(double* mj, double* wall_ms, double* power_w) {
  if (!inner_.energy_reading(mj, wall_ms, power_w)) return false;
  energy_.push_back(*mj);
  energy_.push_back(*wall_ms);
  energy_.push_back(*power_w);
  return true;
}

double RecordingSeam::run_batch(int bs) {
  const double v = inner_.run_batch(bs);
  tape_.push_back(v);
  return v;
}

double RecordingSeam::run_mt_request() {
  const double v = inner_.run_mt_request();
  tape_.push_back(v);
  return v;
}

double RecordingSeam::apply_instance_change(int delta) {
  const double v = inner_.apply_instance_change(delta);
  if (delta != 0) tape_.push_back(v);
  return v;
}

void RecordingSeam::run_batches(int bs, int count, double* out) {
  inner_.run_batches(bs, count, out);
  tape_.insert(tape_.end(), out, out + count);
}

void RecordingSeam::run_mt_requests(int count, double* out) {
  inner_.run_mt_requests(count, out);
  tape_.insert(tape_.end(), out, out + count);
}

}  // namespace ds
