// Host control plane of the B200 framework: the reference's Profiler,
// Scaler, matrix completion, Clipper baseline and closed-loop harness,
// restated over an abstract device seam so the same code drives the real
// B200 backend, the reference's analytic model, or a recorded tape.
//
// Every function keeps the reference's semantics, error messages and
// floating-point operation order (cited per declaration), compiled with
// -ffp-contract=off, so Profiler decisions and Scaler trajectories replay
// bit-exactly against the reference on the same latency tape.
#pragma once

#include <cstddef>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <string>
#include <utility>
#include <vector>

namespace ds {

// ------------------------------------------------------------- domain
// reference domain.hpp:12-86, domain.cpp:10-52

enum class KnobKind { kBatching, kMultiTenancy };
const char* knob_kind_name(KnobKind kind);

struct Knob {
  KnobKind kind = KnobKind::kBatching;
  int value = 1;
  bool operator==(const Knob&) const = default;
};

struct DnnProfile {
  std::string id;
  double params_millions = 0.0;
  double mflops = 0.0;
  std::vector<std::pair<int, double>> batching_points;
  std::vector<std::pair<int, double>> mt_points;
  std::optional<double> sigma;
  std::optional<double> u1;
};

struct SloStep {
  double at_s = 0.0;
  double slo_ms = 0.0;
};

struct JobSpec {
  int job_id = 0;
  std::string dnn_id;
  std::string dataset_tag;
  double slo_ms = 0.0;
  double duration_s = 0.0;
  std::vector<SloStep> slo_schedule;
};

struct MetricsRecord {
  double time_s = 0.0;
  int job_id = 0;
  Knob knob;
  double p95_ms = 0.0;
  double mean_ms = 0.0;
  double throughput = 0.0;
  double power_w = 0.0;
  double slo_ms = 0.0;
  bool violated = false;
};

double percentile(const std::vector<double>& samples, double q);  // domain.cpp:14-24
double throughput_improvement(double tput_new, double tput_base);  // domain.cpp:26-29

class LatencyWindow {  // domain.cpp:31-52
 public:
  explicit LatencyWindow(size_t capacity = 100);
  void push(double latency_ms);
  void clear();
  bool full() const { return samples_.size() == capacity_; }
  size_t size() const { return samples_.size(); }
  size_t capacity() const { return capacity_; }
  std::vector<double> to_vector() const;
  double p95() const;
  double mean() const;

 private:
  size_t capacity_;
  std::deque<double> samples_;
};

// ------------------------------------------------------------- random
// reference random.hpp:10-47 (also used for synthetic weights/images)
uint64_t mix_seed_u64(uint64_t seed, uint64_t salt);

class NoiseStream {
 public:
  explicit NoiseStream(uint64_t seed = 0) : eng_(seed) {}
  double uniform();
  double gaussian();
  uint64_t next_u64() { return eng_(); }

 private:
  std::mt19937_64 eng_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

// ------------------------------------------------------------- perf model
// reference perf_model.hpp:13-52, perf_model.cpp:11-101. On the B200 path
// it no longer produces latencies; it calibrates catalog curves (donor rows
// for mt_init, harness power/ramp accounting) and backs AnalyticSeam.
struct BatchingModel {
  double a_ms = 0.0;
  double b_ms = 0.0;
  double sigma = 0.05;
};

struct MtModel {
  double l1_ms = 0.0;
  double capacity = 1.0;
  double sigma = 0.05;
  double launch_delay_ms = 500.0;
  double terminate_delay_ms = 100.0;
};

struct PowerModel {
  double p_idle_w = 50.0;
  double p_max_w = 250.0;
  double u1 = 0.12;
  double s_bs = 1.0;
};

BatchingModel calibrate_batching(const std::vector<std::pair<int, double>>& points,
                                 double sigma = 0.05);
MtModel calibrate_mt(const std::vector<std::pair<int, double>>& points, double sigma = 0.05);
double mean_batch_latency(const BatchingModel& m, int bs);
double mean_mt_latency(const MtModel& m, int mtl);
double batch_latency(const BatchingModel& m, int bs, NoiseStream& rng);
double mt_latency(const MtModel& m, int mtl, NoiseStream& rng);
double utilization(const PowerModel& pm, const Knob& knob, const BatchingModel& bm);
double power_draw(const PowerModel& pm, double utilization);

// ------------------------------------------------------------- seam
// The device seam: the method set of reference GpuSim (gpu_sim.hpp:13-50).
class Seam {
 public:
  struct Config {
    int abs_max_bs = 128;
    int max_mtl = 10;
  };
  virtual ~Seam() = default;
  virtual double run_batch(int bs) = 0;
  virtual double run_mt_request() = 0;
  virtual double apply_instance_change(int delta) = 0;
  // Ramps one instance at a time (gpu_sim.cpp:39-46).
  virtual double set_mtl(int target);
  virtual int mtl() const = 0;
  virtual double clock_ms() const = 0;
  virtual Config config() const = 0;
  // One control window at a fixed knob; equal to `count` single calls.
  virtual void run_batches(int bs, int count, double* out);
  virtual void run_mt_requests(int count, double* out);
  // Measured board power: the device's cumulative
  // energy counter (mJ), a wall clock (ms) and the current power draw (W).
  // Seams without a power meter (analytic, plain replay) return false and the
  // harness keeps the reference PowerModel (perf_model.cpp:88-101).
  virtual bool energy_reading(double* mj, double* wall_ms, double* power_w) {
    (void)mj;
    (void)wall_ms;
    (void)power_w;
    return false;
  }
};

// The reference's simulated GPU (gpu_sim.cpp:7-46): analytic latency with
// lognormal noise, virtual clock, fixed 500/100 ms ramps.
class AnalyticSeam : public Seam {
 public:
  AnalyticSeam(BatchingModel bm, MtModel mm, Config config, uint64_t seed);
  double run_batch(int bs) override;
  double run_mt_request() override;
  double apply_instance_change(int delta) override;
  int mtl() const override { return mtl_; }
  double clock_ms() const override { return clock_ms_; }
  Config config() const override { return config_; }

 private:
  BatchingModel bm_;
  MtModel mm_;
  Config config_;
  NoiseStream rng_;
  double clock_ms_ = 0.0;
  int mtl_ = 1;
};

// Replays a recorded tape: each call consumes the next value (one per
// run_batch / run_mt_request / non-zero instance change), with the
// reference's validation and clock arithmetic.
class ReplaySeam : public Seam {
 public:
  ReplaySeam(std::vector<double> tape, Config config);
  double run_batch(int bs) override;
  double run_mt_request() override;
  double apply_instance_change(int delta) override;
  int mtl() const override { return mtl_; }
  double clock_ms() const override { return clock_ms_; }
  Config config() const override { return config_; }
  size_t consumed() const { return pos_; }
  // Recorded (mJ, wall ms, W) triples of a device run; replays its measured power.
  void set_energy_tape(std::vector<double> tape) { energy_ = std::move(tape); }
  bool energy_reading(double* mj, double* wall_ms, double* power_w) override;

 private:
  double next();
  std::vector<double> energy_;
  size_t epos_ = 0;
  std::vector<double> tape_;
  size_t pos_ = 0;
  Config config_;
  double clock_ms_ = 0.0;
  int mtl_ = 1;
};

// Records every value an inner seam returns, in call order.
class RecordingSeam : public Seam {
 public:
  explicit RecordingSeam(Seam& inner) : inner_(inner) {}
  double run_batch(int bs) override;
  double run_mt_request() override;
  double apply_instance_change(int delta) override;
  int mtl() const override { return inner_.mtl(); }
  double clock_ms() const override { return inner_.clock_ms(); }
  Config config() const override { return inner_.config(); }
  void run_batches(int bs, int count, double* out) override;
  void run_mt_requests(int count, double* out) override;
  bool energy_reading(double* mj, double* wall_ms, double* power_w) override;
  const std::vector<double>& tape() const { return tape_; }
  const std::vector<double>& energy_tape() const { return energy_; }

 private:
  Seam& inner_;
  std::vector<double> tape_;
  std::vector<double> energy_;
};

// ------------------------------------------------------------- profiler
// reference profiler.hpp:7-38, profiler.cpp:13-64
enum class Approach { kBatching, kMultiTenancy };
const char* approach_name(Approach approach);

struct ProfileReport {
  double tput_base = 0.0;
  double tput_batching = 0.0;
  double tput_mt = 0.0;
  double ti_batching = 0.0;
  double ti_mt = 0.0;
  double base_latency_ms = 0.0;
  double probe_latency_batching_ms = 0.0;
  double probe_latency_mt_ms = 0.0;
  int m = 32;
  int n = 8;
  int batches_per_point = 10;
  double base_elapsed_ms = 0.0;
  double batching_elapsed_ms = 0.0;
  double mt_elapsed_ms = 0.0;
  double transition_ms = 0.0;
  double profiling_cost_ms = 0.0;
  double items_served = 0.0;
};

ProfileReport profile(Seam& gpu, int m = 32, int n = 8, int batches_per_point = 10);
Approach decide(const ProfileReport& report, double eps = 0.5);

// ------------------------------------------------------------- matrix completion
// reference matrix_completion.hpp:12-53, matrix_completion.cpp:19-299
struct LatencyMatrix {
  std::vector<std::vector<double>> values;
  std::vector<std::vector<uint8_t>> observed;
  size_t rows() const { return values.size(); }
  size_t cols() const { return values.empty() ? 0 : values.front().size(); }
  void validate() const;
};

struct CompletionOptions {
  int rank = 2;
  int max_iters = 200;
  double tol = 1e-8;
  double ridge = 1e-6;
  uint64_t seed = 0;
};

struct CompletionResult {
  std::vector<std::vector<double>> estimates;
  int rank_used = 0;
  int iterations = 0;
  bool converged = false;
  double residual = 0.0;
};

CompletionResult complete(const LatencyMatrix& m, const CompletionOptions& opts = {});
std::vector<double> estimate_row(const std::vector<std::vector<double>>& catalog_rows,
                                 const std::map<int, double>& observed, int n,
                                 const CompletionOptions& opts = {});
int pick_mtl(const std::vector<double>& estimates, double slo_ms, int max_mtl);

// ------------------------------------------------------------- scaler
// reference scaler.hpp:11-70, scaler.cpp:9-128
enum class BandVerdict { kBelow, kInBand, kAbove };
BandVerdict band_verdict(double p95_ms, double slo_ms, double alpha = 0.85);

struct BatchScalerState {
  int min_bs = 1;
  int max_bs = 128;
  int current_bs = 1;
  int abs_max_bs = 128;
  bool infeasible = false;
  LatencyWindow window{100};
};
BatchScalerState make_batch_scaler(int abs_max_bs, size_t window_capacity = 100);

struct BatchDecision {
  BandVerdict verdict = BandVerdict::kInBand;
  int previous_bs = 1;
  int new_bs = 1;
  bool changed = false;
};
BatchDecision batch_step(BatchScalerState& st, double p95_ms, double slo_ms, double alpha = 0.85);

enum class MtAction { kHold, kAdd, kRemoveLast };

struct MtScalerState {
  int mtl = 1;
  int max_mtl = 10;
  MtAction last_action = MtAction::kHold;
  bool damped = false;
  LatencyWindow window{100};
};
MtScalerState make_mt_scaler(int initial_mtl, int max_mtl, size_t window_capacity = 100);

struct MtDecision {
  BandVerdict verdict = BandVerdict::kInBand;
  MtAction action = MtAction::kHold;
  int previous_mtl = 1;
  int new_mtl = 1;
  bool infeasible = false;
};
MtDecision mt_step(MtScalerState& st, double p95_ms, double slo_ms, double alpha = 0.85);

int mt_init(double lat1_ms, double latn_ms, int n_probe,
            const std::vector<std::vector<double>>& catalog_rows, double slo_ms, int max_mtl,
            const CompletionOptions& opts = {});

// ------------------------------------------------------------- clipper
// reference clipper.hpp:10-28, clipper.cpp:9-35 (comparison baseline)
struct ClipperState {
  int current_bs = 1;
  int abs_max_bs = 128;
  int step = 4;
  double backoff = 0.10;
  bool converged = false;
  LatencyWindow window{100};
};
ClipperState make_clipper(int abs_max_bs, size_t window_capacity = 100);

struct ClipperDecision {
  int previous_bs = 1;
  int new_bs = 1;
  bool changed = false;
  bool violated = false;
};
ClipperDecision clipper_step(ClipperState& st, double p95_ms, double slo_ms);

// ------------------------------------------------------------- harness
// reference scenario.hpp:11-35, harness.hpp:14-80, harness.cpp:16-386
enum class ControllerKind { kDnnScaler, kClipper, kStaticKnob };
const char* controller_name(ControllerKind kind);

struct Scenario {
  std::vector<JobSpec> jobs;
  ControllerKind controller = ControllerKind::kDnnScaler;
  Knob static_knob;
  uint64_t seed = 42;
  double alpha = 0.85;
  int m = 32;
  int n = 8;
  int abs_max_bs = 128;
  int max_mtl = 10;
  size_t window = 100;
  double sigma = 0.05;
};

struct Readaptation {
  double at_s = 0.0;
  int periods = -1;
};

struct JobSummary {
  int job_id = 0;
  std::string dnn_id;
  std::string controller;
  std::string approach;
  bool profiled = false;
  double ti_batching = 0.0;
  double ti_mt = 0.0;
  double profiling_cost_ms = 0.0;
  Knob steady_knob;
  bool converged = false;
  int knob_changes = 0;
  int settle_period = 0;
  int periods = 0;
  double duration_s = 0.0;
  double total_items = 0.0;
  double avg_throughput = 0.0;
  double steady_throughput = 0.0;
  double p95_overall_ms = 0.0;
  double slo_compliance = 0.0;
  double avg_power_w = 0.0;
  double power_efficiency = 0.0;
  // true: avg_power_w / power_efficiency / records' power_w come from the
  // device's measured energy counter (board average power over the job's wall
  // time; efficiency = items per joule), else from the reference PowerModel
  bool power_measured = false;
  double final_slo_ms = 0.0;
  std::vector<Readaptation> readaptations;
  std::string error;
};

struct JobTrace {
  JobSpec spec;
  std::vector<MetricsRecord> records;
  JobSummary summary;
  ProfileReport report;
  std::vector<double> tape;  // every seam value, in call order
  std::vector<double> energy_tape;  // (mJ, wall ms, W) per energy reading (device runs)
  std::vector<double> latencies;  // all served latencies, in order
};

// Makes the seam a job runs on. The analytic factory reproduces the
// reference exactly (GpuSim(bm, mm, pm, cfg, mix_seed(seed, job_id))).
using SeamFactory = std::function<std::unique_ptr<Seam>(
    const Scenario&, const JobSpec&, const BatchingModel&, const MtModel&)>;
SeamFactory analytic_seam_factory();

// B x MT grid on the analytic model (reference harness.cpp:356-386): per
// cell `samples` draws of the instance's mean batch latency x lognormal noise
// from one RandomStream(seed) in bs-major order.
struct SweepCell {
  int bs = 0, mtl = 0;
  double mean_ms = 0.0, p95_ms = 0.0, throughput = 0.0;
};
std::vector<SweepCell> combination_sweep(const BatchingModel& bm, const MtModel& mm,
                                         const std::vector<int>& bs_list,
                                         const std::vector<int>& mtl_list, int samples,
                                         uint64_t seed);

std::vector<std::vector<double>> derive_mt_rows(const std::vector<DnnProfile>& catalog,
                                                const std::string& exclude_id, int width);
const DnnProfile& find_dnn(const std::vector<DnnProfile>& catalog, const std::string& id);
void validate_scenario(const Scenario& s);

JobTrace run_job(const Scenario& scenario, const JobSpec& job,
                 const std::vector<DnnProfile>& catalog, const SeamFactory& make_seam);

// The same job, driven one control period at a time (used by the bench to
// time steady-state periods): start() profiles and seeds the knob, step()
// applies due SLO steps and serves one period, finish() summarises.
class JobSession {
 public:
  JobSession(const Scenario& scenario, const JobSpec& job, const std::vector<DnnProfile>& catalog,
             const SeamFactory& make_seam);
  ~JobSession();
  void start();
  const MetricsRecord& step();
  bool done() const;  // seam clock reached the job duration
  Knob knob() const;
  double clock_ms() const;
  JobTrace finish();

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};
std::vector<JobTrace> run_scenario(const Scenario& scenario,
                                   const std::vector<DnnProfile>& catalog,
                                   const SeamFactory& make_seam);

}  // namespace ds
