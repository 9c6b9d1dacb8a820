// C entry points into the UNMODIFIED reference control plane, linked with
// tape_gpu_sim.cpp — TEST INFRASTRUCTURE ONLY (tests/ and bench.py's
// reference leg). Scenario and catalog are read by the reference's own
// strict loaders (scenario.cpp, catalog.cpp).
#include <cstring>
#include <string>
#include <vector>

#include "dnnscaler/catalog.hpp"
#include "dnnscaler/gpu_sim.hpp"
#include "dnnscaler/harness.hpp"
#include "dnnscaler/perf_model.hpp"
#include "dnnscaler/profiler.hpp"
#include "dnnscaler/report.hpp"
#include "dnnscaler/scenario.hpp"
#include "tape_control.hpp"

using namespace dnnscaler;

namespace {

void set_err(char* err, size_t cap, const std::string& msg) {
  if (!err || cap == 0) return;
  std::strncpy(err, msg.c_str(), cap - 1);
  err[cap - 1] = '\0';
}

void set_mode(int mode, const double* tape, size_t tape_len) {
  auto& s = refseam::state();
  s.mode = mode == 3   ? refseam::Mode::kCallback
           : mode == 2 ? refseam::Mode::kReplay
                       : (mode == 1 ? refseam::Mode::kRecord : refseam::Mode::kStock);
  s.tape.clear();
  s.pos = 0;
  if (mode == 2) s.tape.assign(tape, tape + tape_len);
}

constexpr int kRecordWidth = 10;
constexpr int kSummaryWidth = 24;

void pack_summary(const JobSummary& s, double* o) {
  const double v[kSummaryWidth] = {static_cast<double>(s.job_id),
                                   s.approach == "multi-tenancy" ? 1.0 : 0.0,
                                   s.profiled ? 1.0 : 0.0,
                                   s.ti_batching,
                                   s.ti_mt,
                                   s.profiling_cost_ms,
                                   s.steady_knob.kind == KnobKind::kMultiTenancy ? 1.0 : 0.0,
                                   static_cast<double>(s.steady_knob.value),
                                   s.converged ? 1.0 : 0.0,
                                   static_cast<double>(s.knob_changes),
                                   static_cast<double>(s.settle_period),
                                   static_cast<double>(s.periods),
                                   s.duration_s,
                                   s.total_items,
                                   s.avg_throughput,
                                   s.steady_throughput,
                                   s.p95_overall_ms,
                                   s.slo_compliance,
                                   s.avg_power_w,
                                   s.power_efficiency,
                                   s.final_slo_ms,
                                   static_cast<double>(s.readaptations.size()),
                                   s.error.empty() ? 0.0 : 1.0,
                                   0.0};
  std::memcpy(o, v, sizeof(v));
}

}  // namespace

extern "C" {

int ref_record_width(void) { return kRecordWidth; }

// Callback seam (mode 3 of ref_run_job): latencies come from host functions.
void ref_set_callbacks(refseam::BatchFn batch, refseam::MtFn mt, refseam::ChangeFn change) {
  auto& s = refseam::state();
  s.batch_fn = batch;
  s.mt_fn = mt;
  s.change_fn = change;
}
int ref_summary_width(void) { return kSummaryWidth; }

// Runs job `job_index` of a scenario file through reference run_job.
// mode: 0 stock simulator, 1 stock + record tape, 2 replay `tape`.
// records_out: kRecordWidth doubles per period
//   [time_s, job_id, knob_kind, knob_value, p95, mean, throughput, power, slo, violated]
// readapt_out: pairs [at_s, periods]. Returns 0, or 2 if the job threw.
int ref_run_job(const char* scenario_path, int job_index, int mode, const double* tape,
                size_t tape_len, double* records_out, size_t rec_cap, size_t* n_rec,
                double* summary_out, double* tape_out, size_t tape_cap, size_t* tape_n,
                double* readapt_out, size_t readapt_cap, size_t* n_readapt, size_t* consumed,
                char* err, size_t err_cap) {
  try {
    const Scenario sc = load_scenario(scenario_path);
    const auto catalog = load_catalog(sc.catalog_path);
    set_mode(mode, tape, tape_len);
    const JobTrace t = run_job(sc, sc.jobs.at(static_cast<size_t>(job_index)), catalog);
    const auto& st = refseam::state();
    if (consumed) *consumed = st.pos;
    if (n_rec) *n_rec = t.records.size();
    for (size_t i = 0; records_out && i < t.records.size() && i < rec_cap; ++i) {
      const MetricsRecord& r = t.records[i];
      double* o = records_out + i * kRecordWidth;
      o[0] = r.time_s;
      o[1] = r.job_id;
      o[2] = r.knob.kind == KnobKind::kMultiTenancy ? 1.0 : 0.0;
      o[3] = r.knob.value;
      o[4] = r.p95_ms;
      o[5] = r.mean_ms;
      o[6] = r.throughput;
      o[7] = r.power_w;
      o[8] = r.slo_ms;
      o[9] = r.violated ? 1.0 : 0.0;
    }
    if (summary_out) pack_summary(t.summary, summary_out);
    if (tape_n) *tape_n = st.tape.size();
    if (tape_out && mode == 1)
      std::memcpy(tape_out, st.tape.data(), std::min(tape_cap, st.tape.size()) * sizeof(double));
    if (n_readapt) *n_readapt = t.summary.readaptations.size();
    for (size_t i = 0; readapt_out && i < t.summary.readaptations.size() && i < readapt_cap; ++i) {
      readapt_out[2 * i] = t.summary.readaptations[i].at_s;
      readapt_out[2 * i + 1] = t.summary.readaptations[i].periods;
    }
    set_mode(0, nullptr, 0);
    return 0;
  } catch (const std::exception& e) {
    set_mode(0, nullptr, 0);
    set_err(err, err_cap, e.what());
    return 2;
  }
}

// Reference profile() + decide() on a tape (GpuSim models are unused in replay).
// report_out: the 17 ProfileReport fields in declaration order.
int ref_profile_tape(const double* tape, size_t tape_len, int m, int n, int bpp, int abs_max_bs,
                     int max_mtl, double* report_out, int* approach, char* err, size_t err_cap) {
  try {
    set_mode(2, tape, tape_len);
    GpuSim gpu(BatchingModel{1.0, 1.0, 0.0}, MtModel{}, PowerModel{},
               GpuSim::Config{abs_max_bs, max_mtl}, 0);
    const ProfileReport r = profile(gpu, m, n, bpp);
    const double v[17] = {r.tput_base,
                          r.tput_batching,
                          r.tput_mt,
                          r.ti_batching,
                          r.ti_mt,
                          r.base_latency_ms,
                          r.probe_latency_batching_ms,
                          r.probe_latency_mt_ms,
                          static_cast<double>(r.m),
                          static_cast<double>(r.n),
                          static_cast<double>(r.batches_per_point),
                          r.base_elapsed_ms,
                          r.batching_elapsed_ms,
                          r.mt_elapsed_ms,
                          r.transition_ms,
                          r.profiling_cost_ms,
                          r.items_served};
    std::memcpy(report_out, v, sizeof(v));
    *approach = decide(r) == Approach::kMultiTenancy ? 1 : 0;
    set_mode(0, nullptr, 0);
    return 0;
  } catch (const std::exception& e) {
    set_mode(0, nullptr, 0);
    set_err(err, err_cap, e.what());
    return 2;
  }
}

// Whole scenario on the stock simulator, rendered with the reference's
// byte-stable writers (report.cpp:62-102). Returns needed sizes when short.
int ref_render_scenario(const char* scenario_path, char* csv, size_t csv_cap, size_t* csv_len,
                        char* json, size_t json_cap, size_t* json_len, char* err, size_t err_cap) {
  try {
    const Scenario sc = load_scenario(scenario_path);
    const auto catalog = load_catalog(sc.catalog_path);
    set_mode(0, nullptr, 0);
    const auto traces = run_scenario(sc, catalog);
    const std::string c = render_metrics_csv(traces);
    const std::string j = render_summary_json(sc, traces);
    *csv_len = c.size();
    *json_len = j.size();
    if (csv && csv_cap >= c.size()) std::memcpy(csv, c.data(), c.size());
    if (json && json_cap >= j.size()) std::memcpy(json, j.data(), j.size());
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_cap, e.what());
    return 2;
  }
}

// The reference CLI's profile subcommand body (tools/dnnscaler_main.cpp:88-99)
// on the stock simulator, rendered with render_profile_json (report.cpp).
int ref_render_profile(const char* catalog_path, const char* dnn_id, int m, int n, int batches,
                       uint64_t seed, double sigma, char* json, size_t json_cap, size_t* json_len,
                       char* err, size_t err_cap) {
  try {
    set_mode(0, nullptr, 0);
    const auto catalog = load_catalog(catalog_path);
    const auto& dnn = find_dnn(catalog, dnn_id);
    const double used_sigma = sigma >= 0.0 ? sigma : dnn.sigma.value_or(0.05);
    PowerModel pm;
    if (dnn.u1) pm.u1 = *dnn.u1;
    GpuSim gpu(calibrate_batching(dnn.batching_points, used_sigma),
               calibrate_mt(dnn.mt_points, used_sigma), pm, GpuSim::Config{}, seed);
    const auto report = profile(gpu, m, n, batches);
    const std::string j = render_profile_json(report, dnn.id, approach_name(decide(report)));
    *json_len = j.size();
    if (json && json_cap >= j.size()) std::memcpy(json, j.data(), j.size());
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_cap, e.what());
    return 2;
  }
}

// The reference CLI's sweep subcommand body (tools/dnnscaler_main.cpp:186-199)
// rendered with render_sweep_csv (report.cpp:104-119).
int ref_render_sweep(const char* catalog_path, const char* dnn_id, const int* bs, int n_bs,
                     const int* mtl, int n_mtl, int samples, uint64_t seed, double sigma, char* csv,
                     size_t cap, size_t* len, char* err, size_t err_cap) {
  try {
    const auto catalog = load_catalog(catalog_path);
    const auto& dnn = find_dnn(catalog, dnn_id);
    const double used_sigma = sigma >= 0.0 ? sigma : 0.0;
    const auto cells = combination_sweep(calibrate_batching(dnn.batching_points, used_sigma),
                                         calibrate_mt(dnn.mt_points, used_sigma),
                                         std::vector<int>(bs, bs + n_bs),
                                         std::vector<int>(mtl, mtl + n_mtl), samples, seed);
    const std::string c = render_sweep_csv(cells);
    *len = c.size();
    if (csv && cap >= c.size()) std::memcpy(csv, c.data(), c.size());
    return 0;
  } catch (const std::exception& e) {
    set_err(err, err_cap, e.what());
    return 2;
  }
}

}  // extern "C"

// The reference's generator (random.hpp:10-47), for pinning the oracles'
// restatements: n raw 64-bit draws of RandomStream(seed) (next_u64), then n
// gaussians of a fresh RandomStream(seed), and mix_seed(seed, 0..n-1).
extern "C" void ref_random(uint64_t seed, int n, uint64_t* u64_out, double* gauss_out,
                           uint64_t* mix_out) {
  dnnscaler::RandomStream a(seed), b(seed);
  for (int i = 0; i < n; ++i) {
    u64_out[i] = a.next_u64();
    gauss_out[i] = b.gaussian();
    mix_out[i] = dnnscaler::mix_seed(seed, static_cast<uint64_t>(i));
  }
}
