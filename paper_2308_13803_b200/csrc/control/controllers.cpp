// Profiler (Eqs. 3-5), Scaler (Algorithm 1) and the Clipper baseline.
// Restated from reference profiler.cpp, scaler.cpp, clipper.cpp.
#include <algorithm>
#include <cmath>
#include <map>
#include <stdexcept>
#include <vector>

#include "../../../include/dnnscaler_b200/control.hpp"

namespace ds {

const char* approach_name(Approach a) {  // profiler.cpp:9-11
  return a == Approach::kBatching ? "batching" : "multi-tenancy";
}

// profiler.cpp:13-55. The probes go through the seam's window calls (one
// window per probe point); the values are then folded in call order so the
// sums are the same double additions the reference performs.
ProfileReport profile(Seam& gpu, int m, int n, int batches_per_point) {
  if (m < 2) throw std::invalid_argument("batch probe needs m > 1");
  if (n < 2) throw std::invalid_argument("instance probe needs n > 1");
  if (m > gpu.config().abs_max_bs) throw std::invalid_argument("batch probe above device limit");
  if (n > gpu.config().max_mtl) throw std::invalid_argument("instance probe above device limit");
  if (batches_per_point < 1) throw std::invalid_argument("batches_per_point must be positive");
  if (gpu.mtl() != 1) throw std::invalid_argument("profiling starts from a single instance");

  ProfileReport r;
  r.m = m;
  r.n = n;
  r.batches_per_point = batches_per_point;
  const double start_ms = gpu.clock_ms();
  const double w = static_cast<double>(batches_per_point);
  std::vector<double> lat(static_cast<size_t>(batches_per_point));

  gpu.run_batches(1, batches_per_point, lat.data());
  double base_sum = 0.0;
  for (double v : lat) base_sum += v;
  r.base_elapsed_ms = base_sum;
  r.base_latency_ms = base_sum / w;
  r.tput_base = w * 1000.0 / base_sum;

  gpu.run_batches(m, batches_per_point, lat.data());
  double batch_sum = 0.0;
  for (double v : lat) batch_sum += v;
  r.batching_elapsed_ms = batch_sum;
  r.probe_latency_batching_ms = batch_sum / w;
  r.tput_batching = w * static_cast<double>(m) * 1000.0 / batch_sum;

  r.transition_ms += gpu.set_mtl(n);
  const int requests = batches_per_point * n;
  std::vector<double> mt(static_cast<size_t>(requests));
  gpu.run_mt_requests(requests, mt.data());
  double mt_sum = 0.0;
  for (double v : mt) mt_sum += v;
  r.mt_elapsed_ms = mt_sum / static_cast<double>(n);
  r.probe_latency_mt_ms = mt_sum / static_cast<double>(requests);
  r.tput_mt = static_cast<double>(requests) * 1000.0 / r.mt_elapsed_ms;
  r.transition_ms += gpu.set_mtl(1);

  r.ti_batching = throughput_improvement(r.tput_batching, r.tput_base);
  r.ti_mt = throughput_improvement(r.tput_mt, r.tput_base);
  r.profiling_cost_ms = gpu.clock_ms() - start_ms;
  r.items_served = w * (1.0 + static_cast<double>(m)) + static_cast<double>(requests);
  return r;
}

Approach decide(const ProfileReport& report, double eps) {  // profiler.cpp:57-64
  if (eps < 0.0) throw std::invalid_argument("eps must be non-negative");
  if (report.ti_batching > report.ti_mt + eps) return Approach::kBatching;
  if (report.ti_mt > report.ti_batching + eps) return Approach::kMultiTenancy;
  return report.probe_latency_batching_ms <= report.probe_latency_mt_ms ? Approach::kBatching
                                                                       : Approach::kMultiTenancy;
}

BandVerdict band_verdict(double p95_ms, double slo_ms, double alpha) {  // scaler.cpp:9-15
  if (!(slo_ms > 0.0)) throw std::invalid_argument("invalid slo");
  if (!(alpha > 0.0) || alpha > 1.0) throw std::invalid_argument("alpha out of range");
  if (p95_ms > slo_ms) return BandVerdict::kAbove;
  if (p95_ms < alpha * slo_ms) return BandVerdict::kBelow;
  return BandVerdict::kInBand;
}

BatchScalerState make_batch_scaler(int abs_max_bs, size_t window_capacity) {  // scaler.cpp:17-26
  if (abs_max_bs < 1) throw std::invalid_argument("invalid batch size limit");
  BatchScalerState st;
  st.min_bs = 1;
  st.max_bs = abs_max_bs;
  st.current_bs = 1;
  st.abs_max_bs = abs_max_bs;
  st.window = LatencyWindow(window_capacity);
  return st;
}

// scaler.cpp:28-63: pseudo-binary search (Algorithm 1, batching branch).
BatchDecision batch_step(BatchScalerState& st, double p95_ms, double slo_ms, double alpha) {
  BatchDecision d;
  d.verdict = band_verdict(p95_ms, slo_ms, alpha);
  d.previous_bs = st.current_bs;
  if (d.verdict == BandVerdict::kInBand) {
    st.infeasible = false;
  } else if (d.verdict == BandVerdict::kBelow) {
    // Headroom: search the upper half up to the absolute cap.
    st.infeasible = false;
    st.min_bs = st.current_bs;
    st.max_bs = st.abs_max_bs;
    st.current_bs = (st.min_bs + st.max_bs + 1) / 2;
  } else if (st.current_bs == 1) {
    st.infeasible = true;  // violating at size 1: keep probing for a later relaxation
  } else if (st.current_bs == st.min_bs) {
    // Violation at the lower bound: restart the search below it.
    st.max_bs = st.current_bs;
    st.min_bs = 1;
    st.current_bs = (st.min_bs + st.max_bs) / 2;
  } else {
    st.max_bs = st.current_bs;
    st.current_bs = (st.min_bs + st.max_bs) / 2;
  }
  d.new_bs = st.current_bs;
  d.changed = d.new_bs != d.previous_bs;
  if (d.changed) st.window.clear();
  return d;
}

MtScalerState make_mt_scaler(int initial_mtl, int max_mtl, size_t window_capacity) {
  // scaler.cpp:65-74
  if (max_mtl < 1) throw std::invalid_argument("invalid instance limit");
  if (initial_mtl < 1 || initial_mtl > max_mtl)
    throw std::invalid_argument("initial instance count out of range");
  MtScalerState st;
  st.mtl = initial_mtl;
  st.max_mtl = max_mtl;
  st.window = LatencyWindow(window_capacity);
  return st;
}

// scaler.cpp:76-109: one instance at a time; a removal right after an
// addition arms the damper, which holds through headroom until the verdict
// returns to the band.
MtDecision mt_step(MtScalerState& st, double p95_ms, double slo_ms, double alpha) {
  MtDecision d;
  d.verdict = band_verdict(p95_ms, slo_ms, alpha);
  d.previous_mtl = st.mtl;
  MtAction action = MtAction::kHold;
  if (d.verdict == BandVerdict::kInBand) {
    st.damped = false;
  } else if (d.verdict == BandVerdict::kBelow) {
    if (!st.damped && st.mtl < st.max_mtl) action = MtAction::kAdd;
  } else if (st.mtl > 1) {
    action = MtAction::kRemoveLast;
    st.damped = st.last_action == MtAction::kAdd;
  } else {
    st.damped = false;
    d.infeasible = true;
  }
  if (action == MtAction::kAdd) st.mtl += 1;
  if (action == MtAction::kRemoveLast) st.mtl -= 1;
  if (action != MtAction::kHold) st.window.clear();
  st.last_action = action;
  d.action = action;
  d.new_mtl = st.mtl;
  return d;
}

// scaler.cpp:111-128
int mt_init(double lat1_ms, double latn_ms, int n_probe,
            const std::vector<std::vector<double>>& catalog_rows, double slo_ms, int max_mtl,
            const CompletionOptions& opts) {
  if (!(lat1_ms > 0.0) || !(latn_ms > 0.0)) throw std::invalid_argument("invalid probe latency");
  if (n_probe < 2) throw std::invalid_argument("instance probe needs n > 1");
  if (max_mtl < 1) throw std::invalid_argument("invalid instance limit");
  const int width = std::max(max_mtl, n_probe);
  if (catalog_rows.empty()) {
    // No donors: unobserved levels are assumed to sit exactly at the SLO,
    // which the strict pick_mtl test rejects.
    std::vector<double> sparse(static_cast<size_t>(width), slo_ms);
    sparse[0] = lat1_ms;
    sparse[static_cast<size_t>(n_probe) - 1] = latn_ms;
    return pick_mtl(sparse, slo_ms, max_mtl);
  }
  const std::map<int, double> observed{{1, lat1_ms}, {n_probe, latn_ms}};
  return pick_mtl(estimate_row(catalog_rows, observed, width, opts), slo_ms, max_mtl);
}

ClipperState make_clipper(int abs_max_bs, size_t window_capacity) {  // clipper.cpp:9-15
  if (abs_max_bs < 1) throw std::invalid_argument("invalid batch size limit");
  ClipperState st;
  st.abs_max_bs = abs_max_bs;
  st.window = LatencyWindow(window_capacity);
  return st;
}

ClipperDecision clipper_step(ClipperState& st, double p95_ms, double slo_ms) {  // clipper.cpp:17-35
  if (!(slo_ms > 0.0)) throw std::invalid_argument("invalid slo");
  ClipperDecision d;
  d.previous_bs = st.current_bs;
  d.violated = p95_ms > slo_ms;
  if (d.violated) {
    st.current_bs =
        std::max(1, static_cast<int>(std::floor(st.current_bs * (1.0 - st.backoff))));
    st.converged = true;
  } else if (!st.converged) {
    st.current_bs = std::min(st.abs_max_bs, st.current_bs + st.step);
  }
  d.new_bs = st.current_bs;
  d.changed = d.new_bs != d.previous_bs;
  if (d.changed) st.window.clear();
  return d;
}

}  // namespace ds
