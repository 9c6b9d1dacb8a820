// Drop-in proof (test infrastructure): the reference's UNMODIFIED scenario
// loader, harness (run_scenario), Profiler, Scaler and report writers,
// compiled against include/dnnscaler_b200/drop_in/dnnscaler/gpu_sim.hpp and
// linked with libdnnscaler_b200.so — i.e. the reference serving on a B200.
//
//   ref_on_b200 <scenario.json> [metrics.csv] [summary.json]
//   (model: DNNSCALER_B200_MODEL, device: DNNSCALER_B200_DEVICE)
#include <cstdio>
#include <exception>
#include <stdexcept>

#include "dnnscaler/catalog.hpp"
#include "dnnscaler/harness.hpp"
#include "dnnscaler/report.hpp"
#include "dnnscaler/scenario.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s scenario.json [metrics.csv] [summary.json]\n", argv[0]);
    return 2;
  }
  try {
    const auto scenario = dnnscaler::load_scenario(argv[1]);
    const auto catalog = dnnscaler::load_catalog(scenario.catalog_path);
    const auto traces = dnnscaler::run_scenario(scenario, catalog);
    const std::string summary = dnnscaler::render_summary_json(scenario, traces);
    if (argc > 2) dnnscaler::write_file(argv[2], dnnscaler::render_metrics_csv(traces));
    if (argc > 3) dnnscaler::write_file(argv[3], summary);
    std::printf("%s\n", summary.c_str());
    return 0;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
