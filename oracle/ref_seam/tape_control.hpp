// Mode switch of the tape seam (test infrastructure).
#pragma once

#include <cstddef>
#include <vector>

namespace refseam {

enum class Mode { kStock, kRecord, kReplay };

struct TapeState {
  Mode mode = Mode::kStock;
  std::vector<double> tape;
  size_t pos = 0;
};

TapeState& state();

}  // namespace refseam
