// Mode switch of the tape seam (test infrastructure).
#pragma once

#include <cstddef>
#include <vector>

namespace refseam {

enum class Mode { kStock, kRecord, kReplay, kCallback };

// kCallback: every seam value comes from a host function (the CPU serving
// path of bench.py's reference arm: a CPU forward pass timed per call).
using BatchFn = double (*)(int bs);
using MtFn = double (*)(int mtl);
using ChangeFn = double (*)(int delta);

struct TapeState {
  Mode mode = Mode::kStock;
  std::vector<double> tape;
  size_t pos = 0;
  BatchFn batch_fn = nullptr;
  MtFn mt_fn = nullptr;
  ChangeFn change_fn = nullptr;
};

TapeState& state();

}  // namespace refseam
