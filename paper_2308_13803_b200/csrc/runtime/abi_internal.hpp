// Shared between the C-ABI translation units.
#pragma once

#include <string>

#include "engine.hpp"

struct ds_backend {
  ds::Backend* impl;
};

// Sets the thread-local message returned by ds_last_error().
void ds_internal_set_error(const std::string& msg);
