// Shared host-side helpers for the cprb C ABI.
#pragma once
#include <string>

#include "../../include/cpr_b200.h"

namespace cprb {
int set_error(int code, const std::string& msg);
double pairwise_sum(const double* a, int64_t n);
double segment_sum(const double* a, int64_t n);
}  // namespace cprb
