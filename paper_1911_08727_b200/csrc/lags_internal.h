// Host-side helpers shared by the translation units of liblagsb200.so (not part of the ABI).
#pragma once
#include <string>

namespace lags {
// Record the thread-local message returned by lags_last_error() and return `code`.
int host_fail(int code, const std::string& msg);
// Add to the process-wide kernel launch counter (lags_kernel_launches).
void host_count_launches(int n);
}  // namespace lags
