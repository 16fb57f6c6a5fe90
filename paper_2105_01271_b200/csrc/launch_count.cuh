// Per-thread count of kernels launched by this library (reported by the
// pipelines in info[SP_INFO_LAUNCHES] and by sp_launch_count()).
#pragma once
#include <stdint.h>
#include <algorithm>

namespace spb {
void count_launch(int n = 1);
int64_t launches();
}  // namespace spb
