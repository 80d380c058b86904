// Live per-kernel timing for bench.py's roofline: when enabled, tagged launch
// sites bracket their kernel with CUDA events on the library stream and add
// the launch's algorithmic work (bytes or flops, per the tag's definition in
// DESIGN.md); pairs are resolved lazily (no synchronisation on the launch path).
#pragma once

#include "core.h"

#include <string>

namespace mdnn {

void prof_enable(bool on);
bool prof_enabled();
// totals since the last reset for one tag: launches, summed device ms, summed work
bool prof_read(const std::string& tag, long* count, double* total_ms, double* total_work);
void prof_reset();

class ProfScope {
public:
    explicit ProfScope(const char* tag, double work = 0.0);
    ~ProfScope();
    ProfScope(const ProfScope&) = delete;
    ProfScope& operator=(const ProfScope&) = delete;

private:
    const char* tag_;
    double work_;
    cudaEvent_t start_ = nullptr;
};

} // namespace mdnn
