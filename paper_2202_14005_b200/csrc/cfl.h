// cfl file pairs and weight bundles on device arrays (reference cfl.hpp:15-142).
#pragma once

#include "core.h"

#include <map>
#include <string>

namespace mdnn {

// header dims of <base>.hdr, padded to 16 (IoError on missing / corrupt files)
Dims cfl_read_dims(const std::string& base);
// <base>.cfl into a new device array (pinned double-buffered staging)
DArray cfl_read(const std::string& base);
// device array (any layout) to <base>.hdr / <base>.cfl
void cfl_write(const std::string& base, const DArray& a);

struct WeightsBundle {
    std::map<std::string, std::string> meta;
    std::map<std::string, DArray> arrays;

    void save(const std::string& dir) const;
    static WeightsBundle load(const std::string& dir);
    std::string meta_or(const std::string& key, const std::string& fallback) const;
};

} // namespace mdnn
