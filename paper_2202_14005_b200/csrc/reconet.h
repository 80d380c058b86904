// reconet driver (cli.hpp:52-265) on device arrays.
#pragma once

#include "core.h"

#include <string>

namespace mdnn {

struct ReconetOptions {
    std::string network = "varnet";
    bool do_train = false, do_apply = false;
    bool normalize = false;
    std::string pattern_file, init_weights;
    long iterations = -1, filters = -1, kernel = -1, rbf = -1;
    long layers = -1, cg_iter = -1;
    long epochs = 10, batch_size = 10;
    double lr = -1;
    std::string optimizer;
    uint64_t seed = 42;
    bool verbose = true;
    std::string kspace_file, coils_file, weights_dir, target_file;
};

// estimate_pattern (cli.hpp:28-50): a phase-encode line is sampled iff any
// coil of any item has a nonzero value on it
DArray estimate_pattern(const DArray& kspace);

// cmd_reconet (cli.hpp:94-265)
int run_reconet(ReconetOptions o);

} // namespace mdnn
