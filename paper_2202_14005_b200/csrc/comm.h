// Data-parallel gradient exchange inside the library: an NCCL
// communicator per replica, resolved from libnccl.so.2 at run time (the one
// torch already mapped when it is in the process, else the system library),
// so a C++ caller of the C ABI can train data-parallel without Python.
//
// The payload is the trainer's flat fp32 buffer [weight gradients | moving
// statistics] (train.h); buckets of it are all-reduced (sum) on a dedicated
// comm stream while the reverse sweep is still running (Trainer::on_final).
#pragma once

#include "core.h"

#include <cstdint>

namespace mdnn {

constexpr int nccl_id_bytes = 128; // NCCL_UNIQUE_ID_BYTES

bool nccl_available(std::string* why = nullptr);
void nccl_unique_id(uint8_t* out);

class Comm {
public:
    Comm(const uint8_t* id, int nranks, int rank);
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    int nranks() const { return nranks_; }
    int rank() const { return rank_; }
    cudaStream_t stream() const { return stream_; }
    // in-place sum over ranks of n floats at p, enqueued on the comm stream
    void allreduce_sum(float* p, long n);

private:
    void* comm_ = nullptr;
    cudaStream_t stream_ = nullptr;
    int nranks_ = 1, rank_ = 0;
};

} // namespace mdnn
