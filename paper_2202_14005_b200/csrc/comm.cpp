#include "comm.h"

#include <nccl.h>

#include <dlfcn.h>

#include <cstring>
#include <mutex>

namespace mdnn {

namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string why;
    bool ok = false;
};

const NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // the soname torch's bundled NCCL registers, so an already-mapped copy is reused
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen(libnccl.so.2): ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.get_unique_id && api.init_rank && api.all_reduce && api.destroy && api.error_string;
        if (!api.ok)
            api.why = "libnccl.so.2 lacks the NCCL 2 entry points";
    });
    return api;
}

void check(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess)
        throw CudaError(std::string(what) + ": " + nccl().error_string(r));
}

const NcclApi& need()
{
    const NcclApi& a = nccl();
    if (!a.ok)
        throw ConfigError("NCCL unavailable: " + a.why);
    return a;
}

} // namespace

bool nccl_available(std::string* why)
{
    const NcclApi& a = nccl();
    if (why)
        *why = a.why;
    return a.ok;
}

void nccl_unique_id(uint8_t* out)
{
    static_assert(sizeof(ncclUniqueId) == nccl_id_bytes, "NCCL unique id size");
    ncclUniqueId id;
    check(need().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, nccl_id_bytes);
}

Comm::Comm(const uint8_t* id, int nranks, int rank) : nranks_(nranks), rank_(rank)
{
    if (nranks < 1 || rank < 0 || rank >= nranks)
        throw ConfigError("communicator: rank " + std::to_string(rank) + " of " + std::to_string(nranks));
    const NcclApi& a = need();
    ncclUniqueId uid;
    std::memcpy(&uid, id, nccl_id_bytes);
    ctx(); // the device of this replica is current
    ncclComm_t c = nullptr;
    check(a.init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
    comm_ = c;
    CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
}

Comm::~Comm()
{
    if (stream_)
        cudaStreamSynchronize(stream_);
    if (comm_)
        nccl().destroy(static_cast<ncclComm_t>(comm_));
    if (stream_)
        cudaStreamDestroy(stream_);
}

void Comm::allreduce_sum(float* p, long n)
{
    if (n <= 0)
        return;
    check(nccl().all_reduce(p, p, size_t(n), ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm_), stream_),
          "ncclAllReduce");
}

} // namespace mdnn
