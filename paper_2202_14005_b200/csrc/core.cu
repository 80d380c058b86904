#include "core.h"

#include <cstdlib>
#include "kernels.h"

#include <atomic>
#include <cstring>
#include <map>
#include <mutex>

namespace mdnn {

bool g_pdl = true;


void cuda_check(cudaError_t e, const char* what, const char* file, int line)
{
    if (e != cudaSuccess)
        throw CudaError(std::string("CUDA error '") + cudaGetErrorString(e) + "' in " + what + " (" + file + ":"
                        + std::to_string(line) + ")");
}

static std::atomic<long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long launch_count() { return g_launches.load(); }

long md_size(const Dims& d)
{
    long n = 1;
    for (long v : d)
        n *= v;
    return n;
}

std::string dims_to_string(const Dims& d)
{
    std::string s = "[";
    for (size_t i = 0; i < d.size(); i++)
        s += (i ? "," : "") + std::to_string(d[i]);
    return s + "]";
}

void check_rank(const Dims& d)
{
    if (d.empty() || d.size() > size_t(max_rank))
        throw ShapeError("rank must be in 1.." + std::to_string(max_rank) + ", got " + std::to_string(d.size()));
    for (long v : d)
        if (v < 1)
            throw ShapeError("dimensions must be positive, got " + dims_to_string(d));
}

Dims default_strides(const Dims& d)
{
    check_rank(d);
    Dims s(d.size());
    long acc = 1;
    for (size_t i = 0; i < d.size(); i++) {
        s[i] = acc;
        acc *= d[i];
    }
    return s;
}

Dims dims16(std::initializer_list<long> head)
{
    Dims d(head);
    d.resize(max_rank, 1);
    return d;
}

// ---------------------------------------------------------------------------

namespace {
std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<Context>> g_ctx;
thread_local int t_device = -1;

Context* make_ctx(int dev)
{
    auto c = std::make_unique<Context>();
    c->device = dev;
    CUDA_CHECK(cudaSetDevice(dev));
    CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    cudaDeviceProp prop;
    CUDA_CHECK(cudaGetDeviceProperties(&prop, dev));
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    // keep freed blocks cached in the default pool (stream-ordered allocator)
    cudaMemPool_t pool;
    CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thresh = UINT64_MAX;
    CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    // optional up-front reservation (MDNN_POOL_RESERVE_GB): the pool maps its
    // physical memory once instead of growing while steps are in flight
    if (const char* r = std::getenv("MDNN_POOL_RESERVE_GB")) {
        const size_t bytes = size_t(std::atof(r) * 1e9);
        if (bytes) {
            void* p = nullptr;
            CUDA_CHECK(cudaMallocAsync(&p, bytes, c->stream));
            CUDA_CHECK(cudaFreeAsync(p, c->stream));
            CUDA_CHECK(cudaStreamSynchronize(c->stream));
            c->pool_reserved = bytes;
        }
    }
    CUDA_CHECK(cudaMalloc(&c->d_errflags, 64));
    CUDA_CHECK(cudaMemset(c->d_errflags, 0, 64));
    CUDA_CHECK(cudaMalloc(&c->d_zero, 16));
    CUDA_CHECK(cudaMemset(c->d_zero, 0, 16));
    return c.release();
}
} // namespace

Context& ctx()
{
    if (t_device < 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess)
            dev = 0;
        t_device = dev;
    }
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    auto it = g_ctx.find(t_device);
    if (it == g_ctx.end())
        it = g_ctx.emplace(t_device, std::unique_ptr<Context>(make_ctx(t_device))).first;
    else
        cudaSetDevice(t_device);
    return *it->second;
}

void allow_max_dyn_smem(const void* func)
{
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, bool> done;
    auto& c = ctx();
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(c.device, func);
    if (done.count(key))
        return;
    cudaFuncAttributes fa;
    CUDA_CHECK(cudaFuncGetAttributes(&fa, func));
    int dyn = int(c.smem_optin) - int(fa.sharedSizeBytes);
    CUDA_CHECK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    done[key] = true;
}

void set_device(int dev)
{
    CUDA_CHECK(cudaSetDevice(dev));
    t_device = dev;
    (void)ctx();
}

void sync_and_check()
{
    auto& c = ctx();
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    unsigned flags = 0;
    CUDA_CHECK(cudaMemcpy(&flags, c.d_errflags, sizeof(unsigned), cudaMemcpyDeviceToHost));
    if (flags) {
        CUDA_CHECK(cudaMemset(c.d_errflags, 0, sizeof(unsigned)));
        if (flags & ERRF_PATTERN) // raised before any result is used, as the reference's check (recon.hpp:67-77)
            throw ConfigError("sense: sampling pattern must be binary");
        if (flags & ERRF_CG_BREAKDOWN)
            throw SolverError("cg: numerical breakdown (p^H A p <= 0 or non-finite)");
        if (flags & ERRF_CG_NONFINITE)
            throw SolverError("cg: non-finite residual");
        if (flags & ERRF_NONFINITE_GRAD)
            throw SolverError("non-finite gradient");
        if (flags & ERRF_GRID_BARRIER)
            throw CudaError("A^H A: fused CG update grid barrier timed out (CTAs not co-resident)");
        throw SolverError("device error flags set");
    }
}

Buffer::~Buffer()
{
    if (ptr && owned) {
        auto& c = ctx();
        cudaFreeAsync(ptr, c.stream);
    }
}

DArray::DArray(Dims d, bool zero_init, Layout l) : dims(std::move(d)), layout(l)
{
    check_rank(dims);
    auto& c = ctx();
    buf = std::make_shared<Buffer>();
    buf->bytes = size_t(md_size(dims)) * sizeof(cfloat);
    buf->device = c.device;
    CUDA_CHECK(cudaMallocAsync(&buf->ptr, buf->bytes, c.stream));
    if (zero_init)
        zero();
}

void DArray::zero() const
{
    CUDA_CHECK(cudaMemsetAsync(buf->ptr, 0, buf->bytes, ctx().stream));
}

DArray DArray::clone() const
{
    DArray o(dims, false, layout);
    CUDA_CHECK(cudaMemcpyAsync(o.buf->ptr, buf->ptr, buf->bytes, cudaMemcpyDeviceToDevice, ctx().stream));
    return o;
}

namespace {
__global__ void k_set_scalar(float2* p, float re, float im) {
    MDNN_PDL_ENTRY(); *p = float2{re, im}; }
} // namespace

DArray DArray::scalar(float re, float im)
{
    // value travels as a kernel argument: no host staging, no stream synchronisation
    DArray a(Dims{1}, false);
    pdl_launch(k_set_scalar, 1, 1, 0, ctx().stream, a.data(), re, im);
    KERNEL_CHECK();
    return a;
}

void reserve_pool(size_t bytes)
{
    auto& c = ctx();
    if (c.pool_reserved >= bytes)
        return;
    void* p = nullptr;
    CUDA_CHECK(cudaMallocAsync(&p, bytes, c.stream));
    CUDA_CHECK(cudaFreeAsync(p, c.stream));
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    c.pool_reserved = bytes;
}

DArray DArray::view(cfloat* p, Dims d)
{
    DArray a;
    a.dims = std::move(d);
    a.buf = std::make_shared<Buffer>();
    a.buf->ptr = p;
    a.buf->bytes = size_t(md_size(a.dims)) * sizeof(cfloat);
    a.buf->device = ctx().device;
    a.buf->owned = false;
    return a;
}

DArray to_layout(const DArray& a, Layout l)
{
    if (a.layout == l)
        return a;
    if (a.dims.size() < 3 || a.dims[2] == 1) {
        // one channel: CANON and CHLAST coincide byte for byte -> relabel, no copy
        DArray o = a;
        o.layout = l;
        return o;
    }
    DArray o(a.dims, false, l);
    o.tf32 = a.tf32;
    launch_layout_convert(a, o);
    return o;
}

static bool is_default(const Dims& d, const Dims& s) { return s.empty() || s == default_strides(d); }

DArray import_array(const HostView& v)
{
    DArray a(v.dims, false);
    auto& c = ctx();
    const size_t bytes = a.buf->bytes;
    if (is_default(v.dims, v.strides)) {
        CUDA_CHECK(cudaMemcpyAsync(a.buf->ptr, v.data, bytes,
                                   v.device >= 0 ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
        if (v.device < 0)
            CUDA_CHECK(cudaStreamSynchronize(c.stream));
        return a;
    }
    if (v.device >= 0) {
        launch_strided_copy(v.dims, a.data(), default_strides(v.dims), reinterpret_cast<const cfloat*>(v.data),
                            v.strides);
        return a;
    }
    // host gather into a packed staging buffer
    std::vector<std::complex<float>> tmp(size_t(md_size(v.dims)));
    Dims idx(v.dims.size(), 0);
    for (size_t k = 0; k < tmp.size(); k++) {
        long off = 0;
        for (size_t i = 0; i < idx.size(); i++)
            off += idx[i] * v.strides[i];
        tmp[k] = {v.data[2 * off], v.data[2 * off + 1]};
        for (size_t i = 0; i < idx.size(); i++) {
            if (++idx[i] < v.dims[i])
                break;
            idx[i] = 0;
        }
    }
    CUDA_CHECK(cudaMemcpyAsync(a.buf->ptr, tmp.data(), bytes, cudaMemcpyHostToDevice, c.stream));
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    return a;
}

DArray borrow_array(const HostView& v)
{
    if (v.device != ctx().device || !is_default(v.dims, v.strides))
        return import_array(v);
    check_rank(v.dims);
    DArray a;
    a.dims = v.dims;
    a.buf = std::make_shared<Buffer>();
    a.buf->ptr = const_cast<float*>(v.data);
    a.buf->bytes = size_t(md_size(v.dims)) * sizeof(cfloat);
    a.buf->device = v.device;
    a.buf->owned = false;
    return a;
}

DArray import_array_async(const HostView& v, cudaEvent_t done)
{
    if (v.device >= 0 || !is_default(v.dims, v.strides))
        throw ConfigError("stage_data: a dense host array is required");
    check_rank(v.dims);
    auto& c = ctx();
    DArray a;
    a.dims = v.dims;
    a.buf = std::make_shared<Buffer>();
    a.buf->bytes = size_t(md_size(v.dims)) * sizeof(cfloat);
    a.buf->device = c.device;
    // allocated in the copy stream's order; freed later on the compute stream,
    // which only touches it after waiting on `done`
    CUDA_CHECK(cudaMallocAsync(&a.buf->ptr, a.buf->bytes, c.copy_stream));
    CUDA_CHECK(cudaMemcpyAsync(a.buf->ptr, v.data, a.buf->bytes, cudaMemcpyHostToDevice, c.copy_stream));
    CUDA_CHECK(cudaEventRecord(done, c.copy_stream));
    return a;
}

void export_array(const DArray& a0, const HostView& v)
{
    if (v.dims != a0.dims)
        throw ShapeError("output buffer dims " + dims_to_string(v.dims) + " != " + dims_to_string(a0.dims));
    DArray a = to_layout(a0, Layout::CANON);
    auto& c = ctx();
    if (is_default(v.dims, v.strides)) {
        CUDA_CHECK(cudaMemcpyAsync(v.data, a.buf->ptr, a.buf->bytes,
                                   v.device >= 0 ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.stream));
        if (v.device < 0)
            sync_and_check();
        return;
    }
    if (v.device >= 0) {
        launch_strided_copy(v.dims, reinterpret_cast<cfloat*>(v.data), v.strides, a.data(), default_strides(v.dims));
        return;
    }
    auto tmp = to_host(a);
    Dims idx(v.dims.size(), 0);
    for (size_t k = 0; k < tmp.size(); k++) {
        long off = 0;
        for (size_t i = 0; i < idx.size(); i++)
            off += idx[i] * v.strides[i];
        v.data[2 * off] = tmp[k].real();
        v.data[2 * off + 1] = tmp[k].imag();
        for (size_t i = 0; i < idx.size(); i++) {
            if (++idx[i] < v.dims[i])
                break;
            idx[i] = 0;
        }
    }
}

std::vector<std::complex<float>> to_host(const DArray& a0)
{
    DArray a = to_layout(a0, Layout::CANON);
    std::vector<std::complex<float>> h(size_t(a.size()));
    CUDA_CHECK(cudaMemcpyAsync(h.data(), a.buf->ptr, a.buf->bytes, cudaMemcpyDeviceToHost, ctx().stream));
    sync_and_check();
    return h;
}

DArray from_host(const Dims& d, const std::complex<float>* v)
{
    DArray a(d, false);
    CUDA_CHECK(cudaMemcpyAsync(a.buf->ptr, v, a.buf->bytes, cudaMemcpyHostToDevice, ctx().stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx().stream));
    return a;
}

} // namespace mdnn
