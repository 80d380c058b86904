// Core types of the B200 host engine: errors, dims, per-device context
// (stream + stream-ordered memory pool) and DArray, the device md-array.
//
// Reference correspondences:
//   error taxonomy          common.hpp:15-26
//   Dims / default strides  common.hpp:35-68 (column-major, element strides)
//   MdArray<R>              mdarray.hpp:23-200 (shared buffer, immutable here)
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mdnn {

constexpr int max_rank = 16;
// BART dimension convention (recon.hpp:10-16)
constexpr int dim_x = 0, dim_y = 1, dim_chan = 2, dim_coil = 3, dim_maps = 4, dim_batch = 15;

class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
    virtual int code() const { return 1; }
};
#define MDNN_ERR(NAME, CODE)                                        \
    class NAME : public Error {                                     \
    public:                                                         \
        using Error::Error;                                         \
        int code() const override { return CODE; }                  \
    };
MDNN_ERR(ShapeError, 2)
MDNN_ERR(IoError, 3)
MDNN_ERR(ConfigError, 4)
MDNN_ERR(SolverError, 5)
MDNN_ERR(BoundsError, 6)
MDNN_ERR(AliasError, 7)
MDNN_ERR(StaleDerivativeError, 8)
MDNN_ERR(CudaError, 9)
#undef MDNN_ERR

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
void count_launch(); // every kernel launch site reports here (bench gpu_launches)
long launch_count();
#define CUDA_CHECK(x) ::mdnn::cuda_check((x), #x, __FILE__, __LINE__)
#define KERNEL_CHECK()                                                                \
    do {                                                                              \
        ::mdnn::count_launch();                                                       \
        ::mdnn::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);  \
    } while (0)

// Programmatic dependent launch (option "pdl", default on): every library kernel
// starts with MDNN_PDL_ENTRY() -- wait until the previous kernel in the stream has
// completed and its memory is visible, then let the next kernel be scheduled --
// and is launched with the programmatic-stream-serialisation attribute, so its
// launch and CTA start overlap the previous kernel's tail.
extern bool g_pdl;
template<class... KArgs, class... Args>
inline void pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}
#define MDNN_PDL_ENTRY() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

using Dims = std::vector<long>;
long md_size(const Dims& d);
std::string dims_to_string(const Dims& d);
void check_rank(const Dims& d);
Dims default_strides(const Dims& d);
Dims dims16(std::initializer_list<long> head);

using cfloat = float2; // interleaved complex64 on the device

// ---------------------------------------------------------------------------
// Per-device context: one compute stream per device (the replica's stream) and
// a stream-ordered pool allocator (cudaMallocAsync) that keeps freed blocks
// cached, so per-step allocations never reach the driver after warm-up.
// ---------------------------------------------------------------------------
struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr; // host->device input staging (overlaps the compute stream)
    int sm_count = 148;
    size_t smem_optin = 227 * 1024;
    size_t pool_reserved = 0; // bytes mapped into the stream-ordered pool up front
    // device-side error word: kernels OR in error bits (CG breakdown, ...)
    // which the host checks at synchronisation points (no per-iteration sync)
    unsigned* d_errflags = nullptr;
    unsigned* d_zero = nullptr; // a device word that stays 0 ("no imaginary part" flag for known-real operands)
    std::string err_detail;
};
Context& ctx();             // context of the current device (creates on first use)
// opt a kernel into the largest dynamic shared memory the device allows
// (opt-in limit minus the kernel's static shared memory); once per device
void allow_max_dyn_smem(const void* func);
// Map `bytes` of physical memory into the stream-ordered pool once (release
// threshold is infinite, so it stays).  Growing the pool while a training step
// is in flight costs 0.1-0.8 s stalls on B200 (measured); trainers reserve up
// front.
void reserve_pool(size_t bytes);
void set_device(int dev);
void sync_and_check();      // cudaStreamSynchronize + device error flags
enum ErrFlag : unsigned { ERRF_CG_BREAKDOWN = 1u, ERRF_CG_NONFINITE = 2u, ERRF_NONFINITE_GRAD = 4u, ERRF_PATTERN = 8u,
                        ERRF_GRID_BARRIER = 16u };

struct Buffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    int device = 0;
    bool owned = true;
    ~Buffer();
};

// Physical storage order of a feature-map array [X,Y,C,1,..,B]:
//   CANON  : reference column-major complex interleaved (x fastest)
//   CHLAST : per pixel 2*C floats (C real parts, then C imaginary parts),
//            pixels ordered x fastest, then y, then batch; the K-major operand
//            order of the tcgen05 implicit-GEMM convolution.  Only ever used on
//            internal graph edges between nodes that request it.
enum class Layout : uint8_t { CANON = 0, CHLAST = 1 };

struct DArray {
    Dims dims;
    std::shared_ptr<Buffer> buf;
    Layout layout = Layout::CANON;
    // values are already rounded RN to TF32 (set by producers that feed a
    // tensor-core convolution; lets the consumer skip its operand conversion)
    bool tf32 = false;
    // optional per-channel partial sums of these values written by the
    // producer kernel (tcgen05 conv epilogue): chstats_blocks blocks x
    // 2C real channels (re | im) x {sum, sum of squares}, doubles; lets a
    // batch-norm consumer skip its statistics pass
    std::shared_ptr<DArray> chstats;
    int chstats_blocks = 0;
    // 1: forward statistics [blk][2C][sum, sum sq]; 2: batch-norm backward
    // partials [blk][2C][3] for the consumer identified by chstats_tag
    int chstats_kind = 0;
    // the producer guarantees zero imaginary parts (real-channel split, Re, RBF,
    // real-weight arguments, convolutions of known-real operands); lets a consumer
    // skip its device-side imaginary-part scan
    bool known_real = false;
    const void* chstats_tag = nullptr;
    void drop_chstats()
    {
        chstats.reset();
        chstats_blocks = chstats_kind = 0;
        chstats_tag = nullptr;
    }

    DArray() = default;
    explicit DArray(Dims d, bool zero = true, Layout l = Layout::CANON);
    bool valid() const { return bool(buf); }
    long size() const { return md_size(dims); }
    int rank() const { return int(dims.size()); }
    cfloat* data() const { return static_cast<cfloat*>(buf->ptr); }
    float* fdata() const { return static_cast<float*>(buf->ptr); }
    void zero() const;
    DArray clone() const;
    static DArray scalar(float re, float im = 0.f);
    // non-owning view of caller memory (lifetime managed by the caller)
    static DArray view(cfloat* p, Dims d);
};

// Layout conversion (feature maps only; dims[2] is the channel axis)
DArray to_layout(const DArray& a, Layout l);

// Host <-> device copies for the C ABI (honour caller strides)
struct HostView {
    float* data;
    int device;
    Dims dims;
    Dims strides; // element strides
};
DArray import_array(const HostView& v);
// a dense device array on the current device is borrowed (no copy, not freed):
// for calls that do not retain their inputs past the call (standalone SENSE / CG)
DArray borrow_array(const HostView& v);
// asynchronous host->device copy on the context's copy stream into a fresh
// array; `done` is recorded on the copy stream after the copy (the caller
// makes the compute stream wait on it and keeps the host buffer alive until
// then).  Dense (default-stride) host views only.
DArray import_array_async(const HostView& v, cudaEvent_t done);
void export_array(const DArray& a, const HostView& v);
std::vector<std::complex<float>> to_host(const DArray& a);
DArray from_host(const Dims& d, const std::complex<float>* v);

} // namespace mdnn
