// cfl file pairs and weight bundles (reference: cfl.hpp:15-142).
//
// Same on-disk format as the reference, byte for byte: `<base>.hdr` is a text
// header ("# Dimensions" then 16 dimensions), `<base>.cfl` the raw interleaved
// complex64 payload in column-major order.  A weights bundle is a directory
// of cfl pairs plus `manifest.txt` ("format 1", sorted meta keys, one
// "array <name>" line per array in sorted order), so identical contents give
// identical bytes.
//
// B200 side: payloads move between the file and device memory through two
// pinned staging buffers, chunk k+1 read from (or written to) the file while
// chunk k is on the copy engine; no pageable host copy of the whole array.
#include "cfl.h"

#include <algorithm>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>

namespace mdnn {

namespace {

constexpr size_t kChunk = size_t(16) << 20; // bytes per staging buffer

struct Staging {
    char* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    Staging()
    {
        for (int i = 0; i < 2; i++) {
            CUDA_CHECK(cudaMallocHost(&buf[i], kChunk));
            CUDA_CHECK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        }
    }
};

Staging& staging()
{
    // one pair per host thread (the ABI is synchronous per call)
    thread_local std::unique_ptr<Staging> s;
    if (!s)
        s = std::make_unique<Staging>();
    return *s;
}

} // namespace

Dims cfl_read_dims(const std::string& base)
{
    std::ifstream hdr(base + ".hdr");
    if (!hdr)
        throw IoError("missing file " + base + ".hdr");
    Dims dims;
    std::string line;
    while (std::getline(hdr, line)) {
        if (line.empty() || line[0] == '#')
            continue;
        std::istringstream is(line);
        long v;
        while (is >> v)
            dims.push_back(v);
        if (!dims.empty())
            break;
    }
    if (dims.empty())
        throw IoError("corrupt header in " + base + ".hdr");
    if (dims.size() > size_t(max_rank))
        throw IoError("corrupt header in " + base + ".hdr: too many dimensions");
    dims.resize(max_rank, 1);
    for (long d : dims)
        if (d < 1)
            throw IoError("corrupt header in " + base + ".hdr: nonpositive dimension");
    return dims;
}

DArray cfl_read(const std::string& base)
{
    const Dims dims = cfl_read_dims(base);
    std::ifstream cfl(base + ".cfl", std::ios::binary | std::ios::ate);
    if (!cfl)
        throw IoError("missing file " + base + ".cfl");
    const long expect = md_size(dims) * long(sizeof(cfloat));
    if (long(cfl.tellg()) != expect)
        throw IoError("corrupt file " + base + ".cfl: payload is " + std::to_string(long(cfl.tellg()))
                      + " bytes, header implies " + std::to_string(expect));
    cfl.seekg(0);
    DArray a(dims, false);
    auto& c = ctx();
    Staging& st = staging();
    char* dst = reinterpret_cast<char*>(a.buf->ptr);
    size_t off = 0;
    for (int k = 0; off < size_t(expect); k++) {
        const int s = k & 1;
        const size_t n = std::min(kChunk, size_t(expect) - off);
        CUDA_CHECK(cudaEventSynchronize(st.done[s])); // the copy that last used this buffer
        cfl.read(st.buf[s], std::streamsize(n));
        if (!cfl)
            throw IoError("short read from " + base + ".cfl");
        CUDA_CHECK(cudaMemcpyAsync(dst + off, st.buf[s], n, cudaMemcpyHostToDevice, c.stream));
        CUDA_CHECK(cudaEventRecord(st.done[s], c.stream));
        off += n;
    }
    return a;
}

void cfl_write(const std::string& base, const DArray& a0)
{
    const DArray a = to_layout(a0, Layout::CANON);
    Dims dims(max_rank, 1);
    for (size_t d = 0; d < a.dims.size() && d < size_t(max_rank); d++)
        dims[d] = a.dims[d];
    auto parent = std::filesystem::path(base).parent_path();
    if (!parent.empty())
        std::filesystem::create_directories(parent);
    {
        std::ofstream hdr(base + ".hdr");
        if (!hdr)
            throw IoError("cannot write " + base + ".hdr");
        hdr << "# Dimensions\n";
        for (int d = 0; d < max_rank; d++)
            hdr << dims[d] << (d + 1 < max_rank ? " " : "\n");
    }
    std::ofstream cfl(base + ".cfl", std::ios::binary);
    if (!cfl)
        throw IoError("cannot write " + base + ".cfl");
    auto& c = ctx();
    Staging& st = staging();
    const char* src = reinterpret_cast<const char*>(a.buf->ptr);
    const size_t total = size_t(md_size(a.dims)) * sizeof(cfloat);
    // D2H of chunk k+1 overlaps the file write of chunk k
    size_t off = 0, pend_off = 0, pend_n = 0;
    int pend = -1;
    for (int k = 0; off < total || pend >= 0; k++) {
        const int s = k & 1;
        size_t n = 0;
        if (off < total) {
            n = std::min(kChunk, total - off);
            CUDA_CHECK(cudaMemcpyAsync(st.buf[s], src + off, n, cudaMemcpyDeviceToHost, c.stream));
            CUDA_CHECK(cudaEventRecord(st.done[s], c.stream));
        }
        if (pend >= 0) {
            CUDA_CHECK(cudaEventSynchronize(st.done[pend]));
            cfl.write(st.buf[pend], std::streamsize(pend_n));
            if (!cfl)
                throw IoError("short write to " + base + ".cfl");
        }
        (void)pend_off;
        if (n) {
            pend = s;
            pend_off = off;
            pend_n = n;
            off += n;
        } else {
            pend = -1;
        }
    }
}

void WeightsBundle::save(const std::string& dir) const
{
    std::filesystem::create_directories(dir);
    std::ofstream mf(dir + "/manifest.txt");
    if (!mf)
        throw IoError("cannot write " + dir + "/manifest.txt");
    mf << "format 1\n";
    for (const auto& [k, v] : meta)
        mf << k << " " << v << "\n";
    for (const auto& [name, arr] : arrays) {
        mf << "array " << name << "\n";
        cfl_write(dir + "/" + name, arr);
    }
}

WeightsBundle WeightsBundle::load(const std::string& dir)
{
    std::ifstream mf(dir + "/manifest.txt");
    if (!mf)
        throw IoError("missing weights manifest in " + dir);
    WeightsBundle b;
    std::string line;
    while (std::getline(mf, line)) {
        if (line.empty())
            continue;
        const auto sp = line.find(' ');
        const std::string key = line.substr(0, sp);
        const std::string val = sp == std::string::npos ? "" : line.substr(sp + 1);
        if (key == "format") {
            if (val != "1")
                throw IoError("unsupported weights format " + val);
        } else if (key == "array") {
            b.arrays.emplace(val, cfl_read(dir + "/" + val));
        } else {
            b.meta[key] = val;
        }
    }
    return b;
}

std::string WeightsBundle::meta_or(const std::string& key, const std::string& fallback) const
{
    auto it = meta.find(key);
    return it == meta.end() ? fallback : it->second;
}

} // namespace mdnn
