#include "profile.h"

#include <map>
#include <mutex>
#include <vector>

namespace mdnn {

namespace {
struct Pending {
    std::string tag;
    cudaEvent_t a, b;
    double work;
};
struct Stat {
    long count = 0;
    double ms = 0, work = 0;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Pending> g_pending;
std::map<std::string, Stat> g_stats;

void resolve_locked()
{
    for (auto& p : g_pending) {
        float ms = 0;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            auto& s = g_stats[p.tag];
            s.count++;
            s.ms += ms;
            s.work += p.work;
        }
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    g_pending.clear();
}
} // namespace

void prof_enable(bool on)
{
    std::lock_guard<std::mutex> lk(g_mu);
    g_on = on;
}

bool prof_enabled() { return g_on; }

bool prof_read(const std::string& tag, long* count, double* total_ms, double* total_work)
{
    std::lock_guard<std::mutex> lk(g_mu);
    resolve_locked();
    auto it = g_stats.find(tag);
    if (it == g_stats.end()) {
        *count = 0;
        *total_ms = 0;
        if (total_work)
            *total_work = 0;
        return false;
    }
    *count = it->second.count;
    *total_ms = it->second.ms;
    if (total_work)
        *total_work = it->second.work;
    return true;
}

void prof_reset()
{
    std::lock_guard<std::mutex> lk(g_mu);
    resolve_locked();
    g_stats.clear();
}

ProfScope::ProfScope(const char* tag, double work) : tag_(tag), work_(work)
{
    if (!g_on)
        return;
    cudaEventCreate(&start_);
    cudaEventRecord(start_, ctx().stream);
}

ProfScope::~ProfScope()
{
    if (!start_)
        return;
    cudaEvent_t stop;
    cudaEventCreate(&stop);
    cudaEventRecord(stop, ctx().stream);
    std::lock_guard<std::mutex> lk(g_mu);
    g_pending.push_back({tag_, start_, stop, work_});
}

} // namespace mdnn
