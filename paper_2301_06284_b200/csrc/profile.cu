// profile.cu -- optional phase timing with CUDA events on the caller's stream
// (the bench reads the dominant kernel's live duration from here).
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"

namespace rgnn {

struct PhaseRec {
  cudaEvent_t a, b;
  std::string name;
};
static std::mutex g_mu;
static bool g_on = false;
static std::vector<PhaseRec> g_pending;
static std::vector<cudaEvent_t> g_pool;
static std::map<std::string, std::pair<double, int64_t>> g_acc;

static cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

bool profile_on() { return g_on; }

void* profile_begin(const char* name, cudaStream_t s) {
  if (!g_on) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  PhaseRec r{get_event(), get_event(), name};
  cudaEventRecord(r.a, s);
  g_pending.push_back(r);
  return reinterpret_cast<void*>(g_pending.size());  // 1-based index
}

void profile_end(void* tok, cudaStream_t s) {
  if (!tok) return;
  std::lock_guard<std::mutex> lk(g_mu);
  size_t i = reinterpret_cast<size_t>(tok) - 1;
  if (i < g_pending.size()) cudaEventRecord(g_pending[i].b, s);
}

}  // namespace rgnn

extern "C" {

void rgnn_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(rgnn::g_mu);
  rgnn::g_on = on != 0;
}

int rgnn_profile_read(char* names, double* ms, int64_t* count, int max) {
  using namespace rgnn;
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& r : g_pending) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    auto& acc = g_acc[r.name];
    acc.first += t;
    acc.second += 1;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_pending.clear();
  int n = 0;
  for (auto& kv : g_acc) {
    if (n >= max) break;
    if (names) {
      memset(names + 32 * n, 0, 32);
      strncpy(names + 32 * n, kv.first.c_str(), 31);
    }
    if (ms) ms[n] = kv.second.first;
    if (count) count[n] = kv.second.second;
    ++n;
  }
  g_acc.clear();
  return n;
}

}  // extern "C"
