// prof.cu -- see prof.h.
#include <map>
#include <string>
#include <vector>

#include "amg.h"
#include "prof.h"

namespace amgb {

std::atomic<int64_t> g_launches{0};
thread_local int64_t t_launches = 0;
bool g_prof = false;

namespace {
struct Rec {
  const char* name;
  double bytes;
  cudaEvent_t a, b;
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
size_t g_pool_next = 0;
}  // namespace

cudaEvent_t prof_event() {
  if (g_pool_next == g_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_pool.push_back(e);
  }
  return g_pool[g_pool_next++];
}

const char* prof_name(const char* base, int b, int vt, int xt) {
  static std::map<std::string, std::string>* names = new std::map<std::string, std::string>();
  char buf[128];
  snprintf(buf, sizeof(buf), "%s_b%d_%s%s", base, b, vt == AMG_F32 ? "f32" : (vt == 2 /* AMG_F16, common.cuh */ ? "f16" : "f64"),
           xt < 0 ? "" : (xt == AMG_F32 ? "xf32" : "xf64"));
  auto it = names->find(buf);
  if (it == names->end()) it = names->emplace(buf, buf).first;
  return it->second.c_str();
}

void prof_record(const char* name, double bytes, cudaEvent_t a, cudaEvent_t b) { g_recs.push_back({name, bytes, a, b}); }

}  // namespace amgb

using namespace amgb;

extern "C" {

int64_t amg_kernel_launches(void) { return g_launches.load(); }

int amg_profile_begin(void) {
  g_recs.clear();
  g_pool_next = 0;
  g_prof = true;
  return AMG_OK;
}

// Aggregate per (kernel, bytes-per-launch): JSON list of
// {"kernel": name, "bytes": B, "launches": n, "total_ms": t}; returns the length written.
int64_t amg_profile_end(char* out, int64_t cap) {
  g_prof = false;
  cudaDeviceSynchronize();
  struct Agg {
    int64_t n = 0;
    double ms = 0.0;
  };
  std::map<std::pair<std::string, double>, Agg> agg;
  for (const Rec& r : g_recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    Agg& g = agg[{r.name, r.bytes}];
    g.n++;
    g.ms += ms;
  }
  std::string s = "[";
  char buf[512];
  bool first = true;
  for (auto& kv : agg) {
    snprintf(buf, sizeof(buf), "%s{\"kernel\": \"%s\", \"bytes\": %.0f, \"launches\": %lld, \"total_ms\": %.6f}",
             first ? "" : ", ", kv.first.first.c_str(), kv.first.second, (long long)kv.second.n, kv.second.ms);
    s += buf;
    first = false;
  }
  s += "]";
  g_recs.clear();
  g_pool_next = 0;
  if (out && cap > 0) {
    int64_t n = (int64_t)s.size() < cap - 1 ? (int64_t)s.size() : cap - 1;
    memcpy(out, s.data(), n);
    out[n] = 0;
  }
  return (int64_t)s.size();
}

}  // extern "C"
