// prof.h -- launch accounting: a global launch counter (always on) and, when enabled
// through amg_profile_begin(), a CUDA-event pair around every launch with the launch's
// algorithmic bytes, aggregated per kernel by amg_profile_end().
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace amgb {

extern std::atomic<int64_t> g_launches;      // all library launches of the process
extern thread_local int64_t t_launches;      // this thread's (graph capture counts its own)
extern bool g_prof;

void prof_record(const char* name, double bytes, cudaEvent_t a, cudaEvent_t b);
// stable C string for a kernel label (interned)
const char* prof_name(const char* base, int b, int vt, int xt);
cudaEvent_t prof_event();

class ProfScope {
 public:
  ProfScope(const char* name, double bytes, cudaStream_t s) : name_(name), bytes_(bytes), s_(s) {
    ++g_launches;
    ++t_launches;
    if (g_prof) {
      a_ = prof_event();
      cudaEventRecord(a_, s_);
    }
  }
  ~ProfScope() {
    if (g_prof) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, s_);
      prof_record(name_, bytes_, a_, b);
    }
  }

 private:
  const char* name_;
  double bytes_;
  cudaStream_t s_;
  cudaEvent_t a_ = nullptr;
};

}  // namespace amgb
