// prof.cu -- see prof.h
#include <cstdlib>
#include <cstring>

#include "prof.h"

namespace tn {

Prof g_prof;

namespace {
struct ProfInit {
  ProfInit() {
    const char* e = std::getenv("TN_PROFILE");
    g_prof.on = e && std::strcmp(e, "0") != 0;
  }
} g_prof_init;
}  // namespace

cudaEvent_t Prof::get() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void Prof::flush() {
  for (auto& r : pending) {
    cudaEventSynchronize(r.b);
    float t = 0;
    cudaEventElapsedTime(&t, r.a, r.b);
    ms[r.cat] += t;
    count[r.cat] += 1;
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  pending.clear();
}

}  // namespace tn

// on: 0 = off, 1 = every category, > 1 = bit mask of the categories to record (e.g. only
// P_TC_KERNEL inside a timed region, keeping the event overhead off the other phases).
extern "C" int tn_debug_set_profile(int on) {
  tn::g_prof.flush();
  tn::g_prof.on = on != 0;
  tn::g_prof.mask = on > 1 ? (unsigned)on : ~0u;
  return 0;
}

extern "C" int tn_debug_profile(double* out_ms, long* out_count, int n, int reset) {
  tn::g_prof.flush();
  for (int i = 0; i < n && i < tn::P_NCAT; ++i) {
    out_ms[i] = tn::g_prof.ms[i];
    if (out_count) out_count[i] = tn::g_prof.count[i];
  }
  if (reset)
    for (int i = 0; i < tn::P_NCAT; ++i) {
      tn::g_prof.ms[i] = 0;
      tn::g_prof.count[i] = 0;
    }
  return tn::g_prof.on ? 1 : 0;
}
