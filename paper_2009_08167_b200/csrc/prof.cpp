#include "prof.h"

#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.h"

namespace riga {

std::atomic<long long> g_launches{0};
bool g_pdl = [] {  // opt-in (RIGA_PDL=1): +8% aggregate in the probe, not in the slice timeline
  const char* e = std::getenv("RIGA_PDL");
  return e && e[0] == '1';
}();
thread_local long long t_launches = 0;

namespace {
struct Rec {
  int cat;
  cudaEvent_t a, b;
  double work;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

bool prof_on() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_on;
}

ProfScope::ProfScope(int c, cudaStream_t st, double w) : cat(c), s(st), work(w) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  e0 = get_event();
  cudaEventRecord(e0, s);
}

ProfScope::~ProfScope() {
  if (!e0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t e1 = get_event();
  cudaEventRecord(e1, s);
  g_recs.push_back(Rec{cat, e0, e1, work});
}

}  // namespace riga

extern "C" {

int riga_launch_count(int64_t* count) {
  if (!count) return RIGA_BAD_ARG;
  *count = riga::g_launches.load();
  return RIGA_OK;
}

int riga_set_pdl(int on) {
  riga::g_pdl = on != 0;
  return RIGA_OK;
}

int riga_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(riga::g_mu);
  riga::g_on = on != 0;
  return RIGA_OK;
}

// Per category: total device ms, total work (flops or bytes), scope count.
int riga_prof_read(double* ms, double* work, int64_t* scopes, int ncat) {
  std::lock_guard<std::mutex> lk(riga::g_mu);
  for (int c = 0; c < ncat; ++c) {
    ms[c] = 0;
    work[c] = 0;
    scopes[c] = 0;
  }
  for (auto& r : riga::g_recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.cat < ncat) {
      ms[r.cat] += t;
      work[r.cat] += r.work;
      scopes[r.cat] += 1;
    }
  }
  return RIGA_OK;
}

int riga_prof_reset(void) {
  std::lock_guard<std::mutex> lk(riga::g_mu);
  for (auto& r : riga::g_recs) {
    cudaEventSynchronize(r.b);
    riga::g_pool.push_back(r.a);
    riga::g_pool.push_back(r.b);
  }
  riga::g_recs.clear();
  return RIGA_OK;
}

}  // extern "C"
