// phases.cu -- per-phase instrumentation of the hot path (SURVEY 8(d)
// "per-phase events for fill, exchange, K3a, K3b and dt"; SURVEY 5 NVTX).
//
// Every phase the library enqueues is bracketed by an NVTX range (host
// timeline; free when no tool is attached) and, while phase timing is on
// (orcha_set_phase_timing), by a pair of CUDA events recorded on the phase's
// stream.  orcha_phase_times synchronizes on the recorded events and returns
// the summed device time per phase since the previous query.  Timing is off
// by default, so the timed bench loop records no extra events.
#include <nvtx3/nvToolsExt.h>

#include <mutex>
#include <vector>

#include "orcha_internal.h"

namespace orcha {

static const char* kPhaseName[PH_COUNT] = {"orcha:fill", "orcha:exchange", "orcha:dt", "orcha:dt-allgather",
                                           "orcha:stage1", "orcha:stage2"};

namespace {
struct Pair {
  int phase;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Pair> g_live;   // recorded (both events), not yet queried
std::vector<Pair> g_free;   // reusable event pairs
}  // namespace

// The scope owns its event pair until it ends; only then does the pair join
// the recorded list, so a query between the two records cannot mismatch it.
PhaseScope::PhaseScope(int phase, cudaStream_t s) : phase_(phase), stream_(s), idx_(-1) {
  nvtxRangePushA(kPhaseName[phase]);
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  Pair p;
  if (!g_free.empty()) {
    p = g_free.back();
    g_free.pop_back();
  } else if (cudaEventCreate(&p.a) != cudaSuccess || cudaEventCreate(&p.b) != cudaSuccess) {
    return;
  }
  if (cudaEventRecord(p.a, s) != cudaSuccess) {
    g_free.push_back(p);
    return;
  }
  a_ = p.a;
  b_ = p.b;
  idx_ = 0;
}

PhaseScope::~PhaseScope() {
  nvtxRangePop();
  if (idx_ < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  Pair p{phase_, a_, b_};
  if (cudaEventRecord(p.b, stream_) == cudaSuccess) g_live.push_back(p);
  else g_free.push_back(p);
}

}  // namespace orcha

using namespace orcha;

extern "C" int32_t orcha_set_phase_timing(int32_t on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on != 0;
  return ORCHA_OK;
}

extern "C" int32_t orcha_phase_times(double* ms, int64_t* counts, int32_t n) {
  if (!ms || n < PH_COUNT) return fail(ORCHA_E_ARG, "orcha_phase_times: need room for ORCHA_NPHASES entries");
  std::vector<Pair> live;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    live.swap(g_live);
  }
  for (int i = 0; i < n; i++) {
    ms[i] = 0.0;
    if (counts) counts[i] = 0;
  }
  int32_t rc = ORCHA_OK;
  for (auto& p : live) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(p.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, p.a, p.b);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "phase event");
      continue;
    }
    ms[p.phase] += t;
    if (counts) counts[p.phase]++;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& p : live) g_free.push_back(p);
  return rc;
}

// FNV-1a 64-bit over host bytes (SPEC S:L433's mesh checksum format:
// "per-variable FNV-1a over raw bytes, hex"), continuing from *hash.
extern "C" int32_t orcha_fnv1a64(const void* data, size_t nbytes, uint64_t* hash) {
  if (!hash || (!data && nbytes)) return fail(ORCHA_E_ARG, "orcha_fnv1a64: null argument");
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h = *hash;
  for (size_t i = 0; i < nbytes; i++) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  *hash = h;
  return ORCHA_OK;
}
