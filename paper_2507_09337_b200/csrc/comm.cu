// comm.cu -- multi-GPU plumbing: NCCL (dlopen'ed from the process, i.e. the
// copy torch already loaded) for the guard exchange and the dt allreduce.
// "The Hydro computation can have either 1 or 2 MPI operations interspersed
// with local node computations" (sec 6); here: one grouped
// send/recv exchange of guard sources + one 8-byte allreduce per step.
#include <dlfcn.h>

#include <cstring>
#include <string>

#include "comm.h"
#include "orcha_internal.h"

namespace orcha {

struct CommPlan {
  int dummy;
};

int32_t comm_build_plan(orcha_comm*, orcha_packet* const*, int, CommPlan** out) {
  *out = nullptr;
  return fail(ORCHA_E_NCCL, "cross-rank guard exchange not available in this build");
}
void comm_free_plan(CommPlan* plan) { delete plan; }
int32_t comm_exchange(orcha_comm*, CommPlan*, cudaStream_t) {
  return fail(ORCHA_E_NCCL, "cross-rank guard exchange not available in this build");
}
int32_t comm_allreduce_dt(orcha_comm*, double*, long long*, bool*, cudaStream_t) {
  return fail(ORCHA_E_NCCL, "allreduce not available in this build");
}

}  // namespace orcha

extern "C" int32_t orcha_comm_unique_id(void*) {
  return orcha::fail(ORCHA_E_NCCL, "NCCL communicator not available in this build");
}
extern "C" int32_t orcha_comm_create(const orcha_grid*, const void*, int32_t, int32_t, const int32_t*,
                                     orcha_comm** out) {
  if (out) *out = nullptr;
  return orcha::fail(ORCHA_E_NCCL, "NCCL communicator not available in this build");
}
extern "C" int32_t orcha_comm_destroy(orcha_comm*) { return ORCHA_OK; }
