// kernels_fused.cu -- the performance advance kernel (placeholder: forwards to
// the reference kernels until the fused z-marching kernel lands).
#include "orcha_internal.h"

namespace orcha {

cudaError_t launch_advance_ref(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                               const double* d_dt, double h_dt, DtRecord* records, long long* nrecords,
                               DevStatus* st, cudaStream_t s);

cudaError_t launch_advance_fused(const DevGrid& G, double* state, double* u1, int nslots, const SlotInfo* slots,
                                 const double* d_dt, double h_dt, DtRecord* records, long long* nrecords,
                                 DevStatus* st, cudaStream_t s) {
  return launch_advance_ref(G, state, u1, nslots, slots, d_dt, h_dt, records, nrecords, st, s);
}

}  // namespace orcha
