// comm.h -- multi-GPU guard exchange and dt allreduce (private to liborcha.so).
#pragma once
#include "orcha_internal.h"

namespace orcha {
struct CommPlan;  // per fill plan: guard cells whose source block lives on another rank

// Build the exchange plan for this rank's packets (host; one device upload).
// buffer 0 = packet state, 1 = stage-1 buffer (per-stage variant).
int32_t comm_build_plan(orcha_comm* comm, orcha_packet* const* pk, int npk, int buffer, CommPlan** out);
void comm_free_plan(CommPlan* plan);
// Forget cached plans that reference a packet being destroyed.
void comm_drop_packet(orcha_packet* p);
// Pack sources, exchange with every peer (grouped ncclSend/ncclRecv), unpack into guards.
int32_t comm_exchange(orcha_comm* comm, CommPlan* plan, cudaStream_t s);
// Global (smax, argmax) with the lowest-g tie-break and the non-physical flag.
int32_t comm_allreduce_dt(orcha_comm* comm, double* smax, long long* g, bool* bad, cudaStream_t s);
// Device-resident dt: allgather this rank's record; *all / *nall = the
// gathered records (every rank's, in rank order).
int32_t comm_allgather_dt_device(orcha_comm* comm, const GatherRec* mine, const GatherRec** all, int* nall,
                                 cudaStream_t s);
// LOCAL transport: push this virtual rank's record to every member.
int32_t comm_push_dt_record(orcha_comm* comm, const GatherRec* mine, cudaStream_t s);
// F2 peer mode: device barrier over the ranks (stage 1 -> stage 2, records
// -> dt), the mode flag and the other ranks' registered packets.
int32_t comm_peer_barrier(orcha_comm* comm, cudaStream_t s);
bool comm_peer_mode(const orcha_comm* comm);
int comm_rank(const orcha_comm* comm);
int32_t comm_peer_packets(const orcha_comm* comm, std::vector<orcha_packet*>* out);
// runtime.cu: drop the fill plans built on a peer-mode communicator being destroyed.
void runtime_drop_comm(const orcha_comm* comm);
}  // namespace orcha
