// xport.h — inter-process message transport between pipeline nodes on one
// NVLink/NVSwitch box: the sender's copy engine writes the payload straight
// into the receiver's HBM (CUDA IPC mapping), records a cross-process CUDA
// event, and publishes a sequence number in host shared memory; the receiver
// enqueues a stream wait on that event. No GPU kernel ever spins on a peer,
// so no stream can be starved by a waiting kernel (the hazard of spinning
// P2P kernels on concurrent streams); every GPU-side wait is on an event that
// is already recorded. NCCL is used only to bootstrap (handle exchange).
//
// Edges: one per (src node, dst node, message kind) crossing ranks; each has
// `cap` payload slots in the receiver's receive arena and `cap` IPC events on
// the sender. Slot = cumulative message index % cap; a step-start barrier
// (host shared memory) guarantees that the previous step's payloads were
// consumed before a slot is overwritten.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

namespace bb {

struct XEdge {
  int src = -1, dst = -1, kind = -1;   // nodes, message kind
  int src_rank = -1, dst_rank = -1;
  int cap = 0;
  size_t slot_bytes = 0;
  size_t recv_off = 0;                 // in the dst rank's receive arena
  int index = -1;                      // shm counter index
  // sender side
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> ev;
  char *peer_base = nullptr;
  uint64_t sent = 0;
  // receiver side
  std::vector<cudaEvent_t> rev;
  uint64_t consumed = 0;
};

struct Xport {
  int rank = 0, world = 1;
  char *arena = nullptr;
  size_t arena_bytes = 0;
  std::vector<char *> peer_arena;      // mapped receive arenas of other ranks
  std::map<std::tuple<int, int, int>, XEdge> edges;
  void *shm = nullptr;
  size_t shm_bytes = 0;
  std::string shm_name;

  volatile uint64_t *counter(int i) const {
    return reinterpret_cast<volatile uint64_t *>(static_cast<char *>(shm) + 64 + 8 * i);
  }
  // Host barrier over all ranks (shared memory, sense-reversing).
  void barrier();
  void post(XEdge &e);                 // after the copy + event are enqueued
  bool available(const XEdge &e) const;
};

// want: the global sorted edge list (identical on every rank) with
// (src, dst, kind); node_rank maps nodes to ranks. slot_bytes(kind) and
// cap(kind) size the slots. world: the NCCL communicator over all ranks.
// Returns an error string (empty on success).
std::string xport_init(Xport &x, ncclComm_t world, int rank, int nranks,
                       const std::vector<std::tuple<int, int, int>> &want,
                       const std::vector<int> &node_rank, const std::vector<size_t> &slot_bytes,
                       const std::vector<int> &cap, const void *id_bytes, int hi_prio);
void xport_destroy(Xport &x);

}  // namespace bb
