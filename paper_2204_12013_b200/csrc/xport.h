// xport.h — inter-process message transport between pipeline nodes on one
// NVLink/NVSwitch box: the sender's copy engine writes the payload straight
// into the receiver's HBM (CUDA IPC mapping of the receiver's arena), and a
// host callback enqueued behind the copy publishes the edge's sequence number
// in host shared memory once the copy has COMPLETED. A receiver that sees the
// number therefore finds the payload whole in its own HBM and needs no GPU
// wait at all; no GPU kernel ever spins on a peer. (Round 1 published at
// enqueue time and had the receiver wait on an interprocess CUDA event; with
// both processes on one GPU that wait sometimes passed before the copy
// landed, so completion is now established on the sender's side.) The ranks
// rendezvous through host shared memory named after a session id (no NCCL),
// so several ranks may share one GPU.
//
// Edges: one per (src node, dst node, message kind) crossing ranks; each has
// `cap` payload slots in the receiver's receive arena. Slot = cumulative
// message index % cap; a step-start barrier (host shared memory) guarantees
// that the previous step's payloads were consumed before a slot is
// overwritten.
#pragma once
#include <cuda_runtime.h>

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
  char *peer_base = nullptr;
  uint64_t sent = 0;
  std::vector<cudaEvent_t> ev;         // per-slot interprocess events (event mode)
  struct Post { volatile uint64_t *ctr; uint64_t value; };
  std::vector<Post> posts;             // host-callback arguments, one per slot (callback mode)
  // receiver side
  std::vector<cudaEvent_t> rev;        // the sender's events, opened here (event mode)
  uint64_t consumed = 0;
};

// Shared segment layout (uint64 words after a 64-byte header): per edge the
// published (completed) count, the intent count (bumped when a send is
// enqueued) and the receiver's consumed count; per rank a heartbeat, a dead
// flag, a blocked flag, a released flag and a step-end arrival stamp; per
// node its published instruction counter (fail-stop cut agreement); then one
// IPC memory handle per rank.
struct Xport {
  int rank = 0, world = 1, nnodes = 0;
  char *arena = nullptr;
  size_t arena_bytes = 0;
  std::vector<char *> peer_arena;      // mapped receive arenas of other ranks
  std::map<std::tuple<int, int, int>, XEdge> edges;
  void *shm = nullptr;
  size_t shm_bytes = 0;
  int nedges = 0;
  std::string shm_name;

  volatile uint64_t *word(size_t i) const {
    return reinterpret_cast<volatile uint64_t *>(static_cast<char *>(shm) + 64) + i;
  }
  volatile uint64_t *counter(int e) const { return word(e); }
  volatile uint64_t *intent(int e) const { return word(nedges + e); }
  volatile uint64_t *consumed_ctr(int e) const { return word(2 * nedges + e); }
  volatile uint64_t *rank_word(int field, int r) const {   // 0 hb 1 dead 2 blocked 3 released 4 arrive
    return word(3 * nedges + field * world + r);
  }
  volatile uint64_t *node_pc(int n) const { return word(3 * nedges + 5 * world + n); }
  size_t words() const { return 3 * nedges + 5 * world + nnodes; }

  // Host barrier over the live ranks (shared memory, sense-reversing).
  void barrier();
  int live() const;                    // ranks not flagged dead
  bool dead(int r) const { return shm && *rank_word(1, r) != 0; }
  // the receiver consumed one message of e (published for quiescence checks)
  void consume(XEdge &e);
  // After the payload copy is enqueued on e.stream, publish the message.
  // Event mode (default): record the slot's interprocess event behind the
  // copy and publish the sequence number at once; the receiver's stream
  // waits on that event (no host in the data path's latency). Callback mode
  // (fail-stop, opts.detect_ms): a host callback behind the copy publishes
  // the number once the copy completed, so the receiver never depends on an
  // event of a process that may have gone silent.
  cudaError_t post(XEdge &e);
  bool callback_mode = false;
  // the event the receiver's stream must wait on before reading slot
  // `slot` of e (nullptr in callback mode: the payload is already there)
  cudaEvent_t wait_event(const XEdge &e, int slot) const {
    return callback_mode ? nullptr : e.rev[slot];
  }
  bool available(const XEdge &e) const;
};

// want: the global sorted edge list (identical on every rank) with
// (src, dst, kind); node_rank maps nodes to ranks. slot_bytes(kind) and
// cap(kind) size the slots. id_bytes: the session id (>= 32 bytes, same on
// every rank). Returns an error string (empty on success).
std::string xport_init(Xport &x, int rank, int nranks, int nnodes,
                       const std::vector<std::tuple<int, int, int>> &want,
                       const std::vector<int> &node_rank, const std::vector<size_t> &slot_bytes,
                       const std::vector<int> &cap, const void *id_bytes, int hi_prio,
                       bool callback_mode = false);
void xport_destroy(Xport &x);

}  // namespace bb
