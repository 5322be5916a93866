// xport.cpp — see xport.h.
#include "xport.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <thread>

namespace bb {

namespace {
struct XErr {
  std::string msg;
};
#define XCK(x)                                                                     \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) throw XErr{std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)
#define XNK(x)                                                                     \
  do {                                                                             \
    ncclResult_t r_ = (x);                                                         \
    if (r_ != ncclSuccess) throw XErr{std::string(#x) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

// Byte-wise all-reduce(sum) of a host table in which every rank filled only
// its own entries (others zero): an all-gather of disjoint entries.
void allgather_bytes(ncclComm_t comm, std::vector<uint8_t> &buf) {
  void *d = nullptr;
  XCK(cudaMalloc(&d, buf.size()));
  XCK(cudaMemcpy(d, buf.data(), buf.size(), cudaMemcpyHostToDevice));
  XNK(ncclAllReduce(d, d, buf.size(), ncclUint8, ncclSum, comm, 0));
  XCK(cudaStreamSynchronize(0));
  XCK(cudaMemcpy(buf.data(), d, buf.size(), cudaMemcpyDeviceToHost));
  XCK(cudaFree(d));
}

void nccl_barrier(ncclComm_t comm) {
  std::vector<uint8_t> one(1, 0);
  allgather_bytes(comm, one);
}
}  // namespace

void Xport::barrier() {
  if (world <= 1) return;
  uint64_t *cnt = reinterpret_cast<uint64_t *>(shm);
  uint64_t *gen = cnt + 1;
  const uint64_t g = __atomic_load_n(gen, __ATOMIC_ACQUIRE);
  if (__atomic_add_fetch(cnt, 1, __ATOMIC_ACQ_REL) == (uint64_t)world) {
    __atomic_store_n(cnt, 0, __ATOMIC_RELAXED);
    __atomic_store_n(gen, g + 1, __ATOMIC_RELEASE);
  } else {
    long spins = 0;
    while (__atomic_load_n(gen, __ATOMIC_ACQUIRE) == g)
      if (++spins > 1000) std::this_thread::yield();
  }
}

void Xport::post(XEdge &e) {
  ++e.sent;
  __atomic_store_n(const_cast<uint64_t *>(counter(e.index)), e.sent, __ATOMIC_RELEASE);
}

bool Xport::available(const XEdge &e) const {
  return __atomic_load_n(const_cast<uint64_t *>(counter(e.index)), __ATOMIC_ACQUIRE) > e.consumed;
}

std::string xport_init(Xport &x, ncclComm_t world, int rank, int nranks,
                       const std::vector<std::tuple<int, int, int>> &want,
                       const std::vector<int> &node_rank, const std::vector<size_t> &slot_bytes,
                       const std::vector<int> &cap, const void *id_bytes, int hi_prio) {
  try {
    x.rank = rank;
    x.world = nranks;
    // ---- edge table and receive-arena layout (identical on every rank)
    std::vector<size_t> arena_size(nranks, 0);
    int idx = 0, max_cap = 0;
    for (auto &w : want) {
      XEdge e;
      e.src = std::get<0>(w);
      e.dst = std::get<1>(w);
      e.kind = std::get<2>(w);
      e.src_rank = node_rank[e.src];
      e.dst_rank = node_rank[e.dst];
      e.cap = cap[e.kind];
      e.slot_bytes = (slot_bytes[e.kind] + 255) / 256 * 256;
      e.recv_off = arena_size[e.dst_rank];
      arena_size[e.dst_rank] += e.slot_bytes * e.cap;
      e.index = idx++;
      max_cap = std::max(max_cap, e.cap);
      x.edges[w] = e;
    }
    x.arena_bytes = std::max<size_t>(arena_size[rank], 256);
    XCK(cudaMalloc(&x.arena, x.arena_bytes));
    // ---- shared host memory: barrier + one sequence counter per edge
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < 32; ++i) h = (h ^ static_cast<const uint8_t *>(id_bytes)[i]) * 1099511628211ull;
    char name[64];
    std::snprintf(name, sizeof(name), "/bamboo_%016llx", (unsigned long long)h);
    x.shm_name = name;
    x.shm_bytes = 64 + 8 * (size_t)std::max(1, idx);
    if (rank == 0) {
      int fd = shm_open(name, O_CREAT | O_RDWR | O_TRUNC, 0600);
      if (fd < 0) throw XErr{"shm_open(create) failed"};
      if (ftruncate(fd, (off_t)x.shm_bytes) != 0) throw XErr{"ftruncate failed"};
      x.shm = mmap(nullptr, x.shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      close(fd);
      if (x.shm == MAP_FAILED) throw XErr{"mmap failed"};
      std::memset(x.shm, 0, x.shm_bytes);
    }
    nccl_barrier(world);
    if (rank != 0) {
      int fd = shm_open(name, O_RDWR, 0600);
      if (fd < 0) throw XErr{"shm_open failed"};
      x.shm = mmap(nullptr, x.shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      close(fd);
      if (x.shm == MAP_FAILED) throw XErr{"mmap failed"};
    }
    nccl_barrier(world);
    if (rank == 0) shm_unlink(name);
    // ---- receive arenas: exchange IPC handles, map the ones we send to
    const size_t HS = sizeof(cudaIpcMemHandle_t);
    std::vector<uint8_t> mh(HS * nranks, 0);
    cudaIpcMemHandle_t mine;
    XCK(cudaIpcGetMemHandle(&mine, x.arena));
    std::memcpy(&mh[HS * rank], &mine, HS);
    allgather_bytes(world, mh);
    x.peer_arena.assign(nranks, nullptr);
    for (auto &kv : x.edges) {
      XEdge &e = kv.second;
      if (e.src_rank != rank || x.peer_arena[e.dst_rank]) continue;
      cudaIpcMemHandle_t ph;
      std::memcpy(&ph, &mh[HS * e.dst_rank], HS);
      void *p = nullptr;
      XCK(cudaIpcOpenMemHandle(&p, ph, cudaIpcMemLazyEnablePeerAccess));
      x.peer_arena[e.dst_rank] = static_cast<char *>(p);
    }
    // ---- per-slot interprocess events, created by the sender
    const size_t ES = sizeof(cudaIpcEventHandle_t);
    std::vector<uint8_t> eh(ES * (size_t)max_cap * std::max(1, idx), 0);
    for (auto &kv : x.edges) {
      XEdge &e = kv.second;
      if (e.src_rank != rank) continue;
      XCK(cudaStreamCreateWithPriority(&e.stream, cudaStreamNonBlocking, hi_prio));
      e.peer_base = x.peer_arena[e.dst_rank];
      for (int s = 0; s < e.cap; ++s) {
        cudaEvent_t ev;
        XCK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess));
        e.ev.push_back(ev);
        cudaIpcEventHandle_t hnd;
        XCK(cudaIpcGetEventHandle(&hnd, ev));
        std::memcpy(&eh[ES * ((size_t)e.index * max_cap + s)], &hnd, ES);
      }
    }
    allgather_bytes(world, eh);
    for (auto &kv : x.edges) {
      XEdge &e = kv.second;
      if (e.dst_rank != rank) continue;
      for (int s = 0; s < e.cap; ++s) {
        cudaIpcEventHandle_t hnd;
        std::memcpy(&hnd, &eh[ES * ((size_t)e.index * max_cap + s)], ES);
        cudaEvent_t ev;
        XCK(cudaIpcOpenEventHandle(&ev, hnd));
        e.rev.push_back(ev);
      }
    }
    XCK(cudaDeviceSynchronize());
    nccl_barrier(world);
    return "";
  } catch (const XErr &e) {
    return e.msg;
  }
}

void xport_destroy(Xport &x) {
  for (auto &kv : x.edges) {
    XEdge &e = kv.second;
    if (e.stream) cudaStreamSynchronize(e.stream);
    for (auto ev : e.ev) cudaEventDestroy(ev);
    for (auto ev : e.rev) cudaEventDestroy(ev);
    if (e.stream) cudaStreamDestroy(e.stream);
  }
  for (auto p : x.peer_arena)
    if (p) cudaIpcCloseMemHandle(p);
  if (x.arena) cudaFree(x.arena);
  if (x.shm) munmap(x.shm, x.shm_bytes);
  x.edges.clear();
  x.peer_arena.clear();
  x.arena = nullptr;
  x.shm = nullptr;
}

}  // namespace bb
