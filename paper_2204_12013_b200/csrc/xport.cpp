// xport.cpp — see xport.h.
#include "xport.h"

#include <fcntl.h>
#include <sys/stat.h>
#include <time.h>
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
}  // namespace

int Xport::live() const {
  int n = 0;
  for (int r = 0; r < world; ++r) n += dead(r) ? 0 : 1;
  return n;
}

void Xport::consume(XEdge &e) {
  ++e.consumed;
  __atomic_store_n(const_cast<uint64_t *>(consumed_ctr(e.index)), e.consumed, __ATOMIC_RELEASE);
}

// Header words: [0] magic, [1] barrier count, [2] barrier generation, [3] world.
void Xport::barrier() {
  if (world <= 1) return;
  uint64_t *cnt = reinterpret_cast<uint64_t *>(shm) + 1;
  uint64_t *gen = cnt + 1;
  const uint64_t g = __atomic_load_n(gen, __ATOMIC_ACQUIRE);
  if (__atomic_add_fetch(cnt, 1, __ATOMIC_ACQ_REL) == (uint64_t)live()) {
    __atomic_store_n(cnt, 0, __ATOMIC_RELAXED);
    __atomic_store_n(gen, g + 1, __ATOMIC_RELEASE);
  } else {
    long spins = 0;
    while (__atomic_load_n(gen, __ATOMIC_ACQUIRE) == g)
      if (++spins > 1000) std::this_thread::yield();
  }
}

namespace {
void CUDART_CB post_cb(void *arg) {
  auto *p = static_cast<XEdge::Post *>(arg);
  __atomic_store_n(const_cast<uint64_t *>(p->ctr), p->value, __ATOMIC_RELEASE);
}
}  // namespace

cudaError_t Xport::post(XEdge &e) {
  if (!callback_mode) {
    const cudaError_t r = cudaEventRecord(e.ev[e.sent % (uint64_t)e.cap], e.stream);
    if (r != cudaSuccess) return r;
    ++e.sent;
    __atomic_store_n(const_cast<uint64_t *>(intent(e.index)), e.sent, __ATOMIC_RELEASE);
    __atomic_store_n(const_cast<uint64_t *>(counter(e.index)), e.sent, __ATOMIC_RELEASE);
    return cudaSuccess;
  }
  XEdge::Post &p = e.posts[e.sent % (uint64_t)e.cap];
  ++e.sent;
  __atomic_store_n(const_cast<uint64_t *>(intent(e.index)), e.sent, __ATOMIC_RELEASE);
  p.ctr = counter(e.index);
  p.value = e.sent;
  return cudaLaunchHostFunc(e.stream, post_cb, &p);
}

bool Xport::available(const XEdge &e) const {
  return __atomic_load_n(const_cast<uint64_t *>(counter(e.index)), __ATOMIC_ACQUIRE) > e.consumed;
}

namespace {
constexpr uint64_t kMagic = 0x62616d626f6f7831ull;   // "bamboox1"
constexpr size_t kHS = 64;                          // IPC mem / event handle bytes

double now_s() {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}
}  // namespace

// Rendezvous through one POSIX shared-memory segment named after the session
// id (no NCCL, no sockets): rank 0 creates it, the others open it when it
// appears. Header | per-edge sequence counters | per-rank heartbeats |
// one IPC memory handle per rank. Ranks fill their own entries and meet at the shm barrier, so
// several ranks may share one GPU (NCCL refuses that: duplicate device).
std::string xport_init(Xport &x, int rank, int nranks, int nnodes,
                       const std::vector<std::tuple<int, int, int>> &want,
                       const std::vector<int> &node_rank, const std::vector<size_t> &slot_bytes,
                       const std::vector<int> &cap, const void *id_bytes, int hi_prio,
                       bool callback_mode) {
  try {
    x.callback_mode = callback_mode;
    x.rank = rank;
    x.world = nranks;
    x.nnodes = nnodes;
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
    x.nedges = idx;
    x.arena_bytes = std::max<size_t>(arena_size[rank], 256);
    XCK(cudaMalloc(&x.arena, x.arena_bytes));
    // ---- the shared segment
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < 32; ++i) h = (h ^ static_cast<const uint8_t *>(id_bytes)[i]) * 1099511628211ull;
    char name[64];
    std::snprintf(name, sizeof(name), "/bamboo_%016llx", (unsigned long long)h);
    x.shm_name = name;
    const size_t off_mh = 64 + 8 * x.words();
    const size_t off_eh = off_mh + kHS * (size_t)nranks;
    x.shm_bytes = off_eh + kHS * (size_t)max_cap * std::max(1, idx);
    auto hdr = [&]() { return static_cast<uint64_t *>(x.shm); };
    const double t0 = now_s();
    if (rank == 0) {
      shm_unlink(name);   // a stale segment of a crashed run with this id
      int fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0) throw XErr{"shm_open(create) failed"};
      if (ftruncate(fd, (off_t)x.shm_bytes) != 0) throw XErr{"ftruncate failed"};
      x.shm = mmap(nullptr, x.shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      close(fd);
      if (x.shm == MAP_FAILED) throw XErr{"mmap failed"};
      std::memset(x.shm, 0, x.shm_bytes);
      hdr()[3] = (uint64_t)nranks;
      __atomic_store_n(&hdr()[0], kMagic, __ATOMIC_RELEASE);
    } else {
      for (;;) {
        int fd = shm_open(name, O_RDWR, 0600);
        if (fd >= 0) {
          struct stat st;
          if (fstat(fd, &st) == 0 && (size_t)st.st_size == x.shm_bytes) {
            x.shm = mmap(nullptr, x.shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
            close(fd);
            if (x.shm == MAP_FAILED) throw XErr{"mmap failed"};
            if (__atomic_load_n(&hdr()[0], __ATOMIC_ACQUIRE) == kMagic) break;
            munmap(x.shm, x.shm_bytes);
            x.shm = nullptr;
          } else {
            close(fd);
          }
        }
        if (now_s() - t0 > 120.0) throw XErr{"rendezvous: rank 0 never created the segment"};
        usleep(1000);
      }
      if (hdr()[3] != (uint64_t)nranks) throw XErr{"rendezvous: world size mismatch"};
    }
    x.barrier();
    if (rank == 0) shm_unlink(name);   // every rank has it mapped now
    char *tab = static_cast<char *>(x.shm);
    // ---- receive arenas: publish our IPC handle, map the ones we send to
    cudaIpcMemHandle_t mine;
    XCK(cudaIpcGetMemHandle(&mine, x.arena));
    std::memcpy(tab + off_mh + kHS * rank, &mine, kHS);
    x.barrier();
    x.peer_arena.assign(nranks, nullptr);
    for (auto &kv : x.edges) {
      XEdge &e = kv.second;
      if (e.src_rank != rank || x.peer_arena[e.dst_rank]) continue;
      if (e.dst_rank == rank) throw XErr{"edge inside one rank"};
      cudaIpcMemHandle_t ph;
      std::memcpy(&ph, tab + off_mh + kHS * e.dst_rank, kHS);
      void *p = nullptr;
      XCK(cudaIpcOpenMemHandle(&p, ph, cudaIpcMemLazyEnablePeerAccess));
      x.peer_arena[e.dst_rank] = static_cast<char *>(p);
    }
    // ---- sender-side streams, host-callback slots and per-slot
    // interprocess events (created by the sender, opened by the receiver)
    for (auto &kv : x.edges) {
      XEdge &e = kv.second;
      if (e.src_rank != rank) continue;
      XCK(cudaStreamCreateWithPriority(&e.stream, cudaStreamNonBlocking, hi_prio));
      e.peer_base = x.peer_arena[e.dst_rank];
      e.posts.assign(e.cap, XEdge::Post{nullptr, 0});
      for (int sl = 0; sl < e.cap; ++sl) {
        cudaEvent_t ev;
        XCK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess));
        e.ev.push_back(ev);
        cudaIpcEventHandle_t hnd;
        XCK(cudaIpcGetEventHandle(&hnd, ev));
        std::memcpy(tab + off_eh + kHS * ((size_t)e.index * max_cap + sl), &hnd, kHS);
      }
    }
    x.barrier();
    for (auto &kv : x.edges) {
      XEdge &e = kv.second;
      if (e.dst_rank != rank) continue;
      for (int sl = 0; sl < e.cap; ++sl) {
        cudaIpcEventHandle_t hnd;
        std::memcpy(&hnd, tab + off_eh + kHS * ((size_t)e.index * max_cap + sl), kHS);
        cudaEvent_t ev;
        XCK(cudaIpcOpenEventHandle(&ev, hnd));
        e.rev.push_back(ev);
      }
    }
    XCK(cudaDeviceSynchronize());
    x.barrier();
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
