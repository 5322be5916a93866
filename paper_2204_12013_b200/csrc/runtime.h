// runtime.h — per-process execution of the pipeline plans on one B200.
//
// One process per GPU hosts one or more pipeline NODES (node n runs stage n
// until a failover moves a stage to its shadow). Each node owns a high-
// priority main stream and a low-priority FRC stream (FRC fills the 1F1B
// bubbles and overlaps the next forward), its parameter copies
// (own stage + the successor's replica with Adam state), saved-set
// slot pools (1F1B stash; full FRC retention, P:524 / Q10), a per-step arena
// for activations and input-gradients (retained for a lazy-BRC resend, Q3) and
// a backward scratch. Nodes on other ranks are reached through xport.h
// (copy-engine writes into the peer's HBM + IPC events; host-shm rendezvous).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <map>
#include <thread>
#include <string>
#include <vector>

#include "bamboo.h"
#include "kernels.h"
#include "plan.h"
#include "xport.h"

namespace bb {

struct Dims {
  int L, H, nh, F, V, S, causal;
  int P, M, mb;
  int D = 1;   // data-parallel pipelines (node d*P + s)
  int R() const { return mb * S; }
  int d() const { return H / nh; }
};

// Parameter tensors of one unit, offsets relative to the stage's flat slice.
struct UnitP {
  int unit, kind;   // kind 0 embedding, 1 block, 2 head
  size_t tok, pos;
  size_t ln1g, ln1b, wqkv, bqkv, wo, bo, ln2g, ln2b, w1, b1, w2, b2;
  size_t lnfg, lnfb, whead;
};
// Saved-set tensors of one unit inside a slot (byte offsets).
struct UnitS {
  size_t out;                                                    // unit output (not last unit)
  size_t h1, mean1, rstd1, qkv, o, lse, x1, h2, mean2, rstd2, pre, act;   // block
  size_t hf, meanf, rstdf, dlog;                                 // head
};
struct StageInfo {
  int X, ua, ub;
  size_t poff, pcount;
  std::vector<UnitP> up;
  std::vector<UnitS> us;
  size_t slot_bytes;
};

struct Entry {
  void *p = nullptr;
  cudaEvent_t ev = nullptr;
  int slot = -1;
};

struct Copy {
  int X = -1;
  bool replica = false;   // kept for the predecessor's successor (false once promoted)
  float *master = nullptr, *m = nullptr, *v = nullptr, *grad = nullptr;
  void *work = nullptr;   // bf16 working copy (== master in fp32 check mode)
  int t = 0;
  // saved-set slot pool: slot i at sp[i]; the FRC scratch slot (saved sets
  // beyond the retention budget) is `scratch`. Chunks are cudaMalloc'ed at
  // init, grown when a replica is promoted, freed when the node dies.
  std::vector<char *> sp;
  char *scratch = nullptr;
  std::vector<std::pair<char *, size_t>> chunks;
  int nslots() const { return (int)sp.size(); }
  std::vector<int> free_slots;
  int retain = 0;              // FRC saved sets kept per step (replica; budget, Q10)
  float *loss = nullptr;  // [M] per-micro-batch losses (stage P-1 only)
  // D > 1: the all-reduced total (AR_SUM writes it, the replica sync and
  // Adam read it; grad keeps the local sum so it can be re-sent) and the
  // receive buffers of the other pipelines' contributions from local nodes
  float *arsum = nullptr;
  std::vector<float *> ar_in;
  // host-swap tier (opts.frc_swap_bytes): pinned host slots for the
  // FRC saved sets beyond the HBM budget, handed out in order each step
  char *hbase = nullptr;
  std::vector<char *> hslots;
  int hnext = 0;
  cudaEvent_t scratch_ev = nullptr;   // the scratch slot's last swap-out (this step)
};

struct Node {
  int n = -1;
  bool alive = true;
  cudaStream_t main = nullptr, frc = nullptr;
  cudaStream_t swap = nullptr;   // device -> host copies of swapped FRC saved sets
  std::map<int, Copy> copies;
  std::map<Key, Entry> store;
  char *arena = nullptr;
  size_t arena_bytes = 0, arena_used = 0;
  std::vector<std::pair<char *, size_t>> arena_spill;   // overflow chunks of this step
  size_t arena_peak = 0;                                // bytes the last step needed
  // opts.timing: [kind (0 FWD, 1 FRC, 2 BWD), start, end] events of this step
  struct TRec { int kind; cudaEvent_t a, b; };
  std::vector<TRec> trec;
  std::vector<cudaEvent_t> tpool;
  size_t tnext = 0;
  // backward scratch: [0] for the main stream, [1] for the FRC stream (EFEB's
  // eager BRC); column-reduction tickets and attention partials are per
  // stream because both streams may run backwards concurrently
  struct Scratch {
    void *sF = nullptr, *s3 = nullptr, *sH[5] = {};
    float *s32[4] = {};   // fp32 [R, H]: LN-input gradients and the residual-gradient chain
    float *s_part = nullptr, *s_attn = nullptr;
  } sc[2];
  float *s_loss_main = nullptr, *s_loss_frc = nullptr;
  int32_t *d_tok = nullptr, *d_tgt = nullptr, *d_csr = nullptr;
  bool needs_csr = false;   // hosts a copy of stage 0: builds the token CSR on the device
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  std::vector<Instr> plan;
  size_t pc = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  cudaEvent_t ev_begin = nullptr;   // after the step-start memsets of this node's buffers
};

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double work;
  int node;
};

struct DbgRec {
  int node, idx;
  Instr ins;
  cudaEvent_t main_ev, frc_ev;
};

struct Ctx {
  std::vector<DbgRec> dbg;
  Dims d{};
  bb_opts o{};
  bool bf16 = true;
  size_t act_bytes = 2;   // sizeof(storage type)
  std::vector<std::pair<int, int>> ranges;
  std::vector<StageInfo> stages;
  size_t total_params = 0;
  Plans plans;
  Topology topo;
  bool failover = false;
  std::vector<int> victims;           // preempted nodes, oldest first (bb_rejoin is LIFO)
  struct Hist { Plans plans; Topology topo; };
  std::vector<Hist> history;          // plans / topology before each failover
  bool fatal = false;
  std::vector<int> node_rank, node_device;
  std::map<int, Node> nodes;          // local nodes only
  Xport x;                            // cross-rank transport (IPC + copy engines)
  cudaStream_t serial = nullptr;      // profile mode: the one stream of all local nodes
  // local mailboxes (per (src node, dst node, kind))
  std::map<ChanKey, std::deque<Entry>> mail;
  // injection / recovery state
  bool armed = false;
  int inj_v = -1, inj_pi = -1;
  bool interrupted = false;
  Cut cut;
  std::map<ChanKey, int> victim_consumed, sent_to_victim;
  Plans continuation;
  RecoveryInfo rinfo;
  std::string recovery_text;
  // host staging
  int32_t *h_tok = nullptr, *h_tgt = nullptr;
  size_t csr_stride = 0;
  long long steps_done = 0;     // completed steps (identical on every rank)
  long long adam_steps = 0;     // Adam steps since bb_load_params (= every copy's t)
  bool resident = false;        // inputs staged on every local node's device (bb_stage_inputs)
  bool resident_step = false;   // this step reuses the resident inputs (no H2D)
  std::string err;
  // profiling
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_next = 0;
  long long launches_at_start = 0;
  uint64_t h2d = 0, d2h = 0;
  float last_step_ms = 0.f;     // host wall time of the last bb_step call
  // fail-stop mode (opts.detect_ms > 0)
  bool failstop = false;
  bool self_dead = false;       // this rank's node was preempted (silent from now on)
  std::thread hb_thread;
  std::atomic<bool> hb_stop{false};
  std::vector<uint64_t> edge_prior;   // messages per cross-rank edge in completed steps
  uint64_t step_id = 0;
  double detect_ms_seen = 0;    // detection latency of the last loss (ms)
  bool recovering = false;      // inside bb_recover's continuation
  int rec_stage = -1;           // the victim's stage (recovery accounting)
  int frc_recomputed = 0;       // forwards recomputed by the current recovery
  int frc_swapped = 0;          // saved sets the current recovery copied back from the host
  uint64_t bytes_rerouted = 0;  // bytes resent / rerouted by the current recovery
};

// Implemented in runtime.cpp
bb_status rt_init(Ctx &c, const bb_model *m, int stages, int microbatches, const bb_opts *o);
bb_status rt_load_params(Ctx &c, const float *host, size_t n);
bb_status rt_step(Ctx &c, const int32_t *tok, const int32_t *tgt, bb_step_stats *st);
bb_status rt_stage_inputs(Ctx &c, const int32_t *tok, const int32_t *tgt);
bb_status rt_preempt(Ctx &c, int stage, int at_instr);
bb_status rt_recover(Ctx &c, bb_recovery_stats *r);
bb_status rt_rejoin(Ctx &c);
bb_status rt_read_state(Ctx &c, int stage, int replica, int what, float *host, size_t n);
bb_status rt_write_state(Ctx &c, int stage, int what, const float *host, size_t n);
bb_status rt_node_stats(Ctx &c, bb_node_stat *out, int cap, int *n);
std::string rt_dump(const Ctx &c);
void rt_destroy(Ctx &c);
bb_status rt_kernel_stats(Ctx &c, bb_kernel_stat *out, int cap, int *n);

// Shared helpers
std::vector<std::pair<size_t, size_t>> unit_param_ranges(const Dims &d);  // per unit [off, n)
size_t unit_param_count(const Dims &d, int unit);

}  // namespace bb
