// plan.h — static pipeline plans, the preemption cut, and the recovery /
// failover plan transforms (host C++, pure integer logic).
//
// Rules (PAPER.md line numbers P:N; readings Q* in DESIGN.md):
//  * contiguous layer shards, remainder on the last stages (Q6);
//  * PipeDream 1F1B per stage;
//  * replica of stage n on node n-1, node P-1 for stage 0, the
//    last node loads the inputs;
//  * FRC_FWD(k) right after SEND_ACT(k); on the last stage before RECV_ACT(k)
//    (Q4);
//  * failover = merge of the victim's and the shadow's lists with the four
//    rules of P:538-545 (Q5), a lost step recomputed by lazy BRC (Q2).
#pragma once
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <vector>

namespace bb {

enum Kind : int8_t {
  LOAD_INPUTS, FWD, FRC_FWD, BWD, SEND_ACT, RECV_ACT, SEND_GRAD, RECV_GRAD, RESEND_GRAD,
  REPLICA_SEND, REPLICA_RECV, APPLY,
  BRC_BWD,                 // EFEB: eager redundant backward of the replica stage
  SEND_DGRAD, RECV_DGRAD,  // EFEB: a stage's input-gradient duplicated to the node two back
  // D > 1 pipelines: the stage's gradient sum to / from the
  // same stage of every other pipeline, then the sum of all D in ascending
  // pipeline order; RESEND_AR gives a lost victim's shadow a contribution again
  AR_SEND, AR_RECV, AR_SUM, RESEND_AR
};
const char *kind_name(Kind k);
bool is_send(Kind k);
bool is_recv(Kind k);
inline bool is_comm(Kind k) { return is_send(k) || is_recv(k); }

struct Instr {
  Kind kind;
  int mb;     // -1 = none
  int peer;   // node id, -1 = none
  int stage;  // logical stage the node acts for, -1 = none
};

enum MsgKind : int8_t { MSG_ACT = 0, MSG_GRAD = 1, MSG_GRADSUM = 2, MSG_STATE = 3 /* rejoin only */,
                        MSG_DGRAD = 4 /* EFEB duplicate gradients */,
                        MSG_AR = 5 /* D > 1 all-reduce contributions */ };
struct Msg {
  MsgKind kind;
  int mb;
  int stage;   // producing stage
  bool operator==(const Msg &o) const { return kind == o.kind && mb == o.mb && stage == o.stage; }
};
Msg message_of(const Instr &i);

// Data keys of the symbolic store (mirrors of the runtime buffers).
enum KeyType : int8_t { K_TOK, K_TGT, K_ACT, K_DACT, K_SAVED, K_LOSS, K_GRADSUM,
                        K_AR /* (stage, pipeline): a received all-reduce contribution */ };
struct Key {
  KeyType t;
  int a, b;
  bool operator<(const Key &o) const { return std::tie(t, a, b) < std::tie(o.t, o.a, o.b); }
  bool operator==(const Key &o) const { return t == o.t && a == o.a && b == o.b; }
};
std::vector<Key> inputs_of(const Instr &i, int P);
std::vector<Key> outputs_of(const Instr &i, int P, int M);

using Plans = std::map<int, std::vector<Instr>>;
using ChanKey = std::tuple<int, int, int>;                  // (src node, dst node, MsgKind)
using Channels = std::map<ChanKey, std::deque<Msg>>;

struct PlanError : std::exception {
  std::string msg;
  explicit PlanError(std::string m) : msg(std::move(m)) {}
  const char *what() const noexcept override { return msg.c_str(); }
};

// Stage unit ranges [a, b] inclusive (units: 0 emb, 1..L blocks, L+1 head).
std::vector<std::pair<int, int>> partition(int n_layer, int P, const int *layers_per_stage);

// mode = bb_rc_mode (0 none, 1 EFLB, 2 LFLB, 3 EFEB); a bool converts to none / EFLB.
// Pipeline d of D: node ids d*P + s (peers inside the pipeline, plus the
// all-reduce partners e*P + s of the other pipelines when D > 1).
std::vector<Instr> stage_plan(int s, int P, int M, int mode, int d = 0, int D = 1);
Plans normal_plans(int P, int M, int mode, int D = 1);

// Round-robin lockstep (one instruction per node per round, ascending node
// id); RECVs wait for their message, SENDs are buffered per (src,dst,kind).
// cap: node -> max instructions. on_exec(node, instr).
void lockstep(const Plans &plans, std::map<int, int> &pcs, Channels &ch,
              const std::map<int, int> &cap,
              const std::function<void(int, const Instr &)> &on_exec = nullptr);

struct Cut {
  std::map<int, int> pcs;   // instructions executed per node
  Channels ch;              // undelivered messages (to the victim removed)
};
Cut cut(const Plans &plans, int victim, int pi);

struct RecoveryInfo {
  int victim = -1, shadow = -1, successor = -1;
  bool commit = false;
  std::vector<int> frc_done, brc_mb, resend;
};
Plans recovery_plans(const Plans &plans, int P, int M, int victim, const std::map<int, int> &pcs,
                     const Channels &ch, RecoveryInfo *info);
// Static failover plans after losing `victim`: the recovery transform of
// `base` (nullptr = the normal plans; after an earlier failover, its plans)
// at an empty cut.
Plans failover_plans(int P, int M, int victim, const Plans *base = nullptr);

// Indexed by global stage g = d*P + s (pipeline d's stage s; its node in the
// normal plans). A node's shadow / successor are its neighbours in its own
// pipeline's ring.
struct Topology {
  std::vector<int> host;        // global stage -> node
  std::vector<int> replica_on;  // global stage -> node holding its replica, -1 none
};
inline int ring_prev(int P, int n) { return n - n % P + (n % P + P - 1) % P; }
inline int ring_next(int P, int n) { return n - n % P + (n % P + 1) % P; }
Topology normal_topology(int P, bool rc, int D = 1);
Topology failover_topology(int P, int victim, int D = 1);
// Topology after node v died and its stage moved to the shadow v-1 (Q21):
// v's stage runs unprotected on the shadow; every stage whose replica lived
// on v loses its protection.
Topology lose_node(int P, const Topology &t, int victim);
// A preemption of node v is recoverable iff v is alive, runs exactly its own
// stage, and that stage's replica lives on its live predecessor (a
// non-adjacent second loss is an independent recovery).
bool recoverable(int P, const Topology &t, const std::vector<int> &dead, int victim);

std::string dump(int P, int M, int rc, const std::vector<std::pair<int, int>> &ranges,
                 const Plans &plans, const Topology &topo, const std::vector<int> &node_device,
                 bool failover, const std::vector<int> &victims);
std::string dump_lines(const Plans &plans);

}  // namespace bb
