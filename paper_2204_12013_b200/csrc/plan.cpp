// plan.cpp — see plan.h. Pure host logic; no CUDA.
#include "plan.h"

#include <algorithm>
#include <set>
#include <sstream>

namespace bb {

const char *kind_name(Kind k) {
  static const char *n[] = {"LOAD_INPUTS", "FWD",          "FRC_FWD",      "BWD",
                            "SEND_ACT",    "RECV_ACT",     "SEND_GRAD",    "RECV_GRAD",
                            "RESEND_GRAD", "REPLICA_SEND", "REPLICA_RECV", "APPLY",
                            "BRC_BWD",     "SEND_DGRAD",   "RECV_DGRAD",   "AR_SEND",
                            "AR_RECV",     "AR_SUM",       "RESEND_AR"};
  return n[k];
}
bool is_send(Kind k) {
  return k == SEND_ACT || k == SEND_GRAD || k == RESEND_GRAD || k == REPLICA_SEND ||
         k == SEND_DGRAD || k == AR_SEND || k == RESEND_AR;
}
bool is_recv(Kind k) {
  return k == RECV_ACT || k == RECV_GRAD || k == REPLICA_RECV || k == RECV_DGRAD ||
         k == AR_RECV;
}

Msg message_of(const Instr &i) {
  switch (i.kind) {
    case SEND_ACT: return {MSG_ACT, i.mb, i.stage};
    case RECV_ACT: return {MSG_ACT, i.mb, i.stage - 1};   // produced by the previous stage
    case SEND_GRAD:
    case RESEND_GRAD: return {MSG_GRAD, i.mb, i.stage};
    case RECV_GRAD: return {MSG_GRAD, i.mb, i.stage + 1}; // produced by the next stage
    case REPLICA_SEND:
    case REPLICA_RECV: return {MSG_GRADSUM, -1, i.stage};
    case SEND_DGRAD: return {MSG_DGRAD, i.mb, i.stage};
    case RECV_DGRAD: return {MSG_DGRAD, i.mb, i.stage + 1};
    case AR_SEND:
    case AR_RECV:
    case RESEND_AR: return {MSG_AR, -1, i.stage};
    default: throw PlanError("message_of on a compute instruction");
  }
}

std::vector<Key> inputs_of(const Instr &i, int P) {
  const int k = i.mb, X = i.stage;
  switch (i.kind) {
    case FWD:
    case FRC_FWD: {
      std::vector<Key> v{X == 0 ? Key{K_TOK, k, 0} : Key{K_ACT, X, k}};
      if (X == P - 1) v.push_back({K_TGT, k, 0});
      return v;
    }
    case BWD:
    case BRC_BWD: {
      std::vector<Key> v{{K_SAVED, X, k}};
      if (X < P - 1) v.push_back({K_DACT, X + 1, k});
      return v;
    }
    case SEND_ACT: return {{K_ACT, X + 1, k}};
    case SEND_GRAD:
    case SEND_DGRAD:
    case RESEND_GRAD: return {{K_DACT, X, k}};
    case REPLICA_SEND:
    case AR_SEND:
    case RESEND_AR:
    case AR_SUM:
    case APPLY: return {{K_GRADSUM, X, 0}};
    default: return {};
  }
}

std::vector<Key> outputs_of(const Instr &i, int P, int M) {
  const int k = i.mb, X = i.stage;
  switch (i.kind) {
    case LOAD_INPUTS: {
      std::vector<Key> v;
      for (int j = 0; j < M; ++j) v.push_back({K_TOK, j, 0});
      for (int j = 0; j < M; ++j) v.push_back({K_TGT, j, 0});
      return v;
    }
    case FWD:
    case FRC_FWD:
      return {{K_SAVED, X, k}, X < P - 1 ? Key{K_ACT, X + 1, k} : Key{K_LOSS, k, 0}};
    case BWD:
    case BRC_BWD: {
      std::vector<Key> v;
      if (X > 0) v.push_back({K_DACT, X, k});
      if (k == M - 1) v.push_back({K_GRADSUM, X, 0});
      return v;
    }
    case RECV_ACT: return {{K_ACT, X, k}};
    case RECV_GRAD:
    case RECV_DGRAD: return {{K_DACT, X + 1, k}};
    case REPLICA_RECV: return {{K_GRADSUM, X, 0}};
    default: return {};
  }
}

// ---------------------------------------------------------------- partition
std::vector<std::pair<int, int>> partition(int L, int P, const int *lps) {
  if (P < 1 || L < P) throw PlanError("need 1 <= stages <= n_layer");
  std::vector<int> cnt(P);
  if (!lps) {
    const int base = L / P, rem = L % P;
    for (int s = 0; s < P; ++s) cnt[s] = base + (s >= P - rem ? 1 : 0);
  } else {
    int sum = 0;
    for (int s = 0; s < P; ++s) {
      cnt[s] = lps[s];
      if (cnt[s] < 0) throw PlanError("bad layers_per_stage");
      if (cnt[s] == 0 && s > 0 && s < P - 1) throw PlanError("interior stage without blocks");
      sum += cnt[s];
    }
    if (sum != L) throw PlanError("layers_per_stage does not sum to n_layer");
  }
  std::vector<std::pair<int, int>> out;
  int nxt = 1;
  for (int s = 0; s < P; ++s) {
    const int a = s == 0 ? 0 : nxt;
    int b = nxt + cnt[s] - 1;
    if (s == P - 1) b = L + 1;
    out.push_back({a, b});
    nxt += cnt[s];
  }
  return out;
}

// -------------------------------------------------------------- normal plan
std::vector<Instr> stage_plan(int s, int P, int M, int mode, int d, int D) {
  // mode = bb_rc_mode: NONE 0, EFLB 1 (replicas + eager FRC), LFLB 2
  // (replicas, no FRC: the forward is recomputed lazily on failure), EFEB 3
  // (eager FRC and eager BRC of the replica stage r = s+1 from the duplicate
  // gradient node s+2 sends, no replica sync)
  const bool rc = mode != 0, frc = mode == 1 || mode == 3, efeb = mode == 3;
  if (rc && P < 2) throw PlanError("RC needs stages >= 2");
  if (D < 1 || d < 0 || d >= D) throw PlanError("bad pipeline index");
  const int r = (s + 1) % P;
  std::vector<Instr> I;
  const bool need_tok = s == 0 || (rc && s == P - 1);
  const bool need_tgt = s == P - 1 || (rc && s == P - 2);
  if (need_tok || need_tgt) I.push_back({LOAD_INPUTS, -1, -1, -1});
  const int W = std::min(P - 1 - s, M);
  auto fwd = [&](int k) {
    if (frc && s == P - 1) I.push_back({FRC_FWD, k, -1, 0});
    if (s > 0) I.push_back({RECV_ACT, k, s - 1, s});
    I.push_back({FWD, k, -1, s});
    if (s < P - 1) {
      I.push_back({SEND_ACT, k, s + 1, s});
      if (frc) I.push_back({FRC_FWD, k, -1, s + 1});
    }
  };
  auto brc = [&](int k) {   // EFEB: the replica stage's backward, eagerly
    if (r < P - 1 && P >= 3) I.push_back({RECV_DGRAD, k, (r + 1) % P, r});
    I.push_back({BRC_BWD, k, -1, r});
  };
  auto bwd = [&](int k) {
    if (efeb && s < P - 1) brc(k);
    if (s < P - 1) I.push_back({RECV_GRAD, k, s + 1, s});
    I.push_back({BWD, k, -1, s});
    if (s > 0) {
      I.push_back({SEND_GRAD, k, s - 1, s});
      if (efeb && P >= 3) I.push_back({SEND_DGRAD, k, (s - 2 + P) % P, s});
    }
  };
  for (int k = 0; k < W; ++k) fwd(k);
  for (int i = 0; i < M - W; ++i) {
    fwd(W + i);
    bwd(i);
  }
  for (int i = M - W; i < M; ++i) bwd(i);
  // D > 1: the stage's gradient sum meets the same stage of the other
  // pipelines before anything reads it (replica sync, update); peers are
  // global node ids, marked here by an offset past the pipeline-local ids
  // EFEB with D > 1: the last node's eager BRCs of stage 0 come before its
  // all-reduce, and every replica is synced with the all-reduced total (the
  // EFLB tail below), since its own eager-BRC gradient is the pipeline's
  // local one
  if (efeb && D > 1 && s == P - 1)
    for (int k = 0; k < M; ++k) brc(k);
  std::vector<int> partners;
  for (int e = 0; e < D; ++e)
    if (e != d) partners.push_back(e * P + s);
  const size_t ar_at = I.size();
  for (int o : partners) I.push_back({AR_SEND, -1, o, s});
  for (int o : partners) I.push_back({AR_RECV, -1, o, s});
  if (D > 1) I.push_back({AR_SUM, -1, -1, s});
  const size_t ar_end = I.size();
  if (efeb && D == 1) {
    if (s == P - 1)   // stage 1's gradients come last: after the own backwards
      for (int k = 0; k < M; ++k) brc(k);
    I.push_back({APPLY, -1, -1, s});
    I.push_back({APPLY, -1, -1, r});
  } else if (rc) {
    I.push_back({REPLICA_SEND, -1, (s - 1 + P) % P, s});
    I.push_back({REPLICA_RECV, -1, (s + 1) % P, (s + 1) % P});
    I.push_back({APPLY, -1, -1, s});
    I.push_back({APPLY, -1, -1, (s + 1) % P});
  } else {
    I.push_back({APPLY, -1, -1, s});
  }
  // pipeline-local peers become global node ids (the all-reduce partners
  // already are)
  for (size_t i = 0; i < I.size(); ++i)
    if (I[i].peer >= 0 && (i < ar_at || i >= ar_end)) I[i].peer += d * P;
  return I;
}

Plans normal_plans(int P, int M, int mode, int D) {
  Plans p;
  for (int d = 0; d < D; ++d)
    for (int s = 0; s < P; ++s) p[d * P + s] = stage_plan(s, P, M, mode, d, D);
  return p;
}

// ----------------------------------------------------------------- lockstep
void lockstep(const Plans &plans, std::map<int, int> &pcs, Channels &ch,
              const std::map<int, int> &cap,
              const std::function<void(int, const Instr &)> &on_exec) {
  for (auto &kv : plans)
    if (!pcs.count(kv.first)) pcs[kv.first] = 0;
  bool progress = true;
  while (progress) {
    progress = false;
    for (auto &kv : plans) {
      const int n = kv.first;
      const auto &seq = kv.second;
      int lim = (int)seq.size();
      auto c = cap.find(n);
      if (c != cap.end()) lim = std::min(lim, c->second);
      int &pc = pcs[n];
      if (pc >= lim) continue;
      const Instr &ins = seq[pc];
      if (is_recv(ins.kind)) {
        const Msg want = message_of(ins);
        auto it = ch.find(ChanKey{ins.peer, n, want.kind});
        if (it == ch.end() || it->second.empty()) continue;
        if (!(it->second.front() == want)) throw PlanError("FIFO order mismatch");
        it->second.pop_front();
      } else if (is_send(ins.kind)) {
        const Msg m = message_of(ins);
        ch[ChanKey{n, ins.peer, m.kind}].push_back(m);
      }
      ++pc;
      progress = true;
      if (on_exec) on_exec(n, ins);
    }
  }
}

Cut cut(const Plans &plans, int v, int pi) {
  auto it = plans.find(v);
  if (it == plans.end() || pi < 0 || pi > (int)it->second.size())
    throw PlanError("injection point out of range");
  Cut c;
  std::map<int, int> cap{{v, pi}};
  lockstep(plans, c.pcs, c.ch, cap);
  if (c.pcs[v] != pi) throw PlanError("victim did not reach its injection point");
  for (auto i = c.ch.begin(); i != c.ch.end();) {
    if (std::get<1>(i->first) == v)
      i = c.ch.erase(i);
    else
      ++i;
  }
  return c;
}

// ----------------------------------------------------------------- recovery
// The continuation after node v is lost (readings Q2-Q5 and the
// EFEB reading in DESIGN.md §2). Written from the rules, independently of the
// oracle's implementation (oracle/plan.py); the two must produce the same
// text (tests/test_plan_parity.py), which is what makes the comparison a
// check of the rules rather than of one transcription.
//
//  shadow u = v-1 (rule set A): keeps its own remaining work, except
//    - its FRC of v (the victim's forward is rerun as a FWD from B),
//    - its sends to v and its receives of messages v never delivered
//      (rule 2: victim <-> shadow traffic becomes local data),
//    - v's APPLY when B brings one (EFLB before v's commit point).
//  victim v (rule set B, run by u): its whole step again, except what was
//    already done elsewhere: inputs (u loads them for its FRC), FRC /
//    replica work (its replica is gone), forwards whose FRC u already ran
//    (the retained FRC result is reused), sends it had delivered, the
//    traffic with u (rule 2); nothing at all once it committed (Q13). EFEB:
//    also not its backward and its gradient receives (u's eager BRC_BWD is
//    that backward, fed by the duplicate gradients w already sends u).
//  every other survivor: EFLB - the successor w re-sends the gradients v
//    received from it (Q3), its other traffic with v goes to u instead, and
//    its replica gradient for v is dropped (w is unprotected now, Q21);
//    EFEB - messages to v are dropped (u has its own copies), receives from
//    v that v had not delivered come from u.
//  A and B are then merged as two sequences (Q5): among the ready heads a
//  communication goes first (rule 1), the victim's first among
//  communications (rule 3); among computations backward before forward
//  (rule 4), then ascending micro-batch, then the victim's.
namespace {

enum Fate { KEEP, DROP, TO_SHADOW };

struct Loss {
  int P, M, v, u, w;
  int sv;   // the victim's stage in its pipeline (instructions name stages)
  bool efeb = false, commit = false;
  bool dp = false;   // D > 1: the victim stage's update follows its all-reduce (in B)
  std::set<int> frc_done;
  const std::map<int, int> *pcs = nullptr;
  const Channels *ch = nullptr;
};

int step_kind_rank(Kind k) {
  if (k == BWD || k == BRC_BWD) return 0;
  if (k == FWD || k == FRC_FWD) return 1;
  return 2;
}

// Messages v had delivered to node n that n has not consumed yet, per kind.
std::map<int, std::deque<Msg>> undelivered_queue(const Loss &x, int n) {
  std::map<int, std::deque<Msg>> q;
  for (auto &kv : *x.ch)
    if (std::get<0>(kv.first) == x.v && std::get<1>(kv.first) == n)
      q[std::get<2>(kv.first)] = kv.second;
  return q;
}

Fate shadow_fate(const Loss &x, const Instr &i) {
  if (i.kind == FRC_FWD && i.stage == x.sv) return DROP;
  if (is_send(i.kind) && i.peer == x.v) return DROP;
  if (i.kind == APPLY && i.stage == x.sv && !x.commit && (!x.efeb || x.dp)) return DROP;
  return KEEP;
}

Fate survivor_fate(const Loss &x, int /*n*/, const Instr &i) {
  if (!is_send(i.kind) || i.peer != x.v) return KEEP;
  if (i.kind == AR_SEND) return TO_SHADOW;   // the shadow replays v's all-reduce
  if (x.efeb) return DROP;
  if (i.kind == REPLICA_SEND) return DROP;   // w's replica on v is gone (Q21)
  return TO_SHADOW;
}

bool victim_work(const Loss &x, const Instr &i, int idx) {
  if (x.commit) return false;
  switch (i.kind) {
    case LOAD_INPUTS:
    case FRC_FWD:
    case BRC_BWD:
    case REPLICA_SEND:
    case REPLICA_RECV:
      return false;
    case APPLY:
      return i.stage == x.sv && (!x.efeb || x.dp);
    case BWD:
      return !x.efeb;
    case RECV_GRAD:
    case RECV_DGRAD:
      if (x.efeb) return false;
      break;
    case FWD:
      return !x.frc_done.count(i.mb);
    default:
      break;
  }
  if (is_comm(i.kind) && i.peer == x.u) return false;
  if (is_send(i.kind) && idx < x.pcs->at(x.v)) return false;
  return true;
}

// Rewrite node n's remaining instructions: fates for the other instructions,
// and every receive from v either stays (its message is already in n's FIFO)
// or, when v never delivered it, is dropped (n == u) or taken from u.
std::vector<Instr> rewrite(const Loss &x, int n, const std::vector<Instr> &rest) {
  auto q = undelivered_queue(x, n);
  std::vector<Instr> out;
  for (Instr i : rest) {
    if (is_recv(i.kind) && i.peer == x.v) {
      auto &d = q[message_of(i).kind];
      if (!d.empty() && d.front() == message_of(i)) {
        d.pop_front();
        out.push_back(i);
      } else if (n != x.u) {
        i.peer = x.u;
        out.push_back(i);
      }
      continue;
    }
    const Fate f = n == x.u ? shadow_fate(x, i) : survivor_fate(x, n, i);
    if (f == DROP) continue;
    if (f == TO_SHADOW) i.peer = x.u;
    out.push_back(i);
  }
  return out;
}

// Merge readiness of a RECV at the shadow, decided on the dependency graph of
// the other survivors' lists instead of by simulating them: the message the
// receive expects is either already in the shadow's FIFO, or it is sent by an
// instruction of its producer that can run given what the shadow has placed
// so far (everything before it on that node can run, and each receive there
// is fed by a message that is pending or sent by something that can run).
struct Readiness {
  const Loss &x;
  const Plans &lists;                          // the other survivors' new lists
  std::map<ChanKey, std::vector<Msg>> pending; // per channel, at the cut
  std::map<ChanKey, std::vector<Msg>> u_sent;  // the shadow's placed sends
  std::map<int, std::vector<int>> memo;        // 0 unknown, 1 yes, 2 no, 3 visiting

  Readiness(const Loss &x_, const Plans &l) : x(x_), lists(l) {
    for (auto &kv : *x.ch) pending[kv.first].assign(kv.second.begin(), kv.second.end());
  }
  void placed_send(const Instr &i) {
    u_sent[ChanKey{x.u, i.peer, message_of(i).kind}].push_back(message_of(i));
    memo.clear();
  }
  // j-th message (0-based, this step's remaining traffic) on channel c, if it
  // can exist given the shadow's placed prefix
  bool message(const ChanKey &c, size_t j, Msg *m) {
    auto p = pending.find(c);
    const size_t np = p == pending.end() ? 0 : p->second.size();
    if (j < np) {
      *m = p->second[j];
      return true;
    }
    j -= np;
    const int src = std::get<0>(c);
    if (src == x.u) {
      auto s = u_sent.find(c);
      if (s == u_sent.end() || j >= s->second.size()) return false;
      *m = s->second[j];
      return true;
    }
    auto it = lists.find(src);
    if (it == lists.end()) return false;
    size_t seen = 0;
    for (size_t i = 0; i < it->second.size(); ++i) {
      const Instr &ins = it->second[i];
      if (!is_send(ins.kind) || ins.peer != std::get<1>(c) ||
          (int)message_of(ins).kind != std::get<2>(c))
        continue;
      if (seen++ == j) {
        if (!can_run(src, (int)i)) return false;
        *m = message_of(ins);
        return true;
      }
    }
    return false;
  }
  bool can_run(int n, int idx) {
    if (idx < 0) return true;
    auto &mv = memo[n];
    if (mv.empty()) mv.assign(lists.at(n).size(), 0);
    if (mv[idx] == 1) return true;
    if (mv[idx] >= 2) return false;   // no, or a cycle
    mv[idx] = 3;
    bool ok = can_run(n, idx - 1);
    const Instr &ins = lists.at(n)[idx];
    if (ok && is_recv(ins.kind)) {
      const ChanKey c{ins.peer, n, message_of(ins).kind};
      size_t j = 0;   // ordinal of this receive on its channel
      for (int i = 0; i < idx; ++i) {
        const Instr &e = lists.at(n)[i];
        if (is_recv(e.kind) && e.peer == ins.peer && message_of(e).kind == message_of(ins).kind) ++j;
      }
      Msg m;
      ok = message(c, j, &m) && m == message_of(ins);
    }
    memo[n][idx] = ok ? 1 : 2;
    return ok;
  }
};

std::vector<Instr> merge_two(const Loss &x, const std::vector<Instr> &A,
                             const std::vector<Instr> &B, std::set<Key> avail,
                             const Plans &others) {
  Readiness rd(x, others);
  std::map<ChanKey, size_t> u_recvd;   // receives the shadow has placed, per channel
  auto ready = [&](const Instr &i) {
    if (is_recv(i.kind)) {
      const ChanKey c{i.peer, x.u, message_of(i).kind};
      Msg m;
      return rd.message(c, u_recvd[c], &m) && m == message_of(i);
    }
    for (const Key &k : inputs_of(i, x.P))
      if (!avail.count(k)) return false;
    return true;
  };
  // side 0 = victim (B), 1 = shadow (A)
  auto order = [&](const Instr &i, int side) {
    return is_comm(i.kind) ? std::make_tuple(0, side, 0, 0)
                           : std::make_tuple(1, step_kind_rank(i.kind), i.mb, side);
  };
  std::vector<Instr> out;
  size_t a = 0, b = 0;
  while (a < A.size() || b < B.size()) {
    const bool ra = a < A.size() && ready(A[a]);
    const bool rb = b < B.size() && ready(B[b]);
    if (!ra && !rb) throw PlanError("merge deadlock");
    const bool pick_a = ra && (!rb || order(A[a], 1) < order(B[b], 0));
    const Instr i = pick_a ? A[a++] : B[b++];
    out.push_back(i);
    for (const Key &k : outputs_of(i, x.P, x.M)) avail.insert(k);
    if (is_recv(i.kind)) ++u_recvd[ChanKey{i.peer, x.u, message_of(i).kind}];
    if (is_send(i.kind)) rd.placed_send(i);
  }
  return out;
}
}  // namespace

Plans recovery_plans(const Plans &plans, int P, int M, int v, const std::map<int, int> &pcs,
                     const Channels &ch, RecoveryInfo *info) {
  Loss x;
  x.P = P;
  x.M = M;
  x.v = v;
  x.sv = v % P;
  x.u = ring_prev(P, v);
  x.w = ring_next(P, v);
  x.pcs = &pcs;
  x.ch = &ch;
  const std::vector<Instr> &pv = plans.at(v), &pu = plans.at(x.u);
  for (int i = 0; i < pcs.at(v); ++i) x.commit = x.commit || pv[i].kind == REPLICA_SEND;
  for (auto &kv : plans)
    for (const Instr &i : kv.second) {
      x.efeb = x.efeb || i.kind == BRC_BWD;
      x.dp = x.dp || i.kind == AR_SEND;
    }
  for (int i = 0; i < pcs.at(x.u); ++i)
    if (pu[i].kind == FRC_FWD && pu[i].stage == x.sv) x.frc_done.insert(pu[i].mb);

  Plans out;
  for (auto &kv : plans) {
    const int n = kv.first;
    if (n == v) continue;
    std::vector<Instr> rest(kv.second.begin() + pcs.at(n), kv.second.end());
    std::vector<Instr> seq = rewrite(x, n, rest);
    if (n == x.w && n != x.u && !x.efeb && !x.commit) {
      // Q3: the gradients w already gave v, again, now to the shadow
      std::vector<Instr> again;
      for (int i = 0; i < pcs.at(n); ++i) {
        const Instr &e = kv.second[i];
        if (e.kind == SEND_GRAD && e.peer == v) again.push_back({RESEND_GRAD, e.mb, x.u, e.stage});
      }
      seq.insert(seq.begin(), again.begin(), again.end());
    }
    if (n / P != v / P && !x.commit) {
      // another pipeline: a contribution v received went down with it; the
      // shadow receives it again when it replays v's all-reduce (nothing to
      // redo after v's commit point, its all-reduce was complete)
      std::vector<Instr> again;
      for (int i = 0; i < pcs.at(n); ++i) {
        const Instr &e = kv.second[i];
        if (e.kind == AR_SEND && e.peer == v) again.push_back({RESEND_AR, -1, x.u, e.stage});
      }
      seq.insert(seq.begin(), again.begin(), again.end());
    }
    out[n] = seq;
  }
  std::vector<Instr> B;
  for (int i = 0; i < (int)pv.size(); ++i)
    if (victim_work(x, pv[i], i)) B.push_back(pv[i]);
  std::set<Key> avail;
  for (int i = 0; i < pcs.at(x.u); ++i)
    for (const Key &k : outputs_of(pu[i], P, M)) avail.insert(k);
  Plans others;
  for (auto &kv : out)
    if (kv.first != x.u) others.insert(kv);
  out[x.u] = merge_two(x, out[x.u], B, avail, others);

  if (info) {
    info->victim = v;
    info->shadow = x.u;
    info->successor = x.w;
    info->commit = x.commit;
    info->frc_done.assign(x.frc_done.begin(), x.frc_done.end());
    info->brc_mb.clear();
    // the victim-stage backwards still to run: B's (EFLB / LFLB) or the
    // shadow's pending eager BRCs (EFEB)
    for (const Instr &i : x.efeb ? out[x.u] : B)
      if ((i.kind == BWD || i.kind == BRC_BWD) && i.stage == x.sv) info->brc_mb.push_back(i.mb);
    info->resend.clear();
    if (out.count(x.w))
      for (const Instr &i : out[x.w])
        if (i.kind == RESEND_GRAD) info->resend.push_back(i.mb);
  }
  return out;
}

Plans failover_plans(int P, int M, int v, const Plans *base) {
  Plans plans = base ? *base : normal_plans(P, M, true);
  std::map<int, int> pcs;
  for (auto &kv : plans) pcs[kv.first] = 0;
  return recovery_plans(plans, P, M, v, pcs, Channels{}, nullptr);
}

Topology normal_topology(int P, bool rc, int D) {
  Topology t;
  for (int g = 0; g < D * P; ++g) {
    t.host.push_back(g);
    t.replica_on.push_back(rc ? ring_prev(P, g) : -1);
  }
  return t;
}

Topology lose_node(int P, const Topology &t0, int v) {
  Topology t = t0;
  t.host[v] = ring_prev(P, v);
  for (int &r : t.replica_on)
    if (r == v) r = -1;
  t.replica_on[v] = -1;
  return t;
}

Topology failover_topology(int P, int v, int D) {
  return lose_node(P, normal_topology(P, true, D), v);
}

bool recoverable(int P, const Topology &t, const std::vector<int> &dead, int v) {
  auto is_dead = [&](int n) { return std::find(dead.begin(), dead.end(), n) != dead.end(); };
  const int G = (int)t.host.size();
  if (v < 0 || v >= G || is_dead(v)) return false;
  for (int g = 0; g < G; ++g)
    if ((t.host[g] == v) != (g == v)) return false;   // v runs exactly its own stage
  const int r = t.replica_on[v];
  return r >= 0 && !is_dead(r) && r == ring_prev(P, v);
}

// --------------------------------------------------------------------- dump
static std::string fld(int x) { return x < 0 ? std::string("-") : std::to_string(x); }

std::string dump_lines(const Plans &plans) {
  std::ostringstream o;
  for (auto &kv : plans) {
    int i = 0;
    for (const Instr &ins : kv.second) {
      o << kv.first << ' ' << i++ << ' ' << kind_name(ins.kind) << ' ' << fld(ins.mb) << ' '
        << fld(ins.peer) << ' ' << fld(ins.stage) << '\n';
    }
  }
  return o.str();
}

std::string dump(int P, int M, int rc, const std::vector<std::pair<int, int>> &ranges,
                 const Plans &plans, const Topology &topo, const std::vector<int> &node_device,
                 bool failover, const std::vector<int> &victims) {
  std::ostringstream o;
  static const char *names[] = {"none", "eflb", "lflb", "efeb"};
  o << "# bamboo-plan v1 P=" << P << " M=" << M << " rc=" << names[rc]
    << " mode=" << (failover ? "failover" : "normal");
  if (failover) {
    o << " victim=";
    for (size_t i = 0; i < victims.size(); ++i) o << (i ? "," : "") << victims[i];
    o << " shadow=";
    for (size_t i = 0; i < victims.size(); ++i) o << (i ? "," : "") << ring_prev(P, victims[i]);
  }
  o << '\n';
  for (int g = 0; g < (int)topo.host.size(); ++g) {
    const int n = topo.host[g];
    o << "# stage " << g << " node " << n << " device " << node_device[n] << " units "
      << ranges[g % P].first << ".." << ranges[g % P].second << " replica_on "
      << fld(topo.replica_on[g]) << '\n';
  }
  o << dump_lines(plans);
  return o.str();
}

}  // namespace bb
