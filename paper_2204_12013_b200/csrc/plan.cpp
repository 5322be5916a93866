// plan.cpp — see plan.h. Pure host logic; no CUDA.
#include "plan.h"

#include <algorithm>
#include <set>
#include <sstream>

namespace bb {

const char *kind_name(Kind k) {
  static const char *n[] = {"LOAD_INPUTS", "FWD",       "FRC_FWD",     "BWD",
                            "SEND_ACT",    "RECV_ACT",  "SEND_GRAD",   "RECV_GRAD",
                            "RESEND_GRAD", "REPLICA_SEND", "REPLICA_RECV", "APPLY"};
  return n[k];
}
bool is_send(Kind k) {
  return k == SEND_ACT || k == SEND_GRAD || k == RESEND_GRAD || k == REPLICA_SEND;
}
bool is_recv(Kind k) { return k == RECV_ACT || k == RECV_GRAD || k == REPLICA_RECV; }

Msg message_of(const Instr &i) {
  switch (i.kind) {
    case SEND_ACT: return {MSG_ACT, i.mb, i.stage};
    case RECV_ACT: return {MSG_ACT, i.mb, i.stage - 1};   // produced by the previous stage
    case SEND_GRAD:
    case RESEND_GRAD: return {MSG_GRAD, i.mb, i.stage};
    case RECV_GRAD: return {MSG_GRAD, i.mb, i.stage + 1}; // produced by the next stage
    case REPLICA_SEND:
    case REPLICA_RECV: return {MSG_GRADSUM, -1, i.stage};
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
    case BWD: {
      std::vector<Key> v{{K_SAVED, X, k}};
      if (X < P - 1) v.push_back({K_DACT, X + 1, k});
      return v;
    }
    case SEND_ACT: return {{K_ACT, X + 1, k}};
    case SEND_GRAD:
    case RESEND_GRAD: return {{K_DACT, X, k}};
    case REPLICA_SEND:
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
    case BWD: {
      std::vector<Key> v;
      if (X > 0) v.push_back({K_DACT, X, k});
      if (k == M - 1) v.push_back({K_GRADSUM, X, 0});
      return v;
    }
    case RECV_ACT: return {{K_ACT, X, k}};
    case RECV_GRAD: return {{K_DACT, X + 1, k}};
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
std::vector<Instr> stage_plan(int s, int P, int M, int mode) {
  // mode = bb_rc_mode: NONE 0, EFLB 1 (replicas + eager FRC), LFLB 2
  // (replicas, no FRC: the forward is recomputed lazily on failure)
  const bool rc = mode != 0, frc = mode == 1;
  if (rc && P < 2) throw PlanError("RC needs stages >= 2");
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
  auto bwd = [&](int k) {
    if (s < P - 1) I.push_back({RECV_GRAD, k, s + 1, s});
    I.push_back({BWD, k, -1, s});
    if (s > 0) I.push_back({SEND_GRAD, k, s - 1, s});
  };
  for (int k = 0; k < W; ++k) fwd(k);
  for (int i = 0; i < M - W; ++i) {
    fwd(W + i);
    bwd(i);
  }
  for (int i = M - W; i < M; ++i) bwd(i);
  if (rc) {
    I.push_back({REPLICA_SEND, -1, (s - 1 + P) % P, s});
    I.push_back({REPLICA_RECV, -1, (s + 1) % P, (s + 1) % P});
    I.push_back({APPLY, -1, -1, s});
    I.push_back({APPLY, -1, -1, (s + 1) % P});
  } else {
    I.push_back({APPLY, -1, -1, s});
  }
  return I;
}

Plans normal_plans(int P, int M, int mode) {
  Plans p;
  for (int s = 0; s < P; ++s) p[s] = stage_plan(s, P, M, mode);
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

// -------------------------------------------------------------------- merge
namespace {
int compute_rank(Kind k) { return k == BWD ? 0 : (k == FWD || k == FRC_FWD) ? 1 : 2; }

std::vector<Instr> merge(const std::vector<Instr> &A, const std::vector<Instr> &B,
                         std::set<Key> avail, int P, int M, int u, const Plans &others,
                         const Channels &channels) {
  Channels och = channels;
  std::map<int, int> opcs;
  const std::map<int, int> nocap;
  lockstep(others, opcs, och, nocap);
  size_t a = 0, b = 0;
  std::vector<Instr> out;
  auto ready = [&](const Instr &ins) {
    if (is_recv(ins.kind)) {
      const Msg want = message_of(ins);
      auto it = och.find(ChanKey{ins.peer, u, want.kind});
      return it != och.end() && !it->second.empty() && it->second.front() == want;
    }
    for (const Key &k : inputs_of(ins, P))
      if (!avail.count(k)) return false;
    return true;
  };
  // priority key: comm first (victim side first), then backward < forward <
  // other, ascending micro-batch, victim side first.
  auto prio = [&](const Instr &ins, int side) {
    if (is_comm(ins.kind)) return std::make_tuple(0, side, 0, 0);
    return std::make_tuple(1, compute_rank(ins.kind), ins.mb, side);
  };
  while (a < A.size() || b < B.size()) {
    bool ra = a < A.size() && ready(A[a]);
    bool rb = b < B.size() && ready(B[b]);
    if (!ra && !rb) throw PlanError("merge deadlock");
    bool takeA;
    if (ra && rb)
      takeA = prio(A[a], 1) < prio(B[b], 0);
    else
      takeA = ra;
    const Instr ins = takeA ? A[a++] : B[b++];
    out.push_back(ins);
    for (const Key &k : outputs_of(ins, P, M)) avail.insert(k);
    if (is_recv(ins.kind)) {
      och[ChanKey{ins.peer, u, message_of(ins).kind}].pop_front();
    } else if (is_send(ins.kind)) {
      const Msg m = message_of(ins);
      och[ChanKey{u, ins.peer, m.kind}].push_back(m);
      lockstep(others, opcs, och, nocap);
    }
  }
  return out;
}
}  // namespace

Plans recovery_plans(const Plans &plans, int P, int M, int v, const std::map<int, int> &pcs,
                     const Channels &ch, RecoveryInfo *info) {
  const int u = (v - 1 + P) % P, w = (v + 1) % P;
  const auto &pv = plans.at(v);
  const int pcv = pcs.at(v);
  bool commit = false;
  for (int i = 0; i < pcv; ++i)
    if (pv[i].kind == REPLICA_SEND) commit = true;

  // Remaining RECVs from v are kept iff their message is already delivered
  // (pending in the per-kind FIFO); otherwise rewritten by `redirect`.
  auto delivered_filter = [&](int n, const std::vector<Instr> &seq, int redirect) {
    std::map<int, std::deque<Msg>> qs;
    for (int kd = 0; kd < 3; ++kd) {
      auto it = ch.find(ChanKey{v, n, kd});
      if (it != ch.end()) qs[kd] = it->second;
    }
    std::vector<Instr> out;
    for (const Instr &ins : seq) {
      if (is_recv(ins.kind) && ins.peer == v) {
        const Msg m = message_of(ins);
        auto &q = qs[m.kind];
        if (!q.empty() && q.front() == m) {
          q.pop_front();
          out.push_back(ins);
        } else if (redirect >= 0) {
          Instr r = ins;
          r.peer = redirect;
          out.push_back(r);
        }
        continue;
      }
      out.push_back(ins);
    }
    return out;
  };

  // A: the shadow's remaining instructions
  std::vector<Instr> A;
  const auto &pu = plans.at(u);
  for (size_t i = pcs.at(u); i < pu.size(); ++i) {
    const Instr &ins = pu[i];
    if (ins.kind == FRC_FWD && ins.stage == v) continue;   // becomes v's FWD in B
    if (is_send(ins.kind) && ins.peer == v) continue;       // rule 2
    if (ins.kind == APPLY && ins.stage == v && !commit) continue;
    A.push_back(ins);
  }
  A = delivered_filter(u, A, -1);

  // B: the victim's whole step, rewritten for the shadow
  std::set<int> frc_done;
  for (int i = 0; i < pcs.at(u); ++i)
    if (pu[i].kind == FRC_FWD && pu[i].stage == v) frc_done.insert(pu[i].mb);
  std::vector<Instr> B;
  if (!commit) {
    for (int idx = 0; idx < (int)pv.size(); ++idx) {
      const Instr &ins = pv[idx];
      const Kind kd = ins.kind;
      if (kd == LOAD_INPUTS || kd == FRC_FWD || kd == REPLICA_SEND || kd == REPLICA_RECV) continue;
      if (kd == APPLY && ins.stage != v) continue;
      if (is_comm(kd) && ins.peer == u) continue;          // rule 2: local data edge
      if (kd == FWD && frc_done.count(ins.mb)) continue;    // reuse retained FRC
      if (kd == SEND_ACT && idx < pcv) continue;            // already delivered
      B.push_back(ins);
    }
  }

  Plans nw;
  for (auto &kv : plans) {
    const int n = kv.first;
    if (n == v) continue;
    std::vector<Instr> seq;
    if (n == u)
      seq = A;
    else
      seq.assign(kv.second.begin() + pcs.at(n), kv.second.end());
    if (n == w) {
      std::vector<Instr> resend;
      if (!commit && w != u) {
        for (int i = 0; i < pcs.at(w); ++i) {
          const Instr &x = plans.at(w)[i];
          if (x.kind == SEND_GRAD && x.peer == v) resend.push_back({RESEND_GRAD, x.mb, u, x.stage});
        }
      }
      std::vector<Instr> s2;
      for (Instr ins : seq) {
        if (ins.kind == REPLICA_SEND && ins.peer == v) continue;
        if (is_send(ins.kind) && ins.peer == v) ins.peer = u;
        s2.push_back(ins);
      }
      if (w != u) {
        auto f = delivered_filter(w, s2, u);
        seq = resend;
        seq.insert(seq.end(), f.begin(), f.end());
      } else {
        seq = s2;
      }
    }
    nw[n] = seq;
  }
  std::set<Key> avail;
  for (int i = 0; i < pcs.at(u); ++i)
    for (const Key &k : outputs_of(pu[i], P, M)) avail.insert(k);
  Plans others;
  for (auto &kv : nw)
    if (kv.first != u) others[kv.first] = kv.second;
  nw[u] = merge(nw[u], B, avail, P, M, u, others, ch);

  if (info) {
    info->victim = v;
    info->shadow = u;
    info->successor = w;
    info->commit = commit;
    info->frc_done.assign(frc_done.begin(), frc_done.end());
    info->brc_mb.clear();
    for (const Instr &i : B)
      if (i.kind == BWD) info->brc_mb.push_back(i.mb);
    info->resend.clear();
    if (nw.count(w))
      for (const Instr &i : nw[w])
        if (i.kind == RESEND_GRAD) info->resend.push_back(i.mb);
  }
  return nw;
}

Plans failover_plans(int P, int M, int v, const Plans *base) {
  Plans plans = base ? *base : normal_plans(P, M, true);
  std::map<int, int> pcs;
  for (auto &kv : plans) pcs[kv.first] = 0;
  return recovery_plans(plans, P, M, v, pcs, Channels{}, nullptr);
}

Topology normal_topology(int P, bool rc) {
  Topology t;
  for (int s = 0; s < P; ++s) {
    t.host.push_back(s);
    t.replica_on.push_back(rc ? (s - 1 + P) % P : -1);
  }
  return t;
}

Topology lose_node(int P, const Topology &t0, int v) {
  Topology t = t0;
  t.host[v] = (v - 1 + P) % P;
  for (int X = 0; X < P; ++X)
    if (t.replica_on[X] == v) t.replica_on[X] = -1;
  t.replica_on[v] = -1;
  return t;
}

Topology failover_topology(int P, int v) { return lose_node(P, normal_topology(P, true), v); }

bool recoverable(int P, const Topology &t, const std::vector<int> &dead, int v) {
  auto is_dead = [&](int n) { return std::find(dead.begin(), dead.end(), n) != dead.end(); };
  if (v < 0 || v >= P || is_dead(v)) return false;
  for (int X = 0; X < P; ++X)
    if ((t.host[X] == v) != (X == v)) return false;   // v runs exactly its own stage
  const int r = t.replica_on[v];
  return r >= 0 && !is_dead(r) && r == (v - 1 + P) % P;
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
    for (size_t i = 0; i < victims.size(); ++i) o << (i ? "," : "") << (victims[i] - 1 + P) % P;
  }
  o << '\n';
  for (int X = 0; X < P; ++X) {
    const int n = topo.host[X];
    o << "# stage " << X << " node " << n << " device " << node_device[n] << " units "
      << ranges[X].first << ".." << ranges[X].second << " replica_on " << fld(topo.replica_on[X])
      << '\n';
  }
  o << dump_lines(plans);
  return o.str();
}

}  // namespace bb
