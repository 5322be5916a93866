"""Oracle plan interpreter with redundant computation, preemption injection and
recovery (O4-O6) — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Semantics:
* Each node n runs its own stage and keeps a replica (parameters AND Adam
  state) of stage (n+1) mod P. The replica is kept identical by
  gradient forwarding: after its last backward, stage n sends its fp32
  gradient sum to node n-1, and both apply the same Adam (Q1 reading).
* D > 1 data-parallel pipelines: node d*P + s runs stage s of
  pipeline d on micro-batches d*M .. d*M+M-1 of the step's batch; the loss is
  the mean over all D*M micro-batches. After its last backward each stage's
  gradient sum is all-reduced over the D pipelines (AR_SEND / AR_RECV, then
  AR_SUM adds the D contributions in ascending pipeline order) before the
  replica sync and the update, so every pipeline applies the same total. A
  failed pipeline's all-reduce is run by its shadow after the recovery: the
  other pipelines wait for it ("all-reduce ... waits").
* FRC_FWD(k) on node n is exactly FNC_{n+1}(k) with the replica weights
  (P:429); its saved set and output are retained for a lazy BRC (P:456,
  P:524; Q10/Q22 readings).
* A preemption of node v at instruction pi (Q12): v executes its first pi
  instructions; the survivors run to quiescence (lockstep round-robin, Q14);
  everything v held is lost; messages v had sent stay delivered.
* Recovery: the shadow u = v-1 promotes the replica, the
  successor w = v+1 is rerouted to u and re-sends the gradients it sent to
  v this step (Q3 reading), u runs the victim's lost work (lazy BRC for every
  micro-batch in ascending order, Q2/Q20) merged with its own, then Adam for
  both stages. Later steps run the static failover plans.

The interpreter stores data under the plan's symbolic keys (plan.inputs_of /
plan.outputs_of), so local data edges created by the merge need no special
casing. Pins: tests/test_oracle_pipeline.py (brute force O2, 1F1B == GPipe,
FRC == FNC and replica == primary exactly, injection sweep == failure-free
exactly, FATAL cases).
"""
from collections import deque

import numpy as np

from . import model
from . import plan as pl


class Node:
    def __init__(self, nid):
        self.nid = nid
        self.copies = {}      # stage -> dict(p, m, v, t, g, role)
        self.store = {}


class Pipeline:
    """P logical nodes executing instruction lists over fp64 numpy data."""

    def __init__(self, cfg, flat_params, rc=True, layers_per_stage=None,
                 lr=1e-4, b1=0.9, b2=0.999, eps=1e-8, D=1):
        self.cfg = cfg
        m = cfg.model
        self.P, self.M, self.D = cfg.stages, cfg.microbatches, D
        self.mode_rc = pl.rc_mode(rc)       # none / eflb / lflb
        self.rc = self.mode_rc != "none"
        self.lay = model.Layout(m)
        self.ranges = pl.partition(m.n_layer, self.P, layers_per_stage)
        self.hp = (lr, b1, b2, eps)
        self.nodes = {n: Node(n) for n in range(self.P * D)}
        self.mode = "normal"
        self.victims = []          # preempted nodes, oldest first (rejoin is LIFO)
        self.history = []          # (plans, host, replica_on) before each failover
        self.dead = set()
        self.plans = pl.normal_plans(self.P, self.M, self.mode_rc, D)
        # keyed by global stage g = d*P + s (its node in the normal plans)
        self.host, self.replica_on = pl.normal_topology(self.P, D)
        if not self.rc:
            self.replica_on = {g: None for g in self.host}
        flat = np.asarray(flat_params, dtype=np.float64)
        for g in range(self.P * D):
            s = g % self.P
            self._install(self.nodes[g], s, flat, "primary")
            if self.rc:
                self._install(self.nodes[self.replica_on[g]], s, flat, "replica")
        self.pending = None        # armed injection (v, pi)
        self.interrupted = None    # state between a preempted step and recover()
        self.step_no = 0

    # ------------------------------------------------------------------ state
    def stage_bounds(self, X):
        a, b = self.ranges[X]
        return self.lay.range_of_units(a, b)

    def _install(self, node, X, flat, role):
        lo, hi = self.stage_bounds(X)
        node.copies[X] = {"p": flat[lo:hi].copy(), "m": np.zeros(hi - lo),
                          "v": np.zeros(hi - lo), "t": 0, "g": np.zeros(hi - lo), "role": role}

    def params(self, X, d=0):
        """Stage X's primary copy in pipeline d."""
        return self.nodes[self.host[d * self.P + X]].copies[X]

    def full_params(self):
        return np.concatenate([self.params(X)["p"] for X in range(self.P)])

    def full_grads(self):
        return np.concatenate([self.params(X)["g"] for X in range(self.P)])

    def full_adam(self):
        return (np.concatenate([self.params(X)["m"] for X in range(self.P)]),
                np.concatenate([self.params(X)["v"] for X in range(self.P)]))

    # ------------------------------------------------------------- execution
    def _stage_fwd(self, X, c, x, k, d=0):
        a, b = self.ranges[X]
        lo, hi = self.stage_bounds(X)
        th = self.lay.tensors(c["p"], lo, hi)
        tok, tgt = self.tokens[d][k], self.targets[d][k]
        saved = []
        for unit in range(a, b + 1):
            x, sv = model.unit_fwd(self.lay, unit, th, x, tok, tgt, self.n_tok)
            saved.append(sv)
        return x, saved

    def _stage_bwd(self, X, c, saved, d, k, dp=0):
        a, b = self.ranges[X]
        lo, hi = self.stage_bounds(X)
        th = self.lay.tensors(c["p"], lo, hi)
        gr = self.lay.tensors(c["g"], lo, hi)
        tok, tgt = self.tokens[dp][k], self.targets[dp][k]
        for unit, sv in zip(reversed(range(a, b + 1)), reversed(saved)):
            d = model.unit_bwd(self.lay, unit, th, gr, sv, d, tok, tgt, self.n_tok)
        return d

    def _exec(self, n, ins, msg):
        node = self.nodes[n]
        st = node.store
        P, k, X = self.P, ins.mb, ins.stage
        dp = n // P          # the node's pipeline (a shadow stays in its own)
        kd = ins.kind
        if kd == pl.LOAD_INPUTS:
            for j in range(self.M):
                st[("tok", j)] = self.tokens[dp][j]
                st[("tgt", j)] = self.targets[dp][j]
        elif kd in (pl.FWD, pl.FRC_FWD):
            c = node.copies[X]
            if kd == pl.FRC_FWD:
                assert c["role"] == "replica" and X == (n % P + 1) % P
            x_in = None if X == 0 else st[("act", X, k)]
            if X == 0:
                assert ("tok", k) in st
            out, saved = self._stage_fwd(X, c, x_in, k, dp)
            st[("saved", X, k)] = saved
            st[("act", X + 1, k) if X < P - 1 else ("loss", k)] = out
        elif kd in (pl.BWD, pl.BRC_BWD):
            c = node.copies[X]
            d = None if X == P - 1 else st[("dact", X + 1, k)]
            din = self._stage_bwd(X, c, st[("saved", X, k)], d, k, dp)
            if X > 0:
                if kd == pl.BWD:
                    st[("dact", X, k)] = din
                else:   # EFEB: the same value the victim would send; keep a received one
                    st.setdefault(("dact", X, k), din)
            if k == self.M - 1:
                st[("gradsum", X)] = c["g"]
        elif kd in pl.SENDS:
            payload = {pl.SEND_ACT: lambda: st[("act", X + 1, k)],
                       pl.SEND_GRAD: lambda: st[("dact", X, k)],
                       pl.SEND_DGRAD: lambda: st[("dact", X, k)],
                       pl.RESEND_GRAD: lambda: st[("dact", X, k)],
                       # the local sum (AR_SUM never overwrites it)
                       pl.AR_SEND: lambda: node.copies[X]["g"].copy(),
                       pl.RESEND_AR: lambda: node.copies[X]["g"].copy(),
                       pl.REPLICA_SEND: lambda: st[("gradsum", X)].copy()}[kd]()
            self.payloads[id(msg)] = payload
        elif kd in pl.RECVS:
            payload = self.payloads.pop(id(msg))
            if kd == pl.RECV_ACT:
                st[("act", X, k)] = payload
            elif kd in (pl.RECV_GRAD, pl.RECV_DGRAD):
                st[("dact", X + 1, k)] = payload
            elif kd == pl.AR_RECV:
                st[("ar", X, ins.peer // P)] = payload   # a shadow's stays its pipeline's
            else:
                c = node.copies[X]
                c["g"][:] = payload
                st[("gradsum", X)] = c["g"]
        elif kd == pl.AR_SUM:
            # the D contributions in ascending pipeline order
            total = np.zeros_like(node.copies[X]["g"])
            for e in range(self.D):
                total = total + (node.copies[X]["g"] if e == dp else st[("ar", X, e)])
            st[("gradsum", X)] = total
        elif kd == pl.APPLY:
            c = node.copies[X]
            lr, b1, b2, eps = self.hp
            c["t"] += 1
            g = st[("gradsum", X)]   # the stage's total (all-reduced when D > 1)
            c["p"], c["m"], c["v"] = model.adam_update(c["p"], g, c["m"], c["v"], c["t"],
                                                       lr, b1, b2, eps)
        else:
            raise ValueError(kd)

    def _run(self, plans, pcs, channels, cap=None):
        return pl.lockstep(plans, pcs, channels, cap, on_exec=self._exec)

    def _begin_step(self, tokens, targets):
        m = self.cfg.model
        mb, M = self.cfg.micro_batch, self.M
        if len(tokens) != self.D * M * mb:
            raise ValueError("tokens: need D*M*micro_batch sequences")
        self.tokens = [[tokens[(d * M + k) * mb:(d * M + k + 1) * mb] for k in range(M)]
                       for d in range(self.D)]
        self.targets = [[targets[(d * M + k) * mb:(d * M + k + 1) * mb] for k in range(M)]
                        for d in range(self.D)]
        self.n_tok = self.D * M * mb * m.seq_len   # the loss is the mean over the whole batch
        self.payloads = {}
        for n, node in self.nodes.items():
            node.store = {}
            for c in node.copies.values():
                c["g"][:] = 0.0

    def _end_step(self):
        loss = 0.0
        for d in range(self.D):
            for k in range(self.M):
                vals = [node.store[("loss", k)] for n, node in self.nodes.items()
                        if n // self.P == d and n not in self.dead and ("loss", k) in node.store]
                # LFLB: a last stage lost after its commit point took the only
                # copy of its losses with it (no FRC recomputed them): the
                # step's loss is unknown (its update is complete)
                loss += vals[0] if vals else float("nan")
        self.step_no += 1
        self.last_stores = {n: node.store for n, node in self.nodes.items()}
        return loss

    # ------------------------------------------------------------ public API
    def preempt(self, v, pi):
        """Arm a preemption of node v after pi instructions of the next step.
        After a failover, another node can be lost if it is not adjacent to a
        dead one (two independent recoveries); P:464's
        consecutive-node case (the double-duty shadow, or a node whose
        replica holder is dead) is Fatal."""
        if not self.rc or not pl.recoverable(self.P, self.host, self.replica_on, self.dead, v):
            raise pl.Fatal("no replica available for the victim")
        self.pending = (v, pi)

    def step(self, tokens, targets):
        """Run one step. Returns ('ok', loss) or ('preempted', cut info)."""
        if self.interrupted is not None:
            raise RuntimeError("recover() pending")
        self._begin_step(tokens, targets)
        live = {n: p for n, p in self.plans.items() if n not in self.dead}
        if self.pending is None:
            pcs, ch = self._run(live, None, None)
            if any(pcs[n] < len(live[n]) for n in live):
                raise pl.PlanError("deadlock in a failure-free step")
            return "ok", self._end_step()
        v, pi = self.pending
        self.pending = None
        pcs, ch = self._run(live, None, None, cap={v: pi})
        assert pcs[v] == pi
        for key in list(ch):
            if key[1] == v:
                for m in ch[key]:
                    self.payloads.pop(id(m), None)
                del ch[key]
        self.dead.add(v)
        self.nodes[v].store = {}
        self.nodes[v].copies = {}
        self.interrupted = (v, pcs, ch)
        return "preempted", {"victim": v, "pcs": dict(pcs)}

    def recover(self):
        """Run the recovery continuation of the interrupted step; install the
        failover plans for later steps. Returns (loss, info)."""
        v, pcs, ch = self.interrupted
        P, M = self.P, self.M
        u = v - v % P + (v % P - 1) % P
        new, info = pl.recovery_plans(self.plans, P, M, v, pcs, ch)
        self.recovery_info = info
        self.continuation = new
        # promote the replica (the shadow executes the victim's work)
        c = self.nodes[u].copies[v % P]
        c["role"] = "primary"
        self.history.append((self.plans, dict(self.host), dict(self.replica_on)))
        self.host, self.replica_on = pl.lose_node(P, self.host, self.replica_on, v)
        self.mode = "failover"
        self.victims.append(v)
        live = {n: p for n, p in new.items()}
        pcs2, ch = self._run(live, {n: 0 for n in live}, ch)
        if any(pcs2[n] < len(live[n]) for n in live):
            raise pl.PlanError("deadlock in recovery continuation")
        self.plans = pl.failover_plans(P, M, v, self.history[-1][0])
        self.interrupted = None
        return self._end_step(), info

    def rejoin(self):
        """The preempted node returns at a step boundary (reconfiguration back
        to full depth): it receives its stage's
        parameters and Adam state from the shadow and its successor's (for its
        replica) from the successor, reusing existing state as much as
        possible; the shadow's copy becomes a replica again and the
        normal plans resume. Values are unchanged by construction."""
        if self.mode != "failover" or self.interrupted is not None:
            raise RuntimeError("rejoin needs a recovered failover pipeline")
        P, v = self.P, self.victims[-1]    # the most recent victim returns first
        base, sv = v - v % P, v % P
        u, w = base + (sv - 1) % P, base + (sv + 1) % P
        sw_ = (sv + 1) % P
        node = self.nodes[v]
        node.copies = {}
        src = self.nodes[u].copies[sv]
        node.copies[sv] = {k: (val.copy() if isinstance(val, np.ndarray) else val)
                           for k, val in src.items()}
        node.copies[sv]["role"] = "primary"
        sw = self.nodes[w].copies[sw_]
        node.copies[sw_] = {k: (val.copy() if isinstance(val, np.ndarray) else val)
                            for k, val in sw.items()}
        node.copies[sw_]["role"] = "replica"
        src["role"] = "replica"
        self.dead.discard(v)
        self.victims.pop()
        self.plans, self.host, self.replica_on = self.history.pop()
        self.mode = "failover" if self.victims else "normal"

    def dump(self):
        host, rep = (self.host, self.replica_on)
        mode = self.mode
        return pl.dump(self.P, self.M, self.mode_rc, self.ranges, self.plans, host, rep, None, mode,
                       self.victims)
