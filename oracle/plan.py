"""Oracle partition, 1F1B + eager-FRC plans, failover/recovery plan transforms
— TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Sources:
* Layer sharding into contiguous stages, "more layers are placed on the last
  few stages" -> even split of blocks with the
  remainder on the LAST stages; embedding on stage 0, LN_f + head + loss on
  stage P-1.
* Static schedule interpreted as an instruction stream, built on
  PipeDream's 1F1B: stage s runs W_s = min(P-1-s, M) warm-up
  forwards, then M-W_s (forward, backward) pairs, then W_s backwards.
* Replica of stage n on node n-1; node P-1 holds node 0's;
  FRC^n_{n+1} is exactly FNC_{n+1}; the last node fetches input
  samples.
* Eager FRC "before the node starts communicating with its successor"
   and FRC(k-1) overlapping FNC(k): FRC_FWD(k) right after
  SEND_ACT(k); on the last stage right before RECV_ACT(k) (Q4 reading).
* Lazy BRC via a failover schedule merging victim and shadow schedules with
  the four rules of P:538-545 (Q5 reading).
* D > 1 data-parallel pipelines: each stage's gradient sum is
  all-reduced over the pipelines after the node's last backward; a failed
  pipeline's share is replayed by its shadow and the others wait (
  DESIGN.md §2 "D > 1 pipelines"). Pinned in tests/test_oracle_dp.py.

Instruction fields: (kind, mb, peer, stage). `stage` is the logical stage on
whose behalf the node acts; `peer` is a NODE id (node n initially runs stage n).
Text dump (parity format, DESIGN.md §Plan dump):
    # bamboo-plan v1 P=<P> M=<M> rc=<none|eflb> mode=<normal|failover> ...
    # stage <X> node <n> device <d> units <a>..<b> replica_on <r|->
    <node> <ordinal> <KIND> <mb|-> <peer|-> <stage|->
"""
from collections import deque, namedtuple

Instr = namedtuple("Instr", "kind mb peer stage")

LOAD_INPUTS, FWD, FRC_FWD, BWD = "LOAD_INPUTS", "FWD", "FRC_FWD", "BWD"
SEND_ACT, RECV_ACT, SEND_GRAD, RECV_GRAD = "SEND_ACT", "RECV_ACT", "SEND_GRAD", "RECV_GRAD"
RESEND_GRAD, REPLICA_SEND, REPLICA_RECV, APPLY = "RESEND_GRAD", "REPLICA_SEND", "REPLICA_RECV", "APPLY"
BRC_BWD = "BRC_BWD"   # EFEB: eager redundant backward of the replica stage
# EFEB: the duplicate of a stage's input-gradient for the node two back (its
# own message kind, so it never shares a FIFO with the normal gradients)
SEND_DGRAD, RECV_DGRAD = "SEND_DGRAD", "RECV_DGRAD"
# D > 1 data-parallel pipelines: each node sends its stage's
# gradient sum to the nodes of the same stage in the other pipelines, receives
# theirs and adds all D in ascending pipeline order (deterministic; the same
# bits on every pipeline). Message kind "ar"; AR_SUM is the local addition.
# AR_SUM leaves the local sum in place (the update reads the total), so a
# contribution the victim consumed can be sent again to its shadow (RESEND_AR).
AR_SEND, AR_RECV, AR_SUM, RESEND_AR = "AR_SEND", "AR_RECV", "AR_SUM", "RESEND_AR"
SENDS = {SEND_ACT, SEND_GRAD, RESEND_GRAD, REPLICA_SEND, SEND_DGRAD, AR_SEND, RESEND_AR}
RECVS = {RECV_ACT, RECV_GRAD, REPLICA_RECV, RECV_DGRAD, AR_RECV}
COMMS = SENDS | RECVS


class PlanError(Exception):
    pass


class Fatal(Exception):
    """Unrecoverable preemption (consecutive nodes)."""


# ----------------------------------------------------------------------------
# partition (A1)
# ----------------------------------------------------------------------------
def partition(n_layer, P, layers_per_stage=None):
    """Unit ranges [(a, b)] inclusive per stage. Units: 0 = embedding,
    1..L = blocks, L+1 = head."""
    if P < 1 or n_layer < P:
        raise PlanError("need 1 <= P <= n_layer")
    if layers_per_stage is None:
        base, rem = divmod(n_layer, P)
        counts = [base + (1 if s >= P - rem else 0) for s in range(P)]
    else:
        counts = list(layers_per_stage)
        if len(counts) != P or sum(counts) != n_layer or min(counts) < 0:
            raise PlanError("bad layers_per_stage")
        if any(c == 0 for c in counts[1:-1]):
            raise PlanError("interior stage without blocks")
    out, nxt = [], 1
    for s, c in enumerate(counts):
        a = 0 if s == 0 else nxt
        b = nxt + c - 1
        if s == P - 1:
            b = n_layer + 1
        out.append((a, b))
        nxt += c
    return out


# ----------------------------------------------------------------------------
# normal plans (A2)
# ----------------------------------------------------------------------------
MODES = ("none", "eflb", "lflb", "efeb")


def rc_mode(rc):
    """RC mode name from a bool (False = none, True = eflb) or a name."""
    if isinstance(rc, str):
        if rc not in MODES:
            raise PlanError(f"unknown RC mode {rc}")
        return rc
    return "eflb" if rc else "none"


def stage_plan(s, P, M, rc, d=0, D=1):
    """Instruction list of node s in a failure-free step. rc: False / "none"
    (no redundancy), True / "eflb" (replica + eager FRC),
    "lflb" (replica kept in sync, no FRC: the victim's forward is recomputed
    lazily on failure, "LFLB") or "efeb" (eager FRC and eager BRC:
    node s also runs the backward of its replica stage r = s+1 every step,
    BRC_BWD(k), from the gradient node r+1 = s+2 sends it next to its normal
    send, "BRC requires the output of BNC_{n+2}"; the replica's own
    gradient then equals the primary's, so there is no replica sync).
    EFEB placement (this build's reading): BRC_BWD(k) (with its RECV_GRAD
    from s+2) right before node s's own RECV_GRAD(k); on the last node (the
    replica of stage 0 needs stage 1's gradient, which comes last) all of
    them after its own backwards.
    d, D: pipeline d of D data-parallel pipelines (node ids d*P + s, peers in
    the same pipeline); with D > 1 the step's gradient sum of the stage is
    all-reduced over the pipelines (AR_SEND to each other pipeline, AR_RECV
    from each, AR_SUM) before the replica sync and the update. EFEB
    with D > 1 (this build's reading): the replica's eager BRC gradient is
    the pipeline's local one, so the replica is synced with the total like
    EFLB's (REPLICA_SEND / RECV after the all-reduce); the eager BRC still
    spares the recovery the lazy backward."""
    mode = rc_mode(rc)
    rc, frc = mode != "none", mode in ("eflb", "efeb")
    efeb = mode == "efeb"
    r = (s + 1) % P
    if rc and P < 2:
        raise PlanError("RC needs P >= 2")
    I = []
    need_tok = s == 0 or (rc and s == P - 1)
    need_tgt = s == P - 1 or (rc and s == P - 2)
    if need_tok or need_tgt:
        I.append(Instr(LOAD_INPUTS, None, None, None))
    W = min(P - 1 - s, M)

    def fwd(k):
        if frc and s == P - 1:
            I.append(Instr(FRC_FWD, k, None, 0))
        if s > 0:
            I.append(Instr(RECV_ACT, k, s - 1, s))
        I.append(Instr(FWD, k, None, s))
        if s < P - 1:
            I.append(Instr(SEND_ACT, k, s + 1, s))
            if frc:
                I.append(Instr(FRC_FWD, k, None, s + 1))

    def brc(k):
        if r < P - 1 and P >= 3:
            I.append(Instr(RECV_DGRAD, k, (r + 1) % P, r))
        I.append(Instr(BRC_BWD, k, None, r))

    def bwd(k):
        if efeb and s < P - 1:
            brc(k)
        if s < P - 1:
            I.append(Instr(RECV_GRAD, k, s + 1, s))
        I.append(Instr(BWD, k, None, s))
        if s > 0:
            I.append(Instr(SEND_GRAD, k, s - 1, s))
            if efeb and P >= 3:   # the gradient node s-2 needs for its BRC of stage s-1
                I.append(Instr(SEND_DGRAD, k, (s - 2) % P, s))

    for k in range(W):
        fwd(k)
    for i in range(M - W):
        fwd(W + i)
        bwd(i)
    for i in range(M - W, M):
        bwd(i)
    base = d * P
    if efeb and s == P - 1 and D > 1:   # the replica stage's eager BRCs, before the all-reduce
        for k in range(M):
            brc(k)
    if D > 1:
        others = [e * P + s - base for e in range(D) if e != d]   # local offsets
        I.extend(Instr(AR_SEND, None, o, s) for o in others)
        I.extend(Instr(AR_RECV, None, o, s) for o in others)
        I.append(Instr(AR_SUM, None, None, s))
    if efeb and D == 1:
        if s == P - 1:
            for k in range(M):
                brc(k)
        I.append(Instr(APPLY, None, None, s))
        I.append(Instr(APPLY, None, None, r))
    elif rc:
        I.append(Instr(REPLICA_SEND, None, (s - 1) % P, s))
        I.append(Instr(REPLICA_RECV, None, (s + 1) % P, (s + 1) % P))
        I.append(Instr(APPLY, None, None, s))
        I.append(Instr(APPLY, None, None, (s + 1) % P))
    else:
        I.append(Instr(APPLY, None, None, s))
    if base:   # peers are node ids: pipeline d's nodes are d*P + s
        I = [i._replace(peer=i.peer + base) if i.peer is not None else i for i in I]
    return I


def normal_plans(P, M, rc, D=1):
    return {d * P + s: stage_plan(s, P, M, rc, d, D) for d in range(D) for s in range(P)}


def gpipe_plan(s, P, M):
    """GPipe: all forwards, then all backwards (no RC); used only as a
    schedule-independence cross-check."""
    I = []
    if s == 0 or s == P - 1:
        I.append(Instr(LOAD_INPUTS, None, None, None))
    for k in range(M):
        if s > 0:
            I.append(Instr(RECV_ACT, k, s - 1, s))
        I.append(Instr(FWD, k, None, s))
        if s < P - 1:
            I.append(Instr(SEND_ACT, k, s + 1, s))
    for k in range(M):
        if s < P - 1:
            I.append(Instr(RECV_GRAD, k, s + 1, s))
        I.append(Instr(BWD, k, None, s))
        if s > 0:
            I.append(Instr(SEND_GRAD, k, s - 1, s))
    I.append(Instr(APPLY, None, None, s))
    return I


# ----------------------------------------------------------------------------
# data keys and messages (used by the merge's readiness and by the cut)
# ----------------------------------------------------------------------------
def inputs_of(ins, P):
    k, X = ins.mb, ins.stage
    if ins.kind in (FWD, FRC_FWD):
        keys = [("tok", k) if X == 0 else ("act", X, k)]
        if X == P - 1:
            keys.append(("tgt", k))
        return keys
    if ins.kind in (BWD, BRC_BWD):
        return [("saved", X, k)] + ([("dact", X + 1, k)] if X < P - 1 else [])
    if ins.kind == SEND_ACT:
        return [("act", X + 1, k)]
    if ins.kind in (SEND_GRAD, RESEND_GRAD, SEND_DGRAD):
        return [("dact", X, k)]
    if ins.kind in (REPLICA_SEND, APPLY, AR_SEND, RESEND_AR, AR_SUM):
        return [("gradsum", X)]
    return []


def outputs_of(ins, P, M):
    k, X = ins.mb, ins.stage
    if ins.kind == LOAD_INPUTS:
        return [("tok", j) for j in range(M)] + [("tgt", j) for j in range(M)]
    if ins.kind in (FWD, FRC_FWD):
        return [("saved", X, k), ("act", X + 1, k) if X < P - 1 else ("loss", k)]
    if ins.kind in (BWD, BRC_BWD):
        out = [("dact", X, k)] if X > 0 else []
        return out + ([("gradsum", X)] if k == M - 1 else [])
    if ins.kind == RECV_ACT:
        return [("act", X, k)]
    if ins.kind in (RECV_GRAD, RECV_DGRAD):
        return [("dact", X + 1, k)]
    if ins.kind == REPLICA_RECV:
        return [("gradsum", X)]
    return []


def message_of(ins):
    """Descriptor of the message a SEND puts on / a RECV expects at the head of
    the (src node, dst node, kind) FIFO: (kind, mb, producer stage)."""
    if ins.kind == SEND_ACT:
        return ("act", ins.mb, ins.stage)
    if ins.kind == RECV_ACT:
        return ("act", ins.mb, ins.stage - 1)
    if ins.kind in (SEND_GRAD, RESEND_GRAD):
        return ("grad", ins.mb, ins.stage)
    if ins.kind == RECV_GRAD:
        return ("grad", ins.mb, ins.stage + 1)
    if ins.kind in (REPLICA_SEND, REPLICA_RECV):
        return ("gradsum", None, ins.stage)
    if ins.kind in (AR_SEND, AR_RECV, RESEND_AR):
        return ("ar", None, ins.stage)
    if ins.kind == SEND_DGRAD:
        return ("dgrad", ins.mb, ins.stage)
    if ins.kind == RECV_DGRAD:
        return ("dgrad", ins.mb, ins.stage + 1)
    raise ValueError(ins)


# ----------------------------------------------------------------------------
# lockstep execution (O4) over symbolic messages; used to find the cut
# ----------------------------------------------------------------------------
def lockstep(plans, pcs=None, channels=None, cap=None, on_exec=None):
    """Round-robin over nodes in ascending id: execute each node's next
    instruction if it is not a RECV whose message is absent. Sends are
    buffered in per-(src, dst, message kind) FIFOs. Runs until no node can progress.
    `cap[n]` limits node n to its first cap[n] instructions (injection).
    `on_exec(node, ins, msg)` is called for every executed instruction.
    Returns (pcs, channels). Asserts FIFO consistency."""
    pcs = {n: 0 for n in plans} if pcs is None else pcs
    channels = {} if channels is None else channels
    cap = cap or {}
    progress = True
    while progress:
        progress = False
        for n in sorted(plans):
            lim = min(len(plans[n]), cap.get(n, len(plans[n])))
            if pcs[n] >= lim:
                continue
            ins = plans[n][pcs[n]]
            msg = None
            if ins.kind in RECVS:
                ch = channels.get((ins.peer, n, message_of(ins)[0]))
                if not ch:
                    continue
                msg = ch.popleft()
                if msg[0] != message_of(ins):
                    raise PlanError(f"FIFO mismatch at node {n}: {ins} got {msg[0]}")
            elif ins.kind in SENDS:
                msg = (message_of(ins), n)
                channels.setdefault((n, ins.peer, msg[0][0]), deque()).append(msg)
            pcs[n] += 1
            progress = True
            if on_exec is not None:
                on_exec(n, ins, msg)
    return pcs, channels


# ----------------------------------------------------------------------------
# failover / recovery transforms (A12/A13)
# ----------------------------------------------------------------------------
def _rank(ins):
    return {BWD: 0, BRC_BWD: 0, FWD: 1, FRC_FWD: 1}.get(ins.kind, 2)


def merge(A, B, avail, P, M, u, others, channels):
    """Two-sequence merge of the shadow's (A) and victim's (B) remaining
    instructions (Q5): each sequence keeps its program order; at
    each point pick among the READY heads: (1) communication before
    computation; (3) among communications the victim's (B) first; (4) among
    computations backward before forward, then ascending micro-batch, then
    the victim's first. Victim<->shadow messages were already deleted by the
    caller (rule 2).

    READY: a computation or send needs its local input keys available; a
    receive needs its message to have arrived. Arrival is decided by
    co-simulating the other survivors' lists (`others`, lockstep) against the
    shadow's placed prefix, so a receive is never placed ahead of a local
    send it transitively waits for (e.g. when the shadow hosts both the last
    and the first stage)."""
    avail = set(avail)
    och = {key: deque(q) for key, q in channels.items()}
    opcs = {n: 0 for n in others}
    pl_others = dict(others)
    lockstep(pl_others, opcs, och)
    a = b = 0
    out = []

    def ready(ins):
        if ins.kind in RECVS:
            q = och.get((ins.peer, u, message_of(ins)[0]))
            if not q:
                return False
            return q[0][0] == message_of(ins)   # the FIFO head is this message
        return all(key in avail for key in inputs_of(ins, P))

    while a < len(A) or b < len(B):
        cand = []
        if a < len(A) and ready(A[a]):
            cand.append((A[a], 1))
        if b < len(B) and ready(B[b]):
            cand.append((B[b], 0))
        if not cand:
            raise PlanError("merge deadlock")

        def key(c):
            ins, side = c
            if ins.kind in COMMS:
                return (0, side, 0, 0)
            return (1, _rank(ins), -1 if ins.mb is None else ins.mb, side)
        ins, side = min(cand, key=key)
        out.append(ins)
        avail.update(outputs_of(ins, P, M))
        if ins.kind in RECVS:
            och[(ins.peer, u, message_of(ins)[0])].popleft()
        elif ins.kind in SENDS:
            och.setdefault((u, ins.peer, message_of(ins)[0]), deque()).append((message_of(ins), u))
            lockstep(pl_others, opcs, och)
        if side == 1:
            a += 1
        else:
            b += 1
    return out


def recovery_plans(plans, P, M, v, pcs, channels):
    """Continuation lists for the surviving nodes after node v died with the
    cut (pcs, channels) (all nodes lockstepped to quiescence with v capped).
    With pcs all 0 and empty channels this yields the static failover plans
    used for the following iterations ("all instructions of the victim node
    must be executed by its shadow node").

    Node ids are d*P + s for pipeline d (D >= 1): the shadow and successor
    are the victim's neighbours in its own pipeline; instructions name the
    pipeline-local stage sv = v % P.

    Returns (new_plans, info). Raises Fatal if unrecoverable."""
    base, sv = v - v % P, v % P
    u, w = base + (sv - 1) % P, base + (sv + 1) % P
    pv = plans[v]
    executed_v = pv[:pcs[v]]
    commit = any(i.kind == REPLICA_SEND for i in executed_v)
    # EFEB (eager BRC): the shadow already runs the victim stage's backward
    # (BRC_BWD) from the duplicate gradients w sends it, so the victim's
    # backward, its APPLY and its receives from w are not replayed; every
    # message to the victim is dropped (the shadow has its copy) and every
    # receive from it is rerouted to the shadow, which takes over the
    # victim's remaining sends (its duplicate gradients for node v-2).
    efeb = any(i.kind == BRC_BWD for seq in plans.values() for i in seq)
    # D > 1: the update reads the all-reduced total, so the victim stage's
    # APPLY follows its all-reduce in B (EFEB too)
    dp = any(i.kind == AR_SEND for seq in plans.values() for i in seq)

    def executed(n):
        return plans[n][:pcs[n]]

    # messages from v that a survivor has not consumed yet (delivered, in FIFO)
    pending_from_v = {n: {kind: [m for m, _ in channels.get((v, n, kind), [])]
                          for kind in ("act", "grad", "gradsum", "dgrad", "ar")}
                      for n in plans if n != v}

    def delivered_filter(n, seq, local_peer_to):
        """Walk n's remaining RECVs from v in order against the delivered FIFO:
        matched ones stay (peer v); unmatched ones are rewritten by
        local_peer_to(ins) (None = delete, else new peer)."""
        qs = {kind: deque(q) for kind, q in pending_from_v[n].items()}
        out = []
        for ins in seq:
            if ins.kind in RECVS and ins.peer == v:
                q = qs[message_of(ins)[0]]
                if q and q[0] == message_of(ins):
                    q.popleft()
                    out.append(ins)
                else:
                    np_ = local_peer_to(ins)
                    if np_ is not None:
                        out.append(ins._replace(peer=np_))
                continue
            out.append(ins)
        return out

    # ---- A: the shadow's remaining instructions
    A = []
    for ins in plans[u][pcs[u]:]:
        if ins.kind == FRC_FWD and ins.stage == sv:
            continue                                  # becomes v's FWD (in B)
        if ins.kind in SENDS and ins.peer == v:
            continue                                  # victim<->shadow (rule 2)
        if ins.kind == APPLY and ins.stage == sv and not commit and (not efeb or dp):
            continue                                  # v's update runs from B
        A.append(ins)
    A = delivered_filter(u, A, lambda ins: None)

    # ---- B: the victim's whole-step instructions, rewritten for the shadow
    B = []
    frc_done = {i.mb for i in executed(u) if i.kind == FRC_FWD and i.stage == sv}
    if not commit:
        for idx, ins in enumerate(pv):
            kd = ins.kind
            if kd in (LOAD_INPUTS, FRC_FWD, REPLICA_SEND, REPLICA_RECV):
                continue
            if kd == APPLY and (ins.stage != sv or (efeb and not dp)):
                continue
            if efeb and kd in (BWD, BRC_BWD, RECV_GRAD, RECV_DGRAD):
                continue                              # the shadow's BRC_BWD does it
            if kd in COMMS and ins.peer == u:
                continue                              # rule 2: becomes local
            if kd == FWD and ins.mb in frc_done:
                continue                              # use the retained FRC result
            if kd in SENDS and idx < pcs[v]:
                continue                              # already delivered
            B.append(ins)

    # ---- W: the successor's remaining instructions, rerouted to the shadow
    new = {}
    for n in plans:
        if n == v:
            continue
        seq = A if n == u else list(plans[n][pcs[n]:])
        if efeb and n != u and n // P == v // P:
            seq = [i for i in seq if not (i.kind in SENDS and i.peer == v)]
            seq = delivered_filter(n, seq, lambda ins: u)
        elif n != w and n != u:
            # another pipeline's node of the victim's stage (D > 1): its
            # all-reduce traffic with v goes to the shadow, which replays v's
            # whole all-reduce; a contribution already sent to v went down
            # with it and is sent again (RESEND_AR, first: the gradient sum
            # it reads is complete and AR_SUM never overwrites it)
            # (not after v's commit point: v's all-reduce was complete)
            resend = [] if commit else [Instr(RESEND_AR, None, u, i.stage) for i in executed(n)
                                        if i.kind == AR_SEND and i.peer == v]
            seq = [i._replace(peer=u) if i.kind in SENDS and i.peer == v else i for i in seq]
            seq = resend + delivered_filter(n, seq, lambda ins: u)
        elif n == w:
            resend = []
            if not commit and w != u:
                resend = [Instr(RESEND_GRAD, i.mb, u, i.stage) for i in executed(w)
                          if i.kind == SEND_GRAD and i.peer == v]
            seq2 = []
            for ins in seq:
                if ins.kind == REPLICA_SEND and ins.peer == v:
                    continue
                if ins.kind in SENDS and ins.peer == v:
                    ins = ins._replace(peer=u)
                seq2.append(ins)
            seq = resend + delivered_filter(w, seq2, lambda ins: u) if w != u else seq2
        new[n] = seq
    avail = set()
    for ins in executed(u):
        avail.update(outputs_of(ins, P, M))
    others = {n: seq for n, seq in new.items() if n != u}
    new[u] = merge(new[u], B, avail, P, M, u, others, channels)
    info = {"victim": v, "shadow": u, "successor": w, "commit": commit,
            "frc_done": sorted(frc_done),
            "brc_mb": sorted(i.mb for i in (A if efeb else B)
                             if i.kind in (BWD, BRC_BWD) and i.stage == sv),
            "resend": [i.mb for i in new.get(w, []) if i.kind == RESEND_GRAD]}
    return new, info


def failover_plans(P, M, v, plans=None):
    """Static failover plans for the iterations after a recovery:
    the recovery transform of `plans` (default: the normal plans; after an
    earlier failover, that failover's plans) at an empty cut."""
    plans = normal_plans(P, M, True) if plans is None else plans
    new, _ = recovery_plans(plans, P, M, v, {n: 0 for n in plans}, {})
    return new


def recoverable(P, host, replica_on, dead, v):
    """A preemption of node v is recoverable iff v is alive, runs exactly its
    own stage (a shadow running two stages loses one with no replica left:
    P:464 "consecutive nodes"), and v's stage has a replica on a live node
    (its predecessor). Non-adjacent preemptions after a failover are two
    independent recoveries."""
    if v in dead or v not in host:
        return False
    if [X for X in host if host[X] == v] != [v]:
        return False
    r = replica_on[v]
    return r is not None and r not in dead and r == v - v % P + (v % P - 1) % P


def cut(plans, v, pi):
    """Lockstep with node v capped at pi instructions (Q12/Q14): the maximal
    progress every survivor can make. Returns (pcs, channels)."""
    if not (0 <= pi <= len(plans[v])):
        raise PlanError("injection point out of range")
    pcs, ch = lockstep(plans, cap={v: pi})
    if pcs[v] != pi:
        raise PlanError("victim did not reach its injection point")
    # messages addressed to the victim are lost with it
    for key in list(ch):
        if key[1] == v:
            del ch[key]
    return pcs, ch


# ----------------------------------------------------------------------------
# text dump
# ----------------------------------------------------------------------------
def _f(x):
    return "-" if x is None else str(x)


def dump(P, M, rc, ranges, plans, host=None, replica_on=None, device=None, mode="normal",
         victim=None):
    """host[X] = node running (global) stage X; replica_on[X] = node holding
    X's replica. With D > 1 pipelines the global stage of pipeline d's stage
    s is d*P + s (pass host / replica_on / device for all of them)."""
    host = host or {s: s for s in range(P)}
    if replica_on is None:
        replica_on = {X: ((X - X % P + (X % P - 1) % P) if rc else None) for X in host}
    device = device or {n: 0 for n in host}
    hdr = f"# bamboo-plan v1 P={P} M={M} rc={rc_mode(rc)} mode={mode}"
    if mode != "normal":
        vs = list(victim) if isinstance(victim, (list, tuple)) else [victim]
        hdr += (f" victim={','.join(map(str, vs))}"
                f" shadow={','.join(str(x - x % P + (x % P - 1) % P) for x in vs)}")
    lines = [hdr]
    for X in sorted(host):
        a, b = ranges[X % P]
        lines.append(f"# stage {X} node {host[X]} device {device[host[X]]} units {a}..{b} "
                     f"replica_on {_f(replica_on[X])}")
    for n in sorted(plans):
        for i, ins in enumerate(plans[n]):
            lines.append(f"{n} {i} {ins.kind} {_f(ins.mb)} {_f(ins.peer)} {_f(ins.stage)}")
    return "\n".join(lines) + "\n"


def lose_node(P, host, replica_on, v):
    """(host, replica_on) after node v died and its stage moved to the shadow
    v-1 (Q21): v's stage runs on the shadow without a replica (the replica was
    promoted), and every stage whose replica lived on v is unprotected."""
    u = v - v % P + (v % P - 1) % P
    host, replica_on = dict(host), dict(replica_on)
    host[v] = u
    for X in replica_on:
        if replica_on[X] == v:
            replica_on[X] = None
    replica_on[v] = None
    return host, replica_on


def normal_topology(P, D=1):
    """(host, replica_on) keyed by global stage d*P + s (= its node)."""
    n = P * D
    return ({g: g for g in range(n)}, {g: g - g % P + (g % P - 1) % P for g in range(n)})


def failover_topology(P, v, D=1):
    """(host, replica_on) after stage v moved to its shadow (Q21)."""
    return lose_node(P, *normal_topology(P, D), v)


# ----------------------------------------------------------------------------
# unit-cost timing replay of a plan (for the schedule pins S:191)
# ----------------------------------------------------------------------------
def simulate_times(plans, P, fwd_t, bwd_t, frc=True):
    """Event replay with compute costs fwd_t[X] / bwd_t[X] per stage, zero-cost
    communication, one compute resource per node (FRC_FWD costs fwd_t of its
    stage when frc is True, else 0). Returns (end time per node, per-node
    list of (kind, mb, start, end))."""
    t_node = {n: 0.0 for n in plans}
    msg_time = {}
    pcs = {n: 0 for n in plans}
    timeline = {n: [] for n in plans}
    progress = True
    while progress:
        progress = False
        for n in sorted(plans):
            if pcs[n] >= len(plans[n]):
                continue
            ins = plans[n][pcs[n]]
            start = t_node[n]
            if ins.kind in RECVS:
                key = (ins.peer, n, message_of(ins))
                if key not in msg_time:
                    continue
                start = max(start, msg_time.pop(key))
                end = start
            elif ins.kind in SENDS:
                msg_time[(n, ins.peer, message_of(ins))] = start
                end = start
            elif ins.kind == FWD:
                end = start + fwd_t[ins.stage]
            elif ins.kind == FRC_FWD:
                end = start + (fwd_t[ins.stage] if frc else 0.0)
            elif ins.kind == BWD:
                end = start + bwd_t[ins.stage]
            else:
                end = start
            timeline[n].append((ins.kind, ins.mb, start, end))
            t_node[n] = end
            pcs[n] += 1
            progress = True
    if any(pcs[n] < len(plans[n]) for n in plans):
        raise PlanError("replay deadlock")
    return t_node, timeline


def dump_lines(plans):
    out = []
    for n in sorted(plans):
        for i, ins in enumerate(plans[n]):
            out.append(f"{n} {i} {ins.kind} {_f(ins.mb)} {_f(ins.peer)} {_f(ins.stage)}")
    return "".join(line + "\n" for line in out)


def recovery_dump(P, M, v, pi, rc=True, D=1):
    """Cut + continuation text of an injection at (v, pi) (DESIGN.md format)."""
    plans = normal_plans(P, M, rc, D)
    pcs, ch = cut(plans, v, pi)
    new, info = recovery_plans(plans, P, M, v, pcs, ch)
    hdr = (f"# bamboo-recovery v1 P={P} M={M} victim={v} shadow={info['shadow']} "
           f"successor={info['successor']} commit={1 if info['commit'] else 0}\n")
    hdr += "# cut" + "".join(f" {n}:{pcs[n]}" for n in sorted(pcs)) + "\n"
    return hdr + dump_lines(new)
