/*
 * bamboo.h — C ABI of the B200-native Bamboo redundant-computation pipeline
 * (arXiv 2204.12013; PAPER.md = /root/reference/PAPER.md line numbers "P:N").
 *
 * The library runs a synchronous 1F1B pipeline-parallel training step of a
 * GPT/BERT-style transformer in which every node also runs
 * a redundant forward (FRC) of its successor's layers in the pipeline bubbles
 * and keeps a replica of the successor's parameters and
 * Adam state. A preempted node's predecessor (its "shadow") promotes
 * that replica, runs the lazy redundant backward (BRC) and the weight update,
 * and the pipeline continues on a merged failover schedule
 * without a checkpoint restart.
 *
 * Processes and devices. One process per GPU. A context hosts the pipeline
 * NODES mapped to its rank (node n runs stage n until a failover); several
 * nodes may share one process/GPU (stages > GPUs), and several processes may
 * share one GPU (tests). Nodes on different ranks exchange activations,
 * gradients and replica gradients through the library's own transport: the
 * sender's copy engine writes the payload into the receiver's HBM over
 * NVLink/NVSwitch (CUDA IPC), records an interprocess event and publishes a
 * sequence number in host shared memory. The ranks rendezvous through a
 * POSIX shared-memory segment named after a session id that the caller
 * creates on rank 0 (bb_session_id) and broadcasts. Each node uses two
 * streams and each cross-rank edge one, so processes should set
 * CUDA_DEVICE_MAX_CONNECTIONS=32 before creating their CUDA context.
 *
 * Conventions for every entry point:
 *  - Returns bb_status (0 = BB_OK). No exception, exit() or abort() crosses
 *    the ABI; CUDA failures map to BB_E_CUDA (BB_E_NCCL is reserved) and the
 *    message is kept per context (bb_last_error).
 *  - Host pointers passed in are borrowed for the duration of the call only
 *    (copied before return). Output host buffers are caller-owned.
 *  - Device pointers (bb_op_* only) are caller-owned CUDA device memory on the
 *    current device; the call is asynchronous on the given stream.
 *  - A context is not thread-safe: one call at a time.
 *  - After BB_E_PREEMPTED only bb_recover, bb_read_state, bb_*_dump,
 *    bb_last_error and bb_destroy are legal; after BB_E_FATAL only
 *    bb_read_state, bb_*_dump, bb_last_error and bb_destroy.
 */
#ifndef BAMBOO_H
#define BAMBOO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BB_OK = 0,
  BB_E_INVAL = -1,        /* bad argument / configuration                                  */
  BB_E_CUDA = -2,         /* CUDA runtime or driver error                                   */
  BB_E_NCCL = -3,         /* NCCL error                                                     */
  BB_E_OOM = -4,          /* device allocation failed                                       */
  BB_E_PREEMPTED = -5,    /* step interrupted by an injected preemption: call bb_recover    */
  BB_E_FATAL = -6,        /* unrecoverable: consecutive / unprotected stage lost    */
  BB_E_STATE = -7,        /* call not legal in the current state                            */
  BB_E_UNSUPPORTED = -8   /* valid request this build does not implement                    */
} bb_status;

/* Redundant-computation modes:
 *  NONE  no replicas, no FRC: a preemption is fatal;
 *  EFLB  eager FRC in the bubbles, lazy BRC on failure (the paper's choice);
 *  LFLB  replicas kept in sync but no FRC: a failure recomputes the victim's
 *        forward (lazy FRC) and backward (lazy BRC) for the whole step;
 *  EFEB  eager FRC and eager BRC: node s also runs stage s+1's backward every
 *        step from the gradient node s+2 sends it ("requires the output
 *        of BNC_{n+2}"), so a failure needs no recomputation at all. */
typedef enum { BB_RC_NONE = 0, BB_RC_EFLB = 1, BB_RC_LFLB = 2, BB_RC_EFEB = 3 } bb_rc_mode;
typedef enum { BB_PREC_BF16 = 0, BB_PREC_FP32_CHECK = 1 } bb_precision;

/* Transformer shape (readings in DESIGN.md): pre-LN GPT-2 block,
 * GELU-tanh, learned positions, untied LM head without bias, LN eps 1e-5.
 * causal = 1 for GPT (causal mask), 0 for BERT (bidirectional). vocab is the
 * padded vocabulary used by the embedding and the head. d_model % n_head == 0
 * and d_model, d_ff, vocab multiples of 8 are required. */
typedef struct {
  int n_layer, d_model, n_head, d_ff, vocab, seq_len, causal;
} bb_model;

typedef struct {
  int micro_batch;              /* sequences per micro-batch (mb)                          */
  bb_rc_mode rc;                /* BB_RC_EFLB needs stages >= 2 (no successor otherwise)   */
  bb_precision prec;            /* bf16 operands + fp32 accumulate, or all-fp32 check mode */
  const int *layers_per_stage;  /* [stages] transformer blocks per stage, NULL = even split
                                   with the remainder on the last stages          */
  float lr, beta1, beta2, eps;  /* Adam, bias-corrected, no weight decay          */
  int world_rank, world_size;   /* this process / number of processes (1 = single process) */
  int device;                   /* CUDA device ordinal this process uses                   */
  const int *node_rank;         /* [stages] process rank hosting node n; NULL = contiguous
                                   blocks of ceil(stages/world_size) nodes per rank        */
  const void *session_id;       /* 32-byte session id (bb_session_id on rank 0, same bytes
                                   on every rank) naming the host-shm rendezvous; NULL
                                   when world_size = 1                                    */
  int profile;                  /* 1 = time every kernel class with CUDA events; the local
                                   nodes then share ONE serialised stream (no FRC overlap),
                                   so use it for per-kernel timing, not for throughput.
                                   Each step first parks that stream for 200 ms of device
                                   time (a spin kernel, outside device_ms) so the host
                                   enqueues ahead: no launch latency inside the brackets */
  size_t frc_retain_bytes;      /* per node: HBM for FRC saved sets kept for a lazy BRC
                                   (SURVEY Q10). 0 = keep all M. Micro-batches past
                                   the budget keep only the stage input and the output;
                                   BRC recomputes their forward (bit-identical)          */
  int frc_persistent;           /* 0 (default): FRC GEMMs launch one CTA per tile, so the
                                   high-priority main stream takes SMs back at tile
                                   granularity; 1: persistent full-device grids (r01)     */
  int timing;                   /* 1 = per-instruction CUDA events on every node for
                                   bb_node_stats (busy / bubble / FRC accounting)        */
  int detect_ms;                /* 0 (default): injected preemptions, bb_preempt called with
                                   the same arguments on every rank. > 0: fail-stop mode
                                   (needs one node per rank, world_size = pipelines *
                                   stages): bb_preempt is called on the
                                   victim's rank only; that rank stops at the injection
                                   point and goes silent (its bb_step returns
                                   BB_E_PREEMPTED; the caller then calls bb_destroy and
                                   exits). The other ranks detect the loss when the
                                   victim's heartbeat in host shared memory is older than
                                   detect_ms (P:417-420 timeouts), run to quiescence,
                                   agree on the cut from the victim's delivered messages
                                   and return BB_E_PREEMPTED from their own bb_step     */
  int pipelines;                /* D data-parallel pipelines, default 1. Node
                                   d*stages + s runs stage s of pipeline d on micro-batches
                                   d*M .. d*M+M-1 of the step's D*M*micro_batch sequences;
                                   its shadow / successor are its ring neighbours inside
                                   pipeline d. After its last backward every stage's fp32
                                   gradient sum is all-reduced with the same stage of the
                                   other pipelines (sum in ascending pipeline order, so
                                   every pipeline applies the same bits) before the replica
                                   sync and Adam; a preempted pipeline's all-reduce is run
                                   by its shadow after the recovery and the others wait for
                                   it. node_rank then has D*stages entries. EFEB:
                                   the replica is synced with the total as in EFLB        */
  size_t frc_swap_bytes;        /* per replica: pinned host memory for the FRC saved sets
                                   beyond frc_retain_bytes ("swap out these data"):
                                   each is copied to the host on its own stream after the
                                   FRC and copied back by a lazy BRC instead of being
                                   recomputed. 0 (default) = recompute. Costs PCIe time
                                   per step                                 */
} bb_opts;

typedef struct {
  float loss;            /* mean token cross-entropy of the step (NaN on ranks without stage P-1;
                            D > 1: the sum over this rank's pipelines of their share, each
                            share = its tokens' CE summed / all D*M*mb*S tokens)           */
  float step_ms;         /* host wall time of the call                                    */
  float device_ms;       /* max over local nodes of main-stream time of the step          */
  int gpu_launches;      /* kernels this process launched during the call                 */
  uint64_t h2d_bytes, d2h_bytes;
} bb_step_stats;

typedef struct {
  int victim, shadow, successor;
  int commit;            /* 1 = victim had already delivered its gradient sum (no BRC)    */
  int brc_mb;            /* micro-batches whose backward was recomputed (lazy BRC)        */
  int frc_done_mb;       /* micro-batches whose retained FRC result was reused            */
  int resent_mb;         /* gradients the successor re-sent to the shadow                 */
  float recover_ms;      /* host wall time of bb_recover                                   */
  float loss;            /* loss of the interrupted step (NaN where not local)           */
  float interrupted_step_ms;  /* host wall time of the bb_step call that was interrupted  */
  int frc_recomputed_mb; /* forwards of the victim's stage recomputed during recovery: FRC
                            catch-up, beyond-budget BRC re-forwards, LFLB lazy FRC        */
  uint64_t bytes_resent; /* bytes re-sent (RESEND_GRAD) or rerouted during the recovery  */
  int frc_swapped_mb;    /* FRC saved sets the lazy BRC copied back from host memory      */
} bb_recovery_stats;

/* Per-node accounting of the last step (opts.timing = 1), from CUDA events
 * around every FWD / BWD (main stream) and FRC_FWD (FRC stream), relative to
 * the node's step start. bubble = step - main busy; frc_hidden = FRC time
 * that ran while the main stream was idle (fig:bubble). */
typedef struct {
  int node;              /* node id                                                        */
  int n_fwd, n_bwd, n_frc;
  float step_ms;         /* node main-stream step time (device)                           */
  float busy_ms;         /* union of main-stream FWD/BWD intervals                         */
  float bubble_ms;       /* step_ms - busy_ms                                              */
  float frc_ms;          /* union of FRC intervals                                         */
  float frc_hidden_ms;   /* FRC time inside main-stream idle time                          */
} bb_node_stat;

/* Fill *o with defaults: micro_batch 1, rc EFLB, bf16, Adam(1e-4, 0.9, 0.999, 1e-8),
 * single process on device 0. */
void bb_default_opts(bb_opts *o);

/* Write a fresh random 32-byte session id into out (cap >= 32; rank 0 only,
 * then broadcast by the caller). */
bb_status bb_session_id(void *out, size_t cap);

/* Create a context for `stages` pipeline stages (P) and `microbatches` (M) per
 * step. Partitions layers, builds every node's static plan
 * (1F1B P:497; eager FRC P:520-521), allocates parameters, replicas
 * (P:429), activation stashes and FRC retention in HBM, creates
 * streams and the cross-rank transport (rendezvous on opts.session_id).
 * Errors: BB_E_INVAL for n_layer < stages, rc with stages < 2, bad shapes;
 * BB_E_UNSUPPORTED for shapes the kernels do not take (bf16 needs
 * d_model >= 64; head dim 64 or 32); BB_E_OOM; BB_E_CUDA. */
bb_status bb_init(const bb_model *m, int stages, int microbatches, const bb_opts *o,
                  void **ctx_out);

/* Load parameters from `host` = the full canonical flat fp32 vector of n
 * values (order in DESIGN.md "Parameter layout"). Every rank passes the same
 * vector; each copies the slices of the stages it hosts and of the replicas
 * it keeps. Resets Adam state and step count. */
bb_status bb_load_params(void *ctx, const float *host, size_t n);

/* One training step over D*M*mb sequences (D = opts.pipelines): tokens,
 * targets = host int32 arrays [D*M*mb, seq_len] row-major (micro-batch j =
 * rows j*mb..j*mb+mb-1; pipeline d takes j = d*M .. d*M+M-1). Every rank
 * passes the full arrays and uploads what its nodes need (the last node
 * fetches inputs for its FRC). Token and target ids must lie in [0, vocab):
 * BB_E_INVAL otherwise (checked before any device work). Returns BB_E_PREEMPTED if an armed injection
 * fired (bb_recover must follow). st may be NULL. tokens = targets = NULL
 * reuses the inputs last staged with bb_stage_inputs (already in HBM: no
 * host-to-device copy inside the call). */
bb_status bb_step(void *ctx, const int32_t *tokens, const int32_t *targets, bb_step_stats *st);

/* Upload tokens/targets (same layout as bb_step) to every local node's HBM
 * now, so that following bb_step(ctx, NULL, NULL, st) calls run on resident
 * inputs. A bb_step with host arrays replaces them. */
bb_status bb_stage_inputs(void *ctx, const int32_t *tokens, const int32_t *targets);

/* Arm a preemption of node `stage` (a node id: 0 <= stage < pipelines *
 * stages, node d*stages + s runs stage s of pipeline d) after it has executed
 * `at_instr` (pi) instructions of its list in the next step (0 <= pi <= list
 * length; BB_E_INVAL otherwise). Must be called with the same arguments on
 * every rank (fail-stop mode: on the victim's rank only). BB_E_FATAL if no
 * redundancy is left for that node: rc off, the node is dead, runs a second
 * stage as a shadow, or its replica holder is dead (P:464 consecutive nodes,
 * SURVEY Q18); a non-adjacent node after a failover is recoverable (SPEC
 * S:537). */
bb_status bb_preempt(void *ctx, int stage, int at_instr);

/* Finish the interrupted step on the survivors: the shadow promotes the
 * replica, runs FRC catch-up, the lazy BRC for every micro-batch of the step,
 * the successor re-sends its retained gradients and is rerouted, and both
 * stages' Adam updates run; later steps use the merged failover
 * plan. Called on every rank (the victim's rank drains and NaN-poisons the
 * victim's memory). r may be NULL. */
bb_status bb_recover(void *ctx, bb_recovery_stats *r);

/* Reconfigure back to full depth at a step boundary after a recovery
 * (SURVEY.md §8(f)-1): the preempted node returns on its rank,
 * receives its stage's parameters and Adam state from the shadow and its
 * successor's (for its replica) from the successor; the shadow's copy
 * becomes a replica again and the normal plans (with full protection)
 * resume, so later preemptions are recoverable again. Called on every rank.
 * BB_E_STATE unless the pipeline is in failover mode with no pending
 * recovery. */
bb_status bb_rejoin(void *ctx);

enum { BB_STATE_PARAMS = 0, BB_STATE_GRADS = 1, BB_STATE_ADAM_M = 2, BB_STATE_ADAM_V = 3 };
/* Copy stage `stage`'s fp32 state (what = BB_STATE_*) into host[n], n = the
 * stage's parameter count. replica = 0 reads the copy the stage runs on
 * (primary; the promoted replica after a failover), 1 reads the replica kept
 * by its predecessor. BB_E_INVAL if that copy is not hosted by this process.
 * With D > 1 pipelines, stage < stages reads the lowest local pipeline's copy
 * and stage = d*stages + s reads pipeline d's copy of stage s; GRADS is the
 * pipeline's local gradient sum (before the all-reduce). */
bb_status bb_read_state(void *ctx, int stage, int replica, int what, float *host, size_t n);

/* Overwrite stage `stage`'s fp32 state (what = BB_STATE_PARAMS, _ADAM_M or
 * _ADAM_V; PARAMS also refreshes the bf16 working copy) in every copy this
 * process hosts (primary and replica, so replica == primary is kept; with
 * D > 1 the copies of every local pipeline), from host[n]. For starting a
 * step from a given state (e.g. an oracle's), at a step boundary. BB_E_INVAL
 * for a bad stage (0 <= stage < stages), kind or size. */
bb_status bb_write_state(void *ctx, int stage, int what, const float *host, size_t n);

/* HBM plan of `stage`: bytes of one saved set (the activations its backward
 * reads, one micro-batch) and how many FRC saved sets its replica keeps per
 * step under opts.frc_retain_bytes (-1 if this process hosts no replica of
 * the stage). Either output may be NULL. */
bb_status bb_stage_memory(void *ctx, int stage, size_t *slot_bytes, int *retained);

/* Number of parameters of `stage` and its offset in the canonical flat vector. */
bb_status bb_stage_params(void *ctx, int stage, size_t *offset, size_t *count);

/* Text dump of the current plans: header, stage
 * assignment, one instruction per line. Writes at most cap bytes (NUL
 * terminated) and the required size (including NUL) into *needed. */
bb_status bb_schedule_dump(void *ctx, char *buf, size_t cap, size_t *needed);

/* Text dump of the last recovery: the cut (instructions executed per node)
 * and the continuation lists, same line format. */
bb_status bb_recovery_dump(void *ctx, char *buf, size_t cap, size_t *needed);

/* Per-node busy / bubble / FRC accounting of the last step (opts.timing = 1):
 * one entry per live local node, *n = count. BB_E_STATE if timing is off. */
bb_status bb_node_stats(void *ctx, bb_node_stat *out, int cap, int *n);

/* Per-kernel-class device time of the last step (profile = 1): for each class
 * c < *n_classes: name, launches, total ms, algorithmic flops or bytes. */
typedef struct { char name[32]; int launches; double ms; double work; } bb_kernel_stat;
bb_status bb_kernel_stats(void *ctx, bb_kernel_stat *out, int cap, int *n_classes);

/* Host-only (no GPU, no context): the plan text of a configuration.
 * victim < 0: the normal plans (same text as bb_schedule_dump after bb_init);
 * victim >= 0 and at_instr >= 0: the cut and continuation lists of an
 * injection at (victim, at_instr) (same text as bb_recovery_dump);
 * victim >= 0 and at_instr < 0: the static failover plans after losing victim. */
bb_status bb_plan_dump(const bb_model *m, int stages, int microbatches, const bb_opts *o,
                       int victim, int at_instr, char *buf, size_t cap, size_t *needed);

/* Transport microbenchmark (no context): two processes (rank 0 / 1, device
 * ordinals of their own, same 32-byte session id) ping-pong `iters`
 * messages of `bytes` through the library's transport (copy-engine write into
 * the peer's HBM, interprocess event, sequence number in host shared
 * memory); each reply's copy waits on the arrival of the message it answers.
 * *us = mean one-way time per message including the data movement, on
 * rank 0. */
bb_status bb_xport_pingpong(int rank, int world, int device, const void *session_id,
                            size_t bytes, int iters, float *us);

bb_status bb_last_error(const void *ctx, char *buf, size_t cap);
void bb_destroy(void *ctx);

/* ---- single-op entry points (kernel parity tests and roofline timing) ----
 * All pointers are device pointers; `stream` is a cudaStream_t (0 = default).
 * bf16 data is passed as uint16 bit patterns. */

/* D[m][n] = sum_k A(m,k) B(n,k) with A(m,k) = A[m*lda+k] (a_mn = 0) or
 * A[k*lda+m] (a_mn = 1), B likewise; epilogue `epi`:
 *   0 STORE      C[m*ldc+n] = D                          (C dtype = act dtype)
 *   1 BIAS       C = D + bias[n]
 *   2 BIAS_RES   C = D + bias[n] + res[m*ldc+n]
 *   3 BIAS_GELU  aux[m*ldc+n] = D + bias[n] (pre-activation), C = gelu_tanh(pre)
 *   4 GELU_BWD   C = D * gelu_tanh'(aux[m*ldc+n])
 *   5 ACC_F32    Cf32[m*ldc+n] += D                      (fp32 output)
 *   6 STORE_F32  Cf32[m*ldc+n]  = D                      (fp32 output)
 * prec = BB_PREC_BF16 (bf16 operands, tcgen05 tensor cores, fp32 accumulate)
 * or BB_PREC_FP32_CHECK (fp32 SIMT). impl: 0 = default, 1 = force SIMT. */
bb_status bb_op_gemm(int prec, int impl, int M, int N, int K, const void *A, int lda, int a_mn,
                     const void *B, int ldb, int b_mn, int epi, void *C, int ldc,
                     const void *bias, const void *res, void *aux, void *stream);

/* Attention over qkv [B*S, 3H] (columns [q|k|v], head h at h*d): o [B*S, H],
 * lse [B, nh, S] fp32. Backward: dqkv [B*S, 3H] from do, o, lse. */
bb_status bb_op_attention_fwd(int prec, int B, int S, int H, int nh, int causal, const void *qkv,
                              void *o, float *lse, void *stream);
bb_status bb_op_attention_bwd(int prec, int B, int S, int H, int nh, int causal, const void *qkv,
                              const void *o, const float *lse, const void *dout, void *dqkv,
                              void *stream);
/* LayerNorm over rows [R, H]: y, mean, rstd; backward dx = dres + LN'(dy)
 * with dy and dres fp32 [R, H] (dres may be NULL), dx in the act dtype,
 * dg/db accumulated (+=) into fp32 [H]. */
bb_status bb_op_layernorm_fwd(int prec, int R, int H, const void *x, const void *g, const void *b,
                              void *y, float *mean, float *rstd, void *stream);
bb_status bb_op_layernorm_bwd(int prec, int R, int H, const float *dy, const void *x,
                              const float *mean, const float *rstd, const void *g,
                              const float *dres, void *dx, float *dg, float *db, void *stream);
/* Cross-entropy over logits [R, V] (overwritten with dlogits = (softmax -
 * onehot)/n_tok), loss_rows[R] fp32 = (lse - logit[target]) / n_tok. */
bb_status bb_op_cross_entropy(int prec, int R, int V, void *logits, const int32_t *targets,
                              float n_tok, float *loss_rows, void *stream);
/* Adam on n fp32 values (bias-corrected, step t >= 1); also writes the bf16
 * working copy when w16 != NULL. */
bb_status bb_op_adam(size_t n, float *p, const float *g, float *m, float *v, uint16_t *w16, int t,
                     float lr, float b1, float b2, float eps, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BAMBOO_H */
