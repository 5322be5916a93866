// api.cpp — the extern "C" boundary declared in include/bamboo.h.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>
#include <time.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include "bamboo.h"
#include "kernels.h"
#include "plan.h"
#include "runtime.h"
#include "xport.h"

using bb::Ctx;

static bb_status copy_text(const std::string &s, char *buf, size_t cap, size_t *needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && cap > 0) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return (buf && cap < s.size() + 1) ? BB_E_INVAL : BB_OK;
}

// No C++ exception may cross the ABI: anything the runtime did not map to a
// status (a library exception) becomes BB_E_STATE with its message.
template <typename F>
static bb_status guarded(void *ctx, F &&f) {
  try {
    return f();
  } catch (const std::exception &e) {
    static_cast<Ctx *>(ctx)->err = std::string("internal: ") + e.what();
    return BB_E_STATE;
  } catch (...) {
    static_cast<Ctx *>(ctx)->err = "internal: unknown exception";
    return BB_E_STATE;
  }
}

extern "C" {

void bb_default_opts(bb_opts *o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->micro_batch = 1;
  o->rc = BB_RC_EFLB;
  o->prec = BB_PREC_BF16;
  o->lr = 1e-4f;
  o->beta1 = 0.9f;
  o->beta2 = 0.999f;
  o->eps = 1e-8f;
  o->world_rank = 0;
  o->world_size = 1;
  o->device = 0;
}

bb_status bb_session_id(void *out, size_t cap) {
  if (!out || cap < 32) return BB_E_INVAL;
  uint8_t b[32] = {};
  int fd = open("/dev/urandom", O_RDONLY);
  size_t got = 0;
  if (fd >= 0) {
    const ssize_t r = read(fd, b, sizeof(b));
    got = r > 0 ? (size_t)r : 0;
    close(fd);
  }
  if (got < sizeof(b)) {   // no urandom: pid and clock are unique enough per launch
    struct timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    const uint64_t v[3] = {(uint64_t)getpid(), (uint64_t)ts.tv_sec, (uint64_t)ts.tv_nsec};
    std::memcpy(b, v, sizeof(v));
  }
  std::memset(out, 0, cap);
  std::memcpy(out, b, sizeof(b));
  return BB_OK;
}

bb_status bb_init(const bb_model *m, int stages, int microbatches, const bb_opts *o,
                  void **ctx_out) {
  if (!ctx_out) return BB_E_INVAL;
  *ctx_out = nullptr;
  Ctx *c = new (std::nothrow) Ctx();
  if (!c) return BB_E_OOM;
  bb_status st = guarded(c, [&] { return bb::rt_init(*c, m, stages, microbatches, o); });
  *ctx_out = c;   // returned even on failure so bb_last_error works; caller destroys
  return st;
}

bb_status bb_load_params(void *ctx, const float *host, size_t n) {
  if (!ctx || !host) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_load_params(*static_cast<Ctx *>(ctx), host, n); });
}

bb_status bb_step(void *ctx, const int32_t *tokens, const int32_t *targets, bb_step_stats *st) {
  if (!ctx) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_step(*static_cast<Ctx *>(ctx), tokens, targets, st); });
}

bb_status bb_stage_inputs(void *ctx, const int32_t *tokens, const int32_t *targets) {
  if (!ctx) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_stage_inputs(*static_cast<Ctx *>(ctx), tokens, targets); });
}

bb_status bb_preempt(void *ctx, int stage, int at_instr) {
  if (!ctx) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_preempt(*static_cast<Ctx *>(ctx), stage, at_instr); });
}

bb_status bb_recover(void *ctx, bb_recovery_stats *r) {
  if (!ctx) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_recover(*static_cast<Ctx *>(ctx), r); });
}

bb_status bb_rejoin(void *ctx) {
  if (!ctx) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_rejoin(*static_cast<Ctx *>(ctx)); });
}

bb_status bb_read_state(void *ctx, int stage, int replica, int what, float *host, size_t n) {
  if (!ctx || !host) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_read_state(*static_cast<Ctx *>(ctx), stage, replica, what, host, n); });
}

bb_status bb_write_state(void *ctx, int stage, int what, const float *host, size_t n) {
  if (!ctx || !host) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_write_state(*static_cast<Ctx *>(ctx), stage, what, host, n); });
}

bb_status bb_node_stats(void *ctx, bb_node_stat *out, int cap, int *n) {
  if (!ctx) return BB_E_INVAL;
  return guarded(ctx, [&] { return bb::rt_node_stats(*static_cast<Ctx *>(ctx), out, cap, n); });
}

bb_status bb_stage_memory(void *ctx, int stage, size_t *slot_bytes, int *retained) {
  if (!ctx) return BB_E_INVAL;
  Ctx &c = *static_cast<Ctx *>(ctx);
  if (stage < 0 || stage >= (int)c.stages.size()) return BB_E_INVAL;
  if (slot_bytes) *slot_bytes = c.stages[stage].slot_bytes;
  if (retained) {
    *retained = -1;
    for (auto &kv : c.nodes)
      for (auto &cc : kv.second.copies)
        if (cc.first == stage && cc.second.replica) *retained = cc.second.retain;
  }
  return BB_OK;
}

bb_status bb_stage_params(void *ctx, int stage, size_t *offset, size_t *count) {
  if (!ctx) return BB_E_INVAL;
  Ctx &c = *static_cast<Ctx *>(ctx);
  if (stage < 0 || stage >= (int)c.stages.size()) return BB_E_INVAL;
  if (offset) *offset = c.stages[stage].poff;
  if (count) *count = c.stages[stage].pcount;
  return BB_OK;
}

bb_status bb_schedule_dump(void *ctx, char *buf, size_t cap, size_t *needed) {
  if (!ctx) return BB_E_INVAL;
  return copy_text(bb::rt_dump(*static_cast<Ctx *>(ctx)), buf, cap, needed);
}

bb_status bb_recovery_dump(void *ctx, char *buf, size_t cap, size_t *needed) {
  if (!ctx) return BB_E_INVAL;
  return copy_text(static_cast<Ctx *>(ctx)->recovery_text, buf, cap, needed);
}

bb_status bb_kernel_stats(void *ctx, bb_kernel_stat *out, int cap, int *n) {
  if (!ctx) return BB_E_INVAL;
  return bb::rt_kernel_stats(*static_cast<Ctx *>(ctx), out, cap, n);
}

bb_status bb_last_error(const void *ctx, char *buf, size_t cap) {
  if (!ctx) return BB_E_INVAL;
  return copy_text(static_cast<const Ctx *>(ctx)->err, buf, cap, nullptr);
}

void bb_destroy(void *ctx) {
  if (!ctx) return;
  Ctx *c = static_cast<Ctx *>(ctx);
  bb::rt_destroy(*c);
  delete c;
}

// Host-only plan dump (no GPU): victim < 0 -> normal plans; victim >= 0 and
// at_instr >= 0 -> cut + continuation of an injection; at_instr < 0 ->
// the static failover plans after losing `victim`.
bb_status bb_plan_dump(const bb_model *m, int stages, int microbatches, const bb_opts *o,
                       int victim, int at_instr, char *buf, size_t cap, size_t *needed) {
  if (!m) return BB_E_INVAL;
  bb_opts def;
  bb_default_opts(&def);
  const bb_opts &op = o ? *o : def;
  const bool rc = op.rc != BB_RC_NONE;
  try {
    const int P = stages, M = microbatches, D = op.pipelines < 1 ? 1 : op.pipelines;
    auto ranges = bb::partition(m->n_layer, P, op.layers_per_stage);
    const int N = D * P;   // nodes
    std::vector<int> dev(N, 0);
    const int ws = op.world_size < 1 ? 1 : op.world_size;
    const int per = (N + ws - 1) / ws;
    for (int n = 0; n < N; ++n) dev[n] = op.node_rank ? op.node_rank[n] : std::min(n / per, ws - 1);
    bb::Plans plans = bb::normal_plans(P, M, (int)op.rc, D);
    std::string s;
    if (victim < 0) {
      s = bb::dump(P, M, (int)op.rc, ranges, plans, bb::normal_topology(P, rc, D), dev, false, {});
    } else {
      if (!rc || victim >= N) return BB_E_INVAL;
      if (at_instr < 0) {
        s = bb::dump(P, M, (int)op.rc, ranges, bb::failover_plans(P, M, victim, &plans),
                     bb::failover_topology(P, victim, D), dev, true, {victim});
      } else {
        bb::Cut cut = bb::cut(plans, victim, at_instr);
        bb::RecoveryInfo info;
        bb::Plans cont = bb::recovery_plans(plans, P, M, victim, cut.pcs, cut.ch, &info);
        std::string o2 = "# bamboo-recovery v1 P=" + std::to_string(P) + " M=" + std::to_string(M) +
                         " victim=" + std::to_string(victim) + " shadow=" +
                         std::to_string(info.shadow) + " successor=" +
                         std::to_string(info.successor) + " commit=" +
                         std::to_string(info.commit ? 1 : 0) + "\n# cut";
        for (auto &kv : cut.pcs) o2 += " " + std::to_string(kv.first) + ":" + std::to_string(kv.second);
        s = o2 + "\n" + bb::dump_lines(cont);
      }
    }
    return copy_text(s, buf, cap, needed);
  } catch (const bb::PlanError &) {
    return BB_E_INVAL;
  }
}

// Transport microbenchmark: two ranks ping-pong `iters` messages of `bytes`
// over the library's transport (copy into the peer's HBM, the sender's
// interprocess event, sequence number in host shared memory). A reply is
// ordered after the arrival of the message it answers (its copy's stream
// waits on that message's event), so the chain of 2 * iters copies is
// serial on the devices and the host time to its end is the one-way latency
// including the data movement; *us = that time / (2 * iters), on rank 0.
// Compare with NCCL send/recv of the same bytes (tools/xport_vs_nccl.py).
bb_status bb_xport_pingpong(int rank, int world, int device, const void *session_id,
                            size_t bytes, int iters, float *us) {
  if (world != 2 || rank < 0 || rank > 1 || !session_id || bytes == 0 || iters < 1)
    return BB_E_INVAL;
  if (cudaSetDevice(device) != cudaSuccess) return BB_E_CUDA;
  bb::Xport x;
  const std::vector<std::tuple<int, int, int>> want{{0, 1, 0}, {1, 0, 0}};
  const std::vector<int> node_rank{0, 1};
  const std::string e = bb::xport_init(x, rank, 2, 2, want, node_rank, {bytes}, {2},
                                       session_id, 0);
  if (!e.empty()) return BB_E_CUDA;
  void *src = nullptr;
  if (cudaMalloc(&src, bytes) != cudaSuccess) return BB_E_OOM;
  bb::XEdge &out = x.edges.at(std::make_tuple(rank, 1 - rank, 0));
  bb::XEdge &in = x.edges.at(std::make_tuple(1 - rank, rank, 0));
  auto send = [&] {
    char *dst = out.peer_base + out.recv_off + (out.sent % out.cap) * out.slot_bytes;
    cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, out.stream);
    x.post(out);
  };
  auto recv = [&] {
    while (!x.available(in)) {
    }
    const int slot = (int)(in.consumed % (uint64_t)in.cap);
    x.consume(in);
    // the next send (and the final synchronise) waits for this payload
    if (cudaEvent_t ev = x.wait_event(in, slot)) cudaStreamWaitEvent(out.stream, ev, 0);
  };
  x.barrier();
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) {
    if (rank == 0) {
      send();
      recv();
    } else {
      recv();
      send();
    }
  }
  cudaStreamSynchronize(out.stream);
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  x.barrier();
  if (us) *us = (float)(1e3 * ms / (2.0 * iters));
  cudaFree(src);
  bb::xport_destroy(x);
  return BB_OK;
}

// ------------------------------------------------------------ single ops
bb_status bb_op_gemm(int prec, int impl, int M, int N, int K, const void *A, int lda, int a_mn,
                     const void *B, int ldb, int b_mn, int epi, void *C, int ldc,
                     const void *bias, const void *res, void *aux, void *stream) {
  if (epi < 0 || epi > 6 || M < 0 || N < 0 || K < 0) return BB_E_INVAL;
  bb::k::Gemm g{M, N, K, A, lda, a_mn != 0, B, ldb, b_mn != 0, epi, C, ldc, bias, res, aux};
  const bool b16 = prec == BB_PREC_BF16;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (b16 && impl == 0) {
    if (!bb::k::gemm_tc_supported(g)) return BB_E_UNSUPPORTED;   // no silent SIMT fallback
    e = bb::k::gemm_tc(g, s);
  } else {
    e = bb::k::gemm_simt(b16, g, s);   // fp32 check mode, or impl = 1 (explicit request)
  }
  return e == cudaSuccess ? BB_OK : BB_E_CUDA;
}

bb_status bb_op_attention_fwd(int prec, int B, int S, int H, int nh, int causal, const void *qkv,
                              void *o, float *lse, void *stream) {
  cudaError_t e = bb::k::attention_fwd(prec == BB_PREC_BF16, B, S, H, nh, causal != 0, qkv, o,
                                       lse, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported) return BB_E_UNSUPPORTED;
  return e == cudaSuccess ? BB_OK : BB_E_CUDA;
}

// Op-level scratch (single-op entry points only: tests and kernel timing):
// one growing device buffer per kind, kept for the process, so a timed call
// measures the kernels, not an allocation. Not thread-safe (like the ops).
static float *op_scratch(int kind, size_t bytes, bool zero, cudaStream_t s) {
  static float *buf[2] = {nullptr, nullptr};
  static size_t cap[2] = {0, 0};
  if (bytes > cap[kind]) {
    cudaStreamSynchronize(s);
    if (buf[kind]) cudaFree(buf[kind]);
    buf[kind] = nullptr;
    cap[kind] = 0;
    if (cudaMalloc((void **)&buf[kind], bytes) != cudaSuccess) return nullptr;
    cap[kind] = bytes;
    zero = true;
  }
  if (zero && cudaMemsetAsync(buf[kind], 0, cap[kind], s) != cudaSuccess) return nullptr;
  return buf[kind];
}

bb_status bb_op_attention_bwd(int prec, int B, int S, int H, int nh, int causal, const void *qkv,
                              const void *o, const float *lse, const void *dout, void *dqkv,
                              void *stream) {
  float *scratch = op_scratch(0, bb::k::attention_bwd_scratch_floats(B, S, H, nh) * 4, false,
                              static_cast<cudaStream_t>(stream));
  if (!scratch) return BB_E_OOM;
  cudaError_t e = bb::k::attention_bwd(prec == BB_PREC_BF16, B, S, H, nh, causal != 0, qkv, o, lse,
                                       dout, dqkv, scratch, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported) return BB_E_UNSUPPORTED;
  return e == cudaSuccess ? BB_OK : BB_E_CUDA;
}

bb_status bb_op_layernorm_fwd(int prec, int R, int H, const void *x, const void *g, const void *b,
                              void *y, float *mean, float *rstd, void *stream) {
  cudaError_t e = bb::k::layernorm_fwd(prec == BB_PREC_BF16, R, H, x, g, b, y, mean, rstd,
                                       static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? BB_OK : BB_E_CUDA;
}

bb_status bb_op_layernorm_bwd(int prec, int R, int H, const float *dy, const void *x,
                              const float *mean, const float *rstd, const void *g,
                              const float *dres, void *dx, float *dg, float *db, void *stream) {
  const bool b16 = prec == BB_PREC_BF16;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // colreduce tickets must start at zero; they reset themselves after a call
  float *part = op_scratch(1, bb::k::colreduce_partial_floats(R, H) * 4, false, s);
  if (!part) return BB_E_OOM;
  cudaError_t e =
      bb::k::layernorm_bwd_dx(b16, R, H, dy, x, mean, rstd, g, dres, nullptr, dx, nullptr, s);
  if (e == cudaSuccess) e = bb::k::colreduce_ln(b16, R, H, dy, x, mean, rstd, part, dg, db, s);
  return e == cudaSuccess ? BB_OK : BB_E_CUDA;
}

bb_status bb_op_cross_entropy(int prec, int R, int V, void *logits, const int32_t *targets,
                              float n_tok, float *loss_rows, void *stream) {
  cudaError_t e = bb::k::cross_entropy(prec == BB_PREC_BF16, R, V, logits, targets, 1.0f / n_tok,
                                       loss_rows, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? BB_OK : BB_E_CUDA;
}

bb_status bb_op_adam(size_t n, float *p, const float *g, float *m, float *v, uint16_t *w16, int t,
                     float lr, float b1, float b2, float eps, void *stream) {
  if (t < 1) return BB_E_INVAL;
  const float bc1 = (float)(1.0 - std::pow((double)b1, t));
  const float bc2 = (float)(1.0 - std::pow((double)b2, t));
  cudaError_t e = bb::k::adam(n, p, g, m, v, w16, lr, b1, b2, eps, bc1, bc2,
                              static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? BB_OK : BB_E_CUDA;
}

}  // extern "C"
