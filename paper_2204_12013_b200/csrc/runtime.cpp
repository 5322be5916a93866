// runtime.cpp — see runtime.h. Interprets the per-node instruction lists of
// plan.h by enqueuing kernels and NCCL P2P on CUDA streams; no host blocking
// on the GPU except at the end of a step.
#include "runtime.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>
#include <cstdio>
#include <ctime>
#include <cstdlib>
#include <sstream>
#include <thread>
#include <unistd.h>

namespace bb {

namespace {
struct RtError {
  bb_status st;
  std::string msg;
};
#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw RtError{e_ == cudaErrorMemoryAllocation ? BB_E_OOM : BB_E_CUDA,                \
                    std::string(#x) + ": " + cudaGetErrorString(e_)};                      \
  } while (0)

constexpr size_t ALIGN = 256;
size_t al(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

void *dmalloc(size_t bytes) {
  void *p = nullptr;
  if (bytes == 0) bytes = ALIGN;
  const cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();   // an allocation failure is not sticky: clear it
    throw RtError{e == cudaErrorMemoryAllocation ? BB_E_OOM : BB_E_CUDA,
                  std::string("cudaMalloc: ") + cudaGetErrorString(e)};
  }
  return p;
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
}  // namespace

// ------------------------------------------------------------ param layout
size_t unit_param_count(const Dims &d, int unit) {
  const size_t H = d.H, F = d.F, V = d.V, S = d.S;
  if (unit == 0) return V * H + S * H;
  if (unit == d.L + 1) return 2 * H + V * H;
  return 2 * H + 3 * H * H + 3 * H + H * H + H + 2 * H + F * H + F + H * F + H;
}

std::vector<std::pair<size_t, size_t>> unit_param_ranges(const Dims &d) {
  std::vector<std::pair<size_t, size_t>> r;
  size_t off = 0;
  for (int u = 0; u < d.L + 2; ++u) {
    const size_t n = unit_param_count(d, u);
    r.push_back({off, n});
    off += n;
  }
  return r;
}

static StageInfo make_stage(const Dims &d, int X, int ua, int ub) {
  StageInfo si;
  si.X = X;
  si.ua = ua;
  si.ub = ub;
  auto ur = unit_param_ranges(d);
  si.poff = ur[ua].first;
  si.pcount = ur[ub].first + ur[ub].second - si.poff;
  const size_t H = d.H, F = d.F, V = d.V, S = d.S;
  const size_t R = d.R(), T = 0;  // placeholder
  (void)T;
  size_t slot = 0;
  for (int u = ua; u <= ub; ++u) {
    UnitP p{};
    p.unit = u;
    size_t o = ur[u].first - si.poff;
    UnitS s{};
    if (u == 0) {
      p.kind = 0;
      p.tok = o;
      p.pos = o + V * H;
    } else if (u == d.L + 1) {
      p.kind = 2;
      p.lnfg = o;
      p.lnfb = o + H;
      p.whead = o + 2 * H;
    } else {
      p.kind = 1;
      p.ln1g = o; o += H;
      p.ln1b = o; o += H;
      p.wqkv = o; o += 3 * H * H;
      p.bqkv = o; o += 3 * H;
      p.wo = o; o += H * H;
      p.bo = o; o += H;
      p.ln2g = o; o += H;
      p.ln2b = o; o += H;
      p.w1 = o; o += F * H;
      p.b1 = o; o += F;
      p.w2 = o; o += H * F;
      p.b2 = o; o += H;
    }
    si.up.push_back(p);
    si.us.push_back(s);
  }
  (void)S;
  (void)R;
  si.slot_bytes = 0;
  return si;
}

// Saved-set layout (needs the storage type size).
static void layout_slots(const Dims &d, size_t tsz, StageInfo &si) {
  const size_t H = d.H, F = d.F, V = d.V, R = d.R();
  const size_t B = d.mb, nh = d.nh, S = d.S;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t r = o;
    o += al(bytes);
    return r;
  };
  for (size_t i = 0; i < si.up.size(); ++i) {
    const UnitP &p = si.up[i];
    UnitS &s = si.us[i];
    const bool last = (int)i == (int)si.up.size() - 1;
    if (p.kind == 1) {
      s.h1 = take(R * H * tsz);
      s.mean1 = take(R * 4);
      s.rstd1 = take(R * 4);
      s.qkv = take(R * 3 * H * tsz);
      s.o = take(R * H * tsz);
      s.lse = take(B * nh * S * 4);
      s.x1 = take(R * H * tsz);
      s.h2 = take(R * H * tsz);
      s.mean2 = take(R * 4);
      s.rstd2 = take(R * 4);
      s.pre = take(R * F * tsz);
      s.act = take(R * F * tsz);
    } else if (p.kind == 2) {
      s.hf = take(R * H * tsz);
      s.meanf = take(R * 4);
      s.rstdf = take(R * 4);
      s.dlog = take(R * V * tsz);
    }
    if (!last && p.kind != 2) s.out = take(R * H * tsz);
  }
  si.slot_bytes = al(o);
}

// ================================================================ helpers
namespace {
double watch_s();
constexpr int kScratchSlot = -2;   // FRC beyond the retention budget
// Entry::slot of a saved set: >= 0 a device slot, -1 gone (a BRC recomputes
// it), <= kHostSlot0 swapped to host slot kHostSlot0 - slot
constexpr int kHostSlot0 = -3;
char *slot_base(const Copy &cp, int slot) {
  return slot == kScratchSlot ? cp.scratch : cp.sp.at(slot);
}

// Append n saved-set slots (one allocation) to a copy's pool.
void grow_slots(Copy &cp, int n, size_t slot_bytes) {
  if (n <= 0) return;
  char *p = (char *)dmalloc(slot_bytes * n);
  cp.chunks.push_back({p, slot_bytes * n});
  for (int i = 0; i < n; ++i) {
    cp.free_slots.insert(cp.free_slots.begin(), cp.nslots());
    cp.sp.push_back(p + (size_t)i * slot_bytes);
  }
}

void free_slots_all(Copy &cp);
// A copy's pool as bb_init sizes it: the 1F1B stash of its own stage, or the
// retention slots (+ scratch) of a replica.
void reset_pool(Ctx &c, Copy &cp, bool scratch) {
  const size_t sb = c.stages[cp.X].slot_bytes;
  grow_slots(cp, cp.replica ? cp.retain : std::min(c.d.M, c.d.P - cp.X), sb);
  if (scratch) {
    cp.scratch = (char *)dmalloc(sb);
    cp.chunks.push_back({cp.scratch, sb});
  }
}

void free_slots_all(Copy &cp) {
  for (auto &ch : cp.chunks) cudaFree(ch.first);
  cp.chunks.clear();
  cp.sp.clear();
  cp.free_slots.clear();
  cp.scratch = nullptr;
}

cudaEvent_t new_event(Node &nd) {
  if (nd.evnext == nd.evpool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    nd.evpool.push_back(e);
  }
  return nd.evpool[nd.evnext++];
}

cudaEvent_t record(Node &nd, cudaStream_t s) {
  cudaEvent_t e = new_event(nd);
  CK(cudaEventRecord(e, s));
  return e;
}

void wait_ev(cudaStream_t s, cudaEvent_t e) {
  if (e) CK(cudaStreamWaitEvent(s, e, 0));
}

// Per-step bump arena. A step that needs more (a failover shadow runs two
// stages; an interrupted step runs its prefix plus the continuation) spills
// into extra chunks; the next begin_step regrows the arena to the peak, so
// only the first step of a new plan pays a cudaMalloc.
void *arena_alloc(Node &nd, size_t bytes) {
  const size_t b = al(bytes);
  nd.arena_peak += b;
  if (nd.arena_used + b <= nd.arena_bytes) {
    void *p = nd.arena + nd.arena_used;
    nd.arena_used += b;
    return p;
  }
  void *p = dmalloc(b);
  nd.arena_spill.push_back({static_cast<char *>(p), b});
  return p;
}

// opts.timing: a timing-enabled event pair around one instruction's work.
cudaEvent_t tevent(Node &nd) {
  if (nd.tnext == nd.tpool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    nd.tpool.push_back(e);
  }
  return nd.tpool[nd.tnext++];
}
struct TMark {
  Ctx &c;
  Node &nd;
  cudaStream_t s;
  int kind;
  cudaEvent_t a = nullptr;
  TMark(Ctx &c_, Node &nd_, cudaStream_t s_, int kind_) : c(c_), nd(nd_), s(s_), kind(kind_) {
    if (!c.o.timing) return;
    a = tevent(nd);
    CK(cudaEventRecord(a, s));
  }
  ~TMark() noexcept(false) {
    if (!a) return;
    cudaEvent_t b = tevent(nd);
    CK(cudaEventRecord(b, s));
    nd.trec.push_back({kind, a, b});
  }
};

const Entry &need(Node &nd, const Key &k) {
  auto it = nd.store.find(k);
  if (it == nd.store.end()) {
    std::ostringstream o;
    o << "node " << nd.n << ": missing data key (" << (int)k.t << "," << k.a << "," << k.b << ")";
    throw RtError{BB_E_STATE, o.str()};
  }
  return it->second;
}

struct Prof {
  Ctx &c;
  Node &nd;
  cudaStream_t s;
  int cls;
  double work;
  cudaEvent_t a = nullptr;
  Prof(Ctx &c_, Node &nd_, cudaStream_t s_, int cls_, double w) : c(c_), nd(nd_), s(s_), cls(cls_), work(w) {
    if (c.o.profile || watch_s() > 0) a = take();
    if (a) CK(cudaEventRecord(a, s));
  }
  cudaEvent_t take() {
    if (c.prof_next == c.prof_pool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c.prof_pool.push_back(e);
    }
    return c.prof_pool[c.prof_next++];
  }
  ~Prof() noexcept(false) {
    if (!a) return;
    cudaEvent_t b = take();
    CK(cudaEventRecord(b, s));
    c.prof.push_back({cls, a, b, work, nd.n});
  }
};

enum ProfCls { PC_GEMM_FWD = 0, PC_GEMM_DX, PC_GEMM_DW, PC_ATTN_FWD, PC_ATTN_BWD, PC_LN, PC_CE,
               PC_EMB, PC_ADAM, PC_REDUCE, PC_N };
const char *prof_names[PC_N] = {"gemm_fwd", "gemm_dx", "gemm_dw", "attn_fwd", "attn_bwd",
                                "layernorm", "cross_entropy", "embedding", "adam", "colreduce"};

void gemm(Ctx &c, Node &nd, cudaStream_t s, int cls, k::Gemm g, bool tile_grid = false) {
  Prof pf(c, nd, s, cls, 2.0 * g.M * (double)g.N * g.K);
  g.tile_grid = tile_grid;
  // bf16: tcgen05 only (no silent SIMT fallback; rt_init rejects shapes the
  // tensor-core path cannot take); fp32 check mode: SIMT FMA by definition.
  if (c.bf16 && !k::gemm_tc_supported(g))
    throw RtError{BB_E_UNSUPPORTED, "GEMM shape/alignment not supported by the tcgen05 path"};
  CK(c.bf16 ? k::gemm_tc(g, s) : k::gemm_simt(false, g, s));
}
}  // namespace

// ============================================================== unit math
namespace {
const void *pw(const Ctx &c, const Copy &cp, size_t off) {
  return static_cast<const char *>(cp.work) + off * c.act_bytes;
}
float *pg(const Copy &cp, size_t off) { return cp.grad + off; }

// Forward of stage X for micro-batch k on stream s. Returns the output
// pointer (activation in the arena) or nullptr for the last stage.
void stage_forward(Ctx &c, Node &nd, Copy &cp, int X, int k, int slot, cudaStream_t s,
                   const void *x_in, void *x_out, float *loss_rows, bool tg = false) {
  const Dims &d = c.d;
  const StageInfo &si = c.stages[X];
  char *sl = slot_base(cp, slot);
  const int R = d.R(), H = d.H, F = d.F;
  const bool b16 = c.bf16;
  const void *x = x_in;
  for (size_t i = 0; i < si.up.size(); ++i) {
    const UnitP &p = si.up[i];
    const UnitS &u = si.us[i];
    const bool last = i + 1 == si.up.size();
    void *out = last ? x_out : (p.kind == 2 ? nullptr : sl + u.out);
    if (p.kind == 0) {
      Prof pf(c, nd, s, PC_EMB, 0);
      CK(k::embed_fwd(b16, R, d.S, H, nd.d_tok + (size_t)k * R, pw(c, cp, p.tok),
                      pw(c, cp, p.pos), out, s));
    } else if (p.kind == 1) {
      {
        Prof pf(c, nd, s, PC_LN, 0);
        CK(k::layernorm_fwd(b16, R, H, x, pw(c, cp, p.ln1g), pw(c, cp, p.ln1b), sl + u.h1,
                            (float *)(sl + u.mean1), (float *)(sl + u.rstd1), s));
      }
      gemm(c, nd, s, PC_GEMM_FWD,
           {R, 3 * H, H, sl + u.h1, H, false, pw(c, cp, p.wqkv), H, false, k::EPI_BIAS,
            sl + u.qkv, 3 * H, pw(c, cp, p.bqkv), nullptr, nullptr}, tg);
      {
        Prof pf(c, nd, s, PC_ATTN_FWD, 0);
        CK(k::attention_fwd(b16, d.mb, d.S, H, d.nh, d.causal, sl + u.qkv, sl + u.o,
                            (float *)(sl + u.lse), s));
      }
      gemm(c, nd, s, PC_GEMM_FWD,
           {R, H, H, sl + u.o, H, false, pw(c, cp, p.wo), H, false, k::EPI_BIAS_RES, sl + u.x1, H,
            pw(c, cp, p.bo), x, nullptr}, tg);
      {
        Prof pf(c, nd, s, PC_LN, 0);
        CK(k::layernorm_fwd(b16, R, H, sl + u.x1, pw(c, cp, p.ln2g), pw(c, cp, p.ln2b),
                            sl + u.h2, (float *)(sl + u.mean2), (float *)(sl + u.rstd2), s));
      }
      gemm(c, nd, s, PC_GEMM_FWD,
           {R, F, H, sl + u.h2, H, false, pw(c, cp, p.w1), H, false, k::EPI_BIAS_GELU, sl + u.act,
            F, pw(c, cp, p.b1), nullptr, sl + u.pre}, tg);
      gemm(c, nd, s, PC_GEMM_FWD,
           {R, H, F, sl + u.act, F, false, pw(c, cp, p.w2), F, false, k::EPI_BIAS_RES, out, H,
            pw(c, cp, p.b2), sl + u.x1, nullptr}, tg);
    } else {
      {
        Prof pf(c, nd, s, PC_LN, 0);
        CK(k::layernorm_fwd(b16, R, H, x, pw(c, cp, p.lnfg), pw(c, cp, p.lnfb), sl + u.hf,
                            (float *)(sl + u.meanf), (float *)(sl + u.rstdf), s));
      }
      gemm(c, nd, s, PC_GEMM_FWD,
           {R, d.V, H, sl + u.hf, H, false, pw(c, cp, p.whead), H, false, k::EPI_STORE,
            sl + u.dlog, d.V, nullptr, nullptr, nullptr}, tg);
      {
        Prof pf(c, nd, s, PC_CE, 0);
        const float inv = 1.0f / (float)((double)d.D * d.M * d.mb * d.S);   // whole-batch mean
        CK(k::cross_entropy(b16, R, d.V, sl + u.dlog, nd.d_tgt + (size_t)k * R, inv, loss_rows,
                            s));
        CK(k::sum_fixed(R, loss_rows, cp.loss + k, s));
      }
    }
    x = out;
  }
}

// Backward of stage X for micro-batch k (main stream). dout = gradient w.r.t.
// the stage output (nullptr for the last stage); x_in = stage input act.
// Writes the gradient w.r.t. the stage input into dx_out (if X > 0).
// Inside the stage the residual-gradient chain is carried in fp32 (s32) next
// to its storage-type copy (a GEMM operand); GEMM outputs that only feed a
// LayerNorm backward are written in fp32.
void stage_backward(Ctx &c, Node &nd, Copy &cp, int X, int k, int slot, cudaStream_t s,
                    const void *x_in, const void *dout, void *dx_out, Node::Scratch &sc) {
  const Dims &d = c.d;
  const StageInfo &si = c.stages[X];
  char *sl = slot_base(cp, slot);
  const int R = d.R(), H = d.H, F = d.F;
  const bool b16 = c.bf16;
  const void *dy = dout;      // storage type
  const float *dy32 = nullptr;
  int flip = 0;
  for (int i = (int)si.up.size() - 1; i >= 0; --i) {
    const UnitP &p = si.up[i];
    const UnitS &u = si.us[i];
    const void *x = i == 0 ? x_in : (const void *)(sl + si.us[i - 1].out);
    void *dx = i == 0 ? dx_out : sc.sH[3 + flip];
    float *dx32 = i == 0 ? nullptr : sc.s32[2 + flip];
    flip ^= 1;
    if (p.kind == 0) {
      Prof pf(c, nd, s, PC_EMB, 0);
      const int32_t *csr = nd.d_csr + (size_t)k * c.csr_stride;
      CK(k::embed_bwd(b16, dy32 != nullptr, R, d.S, H, csr, dy32 ? (const void *)dy32 : dy,
                      pg(cp, p.tok), pg(cp, p.pos), s));
    } else if (p.kind == 2) {
      float *dhf = sc.s32[0];
      gemm(c, nd, s, PC_GEMM_DX,
           {R, H, d.V, sl + u.dlog, d.V, false, pw(c, cp, p.whead), H, true, k::EPI_STORE_F32,
            dhf, H, nullptr, nullptr, nullptr});
      gemm(c, nd, s, PC_GEMM_DW,
           {d.V, H, R, sl + u.dlog, d.V, true, sl + u.hf, H, true, k::EPI_ACC_F32,
            pg(cp, p.whead), H, nullptr, nullptr, nullptr});
      Prof pf(c, nd, s, PC_LN, 0);
      CK(k::layernorm_bwd_dx(b16, R, H, dhf, x, (float *)(sl + u.meanf), (float *)(sl + u.rstdf),
                             pw(c, cp, p.lnfg), nullptr, nullptr, dx, dx32, s));
      CK(k::colreduce_ln(b16, R, H, dhf, x, (float *)(sl + u.meanf), (float *)(sl + u.rstdf),
                         sc.s_part, pg(cp, p.lnfg), pg(cp, p.lnfb), s));
    } else {
      void *dpre = sc.sF, *dx1 = sc.sH[1], *dO = sc.sH[2], *dqkv = sc.s3;
      float *dh2 = sc.s32[0], *dx1_32 = sc.s32[1], *dh1 = sc.s32[0];
      gemm(c, nd, s, PC_GEMM_DX,
           {R, F, H, dy, H, false, pw(c, cp, p.w2), F, true, k::EPI_GELU_BWD, dpre, F, nullptr,
            nullptr, sl + u.pre});
      gemm(c, nd, s, PC_GEMM_DW,
           {H, F, R, dy, H, true, sl + u.act, F, true, k::EPI_ACC_F32, pg(cp, p.w2), F, nullptr,
            nullptr, nullptr});
      {
        Prof pf(c, nd, s, PC_REDUCE, 0);
        CK(k::colreduce(b16, dy32 != nullptr, 0, R, H, dy32 ? (const void *)dy32 : dy, nullptr,
                        nullptr, nullptr, sc.s_part, pg(cp, p.b2), s));
      }
      gemm(c, nd, s, PC_GEMM_DX,
           {R, H, F, dpre, F, false, pw(c, cp, p.w1), H, true, k::EPI_STORE_F32, dh2, H, nullptr,
            nullptr, nullptr});
      gemm(c, nd, s, PC_GEMM_DW,
           {F, H, R, dpre, F, true, sl + u.h2, H, true, k::EPI_ACC_F32, pg(cp, p.w1), H, nullptr,
            nullptr, nullptr});
      {
        Prof pf(c, nd, s, PC_REDUCE, 0);
        CK(k::colreduce(b16, false, 0, R, F, dpre, nullptr, nullptr, nullptr, sc.s_part,
                        pg(cp, p.b1), s));
      }
      {
        Prof pf(c, nd, s, PC_LN, 0);
        CK(k::layernorm_bwd_dx(b16, R, H, dh2, sl + u.x1, (float *)(sl + u.mean2),
                               (float *)(sl + u.rstd2), pw(c, cp, p.ln2g), dy32,
                               dy32 ? nullptr : dy, dx1, dx1_32, s));
        CK(k::colreduce_ln(b16, R, H, dh2, sl + u.x1, (float *)(sl + u.mean2),
                           (float *)(sl + u.rstd2), sc.s_part, pg(cp, p.ln2g), pg(cp, p.ln2b), s));
      }
      gemm(c, nd, s, PC_GEMM_DX,
           {R, H, H, dx1, H, false, pw(c, cp, p.wo), H, true, k::EPI_STORE, dO, H, nullptr,
            nullptr, nullptr});
      gemm(c, nd, s, PC_GEMM_DW,
           {H, H, R, dx1, H, true, sl + u.o, H, true, k::EPI_ACC_F32, pg(cp, p.wo), H, nullptr,
            nullptr, nullptr});
      {
        Prof pf(c, nd, s, PC_REDUCE, 0);
        CK(k::colreduce(b16, true, 0, R, H, dx1_32, nullptr, nullptr, nullptr, sc.s_part,
                        pg(cp, p.bo), s));
      }
      {
        Prof pf(c, nd, s, PC_ATTN_BWD, 0);
        CK(k::attention_bwd(b16, d.mb, d.S, H, d.nh, d.causal, sl + u.qkv, sl + u.o,
                            (float *)(sl + u.lse), dO, dqkv, sc.s_attn, s));
      }
      gemm(c, nd, s, PC_GEMM_DX,
           {R, H, 3 * H, dqkv, 3 * H, false, pw(c, cp, p.wqkv), H, true, k::EPI_STORE_F32, dh1, H,
            nullptr, nullptr, nullptr});
      gemm(c, nd, s, PC_GEMM_DW,
           {3 * H, H, R, dqkv, 3 * H, true, sl + u.h1, H, true, k::EPI_ACC_F32, pg(cp, p.wqkv), H,
            nullptr, nullptr, nullptr});
      {
        Prof pf(c, nd, s, PC_REDUCE, 0);
        CK(k::colreduce(b16, false, 0, R, 3 * H, dqkv, nullptr, nullptr, nullptr, sc.s_part,
                        pg(cp, p.bqkv), s));
      }
      {
        Prof pf(c, nd, s, PC_LN, 0);
        CK(k::layernorm_bwd_dx(b16, R, H, dh1, x, (float *)(sl + u.mean1),
                               (float *)(sl + u.rstd1), pw(c, cp, p.ln1g), dx1_32, nullptr, dx,
                               dx32, s));
        CK(k::colreduce_ln(b16, R, H, dh1, x, (float *)(sl + u.mean1),
                           (float *)(sl + u.rstd1), sc.s_part, pg(cp, p.ln1g), pg(cp, p.ln1b), s));
      }
    }
    dy = dx;
    dy32 = dx32;
  }
}
}  // namespace


// ============================================================ interpreter
namespace {
bool is_local(const Ctx &c, int n) { return c.node_rank[n] == c.o.world_rank; }

XEdge &xedge(Ctx &c, int src, int dst, int kind) {
  auto it = c.x.edges.find(std::make_tuple(src, dst, kind));
  if (it == c.x.edges.end())
    throw RtError{BB_E_STATE, "no transport edge " + std::to_string(src) + " -> " +
                                  std::to_string(dst) + " kind " + std::to_string(kind)};
  return it->second;
}

size_t msg_count(const Ctx &c, MsgKind kind, int stage) {
  if (kind == MSG_GRADSUM || kind == MSG_AR) return c.stages[stage].pcount;
  return (size_t)c.d.R() * c.d.H;
}
size_t msg_bytes(const Ctx &c, MsgKind kind, int stage) {
  const bool f32 = kind == MSG_GRADSUM || kind == MSG_AR;
  return msg_count(c, kind, stage) * (f32 ? sizeof(float) : c.act_bytes);
}

Key payload_key(const Instr &ins) {
  switch (ins.kind) {
    case SEND_ACT: return {K_ACT, ins.stage + 1, ins.mb};
    case SEND_GRAD:
    case SEND_DGRAD:
    case RESEND_GRAD: return {K_DACT, ins.stage, ins.mb};
    default: return {K_GRADSUM, ins.stage, 0};
  }
}

struct Phase {
  bool drop_to_victim = false;   // prefix of an interrupted step
  int victim = -1;
};

bool debug_on() {
  static const bool on = [] {
    const char *e = std::getenv("BB_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}
// BB_WATCH=<seconds>: record an event pair per instruction and, when a step's
// device work has not finished after that long, report the first unfinished
// instruction of every node and fail the call (diagnosing device hangs).
double watch_s() {
  static const double w = [] {
    const char *e = std::getenv("BB_WATCH");
    return e ? std::atof(e) : 0.0;
  }();
  return w;
}

// Input of stage X for micro-batch k on node nd: tokens (X = 0) or the
// activation key; makes stream s wait for it (and for the targets on the last
// stage). Returns the activation pointer (nullptr for X = 0).
const void *stage_input(Ctx &c, Node &nd, cudaStream_t s, int X, int k) {
  const void *x_in = nullptr;
  if (X == 0) {
    wait_ev(s, need(nd, {K_TOK, k, 0}).ev);
  } else {
    const Entry &e = need(nd, {K_ACT, X, k});
    wait_ev(s, e.ev);
    x_in = e.p;
  }
  if (X == c.d.P - 1) wait_ev(s, need(nd, {K_TGT, k, 0}).ev);
  return x_in;
}

// Execute one instruction of node nd; false = blocked on a local message.
bool exec(Ctx &c, Node &nd, const Instr &ins, const Phase &ph) {
  if (debug_on())
    std::fprintf(stderr, "[bb rank %d node %d] %s mb=%d peer=%d stage=%d\n", c.o.world_rank, nd.n,
                 kind_name(ins.kind), ins.mb, ins.peer, ins.stage);
  const Dims &d = c.d;
  const int P = d.P, M = d.M, k = ins.mb, X = ins.stage;
  switch (ins.kind) {
    case LOAD_INPUTS: {
      const size_t n = (size_t)M * d.R();
      const size_t off = (size_t)(nd.n / P) * n;   // pipeline d's micro-batches d*M ..
      if (!c.resident_step) {   // the last node fetches its inputs itself
        CK(cudaMemcpyAsync(nd.d_tok, c.h_tok + off, n * 4, cudaMemcpyHostToDevice, nd.main));
        CK(cudaMemcpyAsync(nd.d_tgt, c.h_tgt + off, n * 4, cudaMemcpyHostToDevice, nd.main));
        if (nd.needs_csr) CK(k::embed_csr(M, d.R(), nd.d_tok, nd.d_csr, nd.main));
        c.h2d += 2 * n * 4;
      }
      cudaEvent_t e = record(nd, nd.main);
      for (int j = 0; j < M; ++j) {
        nd.store[{K_TOK, j, 0}] = {nd.d_tok + (size_t)j * d.R(), e};
        nd.store[{K_TGT, j, 0}] = {nd.d_tgt + (size_t)j * d.R(), e};
      }
      return true;
    }
    case FWD:
    case FRC_FWD: {
      Copy &cp = nd.copies.at(X);
      const bool frc = ins.kind == FRC_FWD;
      cudaStream_t s = frc ? nd.frc : nd.main;
      const void *x_in = stage_input(c, nd, s, X, k);
      // FRC retention budget (Q10): an FRC keeps its saved set for a
      // lazy BRC while the replica's pool (cp.retain slots) has a free slot;
      // beyond that it runs in the scratch slot and keeps only its input and
      // output (the BRC recomputes the forward).
      bool keep = true, swap = false;
      int slot;
      if (frc && cp.free_slots.empty() && cp.scratch) {
        keep = false;
        slot = kScratchSlot;
        // host-swap tier: the saved set goes to pinned host memory instead
        swap = cp.hnext < (int)cp.hslots.size();
        if (cp.scratch_ev) wait_ev(s, cp.scratch_ev);   // the last swap-out read it
      } else {
        if (cp.free_slots.empty()) throw RtError{BB_E_STATE, "saved-set pool exhausted"};
        slot = cp.free_slots.back();
        cp.free_slots.pop_back();
      }
      void *out = X < P - 1 ? arena_alloc(nd, msg_bytes(c, MSG_ACT, X)) : nullptr;
      {
        TMark tm(c, nd, s, frc ? 1 : 0);
        stage_forward(c, nd, cp, X, k, slot, s, x_in, out,
                      s == nd.main ? nd.s_loss_main : nd.s_loss_frc,
                      frc && !c.o.frc_persistent && !c.o.profile);
      }
      if (c.recovering && !frc && X == c.rec_stage) ++c.frc_recomputed;
      cudaEvent_t e = record(nd, s);
      nd.store[{K_SAVED, X, k}] = {nullptr, e, keep ? slot : -1};
      if (swap) {
        const int h = cp.hnext++;
        wait_ev(nd.swap, e);
        CK(cudaMemcpyAsync(cp.hslots[h], cp.scratch, c.stages[X].slot_bytes,
                           cudaMemcpyDeviceToHost, nd.swap));
        cp.scratch_ev = record(nd, nd.swap);
        nd.store[{K_SAVED, X, k}] = {cp.hslots[h], cp.scratch_ev, kHostSlot0 - h};
      }
      if (X < P - 1)
        nd.store[{K_ACT, X + 1, k}] = {out, e};
      else
        nd.store[{K_LOSS, k, 0}] = {cp.loss + k, e};
      return true;
    }
    case BWD:
    case BRC_BWD: {
      // BRC_BWD (EFEB): the replica stage's backward, eagerly, on the FRC
      // stream with its own scratch; it accumulates the replica's gradient and
      // its input-gradient stands in for the victim's only if none arrived
      Copy &cp = nd.copies.at(X);
      const bool brc = ins.kind == BRC_BWD;
      cudaStream_t s = brc ? nd.frc : nd.main;
      const Entry sv = need(nd, {K_SAVED, X, k});
      wait_ev(s, sv.ev);
      const void *dout = nullptr;
      if (X < P - 1) {
        const Entry &e = need(nd, {K_DACT, X + 1, k});
        wait_ev(s, e.ev);
        dout = e.p;
      }
      const void *x_in = X == 0 ? nullptr : need(nd, {K_ACT, X, k}).p;
      void *dx = X > 0 ? arena_alloc(nd, msg_bytes(c, MSG_GRAD, X)) : nullptr;
      TMark tm(c, nd, s, brc ? 1 : 2);
      int slot = sv.slot;
      if (slot <= kHostSlot0) {
        // swapped to the host: copy it back into a device slot
        if (cp.free_slots.empty()) throw RtError{BB_E_STATE, "saved-set pool exhausted"};
        slot = cp.free_slots.back();
        cp.free_slots.pop_back();
        CK(cudaMemcpyAsync(slot_base(cp, slot), sv.p, c.stages[X].slot_bytes,
                           cudaMemcpyHostToDevice, s));
        if (c.recovering) ++c.frc_swapped;
      } else if (slot < 0) {
        // an FRC saved set beyond the retention budget: recompute the forward
        // from the retained stage input (same kernels, same order: the saved
        // set is bit-identical to the one FNC / FRC produced)
        if (cp.free_slots.empty()) throw RtError{BB_E_STATE, "saved-set pool exhausted"};
        slot = cp.free_slots.back();
        cp.free_slots.pop_back();
        const void *xi = stage_input(c, nd, s, X, k);
        void *tmp = X < P - 1 ? arena_alloc(nd, msg_bytes(c, MSG_ACT, X)) : nullptr;
        stage_forward(c, nd, cp, X, k, slot, s, xi, tmp, brc ? nd.s_loss_frc : nd.s_loss_main);
        if (c.recovering) ++c.frc_recomputed;
      }
      stage_backward(c, nd, cp, X, k, slot, s, x_in, dout, dx, nd.sc[brc ? 1 : 0]);
      cudaEvent_t e = record(nd, s);
      cp.free_slots.push_back(slot);
      if (X > 0 && (!brc || !nd.store.count({K_DACT, X, k}))) nd.store[{K_DACT, X, k}] = {dx, e};
      if (k == M - 1) nd.store[{K_GRADSUM, X, 0}] = {cp.grad, e};
      return true;
    }
    case SEND_ACT:
    case SEND_GRAD:
    case SEND_DGRAD:
    case RESEND_GRAD:
    case REPLICA_SEND:
    case AR_SEND:
    case RESEND_AR: {
      const Msg m = message_of(ins);
      const ChanKey ck{nd.n, ins.peer, (int)m.kind};
      if (ph.drop_to_victim && ins.peer == ph.victim) {
        // the victim never receives it: a survivor cannot deliver to a dead node
        const int sent = ++c.sent_to_victim[ck];
        auto it = c.victim_consumed.find(ck);
        if (it == c.victim_consumed.end() || sent > it->second) return true;
      }
      Entry pl = need(nd, payload_key(ins));
      // an all-reduce contribution is the local sum, never the total
      if (m.kind == MSG_AR) pl.p = nd.copies.at(X).grad;
      const size_t bytes = msg_bytes(c, m.kind, m.stage);
      if (c.recovering && (ins.kind == RESEND_GRAD || ins.kind == RESEND_AR ||
                           (ins.kind == SEND_ACT && X == c.rec_stage)))
        c.bytes_rerouted += bytes;
      if (is_local(c, ins.peer)) {
        Node &dst = c.nodes.at(ins.peer);
        // a replica gradient sum lands in the replica's accumulator, except
        // under EFEB (D > 1), where the replica's own eager BRC may still be
        // accumulating there on the receiver's FRC stream: then it is a
        // message of its own and the update reads it from there
        const bool into_grad = m.kind == MSG_GRADSUM && c.o.rc != BB_RC_EFEB;
        void *dp = into_grad               ? (void *)dst.copies.at(X).grad
                   : m.kind == MSG_AR      ? (void *)dst.copies.at(X).ar_in.at(nd.n / P)
                                           : arena_alloc(dst, bytes);
        wait_ev(nd.main, pl.ev);
        // the receiver's step-start memset of that buffer ran on ITS stream:
        // order this cross-node write after it explicitly
        wait_ev(nd.main, dst.ev_begin);
        CK(cudaMemcpyAsync(dp, pl.p, bytes, cudaMemcpyDeviceToDevice, nd.main));
        c.mail[ck].push_back({dp, record(nd, nd.main)});
      } else {
        XEdge &e = xedge(c, nd.n, ins.peer, m.kind);
        const int slot = (int)(e.sent % (uint64_t)e.cap);
        if (bytes > e.slot_bytes) throw RtError{BB_E_STATE, "message larger than its slot"};
        char *dst = e.peer_base + e.recv_off + (size_t)slot * e.slot_bytes;
        wait_ev(e.stream, pl.ev);
        CK(cudaMemcpyAsync(dst, pl.p, bytes, cudaMemcpyDeviceToDevice, e.stream));
        CK(c.x.post(e));   // published once the copy has completed
      }
      return true;
    }
    case RECV_ACT:
    case RECV_GRAD:
    case RECV_DGRAD:
    case REPLICA_RECV:
    case AR_RECV: {
      const Msg m = message_of(ins);
      const ChanKey ck{ins.peer, nd.n, (int)m.kind};
      Entry got;
      if (is_local(c, ins.peer)) {
        auto it = c.mail.find(ck);
        if (it == c.mail.end() || it->second.empty()) return false;
        got = it->second.front();
        it->second.pop_front();
      } else {
        XEdge &e = xedge(c, ins.peer, nd.n, m.kind);
        if (!c.x.available(e)) return false;       // the sender has not posted it yet
        const int slot = (int)(e.consumed % (uint64_t)e.cap);
        c.x.consume(e);
        char *src = c.x.arena + e.recv_off + (size_t)slot * e.slot_bytes;
        // event mode: consumers wait on the sender's event for this slot;
        // callback mode: the number was published after the payload landed
        cudaEvent_t ready = c.x.wait_event(e, slot);
        if (m.kind == MSG_GRADSUM && c.o.rc != BB_RC_EFEB) {   // (EFEB: read in place)
          wait_ev(nd.main, ready);
          CK(cudaMemcpyAsync(nd.copies.at(X).grad, src, msg_bytes(c, m.kind, m.stage),
                             cudaMemcpyDeviceToDevice, nd.main));
          got = {nd.copies.at(X).grad, record(nd, nd.main)};
        } else {
          got = {src, ready};
        }
      }
      if (ins.kind == RECV_ACT)
        nd.store[{K_ACT, X, k}] = got;
      else if (ins.kind == AR_RECV)
        nd.store[{K_AR, X, ins.peer / P}] = got;   // a shadow's stays its pipeline's
      else if (ins.kind == RECV_GRAD || ins.kind == RECV_DGRAD)
        nd.store[{K_DACT, X + 1, k}] = got;
      else
        nd.store[{K_GRADSUM, X, 0}] = {c.o.rc == BB_RC_EFEB ? got.p : nd.copies.at(X).grad, got.ev};
      return true;
    }
    case AR_SUM: {
      // the D contributions in ascending pipeline order: every
      // pipeline adds the same operands in the same order, same bits
      Copy &cp = nd.copies.at(X);
      std::vector<const float *> src(d.D);
      const int own = nd.n / P;
      for (int e = 0; e < d.D; ++e) {
        const Entry &en = need(nd, e == own ? Key{K_GRADSUM, X, 0} : Key{K_AR, X, e});
        wait_ev(nd.main, en.ev);
        src[e] = e == own ? cp.grad : (const float *)en.p;
      }
      CK(k::sum_pipelines(c.stages[X].pcount, src.data(), d.D, cp.arsum, nd.main));
      nd.store[{K_GRADSUM, X, 0}] = {cp.arsum, record(nd, nd.main)};
      return true;
    }
    case APPLY: {
      Copy &cp = nd.copies.at(X);
      const Entry gs = need(nd, {K_GRADSUM, X, 0});   // the local sum, or the total (D > 1)
      wait_ev(nd.main, gs.ev);
      wait_ev(nd.main, record(nd, nd.frc));   // the FRC stream read these parameters
      cp.t += 1;
      const double b1 = c.o.beta1, b2 = c.o.beta2;
      const float bc1 = (float)(1.0 - std::pow(b1, cp.t)), bc2 = (float)(1.0 - std::pow(b2, cp.t));
      Prof pf(c, nd, nd.main, PC_ADAM, 16.0 * c.stages[X].pcount);
      CK(k::adam(c.stages[X].pcount, cp.master, (const float *)gs.p, cp.m, cp.v,
                 c.bf16 ? cp.work : nullptr,
                 c.o.lr, c.o.beta1, c.o.beta2, c.o.eps, bc1, bc2, nd.main));
      return true;
    }
  }
  return true;
}

// Run the local nodes' lists; lim[n] caps node n (prefix of an interrupted step).
void run(Ctx &c, const Plans &lists, const std::map<int, int> *lim, const Phase &ph) {
  std::map<int, size_t> pc;
  for (auto &kv : c.nodes)
    if (kv.second.alive && lists.count(kv.first)) pc[kv.first] = 0;
  const double t_start = now_ms();
  for (;;) {
    bool progress = false, pending = false;
    for (auto &kv : pc) {
      Node &nd = c.nodes.at(kv.first);
      const auto &seq = lists.at(kv.first);
      size_t cap = seq.size();
      if (lim) cap = std::min(cap, (size_t)lim->at(kv.first));
      if (kv.second < cap) pending = true;
      while (kv.second < cap && exec(c, nd, seq[kv.second], ph)) {
        if (debug_on() || watch_s() > 0) {
          cudaEvent_t e1, e2;
          cudaEventCreateWithFlags(&e1, cudaEventDisableTiming);
          cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
          cudaEventRecord(e1, nd.main);
          cudaEventRecord(e2, nd.frc);
          c.dbg.push_back({nd.n, (int)kv.second, seq[kv.second], e1, e2});
        }
        ++kv.second;
        progress = true;
      }
    }
    if (!pending) break;
    if (!progress) {
      // waiting for a peer rank's message (or a genuine local deadlock)
      if (c.o.world_size == 1 || now_ms() - t_start > 300000.0) break;
      std::this_thread::yield();
    }
  }
  for (auto &kv : pc) {
    const auto &seq = lists.at(kv.first);
    size_t cap = seq.size();
    if (lim) cap = std::min(cap, (size_t)lim->at(kv.first));
    if (kv.second < cap) {
      std::ostringstream o;
      o << "local deadlock at node " << kv.first << " instruction " << kv.second;
      throw RtError{BB_E_STATE, o.str()};
    }
  }
}

void debug_wait(Ctx &c, bool comm_too) {
  // BB_DEBUG: poll instead of blocking and report the streams still busy
  for (int iter = 0;; ++iter) {
    bool busy = false;
    std::ostringstream o;
    for (auto &kv : c.nodes) {
      if (cudaStreamQuery(kv.second.main) == cudaErrorNotReady) { busy = true; o << " main" << kv.first; }
      if (cudaStreamQuery(kv.second.frc) == cudaErrorNotReady) { busy = true; o << " frc" << kv.first; }
    }
    if (comm_too)
      for (auto &kv : c.x.edges)
        if (kv.second.stream && cudaStreamQuery(kv.second.stream) == cudaErrorNotReady) {
          busy = true;
          o << " edge" << std::get<0>(kv.first) << "->" << std::get<1>(kv.first) << "k"
            << std::get<2>(kv.first) << "(sent " << kv.second.sent << ")";
        }
    if (!busy) return;
    if (iter % 50 == 49) {
      std::fprintf(stderr, "[bb rank %d] busy:%s\n", c.o.world_rank, o.str().c_str());
      std::map<int, int> shown;
      for (auto &d : c.dbg) {
        const bool m_ok = cudaEventQuery(d.main_ev) == cudaSuccess;
        const bool f_ok = cudaEventQuery(d.frc_ev) == cudaSuccess;
        if ((!m_ok || !f_ok) && shown[d.node]++ < 2)
          std::fprintf(stderr, "[bb rank %d] node %d first pending #%d %s mb=%d peer=%d stage=%d main=%d frc=%d\n",
                       c.o.world_rank, d.node, d.idx, kind_name(d.ins.kind), d.ins.mb, d.ins.peer,
                       d.ins.stage, m_ok, f_ok);
      }
    }
    struct timespec ts{0, 100000000};
    nanosleep(&ts, nullptr);
  }
}

void watch_wait(Ctx &c, bool comm_too) {
  const double t0 = now_ms();
  for (;;) {
    bool busy = false;
    for (auto &kv : c.nodes)
      busy = busy || cudaStreamQuery(kv.second.main) == cudaErrorNotReady ||
             cudaStreamQuery(kv.second.frc) == cudaErrorNotReady;
    if (comm_too)
      for (auto &kv : c.x.edges)
        busy = busy || (kv.second.stream && cudaStreamQuery(kv.second.stream) == cudaErrorNotReady);
    if (!busy) return;
    if (now_ms() - t0 > 1000.0 * watch_s()) {
      std::ostringstream o;
      o << "device watchdog: step not finished after " << watch_s() << " s;";
      std::map<int, int> shown;
      for (auto &d : c.dbg) {
        const bool m_ok = cudaEventQuery(d.main_ev) == cudaSuccess;
        const bool f_ok = cudaEventQuery(d.frc_ev) == cudaSuccess;
        if ((!m_ok || !f_ok) && shown[d.node]++ < 1)
          o << " node " << d.node << " #" << d.idx << ' ' << kind_name(d.ins.kind) << " mb "
            << d.ins.mb << " stage " << d.ins.stage << (m_ok ? "" : " main") << (f_ok ? "" : " frc")
            << ';';
      }
      std::fprintf(stderr, "[bb rank %d] %s\n", c.o.world_rank, o.str().c_str());
      throw RtError{BB_E_CUDA, o.str()};
    }
    struct timespec ts{0, 20000000};
    nanosleep(&ts, nullptr);
  }
}

// BB_WATCH: a host thread that outlives a hung device. When the launch
// queue fills behind a kernel that never finishes, the step's own thread
// blocks inside a launch and cannot report; this one prints the first
// unfinished instruction of every node and ends the process.
struct Watchdog {
  Ctx &c;
  std::atomic<bool> done{false};
  std::thread t;
  explicit Watchdog(Ctx &c_) : c(c_) {
    if (watch_s() <= 0) return;
    t = std::thread([this] {
      const double t0 = now_ms();
      while (!done.load()) {
        if (now_ms() - t0 > 1000.0 * (watch_s() + 5.0)) {
          std::fprintf(stderr, "[bb rank %d] watchdog: step running for %.0f s; first unfinished:",
                       c.o.world_rank, (now_ms() - t0) / 1000.0);
          std::map<int, int> shown;
          for (size_t i = 0; i < c.dbg.size(); ++i) {
            const DbgRec d = c.dbg[i];
            const bool m_ok = cudaEventQuery(d.main_ev) == cudaSuccess;
            const bool f_ok = cudaEventQuery(d.frc_ev) == cudaSuccess;
            if ((!m_ok || !f_ok) && shown[d.node]++ < 1)
              std::fprintf(stderr, " node %d #%d %s mb %d stage %d%s%s;", d.node, d.idx,
                           kind_name(d.ins.kind), d.ins.mb, d.ins.stage, m_ok ? "" : " main",
                           f_ok ? "" : " frc");
          }
          std::fprintf(stderr, " (%zu instructions issued); first unfinished kernel:",
                       c.dbg.size());
          std::map<int, int> shown_k;
          for (size_t i = 0; i < c.prof.size(); ++i) {
            const ProfRec r = c.prof[i];
            if (cudaEventQuery(r.b) != cudaSuccess && shown_k[r.node]++ < 1)
              std::fprintf(stderr, " node %d %s %.3g flop (%s, record %zu);", r.node,
                           prof_names[r.cls], r.work,
                           cudaEventQuery(r.a) == cudaSuccess ? "started" : "not started", i);
          }
          std::fprintf(stderr, "\n");
          k::gemm_trace_dump();
          std::fflush(stderr);
          _exit(3);
        }
        struct timespec ts{0, 50000000};
        nanosleep(&ts, nullptr);
      }
    });
  }
  ~Watchdog() {
    done = true;
    if (t.joinable()) t.join();
  }
};

void sync_all(Ctx &c, bool comm_too) {
  if (debug_on()) debug_wait(c, comm_too);
  else if (watch_s() > 0) watch_wait(c, comm_too);
  for (auto &kv : c.nodes) {
    CK(cudaStreamSynchronize(kv.second.main));
    CK(cudaStreamSynchronize(kv.second.frc));
    if (kv.second.swap) CK(cudaStreamSynchronize(kv.second.swap));
  }
  if (comm_too)
    for (auto &kv : c.x.edges)
      if (kv.second.stream) CK(cudaStreamSynchronize(kv.second.stream));
}

void begin_step(Ctx &c) {
  for (auto &d : c.dbg) {
    cudaEventDestroy(d.main_ev);
    cudaEventDestroy(d.frc_ev);
  }
  c.dbg.clear();
  if (watch_s() > 0) {   // the watchdog thread reads these: no reallocation
    c.dbg.reserve(1 << 18);
    c.prof.reserve(1 << 20);
  }
  c.mail.clear();
  c.prof.clear();
  c.prof_next = 0;
  c.h2d = c.d2h = 0;
  c.launches_at_start = k::g_launches;
  for (auto &kv : c.nodes) {
    Node &nd = kv.second;
    if (!nd.alive) continue;
    for (auto &cc : nd.copies) {   // host-swap slots are free again (sync_all at step end)
      cc.second.hnext = 0;
      cc.second.scratch_ev = nullptr;
    }
    nd.evnext = 0;
    nd.store.clear();
    nd.arena_used = 0;
    if (!nd.arena_spill.empty()) {   // the last step overflowed: regrow to its peak
      for (auto &ch : nd.arena_spill) CK(cudaFree(ch.first));
      nd.arena_spill.clear();
      CK(cudaFree(nd.arena));
      nd.arena_bytes = al(nd.arena_peak + nd.arena_peak / 8);
      nd.arena = (char *)dmalloc(nd.arena_bytes);
    }
    nd.arena_peak = 0;
    nd.trec.clear();
    nd.tnext = 0;
    for (auto &cc : nd.copies) {
      Copy &cp = cc.second;

      // a loss nobody computes this step reads NaN (LFLB: the last stage
      // lost after its commit point took the only copy of its losses)
      if (cp.loss) CK(k::fill_nan(cp.loss, (size_t)c.d.M * 4, nd.main));
      cp.free_slots.clear();
      for (int i = cp.nslots() - 1; i >= 0; --i) cp.free_slots.push_back(i);
      CK(cudaMemsetAsync(cp.grad, 0, c.stages[cp.X].pcount * sizeof(float), nd.main));
    }
    CK(cudaEventRecord(nd.ev_begin, nd.main));
    CK(cudaEventRecord(nd.t0, nd.main));
  }
}

// Host staging: tokens, targets and the per-micro-batch token CSR used by the
// deterministic embedding backward.
void stage_inputs(Ctx &c, const int32_t *tok, const int32_t *tgt) {
  const Dims &d = c.d;
  const size_t R = d.R();
  // ids index the embedding / head rows on the device: reject out-of-range
  // ids here rather than read or write outside the tensors
  const size_t n = (size_t)d.D * d.M * R;   // every pipeline's micro-batches
  for (size_t i = 0; i < n; ++i)
    if (tok[i] < 0 || tok[i] >= d.V || tgt[i] < 0 || tgt[i] >= d.V)
      throw RtError{BB_E_INVAL, "token or target id outside [0, vocab)"};
  std::memcpy(c.h_tok, tok, n * 4);
  std::memcpy(c.h_tgt, tgt, n * 4);
}

float read_loss_of(Ctx &c, int pipe);

// The step's loss: the sum of the local pipelines' shares (each is its
// micro-batches' token CE over the whole batch's token count); NaN without a
// local last stage.
float read_loss(Ctx &c) {
  float sum = 0.f;
  bool any = false;
  for (int p = 0; p < c.d.D; ++p) {
    const float l = read_loss_of(c, p);
    if (std::isnan(l) && !c.nodes.count(c.topo.host[p * c.d.P + c.d.P - 1])) continue;
    sum += l;
    any = true;
  }
  return any ? sum : NAN;
}

float read_loss_of(Ctx &c, int pipe) {
  const int X = c.d.P - 1;
  const int n = c.topo.host[pipe * c.d.P + X];
  if (!c.nodes.count(n) || !c.nodes.at(n).alive) return NAN;
  Node &nd = c.nodes.at(n);
  Copy &cp = nd.copies.at(X);
  float *tmp = nd.s_loss_main;   // scratch: loss rows are no longer needed
  if (std::getenv("BB_DEBUG_LOSS")) {
    std::vector<float> h(c.d.M);
    CK(cudaMemcpy(h.data(), cp.loss, c.d.M * 4, cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "[bb rank %d] loss of stage %d on node %d:", c.o.world_rank, X, n);
    for (float f : h) std::fprintf(stderr, " %g", f);
    std::fprintf(stderr, "\n");
  }
  CK(k::sum_fixed(c.d.M, cp.loss, tmp, nd.main));
  float h = NAN;
  CK(cudaMemcpyAsync(&h, tmp, 4, cudaMemcpyDeviceToHost, nd.main));
  CK(cudaStreamSynchronize(nd.main));
  c.d2h += 4;
  return h;
}

// A preempted node's memory is lost: NaN-fill everything the node
// owns (parameter copies, Adam state, saved sets, step arena, scratch) and
// mark it dead. Called at the injection, before bb_recover runs, so a
// recovery that read victim memory would poison the results (the bitwise
// recovered == failure-free tests catch it).
void poison_node(Ctx &c, Node &nd) {
  for (auto &cc : nd.copies) {
    Copy &cp = cc.second;
    const size_t n = c.stages[cp.X].pcount;
    CK(k::fill_nan(cp.master, n * 4, nd.main));
    CK(k::fill_nan(cp.m, n * 4, nd.main));
    CK(k::fill_nan(cp.v, n * 4, nd.main));
    CK(k::fill_nan(cp.grad, n * 4, nd.main));
    if (c.bf16) CK(k::fill_nan(cp.work, n * 2, nd.main));
    for (auto &ch : cp.chunks) CK(k::fill_nan(ch.first, ch.second, nd.main));
    if (cp.loss) CK(k::fill_nan(cp.loss, (size_t)c.d.M * 4, nd.main));
  }
  CK(k::fill_nan(nd.arena, nd.arena_bytes, nd.main));
  for (auto &ch : nd.arena_spill) CK(k::fill_nan(ch.first, ch.second, nd.main));
  const size_t R = c.d.R(), H = c.d.H, F = c.d.F;
  for (auto &sc : nd.sc) {
    if (!sc.sF) continue;
    CK(k::fill_nan(sc.sF, R * F * c.act_bytes, nd.main));
    CK(k::fill_nan(sc.s3, R * 3 * H * c.act_bytes, nd.main));
    for (auto p : sc.sH) CK(k::fill_nan(p, R * H * c.act_bytes, nd.main));
    for (auto p : sc.s32) CK(k::fill_nan(p, R * H * 4, nd.main));
  }
  CK(cudaStreamSynchronize(nd.main));
  nd.alive = false;
}

// Step end on every live node's main stream (before the host synchronises).
void mark_end(Ctx &c) {
  for (auto &kv : c.nodes)
    if (kv.second.alive) CK(cudaEventRecord(kv.second.t1, kv.second.main));
}

void finish_stats(Ctx &c, bb_step_stats *st, double t0) {
  c.last_step_ms = (float)(now_ms() - t0);
  if (!st) return;
  float dev = 0.f;
  for (auto &kv : c.nodes) {
    Node &nd = kv.second;
    if (!nd.alive) continue;
    CK(cudaEventSynchronize(nd.t1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, nd.t0, nd.t1));
    dev = std::max(dev, ms);
  }
  st->device_ms = dev;
  st->step_ms = c.last_step_ms;
  st->gpu_launches = (int)(k::g_launches - c.launches_at_start);
  st->h2d_bytes = c.h2d;
  st->d2h_bytes = c.d2h;
}
}  // namespace

// ========================================================== fail-stop mode
// opts.detect_ms > 0: a preempted rank goes silent; the others
// notice that its heartbeat stopped, run to quiescence, agree on the cut from
// the messages it delivered, and recover as in the injected mode.
namespace {
// Messages each cross-rank edge carries when `plans` run for `lim` (or all)
// instructions: every rank derives the same counts from the same plans.
void add_edge_sends(Ctx &c, const Plans &plans, const std::map<int, int> *lim) {
  for (auto &kv : plans) {
    const int n = kv.first;
    size_t cap = kv.second.size();
    if (lim && lim->count(n)) cap = std::min(cap, (size_t)lim->at(n));
    for (size_t i = 0; i < cap; ++i) {
      const Instr &ins = kv.second[i];
      if (!is_send(ins.kind) || c.node_rank[ins.peer] == c.node_rank[n]) continue;
      auto it = c.x.edges.find(std::make_tuple(n, ins.peer, (int)message_of(ins).kind));
      if (it != c.x.edges.end()) ++c.edge_prior[it->second.index];
    }
  }
}

uint64_t hb_now(Ctx &c, int r) { return *c.x.rank_word(0, r); }

// Ranks whose heartbeat has not moved for detect_ms are flagged dead in shm
// (every survivor applies the same rule; the flag makes the verdict shared).
void detect(Ctx &c, std::vector<uint64_t> &seen, std::vector<double> &since) {
  const double t = now_ms();
  for (int r = 0; r < c.o.world_size; ++r) {
    if (r == c.o.world_rank || c.x.dead(r)) continue;
    const uint64_t h = hb_now(c, r);
    if (h != seen[r]) {
      seen[r] = h;
      since[r] = t;
    } else if (t - since[r] > c.o.detect_ms) {
      __atomic_store_n(const_cast<uint64_t *>(c.x.rank_word(1, r)), 1ull, __ATOMIC_RELEASE);
      c.detect_ms_seen = t - since[r];
    }
  }
}

uint64_t inbound_sum(Ctx &c, int rank) {
  uint64_t s = 0;
  for (auto &kv : c.x.edges)
    if (kv.second.dst_rank == rank) s += *c.x.counter(kv.second.index);
  return s;
}

// Quiescent: every live rank is blocked on what it last saw arrive, and every
// copy enqueued between live ranks has completed.
bool quiescent(Ctx &c) {
  for (int r = 0; r < c.o.world_size; ++r) {
    if (c.x.dead(r)) continue;
    const uint64_t b = *c.x.rank_word(2, r);
    if (b == 0 || b - 1 != inbound_sum(c, r)) return false;
  }
  for (auto &kv : c.x.edges) {
    const XEdge &e = kv.second;
    if (c.x.dead(e.src_rank) || c.x.dead(e.dst_rank)) continue;
    if (*c.x.intent(e.index) != *c.x.counter(e.index)) return false;
  }
  return true;
}

// Survivor side of a fail-stop step. Returns -1 when the step completed on
// every live rank, else the dead node (the local lists stopped at quiescence;
// pcs holds how far each local node got).
int run_failstop(Ctx &c, std::map<int, size_t> &pc) {
  const int W = c.o.world_size, me = c.o.world_rank;
  std::vector<uint64_t> seen(W, 0);
  std::vector<double> since(W, now_ms());
  for (int r = 0; r < W; ++r) seen[r] = hb_now(c, r);
  for (auto &kv : c.nodes)
    if (kv.second.alive && c.plans.count(kv.first)) pc[kv.first] = 0;
  auto flag = [&](int f) { return const_cast<uint64_t *>(c.x.rank_word(f, me)); };
  bool arrived = false;
  double stable_since = -1;
  for (;;) {
    bool progress = false, done = true;
    for (auto &kv : pc) {
      Node &nd = c.nodes.at(kv.first);
      const auto &seq = c.plans.at(kv.first);
      while (kv.second < seq.size() && exec(c, nd, seq[kv.second], Phase{})) {
        ++kv.second;
        progress = true;
      }
      if (kv.second < seq.size()) done = false;
    }
    if (done && !arrived) {
      mark_end(c);
      sync_all(c, true);
      __atomic_store_n(flag(4), c.step_id, __ATOMIC_RELEASE);
      arrived = true;
    }
    int dead = -1;   // a rank lost in THIS step (earlier victims stay flagged)
    for (int r = 0; r < W; ++r)
      if (c.x.dead(r) && std::find(c.victims.begin(), c.victims.end(), r) == c.victims.end())
        dead = r;
    if (arrived && dead < 0) {
      bool all = true;
      for (int r = 0; r < W; ++r)
        if (!c.x.dead(r) && *c.x.rank_word(4, r) < c.step_id) all = false;
      if (all) return -1;
    }
    if (progress) {
      __atomic_store_n(flag(2), 0ull, __ATOMIC_RELEASE);
      stable_since = -1;
      continue;
    }
    if (dead < 0) {
      detect(c, seen, since);
      std::this_thread::yield();
      continue;
    }
    // a rank is gone: block here, publish what we have seen, wait for the
    // live ranks to settle
    __atomic_store_n(flag(2), 1 + inbound_sum(c, me), __ATOMIC_RELEASE);
    if (quiescent(c)) {
      if (stable_since < 0) stable_since = now_ms();
      if (now_ms() - stable_since > 20.0) {
        if (!arrived) {
          mark_end(c);
          sync_all(c, true);
        }
        return dead;   // dead RANK; with one node per rank it is the node id
      }
    } else {
      stable_since = -1;
    }
    std::this_thread::yield();
  }
}

// The victim's instruction count as seen from outside: just past the last
// send whose message was delivered (its later instructions left no trace).
int observed_cut(Ctx &c, int v) {
  std::map<int, uint64_t> ordinal;   // per edge index, sends of v so far this step
  const auto &seq = c.plans.at(v);
  int pi = 0;
  for (size_t i = 0; i < seq.size(); ++i) {
    const Instr &ins = seq[i];
    if (!is_send(ins.kind)) continue;
    auto it = c.x.edges.find(std::make_tuple(v, ins.peer, (int)message_of(ins).kind));
    if (it == c.x.edges.end()) continue;
    const int e = it->second.index;
    const uint64_t delivered = *c.x.counter(e) - c.edge_prior[e];
    if (ordinal[e]++ < delivered) pi = (int)i + 1;
  }
  return pi;
}

void heartbeat(Ctx *c) {
  volatile uint64_t *h = c->x.rank_word(0, c->o.world_rank);
  while (!c->hb_stop.load()) {
    __atomic_add_fetch(const_cast<uint64_t *>(h), 1ull, __ATOMIC_RELEASE);
    struct timespec ts{0, 5000000};
    nanosleep(&ts, nullptr);
  }
}
}  // namespace

// ================================================================= API
bb_status rt_init(Ctx &c, const bb_model *m, int P, int M, const bb_opts *o) {
  try {
    if (!m || P < 1 || M < 1) throw RtError{BB_E_INVAL, "bad arguments"};
    bb_opts def;
    bb_default_opts(&def);
    c.o = o ? *o : def;
    if (c.o.world_size < 1 || c.o.world_rank < 0 || c.o.world_rank >= c.o.world_size)
      throw RtError{BB_E_INVAL, "bad world rank/size"};
    if (m->n_layer < P) throw RtError{BB_E_INVAL, "n_layer < stages"};
    if (c.o.rc != BB_RC_NONE && P < 2) throw RtError{BB_E_INVAL, "RC needs stages >= 2"};
    if (c.o.rc < BB_RC_NONE || c.o.rc > BB_RC_EFEB) throw RtError{BB_E_INVAL, "unknown RC mode"};
    if (m->n_head <= 0 || m->d_model % m->n_head) throw RtError{BB_E_INVAL, "d_model % n_head"};
    if (m->d_model % 8 || m->d_ff % 8 || m->vocab % 8)
      throw RtError{BB_E_INVAL, "d_model, d_ff, vocab must be multiples of 8"};
    if (m->d_model / m->n_head != 64 && m->d_model / m->n_head != 32)
      throw RtError{BB_E_UNSUPPORTED, "attention kernels take head dim 64 (or 32)"};
    if (c.o.micro_batch < 1) throw RtError{BB_E_INVAL, "micro_batch < 1"};
    const int D = c.o.pipelines < 1 ? 1 : c.o.pipelines, N = D * P;   // pipelines, nodes
    if (D > k::kMaxPipelines) throw RtError{BB_E_UNSUPPORTED, "at most 8 pipelines"};
    if (c.o.detect_ms > 0 && (c.o.world_size != N || c.o.node_rank))
      // a process death takes all its nodes: only one node per rank is recoverable
      throw RtError{BB_E_INVAL,
                    "fail-stop mode needs one node per rank (world_size == pipelines * stages)"};
    if (c.o.prec == BB_PREC_BF16 && m->d_model < 64)
      // the transposed (MN-major) operands of dX / dW need >= 64 rows
      throw RtError{BB_E_UNSUPPORTED, "bf16 path needs d_model >= 64"};
    c.d = {m->n_layer, m->d_model, m->n_head, m->d_ff, m->vocab, m->seq_len, m->causal ? 1 : 0,
           P, M, c.o.micro_batch, D};
    c.bf16 = c.o.prec == BB_PREC_BF16;
    c.act_bytes = c.bf16 ? 2 : 4;
    const bool rc = c.o.rc != BB_RC_NONE;
    try {
      c.ranges = partition(m->n_layer, P, c.o.layers_per_stage);
      c.plans = normal_plans(P, M, (int)c.o.rc, D);
    } catch (const PlanError &e) {
      throw RtError{BB_E_INVAL, e.msg};
    }
    c.topo = normal_topology(P, rc, D);
    for (int X = 0; X < P; ++X) {
      c.stages.push_back(make_stage(c.d, X, c.ranges[X].first, c.ranges[X].second));
      layout_slots(c.d, c.act_bytes, c.stages.back());
    }
    auto ur = unit_param_ranges(c.d);
    c.total_params = ur.back().first + ur.back().second;
    // node -> rank
    c.node_rank.resize(N);
    const int per = (N + c.o.world_size - 1) / c.o.world_size;
    for (int n = 0; n < N; ++n) {
      c.node_rank[n] = c.o.node_rank ? c.o.node_rank[n] : std::min(n / per, c.o.world_size - 1);
      if (c.node_rank[n] < 0 || c.node_rank[n] >= c.o.world_size)
        throw RtError{BB_E_INVAL, "bad node_rank"};
    }
    c.node_device.assign(N, 0);
    for (int n = 0; n < N; ++n) c.node_device[n] = c.node_rank[n];
    CK(cudaSetDevice(c.o.device));
    const size_t R = c.d.R();
    c.csr_stride = k::embed_csr_ints((int)R);
    CK(cudaMallocHost(&c.h_tok, (size_t)D * M * R * 4));
    CK(cudaMallocHost(&c.h_tgt, (size_t)D * M * R * 4));
    int lo_prio = 0, hi_prio = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    const size_t act = R * c.d.H * c.act_bytes;
    for (int n = 0; n < N; ++n) {
      if (c.node_rank[n] != c.o.world_rank) continue;
      Node &nd = c.nodes[n];
      const int sn = n % P;   // the node's stage
      nd.n = n;
      if (c.o.profile) {
        // profiling: every local node issues into one serialised stream so
        // each kernel's CUDA-event time is its own (no cross-stream overlap)
        if (!c.serial) CK(cudaStreamCreateWithPriority(&c.serial, cudaStreamNonBlocking, hi_prio));
        nd.main = nd.frc = c.serial;
      } else {
        CK(cudaStreamCreateWithPriority(&nd.main, cudaStreamNonBlocking, hi_prio));
        CK(cudaStreamCreateWithPriority(&nd.frc, cudaStreamNonBlocking, lo_prio));
      }
      CK(cudaEventCreate(&nd.t0));
      CK(cudaEventCreate(&nd.t1));
      CK(cudaEventCreateWithFlags(&nd.ev_begin, cudaEventDisableTiming));
      std::vector<std::pair<int, bool>> hosted{{sn, false}};
      if (rc) hosted.push_back({(sn + 1) % P, true});
      for (auto &h : hosted) {
        const int X = h.first;
        const StageInfo &si = c.stages[X];
        Copy &cp = nd.copies[X];
        cp.X = X;
        cp.replica = h.second;
        cp.master = (float *)dmalloc(si.pcount * 4);
        cp.m = (float *)dmalloc(si.pcount * 4);
        cp.v = (float *)dmalloc(si.pcount * 4);
        cp.grad = (float *)dmalloc(si.pcount * 4);
        cp.work = c.bf16 ? dmalloc(si.pcount * 2) : (void *)cp.master;
        if (!h.second) {   // 1F1B stash of the node's own stage: min(M, P - X) in flight
          grow_slots(cp, std::min(M, P - X), si.slot_bytes);
        }
        if (X == P - 1) cp.loss = (float *)dmalloc(M * 4);
        if (D > 1) {   // a replica may be promoted: its node then runs the all-reduce
          cp.arsum = (float *)dmalloc(si.pcount * 4);
          cp.ar_in.assign(D, nullptr);
          for (int e = 0; e < D; ++e)
            if (e != n / P) cp.ar_in[e] = (float *)dmalloc(si.pcount * 4);
        }
      }
      // normal 1F1B step: FWD / FRC outputs, BWD input-gradients, local receives
      nd.arena_bytes = (size_t)(6 * M + 8) * al(act);
      nd.arena = (char *)dmalloc(nd.arena_bytes);
      const size_t F = c.d.F, H = c.d.H;
      for (int si = 0; si < (c.o.rc == BB_RC_EFEB ? 2 : 1); ++si) {
        Node::Scratch &sc = nd.sc[si];
        sc.sF = dmalloc(R * F * c.act_bytes);
        sc.s3 = dmalloc(R * 3 * H * c.act_bytes);
        for (auto &p : sc.sH) p = dmalloc(R * H * c.act_bytes);
        for (auto &p : sc.s32) p = (float *)dmalloc(R * H * 4);
        const size_t pb = k::colreduce_partial_floats((int)R, (int)std::max(F, 3 * H)) * 4;
        sc.s_part = (float *)dmalloc(pb);
        CK(cudaMemset(sc.s_part, 0, pb));   // colreduce tickets start at zero
        sc.s_attn = (float *)dmalloc(
            k::attention_bwd_scratch_floats(c.d.mb, c.d.S, (int)H, c.d.nh) * 4);
      }
      nd.s_loss_main = (float *)dmalloc(R * 4);
      nd.s_loss_frc = (float *)dmalloc(R * 4);
      nd.d_tok = (int32_t *)dmalloc((size_t)M * R * 4);
      nd.d_tgt = (int32_t *)dmalloc((size_t)M * R * 4);
      nd.d_csr = (int32_t *)dmalloc((size_t)M * c.csr_stride * 4);
      // the embedding backward runs where a copy of stage 0 lives (its own
      // node, the replica holder for a lazy BRC)
      nd.needs_csr = sn == 0 || (rc && sn == P - 1);
    }
    // Cross-rank edges, set up before the retention pools so an automatic
    // FRC budget sees the receive arenas: one per (src node, dst node, kind) whose endpoints
    // live on different ranks; ring distance <= 2 covers the normal pipeline,
    // the replica ring and the failover skip edges (xport.h).
    if (c.o.world_size > 1) {
      if (!c.o.session_id) throw RtError{BB_E_INVAL, "session_id required for world_size > 1"};
      std::set<std::tuple<int, int, int>> want;
      // node of pipeline p's stage s (ring inside the pipeline)
      auto node = [&](int p, int s) { return p * P + ((s % P) + P) % P; };
      auto add = [&](int a, int b, int kind) {
        if (a != b && c.node_rank[a] != c.node_rank[b]) want.insert({a, b, kind});
      };
      for (int p = 0; p < D; ++p)
        for (int s = 0; s < P; ++s) {
          const int a = node(p, s);
          if (s < P - 1) add(a, node(p, s + 1), MSG_ACT);
          add(a, node(p, s + 2), MSG_ACT);
          if (s > 0) add(a, node(p, s - 1), MSG_GRAD);
          add(a, node(p, s - 2), MSG_GRAD);
          add(a, node(p, s - 1), MSG_GRADSUM);
          add(node(p, s - 1), a, MSG_STATE);   // rejoin: shadow -> returning node
          add(node(p, s + 1), a, MSG_STATE);   // rejoin: successor -> returning node
          if (c.o.rc == BB_RC_EFEB) {   // eager-BRC gradients; after a loss the shadow
            add(a, node(p, s - 2), MSG_DGRAD);    // takes over the victim's (one hop back)
            add(a, node(p, s - 1), MSG_DGRAD);
          }
          // all-reduce partners, and the shadow that stands in for a lost one
          for (int q = 0; q < D; ++q) {
            if (q == p) continue;
            add(a, node(q, s), MSG_AR);
            add(a, node(q, s - 1), MSG_AR);
            add(node(q, s - 1), a, MSG_AR);
          }
        }
      size_t gmax = 0;
      for (auto &st : c.stages) gmax = std::max(gmax, st.pcount);
      const std::vector<size_t> slot_bytes{act, act, gmax * sizeof(float),
                                           3 * gmax * sizeof(float), act, gmax * sizeof(float)};
      // rejoin sends one state message per edge, two when P == 2 (the shadow
      // and the successor are the same node)
      // (all-reduce: one contribution per stage and step; two when both ends
      // are shadows of the same lost stage and also exchange their own)
      const std::vector<int> caps{2 * M + 4, 2 * M + 4, 4, P == 2 ? 2 : 1, 2 * M + 4, 2};
      const std::vector<std::tuple<int, int, int>> wl(want.begin(), want.end());
      const std::string xe = xport_init(c.x, c.o.world_rank, c.o.world_size, N, wl, c.node_rank,
                                        slot_bytes, caps, c.o.session_id, hi_prio,
                                        /*callback_mode=*/c.o.detect_ms > 0);
      if (!xe.empty()) throw RtError{BB_E_CUDA, "transport init: " + xe};
      c.edge_prior.assign(c.x.nedges, 0);
    }
    // FRC retention pools of the replicas (Q10), allocated last so an
    // automatic budget can take what the rest left free: `retain` slots (the
    // FRC saved sets kept per step) plus a scratch slot for the FRCs beyond
    // them. A promoted replica's pool grows in bb_recover (the 1F1B stash of
    // the victim's stage, min(M, P - X) in flight, plus one BRC re-forward).
    if (rc) {
      size_t budget = c.o.frc_retain_bytes;
      int nrep = 0;
      for (auto &kv : c.nodes)
        for (auto &cc : kv.second.copies) nrep += cc.second.replica ? 1 : 0;
      if (budget == (size_t)-1 && nrep > 0) {   // auto: what is free, minus a reserve
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const size_t reserve = (size_t)8 << 30;
        budget = fr > reserve ? (fr - reserve) / nrep : 0;
      }
      for (auto &kv : c.nodes)
        for (auto &cc : kv.second.copies) {
          Copy &cp = cc.second;
          if (!cp.replica) continue;
          const StageInfo &si = c.stages[cp.X];
          const bool frc = c.o.rc == BB_RC_EFLB || c.o.rc == BB_RC_EFEB;   // LFLB: no FRC
          // (an embedding-only stage saves nothing: every saved set fits)
          const int full = !frc ? 0 : budget == 0 || si.slot_bytes == 0 ? M
                                    : (int)std::min<size_t>(M, budget / si.slot_bytes);
          cp.retain = full;
          grow_slots(cp, full, si.slot_bytes);
          if (frc && full < M) {
            cp.scratch = (char *)dmalloc(si.slot_bytes);
            cp.chunks.push_back({cp.scratch, si.slot_bytes});
            // host-swap tier for the rest
            const size_t nh = std::min<size_t>(M - full, c.o.frc_swap_bytes / si.slot_bytes);
            if (nh > 0) {
              CK(cudaHostAlloc(&cp.hbase, nh * si.slot_bytes, cudaHostAllocDefault));
              for (size_t i = 0; i < nh; ++i) cp.hslots.push_back(cp.hbase + i * si.slot_bytes);
              Node &hn = kv.second;
              if (!hn.swap) CK(cudaStreamCreateWithFlags(&hn.swap, cudaStreamNonBlocking));
            }
          }
        }
    }
    if (c.o.world_size > 1 && c.o.detect_ms > 0) {
      c.failstop = true;
      c.hb_thread = std::thread(heartbeat, &c);
    }
    CK(cudaDeviceSynchronize());
    return BB_OK;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

bb_status rt_load_params(Ctx &c, const float *host, size_t n) {
  try {
    if (n != c.total_params) throw RtError{BB_E_INVAL, "parameter count mismatch"};
    for (auto &kv : c.nodes) {
      Node &nd = kv.second;
      for (auto &cc : nd.copies) {
        Copy &cp = cc.second;
        const StageInfo &si = c.stages[cp.X];
        // Everything on the node's stream, in order. (Round 1 used the legacy
        // stream's cudaMemcpy here: from pageable memory it returns once the
        // data is staged, before the DMA lands, and the cast on the
        // non-blocking node stream could read the old master — a bf16 working
        // copy of zeros, seen as a head-only stage with zero gradients and as
        // uniform logits in multi-process runs on one GPU.)
        CK(cudaMemcpyAsync(cp.master, host + si.poff, si.pcount * 4, cudaMemcpyHostToDevice,
                           nd.main));
        CK(cudaMemsetAsync(cp.m, 0, si.pcount * 4, nd.main));
        CK(cudaMemsetAsync(cp.v, 0, si.pcount * 4, nd.main));
        if (c.bf16) CK(k::cast_f32_to_bf16(si.pcount, cp.master, cp.work, nd.main));
        cp.t = 0;
      }
    }
    c.adam_steps = 0;
    CK(cudaDeviceSynchronize());
    return BB_OK;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

namespace {
bb_status step_failstop(Ctx &c, bb_step_stats *st, double t0) {
  if (c.self_dead) throw RtError{BB_E_STATE, "this rank was preempted"};
  ++c.step_id;
  begin_step(c);
  if (c.armed) {
    // this rank is the victim: run its first pi instructions, let what it sent
    // land, then go silent (no heartbeat, no step-end arrival)
    c.armed = false;
    std::map<int, int> lim{{c.inj_v, c.inj_pi}};
    run(c, c.plans, &lim, Phase{});
    sync_all(c, true);
    c.hb_stop = true;
    if (c.hb_thread.joinable()) c.hb_thread.join();
    c.self_dead = true;
    c.nodes.at(c.inj_v).alive = false;
    finish_stats(c, st, t0);
    if (st) st->loss = NAN;
    return BB_E_PREEMPTED;
  }
  std::map<int, size_t> pc;
  const int dead = run_failstop(c, pc);
  if (dead < 0) {   // every live rank finished the step
    add_edge_sends(c, c.plans, nullptr);
    ++c.steps_done;
    ++c.adam_steps;
    {
      const float loss = read_loss(c);   // its 4-byte read counts in d2h_bytes
      finish_stats(c, st, t0);
      if (st) st->loss = loss;
    }
    return BB_OK;
  }
  // a node died: agree on the cut. Publish how far our nodes got, meet the
  // other survivors, infer the victim's point from what it delivered.
  for (auto &kv : pc) *const_cast<uint64_t *>(c.x.node_pc(kv.first)) = kv.second;
  c.x.barrier();
  const int v = dead;
  if (c.o.rc == BB_RC_NONE || !recoverable(c.d.P, c.topo, c.victims, v)) {
    c.fatal = true;
    throw RtError{BB_E_FATAL, "lost node " + std::to_string(v) + " has no redundancy left"};
  }
  c.inj_v = v;
  c.inj_pi = observed_cut(c, v);
  if (std::getenv("BB_DEBUG_LOSS"))
    std::fprintf(stderr, "[bb rank %d] fail-stop: node %d lost, observed cut %d\n", c.o.world_rank, v,
                 c.inj_pi);
  try {
    c.cut = cut(c.plans, v, c.inj_pi);
  } catch (const PlanError &e) {
    throw RtError{BB_E_STATE, e.msg};
  }
  for (auto &kv : c.cut.pcs) {
    if (kv.first == v) continue;
    const uint64_t got = *c.x.node_pc(kv.first);
    if ((uint64_t)kv.second != got)
      throw RtError{BB_E_STATE, "fail-stop: node " + std::to_string(kv.first) + " stopped at " +
                                    std::to_string(got) + ", the cut says " +
                                    std::to_string(kv.second)};
  }
  std::map<int, int> lim = c.cut.pcs;
  add_edge_sends(c, c.plans, &lim);
  c.interrupted = true;
  finish_stats(c, st, t0);
  if (st) st->loss = NAN;
  return BB_E_PREEMPTED;
}
}  // namespace

bb_status rt_step(Ctx &c, const int32_t *tok, const int32_t *tgt, bb_step_stats *st) {
  const double t0 = now_ms();
  try {
    if (c.fatal) return BB_E_FATAL;
    if (c.interrupted) throw RtError{BB_E_STATE, "bb_recover pending"};
    if ((tok == nullptr) != (tgt == nullptr)) throw RtError{BB_E_INVAL, "null tokens/targets"};
    if (!tok && !c.resident) throw RtError{BB_E_STATE, "no resident inputs (bb_stage_inputs)"};
    CK(cudaSetDevice(c.o.device));
    if (tok) {
      stage_inputs(c, tok, tgt);   // validates ids (BB_E_INVAL) before any rank moves on
      c.resident = false;          // LOAD_INPUTS overwrites the device copies
    }
    c.resident_step = tok == nullptr;
    Watchdog dog(c);
    if (c.failstop) return step_failstop(c, st, t0);
    c.x.barrier();   // every rank finished the previous step: receive slots are free
    // profile mode: park the serialised stream while the host enqueues the
    // step, so host launch latency never sits inside a kernel's event bracket
    if (c.o.profile && c.serial) CK(k::gpu_sleep(200000000ull, c.serial));
    begin_step(c);
    if (!c.armed) {
      run(c, c.plans, nullptr, Phase{});
      mark_end(c);
      sync_all(c, true);
      ++c.steps_done;
      ++c.adam_steps;
      {
        const float loss = read_loss(c);   // its 4-byte read counts in d2h_bytes
        finish_stats(c, st, t0);
        if (st) st->loss = loss;
      }
      return BB_OK;
    }
    // injected preemption: every rank computes the same cut (Q12/Q14)
    c.armed = false;
    const int v = c.inj_v;
    try {
      c.cut = cut(c.plans, v, c.inj_pi);
    } catch (const PlanError &e) {
      throw RtError{BB_E_INVAL, e.msg};
    }
    // messages the victim consumed before dying, per channel
    c.victim_consumed.clear();
    c.sent_to_victim.clear();
    {
      std::map<int, int> pcs;
      Channels ch;
      std::map<int, int> cap{{v, c.inj_pi}};
      lockstep(c.plans, pcs, ch, cap, [&](int n, const Instr &ins) {
        if (n == v && is_recv(ins.kind))
          ++c.victim_consumed[ChanKey{ins.peer, v, (int)message_of(ins).kind}];
      });
    }
    Phase ph;
    ph.drop_to_victim = true;
    ph.victim = v;
    run(c, c.plans, &c.cut.pcs, ph);
    mark_end(c);
    sync_all(c, true);
    // the victim's memory is gone the moment it is preempted: NaN-poison
    // everything its node owned now, so nothing in bb_recover can read it
    if (c.nodes.count(v)) poison_node(c, c.nodes.at(v));
    c.interrupted = true;
    finish_stats(c, st, t0);
    if (st) st->loss = NAN;
    return BB_E_PREEMPTED;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

bb_status rt_stage_inputs(Ctx &c, const int32_t *tok, const int32_t *tgt) {
  try {
    if (!tok || !tgt) throw RtError{BB_E_INVAL, "null tokens/targets"};
    CK(cudaSetDevice(c.o.device));
    stage_inputs(c, tok, tgt);
    const size_t n = (size_t)c.d.M * c.d.R();
    for (auto &kv : c.nodes) {
      Node &nd = kv.second;
      const size_t off = (size_t)(nd.n / c.d.P) * n;   // the node's pipeline's share
      CK(cudaMemcpy(nd.d_tok, c.h_tok + off, n * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(nd.d_tgt, c.h_tgt + off, n * 4, cudaMemcpyHostToDevice));
      if (nd.needs_csr) CK(k::embed_csr(c.d.M, c.d.R(), nd.d_tok, nd.d_csr, nd.main));
      CK(cudaStreamSynchronize(nd.main));
    }
    c.resident = true;
    return BB_OK;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

bb_status rt_preempt(Ctx &c, int stage, int at_instr) {
  if (c.fatal) return BB_E_FATAL;
  if (c.interrupted) {
    c.err = "recovery pending";
    return BB_E_STATE;
  }
  if (stage < 0 || stage >= c.d.D * c.d.P) {
    c.err = "unknown node";
    return BB_E_INVAL;
  }
  if (c.o.rc == BB_RC_NONE || !recoverable(c.d.P, c.topo, c.victims, stage)) {
    // no live replica of the victim's stage (no RC; or the victim is dead, is a
    // double-duty shadow, or lost its replica holder: P:464 consecutive nodes, Q18)
    c.err = "no redundancy left for the victim";
    return BB_E_FATAL;
  }
  if (c.failstop && !is_local(c, stage)) {
    c.err = "fail-stop mode: arm the preemption on the victim's rank only";
    return BB_E_INVAL;
  }
  if (at_instr < 0 || at_instr > (int)c.plans.at(stage).size()) {
    c.err = "injection point beyond the victim's list";
    return BB_E_INVAL;
  }
  c.armed = true;
  c.inj_v = stage;
  c.inj_pi = at_instr;
  return BB_OK;
}

bb_status rt_recover(Ctx &c, bb_recovery_stats *r) {
  const double t0 = now_ms();
  try {
    if (!c.interrupted) throw RtError{BB_E_STATE, "no interrupted step"};
    const int P = c.d.P, M = c.d.M, v = c.inj_v, u = ring_prev(P, v), sv = v % P;
    try {
      c.continuation = recovery_plans(c.plans, P, M, v, c.cut.pcs, c.cut.ch, &c.rinfo);
    } catch (const PlanError &e) {
      throw RtError{BB_E_STATE, e.msg};
    }
    {
      std::ostringstream o;
      o << "# bamboo-recovery v1 P=" << P << " M=" << M << " victim=" << v << " shadow=" << u
        << " successor=" << c.rinfo.successor << " commit=" << (c.rinfo.commit ? 1 : 0) << '\n';
      o << "# cut";
      for (auto &kv : c.cut.pcs) o << ' ' << kv.first << ':' << kv.second;
      o << '\n' << dump_lines(c.continuation);
      c.recovery_text = o.str();
    }
    // promote the replica on the shadow; the victim stops. The
    // promoted pool must also hold the victim stage's 1F1B stash (min(M, P-v)
    // in flight) and one BRC re-forward next to the retained FRC saved sets.
    if (c.nodes.count(u)) {
      Copy &cp = c.nodes.at(u).copies.at(sv);
      cp.replica = false;
      const int need = std::min(M, cp.retain + std::min(M, P - sv) + 1);
      const size_t sb = c.stages[sv].slot_bytes;
      try {
        grow_slots(cp, need - cp.nslots(), sb);
      } catch (const RtError &e) {
        // one GPU hosts the victim too (stages > GPUs): its pools are dead
        // memory now, hand them to the shadow
        if (e.st != BB_E_OOM || !c.nodes.count(v)) throw;
        for (auto &cc : c.nodes.at(v).copies) free_slots_all(cc.second);
        grow_slots(cp, need - cp.nslots(), sb);
      }
    }
    Phase ph;
    c.recovering = true;
    c.rec_stage = sv;
    c.frc_recomputed = 0;
    c.frc_swapped = 0;
    c.bytes_rerouted = 0;
    run(c, c.continuation, nullptr, ph);
    c.recovering = false;
    sync_all(c, true);
    if (c.failstop) {
      add_edge_sends(c, c.continuation, nullptr);
      // the victim's rank may now release its memory (our copies into it are done)
      *const_cast<uint64_t *>(c.x.rank_word(3, c.o.world_rank)) = 1;
    }
    c.history.push_back({c.plans, c.topo});
    c.topo = lose_node(P, c.topo, v);
    try {
      c.plans = failover_plans(P, M, v, &c.history.back().plans);
    } catch (const PlanError &e) {
      throw RtError{BB_E_STATE, e.msg};
    }
    c.failover = true;
    c.victims.push_back(v);
    c.interrupted = false;
    ++c.steps_done;
    ++c.adam_steps;
    if (r) {
      r->victim = v;
      r->shadow = u;
      r->successor = c.rinfo.successor;
      r->commit = c.rinfo.commit ? 1 : 0;
      r->brc_mb = (int)c.rinfo.brc_mb.size();
      r->frc_done_mb = (int)c.rinfo.frc_done.size();
      r->resent_mb = (int)c.rinfo.resend.size();
      r->loss = read_loss(c);
      r->recover_ms = (float)(now_ms() - t0);
      r->interrupted_step_ms = c.last_step_ms;
      r->frc_recomputed_mb = c.frc_recomputed;
      r->bytes_resent = c.bytes_rerouted;
      r->frc_swapped_mb = c.frc_swapped;
    }
    return BB_OK;
  } catch (const RtError &e) {
    c.recovering = false;
    c.err = e.msg;
    c.fatal = e.st != BB_E_INVAL;
    return e.st;
  }
}

// Reconfiguration back to full depth: the
// returning node v receives its stage (params + Adam state) from the shadow
// and its successor's stage (for its replica) from the successor; the
// shadow's promoted copy becomes a replica again; normal plans resume.
bb_status rt_rejoin(Ctx &c) {
  try {
    if (c.fatal) return BB_E_FATAL;
    if (!c.failover || c.interrupted) throw RtError{BB_E_STATE, "rejoin needs a recovered failover pipeline"};
    if (c.failstop) throw RtError{BB_E_UNSUPPORTED, "fail-stop mode: the lost process is gone"};
    CK(cudaSetDevice(c.o.device));
    c.x.barrier();
    // the most recent victim returns first (LIFO): the plans and topology
    // go back to those in force before its preemption
    const int P = c.d.P, v = c.victims.back(), u = ring_prev(P, v), w = ring_next(P, v);
    const int sv = v % P, sw = w % P;   // stages of the returning node and its successor
    auto parts = [&](Copy &cp) {
      return std::vector<float *>{cp.master, cp.m, cp.v};
    };
    // senders
    for (auto pr : std::vector<std::pair<int, int>>{{u, sv}, {w, sw}}) {
      const int from = pr.first, X = pr.second;
      if (!c.nodes.count(from)) continue;
      Node &src = c.nodes.at(from);
      Copy &cp = src.copies.at(X);
      const size_t n = c.stages[X].pcount;
      if (is_local(c, v)) {
        Copy &dc = c.nodes.at(v).copies.at(X);
        auto sp = parts(cp), dp = parts(dc);
        for (int i = 0; i < 3; ++i)
          CK(cudaMemcpyAsync(dp[i], sp[i], n * 4, cudaMemcpyDeviceToDevice, src.main));
      } else {
        XEdge &e = xedge(c, from, v, MSG_STATE);
        const int slot = (int)(e.sent % (uint64_t)e.cap);
        char *dst = e.peer_base + e.recv_off + (size_t)slot * e.slot_bytes;
        wait_ev(e.stream, record(src, src.main));
        auto sp = parts(cp);
        for (int i = 0; i < 3; ++i)
          CK(cudaMemcpyAsync(dst + (size_t)i * n * 4, sp[i], n * 4, cudaMemcpyDeviceToDevice, e.stream));
        CK(c.x.post(e));
      }
    }
    sync_all(c, true);
    // the returning node
    if (c.nodes.count(v)) {
      Node &nd = c.nodes.at(v);
      for (auto pr : std::vector<std::pair<int, int>>{{u, sv}, {w, sw}}) {
        const int from = pr.first, X = pr.second;
        Copy &dc = nd.copies.at(X);
        const size_t n = c.stages[X].pcount;
        if (!is_local(c, from)) {
          XEdge &e = xedge(c, from, v, MSG_STATE);
          const double t0 = now_ms();
          while (!c.x.available(e)) {
            if (now_ms() - t0 > 300000.0) throw RtError{BB_E_STATE, "rejoin: state never arrived"};
            std::this_thread::yield();
          }
          const int slot = (int)(e.consumed % (uint64_t)e.cap);
          c.x.consume(e);
          const char *src = c.x.arena + e.recv_off + (size_t)slot * e.slot_bytes;
          wait_ev(nd.main, c.x.wait_event(e, slot));
          auto dp = parts(dc);
          for (int i = 0; i < 3; ++i)
            CK(cudaMemcpyAsync(dp[i], src + (size_t)i * n * 4, n * 4, cudaMemcpyDeviceToDevice, nd.main));
        }
        if (c.bf16) CK(k::cast_f32_to_bf16(n, dc.master, dc.work, nd.main));
        CK(cudaMemsetAsync(dc.grad, 0, n * 4, nd.main));
        dc.t = (int)c.adam_steps;   // every stage took one Adam step per step since load
        dc.replica = X != sv;
      }
      nd.alive = true;
    }
    if (c.nodes.count(u)) {
      // the shadow's copy is a replica again: back to its retention pool
      Copy &cp = c.nodes.at(u).copies.at(sv);
      cp.replica = true;
      const bool scr = cp.scratch != nullptr;
      free_slots_all(cp);
      reset_pool(c, cp, scr);
    }
    if (c.nodes.count(v))   // pools the returning node gave up under memory pressure
      for (auto &cc : c.nodes.at(v).copies)
        if (cc.second.chunks.empty()) reset_pool(c, cc.second, cc.second.replica && c.o.rc != BB_RC_LFLB && cc.second.retain < c.d.M);
    sync_all(c, true);
    c.plans = c.history.back().plans;
    c.topo = c.history.back().topo;
    c.history.pop_back();
    c.victims.pop_back();
    c.failover = !c.victims.empty();
    return BB_OK;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

bb_status rt_read_state(Ctx &c, int X, int replica, int what, float *host, size_t n) {
  try {
    if (X < 0 || X >= c.d.D * c.d.P) throw RtError{BB_E_INVAL, "bad stage"};
    // X < P: the lowest pipeline whose copy this process hosts (D > 1: the
    // copies of a stage are identical across pipelines, except grads = the
    // local sums); X = d*P + s: pipeline d's copy of stage s
    const int p0 = X < c.d.P ? 0 : X / c.d.P, p1 = X < c.d.P ? c.d.D : p0 + 1;
    X %= c.d.P;
    int node = -1;
    for (int p = p0; p < p1 && node < 0; ++p) {
      const int g = p * c.d.P + X;
      const int nn = replica ? c.topo.replica_on[g] : c.topo.host[g];
      if (nn >= 0 && c.nodes.count(nn) && c.nodes.at(nn).alive) node = nn;
    }
    if (node < 0) throw RtError{BB_E_INVAL, "copy not hosted by this process"};
    Copy &cp = c.nodes.at(node).copies.at(X);
    if (n != c.stages[X].pcount) throw RtError{BB_E_INVAL, "size mismatch"};
    const float *src = what == BB_STATE_PARAMS ? cp.master
                       : what == BB_STATE_GRADS ? cp.grad
                       : what == BB_STATE_ADAM_M ? cp.m
                       : what == BB_STATE_ADAM_V ? cp.v : nullptr;
    if (!src) throw RtError{BB_E_INVAL, "bad state kind"};
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(host, src, n * 4, cudaMemcpyDeviceToHost));
    return BB_OK;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

bb_status rt_write_state(Ctx &c, int X, int what, const float *host, size_t n) {
  try {
    if (X < 0 || X >= c.d.P) throw RtError{BB_E_INVAL, "bad stage"};
    if (n != c.stages[X].pcount) throw RtError{BB_E_INVAL, "size mismatch"};
    if (what != BB_STATE_PARAMS && what != BB_STATE_ADAM_M && what != BB_STATE_ADAM_V)
      throw RtError{BB_E_INVAL, "writable: params, adam_m, adam_v"};
    CK(cudaSetDevice(c.o.device));
    CK(cudaDeviceSynchronize());
    for (auto &kv : c.nodes) {
      Node &nd = kv.second;
      if (!nd.alive || !nd.copies.count(X)) continue;
      Copy &cp = nd.copies.at(X);
      float *dst = what == BB_STATE_PARAMS ? cp.master : what == BB_STATE_ADAM_M ? cp.m : cp.v;
      CK(cudaMemcpyAsync(dst, host, n * 4, cudaMemcpyHostToDevice, nd.main));   // stream-ordered
      if (what == BB_STATE_PARAMS && c.bf16) CK(k::cast_f32_to_bf16(n, cp.master, cp.work, nd.main));
      CK(cudaStreamSynchronize(nd.main));   // host buffer borrowed for this call only
    }
    CK(cudaDeviceSynchronize());
    return BB_OK;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

namespace {
// Total length of the union of [a, b) intervals.
double union_len(std::vector<std::pair<double, double>> v) {
  std::sort(v.begin(), v.end());
  double tot = 0, lo = -1e300, hi = -1e300;
  for (auto &x : v) {
    if (x.first > hi) {
      if (hi > lo) tot += hi - lo;
      lo = x.first;
      hi = x.second;
    } else {
      hi = std::max(hi, x.second);
    }
  }
  if (hi > lo) tot += hi - lo;
  return tot;
}
}  // namespace

bb_status rt_node_stats(Ctx &c, bb_node_stat *out, int cap, int *n) {
  try {
    if (!c.o.timing) throw RtError{BB_E_STATE, "opts.timing is off"};
    int cnt = 0;
    for (auto &kv : c.nodes) {
      Node &nd = kv.second;
      if (!nd.alive) continue;
      CK(cudaEventSynchronize(nd.t1));
      bb_node_stat r{};
      r.node = nd.n;
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, nd.t0, nd.t1));
      r.step_ms = ms;
      std::vector<std::pair<double, double>> mainv, frcv, both;
      for (auto &t : nd.trec) {
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, nd.t0, t.a));
        CK(cudaEventElapsedTime(&b, nd.t0, t.b));
        (t.kind == 1 ? frcv : mainv).push_back({a, b});
        (t.kind == 1 ? r.n_frc : t.kind == 2 ? r.n_bwd : r.n_fwd) += 1;
      }
      r.busy_ms = (float)union_len(mainv);
      r.bubble_ms = r.step_ms - r.busy_ms;
      r.frc_ms = (float)union_len(frcv);
      both = mainv;
      both.insert(both.end(), frcv.begin(), frcv.end());
      // FRC inside main-stream idle time = |main U frc| - |main|
      r.frc_hidden_ms = (float)(union_len(both) - r.busy_ms);
      if (cnt < cap && out) out[cnt] = r;
      ++cnt;
    }
    if (n) *n = cnt;
    return BB_OK;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

std::string rt_dump(const Ctx &c) {
  return dump(c.d.P, c.d.M, (int)c.o.rc, c.ranges, c.plans, c.topo, c.node_device,
              c.failover, c.victims);
}

bb_status rt_kernel_stats(Ctx &c, bb_kernel_stat *out, int cap, int *n) {
  try {
    std::vector<bb_kernel_stat> acc(PC_N);
    for (int i = 0; i < PC_N; ++i) {
      std::memset(&acc[i], 0, sizeof(bb_kernel_stat));
      std::strncpy(acc[i].name, prof_names[i], sizeof(acc[i].name) - 1);
    }
    for (auto &r : c.prof) {
      float ms = 0.f;
      CK(cudaEventSynchronize(r.b));
      CK(cudaEventElapsedTime(&ms, r.a, r.b));
      acc[r.cls].launches += 1;
      acc[r.cls].ms += ms;
      acc[r.cls].work += r.work;
    }
    if (n) *n = PC_N;
    for (int i = 0; i < PC_N && i < cap; ++i) out[i] = acc[i];
    return BB_OK;
  } catch (const RtError &e) {
    c.err = e.msg;
    return e.st;
  }
}

void rt_destroy(Ctx &c) {
  c.hb_stop = true;
  if (c.hb_thread.joinable()) c.hb_thread.join();
  if (c.self_dead && c.x.shm) {
    // a silent victim keeps its memory mapped until every survivor finished
    // the recovery that may still write into it (bounded wait)
    const double t0 = now_ms();
    for (;;) {
      bool all = true;
      for (int r = 0; r < c.o.world_size; ++r)
        if (r != c.o.world_rank && !*c.x.rank_word(3, r) && !c.x.dead(r)) all = false;
      if (all || now_ms() - t0 > 120000.0) break;
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
  }
  cudaDeviceSynchronize();
  xport_destroy(c.x);
  for (auto &kv : c.nodes) {
    Node &nd = kv.second;
    for (auto &cc : nd.copies) {
      Copy &cp = cc.second;
      cudaFree(cp.master);
      cudaFree(cp.m);
      cudaFree(cp.v);
      cudaFree(cp.grad);
      if (c.bf16) cudaFree(cp.work);
      free_slots_all(cp);
      if (cp.loss) cudaFree(cp.loss);
      cudaFree(cp.arsum);
      for (auto p : cp.ar_in) cudaFree(p);
      if (cp.hbase) cudaFreeHost(cp.hbase);
    }
    cudaFree(nd.arena);
    for (auto &sc : nd.sc) {
      if (!sc.sF) continue;
      cudaFree(sc.sF);
      cudaFree(sc.s3);
      for (auto p : sc.sH) cudaFree(p);
      for (auto p : sc.s32) cudaFree(p);
      cudaFree(sc.s_part);
      cudaFree(sc.s_attn);
    }
    cudaFree(nd.s_loss_main);
    cudaFree(nd.s_loss_frc);
    cudaFree(nd.d_tok);
    cudaFree(nd.d_tgt);
    cudaFree(nd.d_csr);
    for (auto e : nd.evpool) cudaEventDestroy(e);
    cudaEventDestroy(nd.t0);
    cudaEventDestroy(nd.t1);
    cudaEventDestroy(nd.ev_begin);
    if (!c.serial) {
      cudaStreamDestroy(nd.main);
      cudaStreamDestroy(nd.frc);
    }
    if (nd.swap) cudaStreamDestroy(nd.swap);
  }
  for (auto e : c.prof_pool) cudaEventDestroy(e);
  if (c.serial) cudaStreamDestroy(c.serial);
  if (c.h_tok) cudaFreeHost(c.h_tok);
  if (c.h_tgt) cudaFreeHost(c.h_tgt);
}

}  // namespace bb
