// Device executor for a compiled 1F1B-RR program (include/pd_b200.h, "executor").
//
// Takes over the reference's discrete-event engine (simulator.py:150-357): instead of
// advancing simulated clocks, each hosted worker (stage replica) owns a CUDA stream and every
// program item (one forward / backward / replica-reduce of one minibatch) becomes that
// worker's kernel chain on the stream.  Readiness (_try_start's ready[] gate,
// simulator.py:255-260) becomes a cudaStreamWaitEvent on the producing item when the
// neighbour lives in this process, or a device-side acquire-poll on the receiver-owned inbox
// flag when it lives in another.  Version selection and commits are resolved ahead of time
// into ring slots (PD_IT_WSLOT / PD_IT_WNEW): the wgrad epilogue (or, for a replicated stage,
// the fused allreduce+SGD kernel) writes the committed version into its slot (simulator.py:315).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "pd_internal.h"

namespace {

using namespace pd;

// Byte layout of a transformer layer's per-minibatch `save` slot and shared `work` scratch.
struct TLayout {
  int64_t T = 0;
  int d = 0, f = 0, H = 0;
  // save (bf16 element offsets, then fp32 float offsets from f32_base)
  int64_t h1 = 0, qkv = 0, a = 0, x2 = 0, h2 = 0, z = 0, u = 0;
  int64_t f32_base = 0;  // bytes
  int64_t lse = 0, mean1 = 0, rstd1 = 0, mean2 = 0, rstd2 = 0;
  int64_t save_bytes = 0;
  // work (bf16 element offsets, fp32 after w32_base)
  int64_t dz1 = 0, dh = 0, dx2 = 0, da = 0, dqkv = 0;
  int64_t w32_base = 0, dq_acc = 0, dvec = 0;
  int64_t work_bytes = 0;
};

inline int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

TLayout tlayout(const pd_layer& y, int batch) {
  TLayout L;
  L.T = (int64_t)batch * y.h;
  L.d = y.kind == PD_LAYER_EMBED ? y.c_out : y.c_in;
  L.f = y.ffn;
  L.H = y.w;
  const int64_t T = L.T, d = L.d, f = L.f;
  if (y.kind == PD_LAYER_BLOCK) {
    int64_t o = 0;
    L.h1 = o; o += T * d;
    L.qkv = o; o += 3 * T * d;
    L.a = o; o += T * d;
    L.x2 = o; o += T * d;
    L.h2 = o; o += T * d;
    L.z = o; o += T * f;
    L.u = o; o += T * f;
    L.f32_base = align256(o * 2);
    int64_t q = 0;
    L.lse = q; q += T * L.H;
    L.mean1 = q; q += T;
    L.rstd1 = q; q += T;
    L.mean2 = q; q += T;
    L.rstd2 = q; q += T;
    L.save_bytes = L.f32_base + q * 4;
    o = 0;
    L.dz1 = o; o += T * f;
    L.dh = o; o += T * d;
    L.dx2 = o; o += T * d;
    L.da = o; o += T * d;
    L.dqkv = o; o += 3 * T * d;
    L.w32_base = align256(o * 2);
    q = 0;
    L.dq_acc = q; q += T * d;
    L.dvec = q; q += T * L.H;
    L.work_bytes = L.w32_base + q * 4;
  } else if (y.kind == PD_LAYER_HEAD) {
    L.h1 = 0;
    L.f32_base = align256(T * d * 2);
    L.mean1 = 0;
    L.rstd1 = T;
    L.save_bytes = L.f32_base + 2 * T * 4;
    L.dh = 0;
    L.work_bytes = T * d * 2;
  }
  return L;
}

struct Layer {
  pd_layer d{};
  std::vector<uint8_t*> argmax;
  std::vector<void*> cols;
  std::vector<void*> save;
  TLayout t;
};

struct Stage {
  pd_stage_desc d{};
  std::vector<Layer> layers;  // empty: MLP stage
  std::vector<int64_t> dims;
  std::vector<float*> w_master, b_master, b_ring, red_grad, red_bgrad;
  std::vector<void*> w_ring, act, act_in, grad_in, dz_last;
  std::vector<const float*> target;
  std::vector<float*> bpart, grad_bpart, dz_bpart;  // fused bias gradient partials (d.fused_bias)
  cudaStream_t stream = nullptr;
  cudaStream_t rstream = nullptr;      // rep > 1: the sharded reduction runs here, under the backward
  cudaEvent_t ev_red = nullptr;        // rep > 1: this round's reduction finished (joined by REDUCE)
  std::vector<cudaEvent_t> ev_layer;   // rep > 1: layer l's gradient is complete (fork to rstream)
  std::vector<cudaEvent_t> ev_upd;     // rep > 1: this replica's layer-l shard is reduced and applied
  int issued_round = 0;                // rep > 1: last round whose reduction has been enqueued
  cudaEvent_t ev_done = nullptr;
  bool fused_signal = false;
  int tag_index = 0;           // this worker's 64-slot block in rt->tags
  int64_t out_bytes = 0;       // forward payload per minibatch (the next stage's input)
  int64_t in_bytes = 0;        // backward payload per minibatch (the previous stage's output gradient)
  bool replicas_local = true;  // rep > 1: every replica of this stage is hosted by this process
  int last_round = 0;          // rep > 1: final allreduce round of the loaded program  // this item's hand-off flag was released by the producing GEMM
};

struct View {
  pd_worker_view v{};
  std::vector<void*> act_in, grad_in;
  std::vector<float*> red_grad, red_bgrad, grad_bpart, w_master, b_master;
};

template <typename T>
std::vector<T> copy_arr(const T* p, int64_t n) {
  return p && n > 0 ? std::vector<T>(p, p + n) : std::vector<T>();
}

}  // namespace

struct pd_runtime {
  int device = 0;
  int epoch = 0;
  std::map<int, Stage> stages;  // hosted workers
  std::map<int, View> views;    // every worker of the plan
  std::vector<int32_t> items;
  std::vector<cudaEvent_t> ev_start, ev_end;
  cudaEvent_t ev0 = nullptr;
  bool traced = false;
  // kernel accounting: launches of our kernels, and optional per-GEMM event timing by class
  int64_t launches = 0;
  bool serial = false;             // all hosted workers on one stream (single-GPU timing mode)
  // CUDA graph of one whole run (single-process programs): captured on the first eligible run,
  // replayed afterwards so the host enqueues one graph instead of thousands of kernels.
  bool graph_mode = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t graph_stream = nullptr;
  int64_t graph_launches = 0;
  cudaStream_t shared = nullptr;
  // end-of-run drain: (worker, peer ack flag, final occupant) of every outbox slot in another
  // process, so the next run cannot overwrite a slot the peer still reads
  struct Drain { int worker; int* flag; int mb; };
  std::vector<Drain> drain;
  bool ltiming = false;  // per-layer fwd / bwd %globaltimer stamps (the layer profiler)
  struct LT { int worker, layer, dir; };
  std::vector<LT> lt;
  size_t lt_used = 0;
  uint64_t* ts = nullptr;  // caller-owned device buffer [2 * ts_cap]
  int ts_cap = 0;
  // device pass records (traced runs, pd_rt_set_records): caller-owned int64 [PD_REC_WIDTH x
  // (1 + items)] (row 0: run-start %globaltimer) and int32 ring-slot version tags [64 per worker]
  int64_t* rec = nullptr;
  int rec_cap = 0;
  int* tags = nullptr;
  int64_t* cur_rec = nullptr;  // record of the item being enqueued (traced runs)
  bool ktiming = false;
  struct KT { int cls; int worker; double flops; cudaEvent_t a, b; };
  int cur_worker = -1;  // worker of the item being enqueued (per-stage kernel statistics)
  std::vector<KT> kt;
  size_t kt_used = 0;
};

static void drop_graph(pd_runtime* rt) {
  if (rt->graph_exec) cudaGraphExecDestroy(rt->graph_exec);
  if (rt->graph) cudaGraphDestroy(rt->graph);
  rt->graph_exec = nullptr;
  rt->graph = nullptr;
}

namespace {

#define PD_CHECK(x)                                                                               \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) return set_error(PD_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)
#define PD_TRY(x)          \
  do {                     \
    int rc_ = (x);         \
    if (rc_) return rc_;   \
  } while (0)

// Flag value of minibatch / round v in run `epoch`: monotone modulo 2^32 (waits compare with a
// wrap-safe signed difference, ptx.cuh flag_before); v < 65536 is enforced by the host.
inline int flag_val(int epoch, int v) { return (int)((uint32_t)epoch * 65536u + (uint32_t)v); }

// Kernel-time classes (pd_rt_kernel_stats): the three GEMM passes, then the non-GEMM kernels.
enum { KC_FWD = 0, KC_DGRAD = 1, KC_WGRAD = 2, KC_ATTN = 3, KC_NORM = 4, KC_LOSS = 5, KC_UPDATE = 6, KC_OTHER = 7,
       KC_N = 8 };

inline cudaStream_t stream_of(pd_runtime* rt, Stage& S) { return rt->serial ? rt->shared : S.stream; }

int timed_gemm(pd_runtime* rt, int cls, int dtype, const void* A, int a_mn, int64_t lda, const void* B, int b_mn,
               int64_t ldb, int M, int N, int K, int kind, const EpiArgs& ep, cudaStream_t st) {
  pd_runtime::KT* slot = nullptr;
  if (rt->ktiming) {
    if (rt->kt_used == rt->kt.size()) {
      pd_runtime::KT k{};
      PD_CHECK(cudaEventCreate(&k.a));
      PD_CHECK(cudaEventCreate(&k.b));
      rt->kt.push_back(k);
    }
    slot = &rt->kt[rt->kt_used++];
    slot->cls = cls;
    slot->worker = rt->cur_worker;
    slot->flops = 2.0 * (double)M * (double)N * (double)K;
    PD_CHECK(cudaEventRecord(slot->a, st));
    g_pre_launch = slot->a;  // re-recorded right before the launch (pd_internal.h)
  }
  const int rc = gemm(dtype, A, a_mn, lda, B, b_mn, ldb, M, N, K, kind, ep, st);
  g_pre_launch = nullptr;
  PD_TRY(rc);
  rt->launches += 1;
  if (slot) PD_CHECK(cudaEventRecord(slot->b, st));
  return 0;
}

// Parameter sizes of layer l (MLP: dims; layered: per kind).
int64_t w_numel(const Stage& S, int l) {
  if (S.layers.empty()) return S.dims[l] * S.dims[l + 1];
  const pd_layer& y = S.layers[l].d;
  if (y.kind == PD_LAYER_LINEAR) return (int64_t)y.c_in * y.c_out;
  if (y.kind == PD_LAYER_EMBED) return (int64_t)(y.c_in + y.h) * y.c_out;
  if (y.kind == PD_LAYER_BLOCK) return (4ll * y.c_in + 2ll * y.ffn) * y.c_in;
  if (y.kind == PD_LAYER_HEAD) return (int64_t)y.c_out * y.c_in;
  return (int64_t)(y.im2col ? 64 : 9 * y.c_in) * y.c_out;
}
int64_t b_numel(const Stage& S, int l) {
  if (S.layers.empty()) return S.dims[l + 1];
  const pd_layer& y = S.layers[l].d;
  if (y.kind == PD_LAYER_EMBED) return 0;
  if (y.kind == PD_LAYER_BLOCK) return 9ll * y.c_in + y.ffn;
  if (y.kind == PD_LAYER_HEAD) return 2ll * y.c_in;
  return y.c_out;
}

// CUDA events around one non-GEMM kernel call on its stream when kernel timing is on.
template <class Fn>
int timed_call(pd_runtime* rt, int cls, cudaStream_t st, Fn&& fn) {
  pd_runtime::KT* slot = nullptr;
  if (rt->ktiming) {
    if (rt->kt_used == rt->kt.size()) {
      pd_runtime::KT k{};
      PD_CHECK(cudaEventCreate(&k.a));
      PD_CHECK(cudaEventCreate(&k.b));
      rt->kt.push_back(k);
    }
    slot = &rt->kt[rt->kt_used++];
    slot->cls = cls;
    slot->worker = rt->cur_worker;
    slot->flops = 0.0;
    PD_CHECK(cudaEventRecord(slot->a, st));
    g_pre_launch = slot->a;  // re-recorded right before the launch (pd_internal.h)
  }
  const int rc = fn();
  g_pre_launch = nullptr;
  if (slot) PD_CHECK(cudaEventRecord(slot->b, st));
  return rc;
}

int wait_flag(pd_runtime* rt, Stage& S, const int* flag, int value) {
  PD_TRY(flag_wait(flag, flag_val(rt->epoch, value), S.d.err_word, stream_of(rt, S)));
  rt->launches += 1;
  return 0;
}
int signal_flag(pd_runtime* rt, Stage& S, int* flag, int value) {
  PD_TRY(flag_signal(flag, flag_val(rt->epoch, value), stream_of(rt, S)));
  rt->launches += 1;
  return 0;
}

// %globaltimer stamps around one layer's pass (fwd dir 0 / bwd dir 1) while layer timing is on:
// tiny kernels on the stage stream, so they also work inside a replayed CUDA graph (the host
// enqueue rate then never starves the timed kernels).  The end stamp is written when the object
// leaves scope (end of the layer's loop iteration).
struct LayerTimer {
  cudaStream_t st = nullptr;
  uint64_t* end = nullptr;
  LayerTimer(pd_runtime* rt, int worker, int layer, int dir, cudaStream_t stream) : st(stream) {
    if (!rt->ltiming || (int)rt->lt_used >= rt->ts_cap) return;
    const size_t i = rt->lt_used++;
    if (i == rt->lt.size()) rt->lt.push_back({});
    rt->lt[i] = {worker, layer, dir};
    timestamp(rt->ts + 2 * i, stream);
    end = rt->ts + 2 * i + 1;
  }
  ~LayerTimer() {
    if (end) timestamp(end, st);
  }
};

// Compute + hand-off fusion: the GEMM whose epilogue stores a stage's payload into a remote
// inbox also releases the receiver's inbox flag from its last CTA (EpiArgs::sig_flag), so no
// separate signal kernel trails the GEMM and the receiver can start as soon as the stores land.
// tcgen05 (bf16) path only; PD_FUSED_HANDOFF=0 falls back to the stand-alone signal kernel.
bool fused_handoff_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PD_FUSED_HANDOFF");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}
void fuse_handoff(pd_runtime* rt, Stage& S, EpiArgs& ep, int* flag, int mb, int counter) {
  if (!flag || S.d.dtype != PD_BF16 || !S.d.sync || !fused_handoff_enabled()) return;
  ep.sig_flag = flag;
  ep.sig_value = flag_val(rt->epoch, mb);
  ep.sig_counter = S.d.sync + counter;
  ep.sig_bytes = rt->cur_rec ? reinterpret_cast<unsigned long long*>(rt->cur_rec + 4) : nullptr;
  S.fused_signal = true;
}

// Replicated stage: before writing round `round`'s parity gradient buffers, every replica's
// reduction that last read them must be done - round-2 of this run, or (rounds 1 and 2, replicas
// in other processes) the final rounds of the previous run, whose flag values are smaller.
// In-process replica sets reset their flags at the start of each run (run_body), so their
// first two rounds have nothing to wait for.
int wait_parity_free(pd_runtime* rt, Stage& S, int round) {
  const pd_stage_desc& d = S.d;
  if (round >= 3) {
    for (int r = 0; r < d.rep; ++r)
      PD_TRY(flag_wait(rt->views.at(d.first_worker + r).v.red_done, flag_val(rt->epoch, round - 2), d.err_word,
                       stream_of(rt, S)));
    rt->launches += d.rep;
  } else if (!S.replicas_local && rt->epoch > 1 && S.last_round > 0) {
    for (int r = 0; r < d.rep; ++r)
      PD_TRY(flag_wait(rt->views.at(d.first_worker + r).v.red_done, flag_val(rt->epoch - 1, S.last_round),
                       d.err_word, stream_of(rt, S)));
    rt->launches += d.rep;
  }
  return 0;
}

// Sharded reduction of a replicated stage.  The backward marks each layer's
// gradient complete (layer_grad_ready: an event, plus the red_lready flag when some replica lives
// in another process).  The round's first REDUCE item then enqueues, for every replica hosted
// here, on its reduction stream: per layer (deepest first) wait for every replica's layer-l
// gradient, reduce-scatter + SGD of the shard it owns (ev_upd / red_lupd), and after all layers
// the all-gather of the other owners' updated shards; red_done and ev_red close the round, and
// each replica's REDUCE item joins ev_red into its stage stream.  On the device a layer's
// reduction starts as soon as the last replica's layer-l gradient exists, under that replica's
// remaining backward.  It is enqueued only once every replica's backward of the round has been
// enqueued (the REDUCE items follow all of them in the issue order), so no wait is ever submitted
// ahead of its producer: in-process waits are events, cross-process waits are flag polls.
// Serial mode (one stream for all workers) cannot overlap replicas: it keeps the whole-tensor
// reduction (run_reduce), which computes the same sums in the same order.
bool sharded_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PD_SHARDED_REDUCE");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}
bool sharded_reduce(const pd_runtime* rt, const Stage& S) {
  return S.d.rep > 1 && !rt->serial && S.rstream && S.d.red_lready && S.d.red_lupd && sharded_enabled();
}

int layer_grad_ready(pd_runtime* rt, Stage& S, int l, int round, cudaStream_t ST) {
  PD_CHECK(cudaEventRecord(S.ev_layer[l], ST));
  if (!S.replicas_local) {
    PD_TRY(flag_signal(S.d.red_lready + l, flag_val(rt->epoch, round), ST));
    rt->launches += 1;
  }
  return 0;
}

int issue_round_reduce(pd_runtime* rt, Stage& S0, int round, int wnew) {
  const pd_stage_desc& d0 = S0.d;
  const int val = flag_val(rt->epoch, round), par = round & 1, L = d0.n_layers;
  std::vector<Stage*> local;
  for (int r = 0; r < d0.rep; ++r) {
    auto f = rt->stages.find(d0.first_worker + r);
    if (f != rt->stages.end()) local.push_back(&f->second);
  }
  auto peer_wait = [&](cudaStream_t R, int q, int l, bool upd) -> int {
    auto f = rt->stages.find(d0.first_worker + q);
    if (f != rt->stages.end()) {
      PD_CHECK(cudaStreamWaitEvent(R, upd ? f->second.ev_upd[l] : f->second.ev_layer[l], 0));
      return 0;
    }
    const View& V = rt->views.at(d0.first_worker + q);
    rt->launches += 1;
    return flag_wait((upd ? V.v.red_lupd : V.v.red_lready) + l, val, S0.d.err_word, R);
  };
  unsigned long long* ctr = rt->traced && rt->rec ? reinterpret_cast<unsigned long long*>(rt->rec + 1) : nullptr;
  std::vector<const float*> g(d0.rep), gb(d0.rep), m(d0.rep), mb(d0.rep);
  for (Stage* Sp : local) {  // pass 1: reduce-scatter + SGD of each local replica's own shard
    Stage& S = *Sp;
    const pd_stage_desc& d = S.d;
    S.issued_round = round;
    cudaStream_t R = S.rstream;
    for (int l = L - 1; l >= 0; --l) {
      for (int q = 0; q < d.rep; ++q) {
        PD_TRY(peer_wait(R, q, l, false));
        const View& V = rt->views.at(d.first_worker + q);
        g[q] = V.red_grad[(size_t)l * 2 + par];
        gb[q] = V.red_bgrad[(size_t)l * 2 + par];
      }
      const int64_t nw = w_numel(S, l), nb = b_numel(S, l);
      PD_TRY(shard_rs_sgd(d.dtype, g.data(), d.rep, d.replica, S.w_master[l], S.w_ring[(size_t)l * d.ring_depth + wnew],
                          nw, d.lr, ctr, R));
      if (nb > 0)
        PD_TRY(shard_rs_sgd(PD_F32, gb.data(), d.rep, d.replica, S.b_master[l], S.b_ring[(size_t)l * d.ring_depth + wnew],
                            nb, d.lr, ctr, R));
      PD_CHECK(cudaEventRecord(S.ev_upd[l], R));
      if (!S.replicas_local) PD_TRY(flag_signal(d.red_lupd + l, val, R));
      rt->launches += 1 + (nb > 0) + (!S.replicas_local);
    }
  }
  for (Stage* Sp : local) {  // pass 2: all-gather the other owners' updated shards
    Stage& S = *Sp;
    const pd_stage_desc& d = S.d;
    cudaStream_t R = S.rstream;
    for (int l = L - 1; l >= 0; --l) {
      for (int q = 0; q < d.rep; ++q) {
        if (q != d.replica) PD_TRY(peer_wait(R, q, l, true));
        const View& V = rt->views.at(d.first_worker + q);
        m[q] = V.w_master[l];
        mb[q] = V.b_master[l];
      }
      const int64_t nw = w_numel(S, l), nb = b_numel(S, l);
      PD_TRY(shard_ag(d.dtype, m.data(), d.rep, d.replica, S.w_master[l], S.w_ring[(size_t)l * d.ring_depth + wnew], nw,
                      ctr, R));
      if (nb > 0)
        PD_TRY(shard_ag(PD_F32, mb.data(), d.rep, d.replica, S.b_master[l], S.b_ring[(size_t)l * d.ring_depth + wnew], nb,
                        ctr, R));
      rt->launches += 1 + (nb > 0);
    }
    PD_TRY(flag_signal(d.red_done, val, R));
    PD_CHECK(cudaEventRecord(S.ev_red, R));
    rt->launches += 1;
  }
  return 0;
}

int run_forward(pd_runtime* rt, Stage& S, const int32_t* it) {
  cudaStream_t ST = stream_of(rt, S);
  const pd_stage_desc& d = S.d;
  const int L = d.n_layers, B = d.batch;
  const int wslot = it[PD_IT_WSLOT], act = it[PD_IT_ACT], mb = it[PD_IT_MB];
  const void* x = d.is_first ? S.act_in[it[PD_IT_BLOCK]] : S.act_in[it[PD_IT_XSLOT]];
  for (int l = 0; l < L; ++l) {
    LayerTimer ltimer(rt, S.d.worker, l, 0, ST);
    const int K = (int)S.dims[l], N = (int)S.dims[l + 1];
    EpiArgs ep{};
    ep.bias = S.b_ring[(size_t)l * d.ring_depth + wslot];
    ep.ldo = N;
    int kind = EPI_STORE;
    if (l < L - 1) {
      ep.out = S.act[(size_t)l * d.act_depth + act];
      ep.relu = 1;
    } else if (d.is_last) {
      kind = EPI_LOSS;
      ep.out = S.dz_last[act];
      ep.target = S.target[it[PD_IT_BLOCK]];
      ep.ldt = N;
      ep.scale = 1.0f / (float)B;
      ep.loss = d.loss + mb;
      if (d.fused_bias) {  // dZ's column-sum partials for this layer's fused bias update
        ep.colsum = S.dz_bpart[act];
        ep.ldc = N;
      }
    } else {
      // the epilogue stores straight into the next stage's inbox slot (peer-mapped if remote)
      const View& V = rt->views.at(it[PD_IT_DST]);
      ep.out = V.act_in[it[PD_IT_OUT]];
      ep.relu = d.relu_last;
      fuse_handoff(rt, S, ep, V.v.remote ? V.v.act_ready + it[PD_IT_OUT] : nullptr, it[PD_IT_MB], 8);
    }
    const void* W = S.w_ring[(size_t)l * d.ring_depth + wslot];
    PD_TRY(timed_gemm(rt, KC_FWD, d.dtype, x, 0, K, W, 0, K, B, N, K, kind, ep, ST));
    x = ep.out;
  }
  return 0;
}

int run_backward(pd_runtime* rt, Stage& S, const int32_t* it) {
  cudaStream_t ST = stream_of(rt, S);
  const pd_stage_desc& d = S.d;
  const int L = d.n_layers, B = d.batch;
  const int wslot = it[PD_IT_WSLOT], wnew = it[PD_IT_WNEW], act = it[PD_IT_ACT], round = it[PD_IT_ROUND];
  const bool replicated = d.rep > 1;
  const int par = round & 1;
  if (replicated) PD_TRY(wait_parity_free(rt, S, round));
  const void* dz = d.is_last ? S.dz_last[act] : S.grad_in[it[PD_IT_GSLOT]];
  for (int l = L - 1; l >= 0; --l) {
    LayerTimer ltimer(rt, S.d.worker, l, 1, ST);
    const int Kin = (int)S.dims[l], Nout = (int)S.dims[l + 1];
    const void* X = (l == 0) ? (d.is_first ? S.act_in[it[PD_IT_BLOCK]] : S.act_in[it[PD_IT_XSLOT]])
                             : S.act[(size_t)(l - 1) * d.act_depth + act];
    const void* Wst = S.w_ring[(size_t)l * d.ring_depth + wslot];
    void* out = nullptr;
    if (!(d.is_first && l == 0)) {
      // dgrad + ReLU-backward: dZ_{l-1} = (dZ_l W_l^{stashed}) * (X_l > 0); the first layer's
      // result goes straight into the previous stage's gradient inbox
      out = (l == 0) ? rt->views.at(it[PD_IT_DST]).grad_in[it[PD_IT_OUT]] : d.tmp[l & 1];
      EpiArgs ep{};
      ep.out = out;
      ep.ldo = Kin;
      ep.mask = X;
      ep.ldm = Kin;
      if (l == 0) {
        const View& V = rt->views.at(it[PD_IT_DST]);
        fuse_handoff(rt, S, ep, V.v.remote ? V.v.grad_ready + it[PD_IT_OUT] : nullptr, it[PD_IT_MB], 9);
        if (V.v.fused_bias) {  // the receiver's bias partials ride along with the gradient
          ep.colsum = V.grad_bpart[it[PD_IT_OUT]];
          ep.ldc = Kin;
        }
      } else if (d.fused_bias) {
        ep.colsum = S.bpart[l - 1];
        ep.ldc = Kin;
      }
      PD_TRY(timed_gemm(rt, KC_DGRAD, d.dtype, dz, 0, Nout, Wst, 1, Kin, B, Kin, Nout, EPI_MASK, ep, ST));
    }
    if (replicated) {
      // this replica's fp32 gradient; the REDUCE item sums all replicas and commits
      EpiArgs ep{};
      ep.out = S.red_grad[(size_t)l * 2 + par];
      ep.ldo = Kin;
      PD_TRY(timed_gemm(rt, KC_WGRAD, d.dtype, dz, 1, Nout, X, 1, Kin, Nout, Kin, B, EPI_GRADF32, ep, ST));
      PD_TRY(timed_call(rt, KC_UPDATE, ST, [&]() { return bias_grad(d.dtype, dz, B, Nout, Nout, S.red_bgrad[(size_t)l * 2 + par], ST); }));
      rt->launches += 1;
      if (sharded_reduce(rt, S)) PD_TRY(layer_grad_ready(rt, S, l, round, ST));
    } else if (wnew >= 0) {
      // wgrad + SGD onto the latest weights, written as version mb into ring slot wnew
      EpiArgs ep{};
      ep.master = S.w_master[l];
      ep.ldw = Kin;
      ep.out = S.w_ring[(size_t)l * d.ring_depth + wnew];
      ep.ldo = Kin;
      ep.lr = d.lr;
      if (d.fused_bias) {
        // the bias update rides in this GEMM's epilogue, from the dZ producer's column sums
        ep.bpart = l < L - 1 ? S.bpart[l] : (d.is_last ? S.dz_bpart[act] : S.grad_bpart[it[PD_IT_GSLOT]]);
        ep.nrb = (B + 31) / 32;
        ep.ldc = Nout;
        ep.bmaster = S.b_master[l];
        ep.bring = S.b_ring[(size_t)l * d.ring_depth + wnew];
      }
      PD_TRY(timed_gemm(rt, KC_WGRAD, d.dtype, dz, 1, Nout, X, 1, Kin, Nout, Kin, B, EPI_SGD, ep, ST));
      if (!d.fused_bias) {
        PD_TRY(timed_call(rt, KC_UPDATE, ST, [&]() { return bias_sgd(d.dtype, dz, B, Nout, Nout, S.b_master[l], S.b_ring[(size_t)l * d.ring_depth + wnew], d.lr,
                        ST); }));
        rt->launches += 1;
      }
    }
    dz = out;
  }
  if (replicated && !sharded_reduce(rt, S)) PD_TRY(signal_flag(rt, S, d.red_ready, round));
  return 0;
}

int timed_conv(pd_runtime* rt, int cls, int pass, const void* act, const void* other, int n, int h, int w, int cin,
               int cout, int kind, const EpiArgs& ep, cudaStream_t st) {
  pd_runtime::KT* slot = nullptr;
  if (rt->ktiming) {
    if (rt->kt_used == rt->kt.size()) {
      pd_runtime::KT k{};
      PD_CHECK(cudaEventCreate(&k.a));
      PD_CHECK(cudaEventCreate(&k.b));
      rt->kt.push_back(k);
    }
    slot = &rt->kt[rt->kt_used++];
    slot->cls = cls;
    slot->worker = rt->cur_worker;
    slot->flops = 2.0 * (double)n * h * w * 9.0 * cin * cout;
    PD_CHECK(cudaEventRecord(slot->a, st));
    g_pre_launch = slot->a;  // re-recorded right before the launch (pd_internal.h)
  }
  const int rc = conv3x3_tc(pass, act, other, n, h, w, cin, cout, kind, ep, st);
  g_pre_launch = nullptr;
  PD_TRY(rc);
  rt->launches += 1;
  if (slot) PD_CHECK(cudaEventRecord(slot->b, st));
  return 0;
}

inline void* bf16_at(void* base, int64_t elems) { return static_cast<__nv_bfloat16*>(base) + elems; }
inline float* f32_at(void* base, int64_t byte_base, int64_t floats) {
  return reinterpret_cast<float*>(static_cast<uint8_t*>(base) + byte_base) + floats;
}

int gemm_t(pd_runtime* rt, int cls, const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M,
           int N, int K, int kind, const EpiArgs& ep, cudaStream_t st) {
  return timed_gemm(rt, cls, PD_BF16, A, a_mn, lda, B, b_mn, ldb, M, N, K, kind, ep, st);
}

// wgrad + SGD of one [M, N] weight matrix inside a flat parameter buffer: dW = A^T B over T rows
// (A = dY [T, M], B = X [T, N], both row-major = MN-major operands).
int wgrad_sgd(pd_runtime* rt, Stage& S, int l, int wnew, int64_t woff, const void* dY, const void* X, int M, int N,
              int64_t T, cudaStream_t st) {
  const pd_stage_desc& d = S.d;
  EpiArgs ep{};
  ep.master = S.w_master[l] + woff;
  ep.ldw = N;
  ep.out = bf16_at(S.w_ring[(size_t)l * d.ring_depth + wnew], woff);
  ep.ldo = N;
  ep.lr = d.lr;
  return gemm_t(rt, KC_WGRAD, dY, 1, M, X, 1, N, M, N, (int)T, EPI_SGD, ep, st);
}

// bias gradient (column sum over T rows) + SGD of a bias slice at boff
int bias_update(pd_runtime* rt, Stage& S, int l, int wnew, int64_t boff, const void* dY, int64_t T, int C,
                cudaStream_t st) {
  const pd_stage_desc& d = S.d;
  rt->launches += 2;
  return bias_grad_tall(dY, T, C, d.part, nullptr, S.b_master[l] + boff,
                        S.b_ring[(size_t)l * d.ring_depth + wnew] + boff, d.lr, st, d.sync);
}

// LayerNorm backward fused with the residual gradient, then the gamma/beta update at goff
int ln_backward(pd_runtime* rt, Stage& S, int l, int wslot, int wnew, int64_t goff, const void* dy, const void* x,
                const float* mean, const float* rstd, const void* dres, void* dx, int64_t T, int D, bool update,
                cudaStream_t st) {
  const pd_stage_desc& d = S.d;
  const float* gb = S.b_ring[(size_t)l * d.ring_depth + wslot] + goff;
  rt->launches += 1;
  // the gamma/beta update is fused: the last block reduces the partials and applies SGD
  return ln_bwd(dy, x, mean, rstd, gb, dres, dx, d.part, T, D, st, update ? d.sync : nullptr,
                update ? S.b_master[l] + goff : nullptr, update ? S.b_ring[(size_t)l * d.ring_depth + wnew] + goff : nullptr,
                d.lr);
}

// Transformer layer forward.  x: layer input (tokens for EMBED), out: layer output [T, d]
// (next layer's stash, or the next stage's inbox slot).
int tfwd(pd_runtime* rt, Stage& S, const Layer& Y, int l, const int32_t* it, const void* x, void* out) {
  cudaStream_t ST = stream_of(rt, S);
  const pd_stage_desc& d = S.d;
  const pd_layer& y = Y.d;
  const int wslot = it[PD_IT_WSLOT], act = it[PD_IT_ACT], mb = it[PD_IT_MB];
  void* W = S.w_ring[(size_t)l * d.ring_depth + wslot];
  const float* b = S.b_ring[(size_t)l * d.ring_depth + wslot];
  const TLayout& L = Y.t;
  const int64_t T = L.T;
  const int D = L.d, F = L.f;
  if (y.kind == PD_LAYER_EMBED) {
    rt->launches += 1;
    return timed_call(rt, KC_OTHER, ST, [&]() { return embed_fwd(static_cast<const int*>(x), W, bf16_at(W, (int64_t)y.c_in * D), out, T, y.h, D, ST); });
  }
  void* sv = Y.save[act];
  if (y.kind == PD_LAYER_HEAD) {
    void* h = bf16_at(sv, 0);
    float* mean = f32_at(sv, L.f32_base, L.mean1);
    float* rstd = f32_at(sv, L.f32_base, L.rstd1);
    PD_TRY(timed_call(rt, KC_NORM, ST, [&]() { return ln_fwd(x, b, h, mean, rstd, T, D, ST); }));
    EpiArgs ep{};
    ep.out = d.logits;
    ep.ldo = y.c_out;
    PD_TRY(gemm_t(rt, KC_FWD, h, 0, D, W, 0, D, (int)T, y.c_out, D, EPI_GRADF32, ep, ST));
    rt->launches += 2;
    return timed_call(rt, KC_LOSS, ST, [&]() { return softmax_ce_v(d.logits, y.c_out, reinterpret_cast<const int*>(S.target[it[PD_IT_BLOCK]]), T, y.vocab, y.c_out,
                        S.dz_last[act], y.c_out, d.loss + mb, ST); });
  }
  // BLOCK (pre-LN): x2 = x + attn(LN1 x) Wo^T + bo ; out = x2 + gelu(LN2 x2 W1^T + b1) W2^T + b2
  const int64_t oWo = 3ll * D * D, oW1 = 4ll * D * D, oW2 = 4ll * D * D + (int64_t)F * D;
  const int64_t obo = 3ll * D, ob1 = 4ll * D, ob2 = 4ll * D + F, oln1 = 5ll * D + F, oln2 = 7ll * D + F;
  void* h1 = bf16_at(sv, L.h1);
  void* qkv = bf16_at(sv, L.qkv);
  void* a = bf16_at(sv, L.a);
  void* x2 = bf16_at(sv, L.x2);
  void* h2 = bf16_at(sv, L.h2);
  void* z = bf16_at(sv, L.z);
  void* u = bf16_at(sv, L.u);
  PD_TRY(timed_call(rt, KC_NORM, ST, [&]() { return ln_fwd(x, b + oln1, h1, f32_at(sv, L.f32_base, L.mean1), f32_at(sv, L.f32_base, L.rstd1), T, D, ST); }));
  EpiArgs ep{};
  ep.out = qkv;
  ep.ldo = 3 * D;
  ep.bias = b;
  PD_TRY(gemm_t(rt, KC_FWD, h1, 0, D, W, 0, D, (int)T, 3 * D, D, EPI_STORE, ep, ST));
  PD_TRY(timed_call(rt, KC_ATTN, ST, [&]() { return attn_fwd(qkv, a, f32_at(sv, L.f32_base, L.lse), (int)(T / y.h), y.h, L.H, ST); }));
  ep = EpiArgs{};
  ep.out = x2;
  ep.ldo = D;
  ep.bias = b + obo;
  ep.mask = x;
  ep.ldm = D;
  PD_TRY(gemm_t(rt, KC_FWD, a, 0, D, bf16_at(W, oWo), 0, D, (int)T, D, D, EPI_RESID, ep, ST));
  PD_TRY(timed_call(rt, KC_NORM, ST, [&]() { return ln_fwd(x2, b + oln2, h2, f32_at(sv, L.f32_base, L.mean2), f32_at(sv, L.f32_base, L.rstd2), T, D, ST); }));
  ep = EpiArgs{};
  ep.out = u;
  ep.aux = z;
  ep.ldo = F;
  ep.bias = b + ob1;
  PD_TRY(gemm_t(rt, KC_FWD, h2, 0, D, bf16_at(W, oW1), 0, D, (int)T, F, D, EPI_GELU, ep, ST));
  ep = EpiArgs{};
  ep.out = out;
  ep.ldo = D;
  ep.bias = b + ob2;
  ep.mask = x2;
  ep.ldm = D;
  PD_TRY(gemm_t(rt, KC_FWD, u, 0, F, bf16_at(W, oW2), 0, F, (int)T, D, F, EPI_RESID, ep, ST));
  rt->launches += 3;
  return 0;
}

// Transformer layer backward.  dout: gradient of the layer output; X: layer input; dst: where the
// input gradient goes (nullptr: none needed).
int tbwd(pd_runtime* rt, Stage& S, const Layer& Y, int l, const int32_t* it, const void* dout, const void* X,
         void* dst) {
  cudaStream_t ST = stream_of(rt, S);
  const pd_stage_desc& d = S.d;
  const pd_layer& y = Y.d;
  const int wslot = it[PD_IT_WSLOT], wnew = it[PD_IT_WNEW], act = it[PD_IT_ACT];
  const bool update = wnew >= 0;
  void* W = S.w_ring[(size_t)l * d.ring_depth + wslot];
  const TLayout& L = Y.t;
  const int64_t T = L.T;
  const int D = L.d, F = L.f;
  if (y.kind == PD_LAYER_EMBED) {
    if (!update) return 0;
    const int64_t n = w_numel(S, l);
    PD_CHECK(cudaMemsetAsync(d.part, 0, sizeof(float) * n, ST));
    PD_TRY(timed_call(rt, KC_UPDATE, ST, [&]() { return embed_bwd(static_cast<const int*>(X), dout, d.part, d.part + (int64_t)y.c_in * D, T, y.h, D, ST); }));
    rt->launches += 2;
    return timed_call(rt, KC_UPDATE, ST, [&]() { return reduce_sgd(PD_BF16, d.part, 1, n, n, nullptr, S.w_master[l], S.w_ring[(size_t)l * d.ring_depth + wnew],
                      d.lr, ST); });
  }
  void* sv = Y.save[act];
  if (y.kind == PD_LAYER_HEAD) {
    void* h = bf16_at(sv, 0);
    void* dh = bf16_at(y.work, L.dh);
    EpiArgs ep{};
    ep.out = dh;
    ep.ldo = D;
    PD_TRY(gemm_t(rt, KC_DGRAD, dout, 0, y.c_out, W, 1, D, (int)T, D, y.c_out, EPI_STORE, ep, ST));
    if (update) PD_TRY(wgrad_sgd(rt, S, l, wnew, 0, dout, h, y.c_out, D, T, ST));
    return ln_backward(rt, S, l, wslot, wnew, 0, dh, X, f32_at(sv, L.f32_base, L.mean1),
                       f32_at(sv, L.f32_base, L.rstd1), nullptr, dst, T, D, update, ST);
  }
  // BLOCK
  const int64_t oWo = 3ll * D * D, oW1 = 4ll * D * D, oW2 = 4ll * D * D + (int64_t)F * D;
  const int64_t obo = 3ll * D, ob1 = 4ll * D, ob2 = 4ll * D + F, oln1 = 5ll * D + F, oln2 = 7ll * D + F;
  void* h1 = bf16_at(sv, L.h1);
  void* qkv = bf16_at(sv, L.qkv);
  void* a = bf16_at(sv, L.a);
  void* x2 = bf16_at(sv, L.x2);
  void* h2 = bf16_at(sv, L.h2);
  void* z = bf16_at(sv, L.z);
  void* u = bf16_at(sv, L.u);
  void* dz1 = bf16_at(y.work, L.dz1);
  void* dh = bf16_at(y.work, L.dh);
  void* dx2 = bf16_at(y.work, L.dx2);
  void* da = bf16_at(y.work, L.da);
  void* dqkv = bf16_at(y.work, L.dqkv);
  // FC2: dz1 = (dout W2) * gelu'(z)
  EpiArgs ep{};
  ep.out = dz1;
  ep.ldo = F;
  ep.mask = z;
  ep.ldm = F;
  PD_TRY(gemm_t(rt, KC_DGRAD, dout, 0, D, bf16_at(W, oW2), 1, F, (int)T, F, D, EPI_GELU_BWD, ep, ST));
  if (update) {
    PD_TRY(wgrad_sgd(rt, S, l, wnew, oW2, dout, u, D, F, T, ST));
    PD_TRY(bias_update(rt, S, l, wnew, ob2, dout, T, D, ST));
  }
  // FC1: dh2 = dz1 W1
  ep = EpiArgs{};
  ep.out = dh;
  ep.ldo = D;
  PD_TRY(gemm_t(rt, KC_DGRAD, dz1, 0, F, bf16_at(W, oW1), 1, D, (int)T, D, F, EPI_STORE, ep, ST));
  if (update) {
    PD_TRY(wgrad_sgd(rt, S, l, wnew, oW1, dz1, h2, F, D, T, ST));
    PD_TRY(bias_update(rt, S, l, wnew, ob1, dz1, T, F, ST));
  }
  // LN2 (+ the residual path): dx2 = dout + LN2'(dh2)
  PD_TRY(ln_backward(rt, S, l, wslot, wnew, oln2, dh, x2, f32_at(sv, L.f32_base, L.mean2),
                     f32_at(sv, L.f32_base, L.rstd2), dout, dx2, T, D, update, ST));
  // out projection: da = dx2 Wo
  ep = EpiArgs{};
  ep.out = da;
  ep.ldo = D;
  PD_TRY(gemm_t(rt, KC_DGRAD, dx2, 0, D, bf16_at(W, oWo), 1, D, (int)T, D, D, EPI_STORE, ep, ST));
  if (update) {
    PD_TRY(wgrad_sgd(rt, S, l, wnew, oWo, dx2, a, D, D, T, ST));
    PD_TRY(bias_update(rt, S, l, wnew, obo, dx2, T, D, ST));
  }
  // attention
  PD_TRY(timed_call(rt, KC_ATTN, ST, [&]() { return attn_bwd(qkv, a, da, f32_at(sv, L.f32_base, L.lse), f32_at(y.work, L.w32_base, L.dvec),
                  f32_at(y.work, L.w32_base, L.dq_acc), dqkv, (int)(T / y.h), y.h, L.H, ST); }));
  rt->launches += 3;
  // QKV: dh1 = dqkv Wqkv
  ep = EpiArgs{};
  ep.out = dh;
  ep.ldo = D;
  PD_TRY(gemm_t(rt, KC_DGRAD, dqkv, 0, 3 * D, W, 1, D, (int)T, D, 3 * D, EPI_STORE, ep, ST));
  if (update) {
    PD_TRY(wgrad_sgd(rt, S, l, wnew, 0, dqkv, h1, 3 * D, D, T, ST));
    PD_TRY(bias_update(rt, S, l, wnew, 0, dqkv, T, 3 * D, ST));
  }
  // LN1 (+ the residual path): dx = dx2 + LN1'(dh1)
  return ln_backward(rt, S, l, wslot, wnew, oln1, dh, X, f32_at(sv, L.f32_base, L.mean1),
                     f32_at(sv, L.f32_base, L.rstd1), dx2, dst, T, D, update, ST);
}

// Layered stage forward (VGG-style): per layer Linear or implicit-GEMM conv (+bias, ReLU fused in
// the epilogue), optional max pool; the stage's last layer writes the next stage's inbox slot,
// or at the model output the loss (MSE epilogue, or fp32 logits + softmax cross-entropy).
int run_forward_layers(pd_runtime* rt, Stage& S, const int32_t* it) {
  cudaStream_t ST = stream_of(rt, S);
  const pd_stage_desc& d = S.d;
  const int L = d.n_layers, B = d.batch;
  const int wslot = it[PD_IT_WSLOT], act = it[PD_IT_ACT], mb = it[PD_IT_MB];
  const void* x = d.is_first ? S.act_in[it[PD_IT_BLOCK]] : S.act_in[it[PD_IT_XSLOT]];
  for (int l = 0; l < L; ++l) {
    LayerTimer ltimer(rt, S.d.worker, l, 0, ST);
    const Layer& Y = S.layers[l];
    const pd_layer& y = Y.d;
    const bool last = l == L - 1;
    void* out = !last ? S.act[(size_t)l * d.act_depth + act]
                      : (d.is_last ? nullptr : rt->views.at(it[PD_IT_DST]).act_in[it[PD_IT_OUT]]);
    const void* W = S.w_ring[(size_t)l * d.ring_depth + wslot];
    const float* bias = S.b_ring[(size_t)l * d.ring_depth + wslot];
    if (y.kind >= PD_LAYER_EMBED) {
      PD_TRY(tfwd(rt, S, Y, l, it, x, out));
      x = out;
      continue;
    }
    EpiArgs ep{};
    ep.bias = bias;
    ep.relu = y.relu;
    if (y.kind == PD_LAYER_LINEAR) {
      ep.ldo = y.c_out;
      int kind = EPI_STORE;
      if (last && d.is_last) {
        if (d.loss_kind == PD_LOSS_CE) {
          kind = EPI_GRADF32;  // fp32 logits (+ bias)
          ep.out = d.logits;
        } else {
          kind = EPI_LOSS;
          ep.out = S.dz_last[act];
          ep.target = S.target[it[PD_IT_BLOCK]];
          ep.ldt = y.c_out;
          ep.scale = 1.0f / (float)B;
          ep.loss = d.loss + mb;
        }
      } else {
        ep.out = out;
      }
      PD_TRY(timed_gemm(rt, KC_FWD, d.dtype, x, 0, y.c_in, W, 0, y.c_in, B, y.c_out, y.c_in, kind, ep, ST));
      if (last && d.is_last && d.loss_kind == PD_LOSS_CE) {
        PD_TRY(timed_call(rt, KC_LOSS, ST, [&]() { return softmax_ce(d.logits, y.c_out, reinterpret_cast<const int*>(S.target[it[PD_IT_BLOCK]]), B, y.c_out,
                          S.dz_last[act], y.c_out, d.loss + mb, ST); }));
        rt->launches += 1;
      }
      x = out;
      continue;
    }
    // CONV3
    if (last && d.is_last) return set_error(PD_ERR_INVALID, "worker %d: a conv layer cannot be the model output", d.worker);
    void* conv_out = y.pool ? d.tmp[0] : out;
    ep.out = conv_out;
    ep.ldo = y.c_out;
    const int pix = B * y.h * y.w;
    if (y.im2col) {
      void* cols = Y.cols[act];
      PD_TRY(timed_call(rt, KC_OTHER, ST, [&]() { return im2col3(x, cols, B, y.h, y.w, y.c_in, 64, ST); }));
      rt->launches += 1;
      PD_TRY(timed_gemm(rt, KC_FWD, d.dtype, cols, 0, 64, W, 1, y.c_out, pix, y.c_out, 64, EPI_STORE, ep, ST));
    } else {
      PD_TRY(timed_conv(rt, KC_FWD, PD_CONV_FWD, x, W, B, y.h, y.w, y.c_in, y.c_out, EPI_STORE, ep, ST));
    }
    if (y.pool) {
      PD_TRY(timed_call(rt, KC_OTHER, ST, [&]() { return maxpool_fwd(conv_out, out, Y.argmax[act], B, y.h, y.w, y.c_out, ST); }));
      rt->launches += 1;
    }
    x = out;
  }
  return 0;
}

int run_backward_layers(pd_runtime* rt, Stage& S, const int32_t* it) {
  cudaStream_t ST = stream_of(rt, S);
  const pd_stage_desc& d = S.d;
  const int L = d.n_layers, B = d.batch;
  const int wslot = it[PD_IT_WSLOT], wnew = it[PD_IT_WNEW], act = it[PD_IT_ACT], round = it[PD_IT_ROUND];
  const bool replicated = d.rep > 1;
  const int par = round & 1;
  if (replicated) PD_TRY(wait_parity_free(rt, S, round));
  const bool update = replicated || wnew >= 0;
  const void* dz = d.is_last ? S.dz_last[act] : S.grad_in[it[PD_IT_GSLOT]];
  auto other_tmp = [&](const void* p) { return p == d.tmp[0] ? d.tmp[1] : d.tmp[0]; };
  for (int l = L - 1; l >= 0; --l) {
    LayerTimer ltimer(rt, S.d.worker, l, 1, ST);
    const Layer& Y = S.layers[l];
    const pd_layer& y = Y.d;
    const void* X = (l == 0) ? (d.is_first ? S.act_in[it[PD_IT_BLOCK]] : S.act_in[it[PD_IT_XSLOT]])
                             : S.act[(size_t)(l - 1) * d.act_depth + act];
    const void* Wst = S.w_ring[(size_t)l * d.ring_depth + wslot];
    const bool need_dx = !(d.is_first && l == 0);
    float* gW = replicated ? S.red_grad[(size_t)l * 2 + par] : nullptr;
    float* gb = replicated ? S.red_bgrad[(size_t)l * 2 + par] : nullptr;
    void* ring_new = (!replicated && wnew >= 0) ? S.w_ring[(size_t)l * d.ring_depth + wnew] : nullptr;
    float* bring_new = (!replicated && wnew >= 0) ? S.b_ring[(size_t)l * d.ring_depth + wnew] : nullptr;
    void* dst = nullptr;
    if (y.kind >= PD_LAYER_EMBED) {
      if (need_dx) dst = (l == 0) ? rt->views.at(it[PD_IT_DST]).grad_in[it[PD_IT_OUT]] : other_tmp(dz);
      PD_TRY(tbwd(rt, S, Y, l, it, dz, X, dst));
      dz = dst;
      continue;
    }
    if (y.kind == PD_LAYER_LINEAR) {
      if (need_dx) {
        dst = (l == 0) ? rt->views.at(it[PD_IT_DST]).grad_in[it[PD_IT_OUT]] : other_tmp(dz);
        EpiArgs ep{};
        ep.out = dst;
        ep.ldo = y.c_in;
        ep.mask = X;
        ep.ldm = y.c_in;
        PD_TRY(timed_gemm(rt, KC_DGRAD, d.dtype, dz, 0, y.c_out, Wst, 1, y.c_in, B, y.c_in, y.c_out, EPI_MASK, ep, ST));
      }
      if (replicated) {
        EpiArgs ep{};
        ep.out = gW;
        ep.ldo = y.c_in;
        PD_TRY(timed_gemm(rt, KC_WGRAD, d.dtype, dz, 1, y.c_out, X, 1, y.c_in, y.c_out, y.c_in, B, EPI_GRADF32, ep, ST));
        PD_TRY(timed_call(rt, KC_UPDATE, ST, [&]() { return bias_grad(d.dtype, dz, B, y.c_out, y.c_out, gb, ST); }));
        rt->launches += 1;
        if (sharded_reduce(rt, S)) PD_TRY(layer_grad_ready(rt, S, l, round, ST));  // after its dgrad
      } else if (update) {
        EpiArgs ep{};
        ep.master = S.w_master[l];
        ep.ldw = y.c_in;
        ep.out = ring_new;
        ep.ldo = y.c_in;
        ep.lr = d.lr;
        PD_TRY(timed_gemm(rt, KC_WGRAD, d.dtype, dz, 1, y.c_out, X, 1, y.c_in, y.c_out, y.c_in, B, EPI_SGD, ep, ST));
        PD_TRY(timed_call(rt, KC_UPDATE, ST, [&]() { return bias_sgd(d.dtype, dz, B, y.c_out, y.c_out, S.b_master[l], bring_new, d.lr, ST); }));
        rt->launches += 1;
      }
      dz = dst;
      continue;
    }
    // CONV3: route the pooled gradient back to the window maxima (dz is already ReLU-masked by
    // the consumer's dgrad epilogue: pooled > 0 <=> the argmax pre-activation > 0)
    const void* dy = dz;
    if (y.pool) {
      void* t = other_tmp(dz);
      PD_TRY(timed_call(rt, KC_OTHER, ST, [&]() { return maxpool_bwd(dz, Y.argmax[act], t, B, y.h, y.w, y.c_out, ST); }));
      rt->launches += 1;
      dy = t;
    }
    const int pix = B * y.h * y.w;
    if (update) {
      // weight gradient: split-K partials into `part`, summed in fixed order by the reduction,
      // which either applies SGD into the new ring slot or hands the sum to the replica reduce
      const int M = y.im2col ? 64 : 9 * y.c_in;
      int splits = 1, per = 0;
      PD_TRY(splitk_plan(M, y.c_out, pix, &splits, &per));
      EpiArgs ep{};
      ep.out = d.part;
      ep.ldo = y.c_out;
      ep.accumulate = 1;  // splits red.add into one zeroed fp32 gradient (no partial round trip)
      PD_CHECK(cudaMemsetAsync(d.part, 0, sizeof(float) * (size_t)M * y.c_out, ST));
      if (y.im2col)
        PD_TRY(timed_conv(rt, KC_WGRAD, PD_GEMM_WGRAD_SPLITK, Y.cols[act], dy, B, y.h, y.w, 64, y.c_out, EPI_GRADF32,
                          ep, ST));
      else
        PD_TRY(timed_conv(rt, KC_WGRAD, PD_CONV_WGRAD, X, dy, B, y.h, y.w, y.c_in, y.c_out, EPI_GRADF32, ep, ST));
      const int64_t n = (int64_t)M * y.c_out;
      PD_TRY(timed_call(rt, KC_UPDATE, ST, [&]() { return reduce_sgd(d.dtype, d.part, 1, n, n, gW, S.w_master[l], ring_new, d.lr, ST); }));
      PD_TRY(bias_grad_tall(dy, pix, y.c_out, d.part, gb, S.b_master[l], bring_new, d.lr, ST, d.sync));
      rt->launches += 3;
    }
    if (need_dx) {
      if (y.im2col) return set_error(PD_ERR_INVALID, "worker %d: im2col layer must be the model input", d.worker);
      dst = (l == 0) ? rt->views.at(it[PD_IT_DST]).grad_in[it[PD_IT_OUT]] : other_tmp(dy);
      EpiArgs ep{};
      ep.out = dst;
      ep.ldo = y.c_in;
      ep.mask = X;
      ep.ldm = y.c_in;
      PD_TRY(timed_conv(rt, KC_DGRAD, PD_CONV_DGRAD, dy, Wst, B, y.h, y.w, y.c_in, y.c_out, EPI_MASK, ep, ST));
    }
    // the layer's new version may overwrite ring slot wnew only after this layer's dgrad read wslot
    if (replicated && sharded_reduce(rt, S)) PD_TRY(layer_grad_ready(rt, S, l, round, ST));
    dz = dst;
  }
  if (replicated && !sharded_reduce(rt, S)) PD_TRY(signal_flag(rt, S, d.red_ready, round));
  return 0;
}

// Replicated stage, round k: wait until every replica's round-k gradients exist, then the fused
// allreduce (peer loads) + SGD kernel commits version k*rep into ring slot wnew on each replica.
int run_reduce(pd_runtime* rt, Stage& S, const int32_t* it) {
  cudaStream_t ST = stream_of(rt, S);
  const pd_stage_desc& d = S.d;
  const int round = it[PD_IT_ROUND], wnew = it[PD_IT_WNEW], par = round & 1;
  if (sharded_reduce(rt, S)) {  // the round's first REDUCE item enqueues it for every local replica
    if (S.issued_round < round) PD_TRY(issue_round_reduce(rt, S, round, wnew));
    PD_CHECK(cudaStreamWaitEvent(ST, S.ev_red, 0));
    return 0;
  }
  for (int r = 0; r < d.rep; ++r) PD_TRY(wait_flag(rt, S, rt->views.at(d.first_worker + r).v.red_ready, round));
  std::vector<const float*> g(d.rep), gb(d.rep);
  for (int l = 0; l < d.n_layers; ++l) {
    for (int r = 0; r < d.rep; ++r) {
      const View& V = rt->views.at(d.first_worker + r);
      g[r] = V.red_grad[(size_t)l * 2 + par];
      gb[r] = V.red_bgrad[(size_t)l * 2 + par];
    }
    const int64_t n = w_numel(S, l);
    PD_TRY(timed_call(rt, KC_UPDATE, ST, [&]() { return allreduce_sgd(d.dtype, g.data(), d.rep, S.w_master[l], S.w_ring[(size_t)l * d.ring_depth + wnew], n,
                         d.lr, ST); }));
    PD_TRY(timed_call(rt, KC_UPDATE, ST, [&]() { return allreduce_sgd(PD_F32, gb.data(), d.rep, S.b_master[l], S.b_ring[(size_t)l * d.ring_depth + wnew],
                         b_numel(S, l), d.lr, ST); }));
    rt->launches += 2;
  }
  PD_TRY(signal_flag(rt, S, d.red_done, round));
  return 0;
}

}  // namespace

extern "C" {

int pd_rt_create(int device, pd_runtime** out) {
  if (!out) return set_error(PD_ERR_INVALID, "pd_rt_create: null out");
  PD_CHECK(cudaSetDevice(device));
  auto* rt = new pd_runtime();
  rt->device = device;
  if (cudaEventCreate(&rt->ev0) != cudaSuccess) {
    delete rt;
    return set_error(PD_ERR_CUDA, "cudaEventCreate failed");
  }
  *out = rt;
  return 0;
}

int pd_rt_add_stage(pd_runtime* rt, const pd_stage_desc* desc) {
  if (!rt || !desc) return set_error(PD_ERR_INVALID, "pd_rt_add_stage: null argument");
  const pd_stage_desc& d = *desc;
  if (d.n_layers < 1 || d.batch < 1 || d.ring_depth < 1 || d.act_depth < 1 || d.rep < 1)
    return set_error(PD_ERR_INVALID, "worker %d: bad descriptor (layers=%d batch=%d ring=%d act=%d rep=%d)",
                     d.worker, d.n_layers, d.batch, d.ring_depth, d.act_depth, d.rep);
  if (d.dtype != PD_F32 && d.dtype != PD_BF16) return set_error(PD_ERR_INVALID, "worker %d: bad dtype", d.worker);
  if (d.init_slot < 0 || d.init_slot >= d.ring_depth)
    return set_error(PD_ERR_INVALID, "worker %d: bad init_slot", d.worker);
  if (d.rep > 1 && (!d.red_grad || !d.red_bgrad || !d.red_ready || !d.red_done))
    return set_error(PD_ERR_INVALID, "worker %d: replicated stage without reduction buffers", d.worker);
  if (rt->stages.count(d.worker)) return set_error(PD_ERR_INVALID, "worker %d added twice", d.worker);
  Stage S;
  S.d = d;
  const int L = d.n_layers;
  S.dims = copy_arr(d.dims, L + 1);
  if (d.layers) {
    for (int l = 0; l < L; ++l) {
      Layer Y;
      Y.d = d.layers[l];
      const pd_layer& y = Y.d;
      if (y.kind < PD_LAYER_LINEAR || y.kind > PD_LAYER_HEAD)
        return set_error(PD_ERR_INVALID, "worker %d layer %d: bad kind %d", d.worker, l, y.kind);
      if (y.c_in < 1 || y.c_out < 1 || (y.kind == PD_LAYER_CONV3 && (y.h < 2 || y.w < 2)))
        return set_error(PD_ERR_INVALID, "worker %d layer %d: bad shape", d.worker, l);
      const bool tkind = y.kind == PD_LAYER_EMBED || y.kind == PD_LAYER_BLOCK || y.kind == PD_LAYER_HEAD;
      if (tkind) {
        if (d.rep > 1) return set_error(PD_ERR_INVALID, "worker %d: transformer stages are not replicated", d.worker);
        if (y.h < 128 || y.h % 128) return set_error(PD_ERR_INVALID, "worker %d layer %d: seq %% 128", d.worker, l);
        if (y.kind == PD_LAYER_BLOCK && (y.w * 64 != y.c_in || y.ffn < 1))
          return set_error(PD_ERR_INVALID, "worker %d layer %d: d = 64 * heads required", d.worker, l);
        if (y.kind == PD_LAYER_HEAD && (y.vocab < 1 || y.vocab > y.c_out || !d.is_last || !d.logits))
          return set_error(PD_ERR_INVALID, "worker %d layer %d: bad head", d.worker, l);
        if (y.kind == PD_LAYER_EMBED && !(d.is_first && l == 0))
          return set_error(PD_ERR_INVALID, "worker %d: the embedding must be the model input", d.worker);
        if (y.kind != PD_LAYER_EMBED && (!y.save || !y.work))
          return set_error(PD_ERR_INVALID, "worker %d layer %d: missing save/work buffers", d.worker, l);
        if (!d.part || !d.sync)
          return set_error(PD_ERR_INVALID, "worker %d: transformer layers need `part` and `sync`", d.worker);
        Y.t = tlayout(y, d.batch);
        if (y.save) Y.save.assign(y.save, y.save + d.act_depth);
      }
      if (d.dtype != PD_BF16) return set_error(PD_ERR_INVALID, "worker %d: layered stages are bf16", d.worker);
      if (y.kind == PD_LAYER_CONV3 && (!d.part || !d.sync))
        return set_error(PD_ERR_INVALID, "worker %d: conv layers need the `part` and `sync` scratch", d.worker);
      if (y.pool) {
        if (!y.argmax) return set_error(PD_ERR_INVALID, "worker %d layer %d: pool without argmax", d.worker, l);
        Y.argmax.assign(y.argmax, y.argmax + d.act_depth);
      }
      if (y.im2col) {
        if (!y.cols) return set_error(PD_ERR_INVALID, "worker %d layer %d: im2col without cols", d.worker, l);
        Y.cols.assign(y.cols, y.cols + d.act_depth);
      }
      Y.d.argmax = nullptr;
      Y.d.cols = nullptr;
      Y.d.save = nullptr;
      S.layers.push_back(Y);
    }
    if (d.is_last && d.loss_kind == PD_LOSS_CE && !d.logits && S.layers.back().d.kind != PD_LAYER_HEAD)
      return set_error(PD_ERR_INVALID, "worker %d: cross-entropy needs the logits buffer", d.worker);
  }
  S.d.layers = nullptr;
  {
    // hand-off payload per minibatch: the stage's output (forward) and input gradient (backward)
    const int64_t esz = d.dtype == PD_F32 ? 4 : 2;
    auto feats = [&](const pd_layer& y, bool out) -> int64_t {
      if (y.kind == PD_LAYER_CONV3)
        return out ? (int64_t)(y.pool ? (y.h / 2) * (y.w / 2) : y.h * y.w) * y.c_out : (int64_t)y.h * y.w * y.c_in;
      if (y.kind == PD_LAYER_LINEAR) return out ? y.c_out : y.c_in;
      if (y.kind == PD_LAYER_EMBED) return out ? (int64_t)y.h * y.c_out : 0;
      return (int64_t)y.h * y.c_in;  // BLOCK / HEAD: [seq, d] per sequence
    };
    if (S.layers.empty()) {
      S.out_bytes = (int64_t)d.batch * S.dims[L] * esz;
      S.in_bytes = (int64_t)d.batch * S.dims[0] * esz;
    } else {
      S.out_bytes = (int64_t)d.batch * feats(S.layers.back().d, true) * esz;
      S.in_bytes = (int64_t)d.batch * feats(S.layers.front().d, false) * esz;
    }
  }
  S.tag_index = (int)rt->stages.size();
  if (d.ring_depth > 64) return set_error(PD_ERR_INVALID, "worker %d: ring depth %d > 64", d.worker, d.ring_depth);
  S.w_master = copy_arr(d.w_master, L);
  S.b_master = copy_arr(d.b_master, L);
  S.w_ring = copy_arr(d.w_ring, (int64_t)L * d.ring_depth);
  S.b_ring = copy_arr(d.b_ring, (int64_t)L * d.ring_depth);
  S.act = copy_arr(d.act, (int64_t)(L - 1) * d.act_depth);
  S.act_in = copy_arr(d.act_in, d.is_first ? d.n_data_blocks : d.in_depth);
  if (!d.is_last) S.grad_in = copy_arr(d.grad_in, d.grad_depth);
  if (d.is_last) {
    S.dz_last = copy_arr(d.dz_last, d.act_depth);
    S.target = copy_arr(d.target, d.n_data_blocks);
  }
  if (d.fused_bias) {
    bool ok = d.dtype == PD_BF16 && d.rep == 1 && !d.layers && (L == 1 || d.bpart) &&
              (d.is_last ? d.dz_bpart != nullptr : d.grad_bpart != nullptr);
    for (int l = 0; l <= L && ok; ++l) ok = S.dims[l] % 32 == 0;
    if (!ok)
      return set_error(PD_ERR_INVALID, "worker %d: fused bias needs a bf16 MLP stage, rep 1, widths %% 32 == 0 "
                       "and its partial buffers", d.worker);
    S.bpart = copy_arr(d.bpart, (int64_t)L - 1);
    if (d.is_last) S.dz_bpart = copy_arr(d.dz_bpart, d.act_depth);
    else S.grad_bpart = copy_arr(d.grad_bpart, d.grad_depth);
  }
  if (d.rep > 1) {
    S.red_grad = copy_arr(d.red_grad, (int64_t)L * 2);
    S.red_bgrad = copy_arr(d.red_bgrad, (int64_t)L * 2);
  }
  S.d.dims = nullptr;
  PD_CHECK(cudaSetDevice(rt->device));
  PD_CHECK(cudaStreamCreateWithFlags(&S.stream, cudaStreamNonBlocking));
  PD_CHECK(cudaEventCreateWithFlags(&S.ev_done, cudaEventDisableTiming));
  if (d.rep > 1 && d.red_lready && d.red_lupd) {
    PD_CHECK(cudaStreamCreateWithFlags(&S.rstream, cudaStreamNonBlocking));
    PD_CHECK(cudaEventCreateWithFlags(&S.ev_red, cudaEventDisableTiming));
    S.ev_layer.assign(L, nullptr);
    S.ev_upd.assign(L, nullptr);
    for (int l = 0; l < L; ++l) {
      PD_CHECK(cudaEventCreateWithFlags(&S.ev_layer[l], cudaEventDisableTiming));
      PD_CHECK(cudaEventCreateWithFlags(&S.ev_upd[l], cudaEventDisableTiming));
    }
  }
  rt->stages.emplace(d.worker, std::move(S));
  return 0;
}

int pd_rt_add_view(pd_runtime* rt, const pd_worker_view* view) {
  if (!rt || !view) return set_error(PD_ERR_INVALID, "pd_rt_add_view: null argument");
  View V;
  V.v = *view;
  V.act_in = copy_arr(view->act_in, view->in_depth);
  V.grad_in = copy_arr(view->grad_in, view->grad_depth);
  V.red_grad = copy_arr(view->red_grad, (int64_t)view->n_layers * 2);
  V.red_bgrad = copy_arr(view->red_bgrad, (int64_t)view->n_layers * 2);
  if (view->w_master) {
    V.w_master = copy_arr(view->w_master, view->n_layers);
    V.b_master = copy_arr(view->b_master, view->n_layers);
  }
  if (view->fused_bias) {
    if (!view->grad_bpart) return set_error(PD_ERR_INVALID, "view of worker %d: fused bias without partials", view->worker);
    V.grad_bpart = copy_arr(view->grad_bpart, view->grad_depth);
  }
  rt->views[view->worker] = std::move(V);
  return 0;
}

int pd_rt_load_program(pd_runtime* rt, const int32_t* items, int n_items) {
  if (!rt || (!items && n_items)) return set_error(PD_ERR_INVALID, "pd_rt_load_program: null argument");
  for (int i = 0; i < n_items; ++i) {
    const int32_t* it = items + (size_t)i * PD_ITEM_WIDTH;
    auto f = rt->stages.find(it[PD_IT_WORKER]);
    if (f == rt->stages.end())
      return set_error(PD_ERR_INVALID, "item %d: worker %d is not hosted here", i, it[PD_IT_WORKER]);
    const Stage& S = f->second;
    const int op = it[PD_IT_OP];
    if (op < 0 || op > 2) return set_error(PD_ERR_INVALID, "item %d: bad op %d", i, op);
    if (it[PD_IT_DEP] >= i || it[PD_IT_WAR] >= i)
      return set_error(PD_ERR_INVALID, "item %d: dependency %d/%d not issued earlier (program not topological)", i,
                       it[PD_IT_DEP], it[PD_IT_WAR]);
    if (it[PD_IT_WSLOT] >= S.d.ring_depth || it[PD_IT_WNEW] >= S.d.ring_depth || it[PD_IT_ACT] >= S.d.act_depth)
      return set_error(PD_ERR_INVALID, "item %d: slot out of range", i);
    if (op == 2 && S.d.rep < 2) return set_error(PD_ERR_INVALID, "item %d: reduce on an unreplicated stage", i);
    const bool sends = (op == 0 && !S.d.is_last) || (op == 1 && !S.d.is_first);
    if (sends) {
      auto v = rt->views.find(it[PD_IT_DST]);
      if (v == rt->views.end()) return set_error(PD_ERR_INVALID, "item %d: no view of worker %d", i, it[PD_IT_DST]);
      const int depth = op == 0 ? v->second.v.in_depth : v->second.v.grad_depth;
      if (it[PD_IT_OUT] < 0 || it[PD_IT_OUT] >= depth)
        return set_error(PD_ERR_INVALID, "item %d: outbox slot %d out of range", i, it[PD_IT_OUT]);
    }
    if (S.d.rep > 1)
      for (int r = 0; r < S.d.rep; ++r)
        if (!rt->views.count(S.d.first_worker + r))
          return set_error(PD_ERR_INVALID, "item %d: no view of replica worker %d", i, S.d.first_worker + r);
  }
  drop_graph(rt);
  rt->items.assign(items, items + (size_t)n_items * PD_ITEM_WIDTH);
  for (auto& kv : rt->stages) {
    Stage& S = kv.second;
    S.last_round = 0;
    S.replicas_local = true;
    for (int r = 0; r < S.d.rep && S.d.rep > 1; ++r)
      if (rt->views.at(S.d.first_worker + r).v.remote) S.replicas_local = false;
  }
  for (int i = 0; i < n_items; ++i) {
    const int32_t* it = items + (size_t)i * PD_ITEM_WIDTH;
    Stage& S = rt->stages.at(it[PD_IT_WORKER]);
    if (S.d.rep > 1) S.last_round = std::max(S.last_round, (int)it[PD_IT_ROUND]);
  }
  // drain list: final occupant of every remote outbox slot
  rt->drain.clear();
  std::map<std::pair<int*, int>, std::pair<int, int>> last;  // (ack array, slot) -> (worker, mb)
  for (int i = 0; i < n_items; ++i) {
    const int32_t* it = items + (size_t)i * PD_ITEM_WIDTH;
    const Stage& S = rt->stages.at(it[PD_IT_WORKER]);
    const int op = it[PD_IT_OP];
    if (!((op == 0 && !S.d.is_last) || (op == 1 && !S.d.is_first))) continue;
    const View& V = rt->views.at(it[PD_IT_DST]);
    if (!V.v.remote) continue;
    int* ack = op == 0 ? V.v.act_ack : V.v.grad_ack;
    auto& e = last[{ack, it[PD_IT_OUT]}];
    if (it[PD_IT_MB] > e.second) e = {it[PD_IT_WORKER], it[PD_IT_MB]};
  }
  for (const auto& kv : last) rt->drain.push_back({kv.second.first, kv.first.first + kv.first.second, kv.second.second});
  for (auto e : rt->ev_start) cudaEventDestroy(e);
  for (auto e : rt->ev_end) cudaEventDestroy(e);
  rt->ev_start.assign(n_items, nullptr);
  rt->ev_end.assign(n_items, nullptr);
  PD_CHECK(cudaSetDevice(rt->device));
  for (int i = 0; i < n_items; ++i) {
    PD_CHECK(cudaEventCreate(&rt->ev_start[i]));
    PD_CHECK(cudaEventCreate(&rt->ev_end[i]));
  }
  return 0;
}

static int run_body(pd_runtime* rt, cudaStream_t main, int trace);

// Graph replay is valid when the run has no cross-process flags (whose values carry the run
// epoch), no tracing and no per-kernel timing: then every run enqueues exactly the same work.
static bool graph_eligible(pd_runtime* rt, int trace) {
  if (!rt->graph_mode || trace || rt->ktiming || !rt->drain.empty()) return false;
  for (const auto& kv : rt->stages)
    if (kv.second.d.remote_prev || kv.second.d.remote_next) return false;
  for (const auto& kv : rt->views)
    if (kv.second.v.remote) return false;
  return true;
}

int pd_rt_run(pd_runtime* rt, void* stream, int trace) {
  if (!rt) return set_error(PD_ERR_INVALID, "pd_rt_run: null runtime");
  cudaStream_t main = static_cast<cudaStream_t>(stream);
  PD_CHECK(cudaSetDevice(rt->device));
  if (!graph_eligible(rt, trace)) return run_body(rt, main, trace);
  if (!rt->graph_exec) {
    // capture on a private stream (the caller's may be the legacy default stream, which cannot
    // be captured); the instantiated graph is then launched into the caller's stream
    if (!rt->graph_stream) PD_CHECK(cudaStreamCreateWithFlags(&rt->graph_stream, cudaStreamNonBlocking));
    const int64_t before = rt->launches;
    rt->lt_used = 0;  // layer-timing events captured into the graph are re-recorded by every replay
    PD_CHECK(cudaStreamBeginCapture(rt->graph_stream, cudaStreamCaptureModeRelaxed));
    const int rc = run_body(rt, rt->graph_stream, 0);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(rt->graph_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return set_error(PD_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
    rt->graph = g;
    PD_CHECK(cudaGraphInstantiate(&rt->graph_exec, g, 0));
    rt->graph_launches = rt->launches - before;
    rt->launches = before;
  }
  PD_CHECK(cudaGraphLaunch(rt->graph_exec, main));
  rt->launches += rt->graph_launches;
  rt->traced = false;
  return 0;
}

static int run_body(pd_runtime* rt, cudaStream_t main, int trace) {
  rt->epoch += 1;
  rt->traced = trace != 0;
  // In-process replica sets: reset their round flags before any stage stream starts.  A captured
  // graph bakes this run's epoch into every flag value, so without the reset a replay would find
  // the previous replay's final values already past every target (and not wait at all).
  for (auto& kv : rt->stages) {
    Stage& S = kv.second;
    if (S.d.rep > 1 && S.replicas_local) {
      PD_CHECK(cudaMemsetAsync(S.d.red_ready, 0, sizeof(int), main));
      PD_CHECK(cudaMemsetAsync(S.d.red_done, 0, sizeof(int), main));
      if (S.d.red_lready) PD_CHECK(cudaMemsetAsync(S.d.red_lready, 0, sizeof(int) * S.d.n_layers, main));
      if (S.d.red_lupd) PD_CHECK(cudaMemsetAsync(S.d.red_lupd, 0, sizeof(int) * S.d.n_layers, main));
    }
  }
  const bool recs = rt->traced && rt->rec;
  if (recs) {
    PD_CHECK(cudaMemsetAsync(rt->rec + 1, 0, sizeof(int64_t), main));  // sharded-reduction peer bytes
    PD_TRY(timestamp(reinterpret_cast<uint64_t*>(rt->rec), main));      // before any stage starts
  }
  for (auto& kv : rt->stages) kv.second.issued_round = 0;
  PD_CHECK(cudaEventRecord(rt->ev0, main));
  int max_mb = 0;
  for (size_t i = 0; i < rt->items.size(); i += PD_ITEM_WIDTH) max_mb = std::max(max_mb, rt->items[i + PD_IT_MB]);
  for (auto& kv : rt->stages) {
    Stage& S = kv.second;
    cudaStream_t ST = stream_of(rt, S);
    PD_CHECK(cudaStreamWaitEvent(ST, rt->ev0, 0));
    // version 0 of this run = the current (latest) weights
    for (int l = 0; l < S.d.n_layers; ++l) {
      const int64_t n = w_numel(S, l);
      PD_TRY(timed_call(rt, KC_OTHER, ST, [&]() { return cast_f32(S.d.dtype, S.w_master[l], S.w_ring[(size_t)l * S.d.ring_depth + S.d.init_slot], n, ST); }));
      rt->launches += 1;
      if (b_numel(S, l) > 0)
        PD_CHECK(cudaMemcpyAsync(S.b_ring[(size_t)l * S.d.ring_depth + S.d.init_slot], S.b_master[l],
                                 sizeof(float) * b_numel(S, l), cudaMemcpyDeviceToDevice, ST));
    }
    if (recs) PD_TRY(set_tags(rt->tags + 64 * S.tag_index, 64, S.d.init_slot, 0, ST));  // slot init_slot = v0
    if (S.d.is_last && S.d.loss)  // losses are indexed by minibatch id
      PD_CHECK(cudaMemsetAsync(S.d.loss, 0, sizeof(float) * (size_t)(max_mb + 1), ST));
  }
  const int n = (int)(rt->items.size() / PD_ITEM_WIDTH);
  for (int i = 0; i < n; ++i) {
    const int32_t* it = rt->items.data() + (size_t)i * PD_ITEM_WIDTH;
    Stage& S = rt->stages[it[PD_IT_WORKER]];
    cudaStream_t ST = stream_of(rt, S);
    const int op = it[PD_IT_OP], mb = it[PD_IT_MB];
    const bool fwd = op == 0;
    rt->cur_worker = it[PD_IT_WORKER];
    const int dep = it[PD_IT_DEP], war = it[PD_IT_WAR];
    if (dep >= 0) PD_CHECK(cudaStreamWaitEvent(ST, rt->ev_end[dep], 0));
    if (war >= 0) PD_CHECK(cudaStreamWaitEvent(ST, rt->ev_end[war], 0));
    if (it[PD_IT_RWAIT] > 0)  // payload produced in another process: acquire my inbox flag
      PD_TRY(wait_flag(rt, S, fwd ? S.d.act_ready + it[PD_IT_XSLOT] : S.d.grad_ready + it[PD_IT_GSLOT],
                       it[PD_IT_RWAIT]));
    if (it[PD_IT_AWAIT] > 0) {  // receiver in another process: its previous occupant must be done
      const View& V = rt->views.at(it[PD_IT_DST]);
      PD_TRY(wait_flag(rt, S, (fwd ? V.v.act_ack : V.v.grad_ack) + it[PD_IT_OUT], it[PD_IT_AWAIT]));
    }
    if (rt->traced) PD_CHECK(cudaEventRecord(rt->ev_start[i], ST));
    int* stag = recs ? rt->tags + 64 * S.tag_index : nullptr;
    const int wslot = it[PD_IT_WSLOT], wnew = it[PD_IT_WNEW];
    rt->cur_rec = recs ? rt->rec + (size_t)(1 + i) * PD_REC_WIDTH : nullptr;
    if (recs) PD_TRY(rec_begin(rt->cur_rec, op != 2 && wslot >= 0 ? stag + wslot : nullptr, ST));
    const bool layered = !S.layers.empty();
    S.fused_signal = false;
    if (op == 0) PD_TRY(layered ? run_forward_layers(rt, S, it) : run_forward(rt, S, it));
    else if (op == 1) PD_TRY(layered ? run_backward_layers(rt, S, it) : run_backward(rt, S, it));
    else PD_TRY(run_reduce(rt, S, it));
    // cross-process hand-off: publish the payload the epilogue stored into the peer inbox
    if ((op == 0 && !S.d.is_last) || (op == 1 && !S.d.is_first)) {
      const View& V = rt->views.at(it[PD_IT_DST]);
      if (V.v.remote && !S.fused_signal) PD_TRY(signal_flag(rt, S, (fwd ? V.v.act_ready : V.v.grad_ready) + it[PD_IT_OUT], mb));
    }
    if (op == 1) {  // my inbox slots are free again: tell producers in other processes
      if (!S.d.is_first && S.d.remote_prev) PD_TRY(signal_flag(rt, S, S.d.act_ack + it[PD_IT_XSLOT], mb));
      if (!S.d.is_last && S.d.remote_next) PD_TRY(signal_flag(rt, S, S.d.grad_ack + it[PD_IT_GSLOT], mb));
    }
    if (recs) {
      // commit: a backward of an unreplicated stage writes version mb, a replica reduce version
      // round * rep (simulator.py:315); the tag follows the committing kernels
      const bool commits = wnew >= 0 && (op == 2 || (op == 1 && S.d.rep == 1));
      const int commit_v = op == 2 ? it[PD_IT_ROUND] * S.d.rep : mb;
      int64_t host_bytes = 0;  // stand-alone signal path: the payload the flag publishes
      if ((op == 0 && !S.d.is_last) || (op == 1 && !S.d.is_first))
        if (rt->views.at(it[PD_IT_DST]).v.remote && !S.fused_signal) {
          host_bytes = op == 0 ? S.out_bytes : S.in_bytes;
          if (op == 1 && rt->views.at(it[PD_IT_DST]).v.fused_bias)  // + the receiver's bias partials
            host_bytes += (int64_t)((S.d.batch + 31) / 32) * S.dims[0] * 4;
        }
      PD_TRY(rec_end(rt->cur_rec, op != 2 && wslot >= 0 ? stag + wslot : nullptr, commits ? stag + wnew : nullptr,
                     commit_v, host_bytes, ST));
      rt->launches += 2;
    }
    rt->cur_rec = nullptr;
    PD_CHECK(cudaEventRecord(rt->ev_end[i], ST));
  }
  for (const auto& dr : rt->drain) PD_TRY(wait_flag(rt, rt->stages[dr.worker], dr.flag, dr.mb));
  for (auto& kv : rt->stages) {
    Stage& S = kv.second;
    PD_CHECK(cudaEventRecord(S.ev_done, stream_of(rt, S)));
    PD_CHECK(cudaStreamWaitEvent(main, S.ev_done, 0));
  }
  return 0;
}

int pd_rt_records(pd_runtime* rt, pd_record* out, int cap, int* n_out) {
  if (!rt || !n_out) return set_error(PD_ERR_INVALID, "pd_rt_records: null argument");
  if (!rt->traced) return set_error(PD_ERR_INVALID, "pd_rt_records: last run was not traced");
  const int n = (int)(rt->items.size() / PD_ITEM_WIDTH);
  PD_CHECK(cudaSetDevice(rt->device));
  int k = 0;
  for (int i = 0; i < n && k < cap; ++i, ++k) {
    float a = 0.f, b = 0.f;
    PD_CHECK(cudaEventSynchronize(rt->ev_end[i]));
    PD_CHECK(cudaEventElapsedTime(&a, rt->ev0, rt->ev_start[i]));
    PD_CHECK(cudaEventElapsedTime(&b, rt->ev0, rt->ev_end[i]));
    out[k].item = i;
    out[k].pad = 0;
    out[k].t_start_ms = a;
    out[k].t_end_ms = b;
  }
  *n_out = k;
  return 0;
}

int pd_rt_set_records(pd_runtime* rt, int64_t* rec, int cap, int32_t* tags) {
  if (!rt) return set_error(PD_ERR_INVALID, "pd_rt_set_records: null runtime");
  if (rec && (!tags || cap < (int)(rt->items.size() / PD_ITEM_WIDTH)))
    return set_error(PD_ERR_INVALID, "pd_rt_set_records: need tags and room for %d items",
                     (int)(rt->items.size() / PD_ITEM_WIDTH));
  rt->rec = rec;
  rt->rec_cap = rec ? cap : 0;
  rt->tags = rec ? tags : nullptr;
  return 0;
}

int pd_rt_set_graph(pd_runtime* rt, int on) {
  if (!rt) return set_error(PD_ERR_INVALID, "pd_rt_set_graph: null runtime");
  rt->graph_mode = on != 0;
  if (!on) drop_graph(rt);
  return 0;
}

int pd_rt_set_serial(pd_runtime* rt, int on) {
  if (!rt) return set_error(PD_ERR_INVALID, "pd_rt_set_serial: null runtime");
  PD_CHECK(cudaSetDevice(rt->device));
  if ((on != 0) != rt->serial) drop_graph(rt);
  if (on && !rt->shared) PD_CHECK(cudaStreamCreateWithFlags(&rt->shared, cudaStreamNonBlocking));
  rt->serial = on != 0;
  return 0;
}

int pd_rt_kernel_timing(pd_runtime* rt, int on) {
  if (!rt) return set_error(PD_ERR_INVALID, "pd_rt_kernel_timing: null runtime");
  rt->ktiming = on != 0;
  rt->kt_used = 0;
  return 0;
}

int pd_rt_kernel_stats(pd_runtime* rt, int worker, double* out9, int n_classes) {
  if (!rt || !out9 || n_classes < 1) return set_error(PD_ERR_INVALID, "pd_rt_kernel_stats: null argument");
  for (int i = 0; i < 3 * n_classes; ++i) out9[i] = 0.0;
  PD_CHECK(cudaSetDevice(rt->device));
  for (size_t i = 0; i < rt->kt_used; ++i) {
    auto& k = rt->kt[i];
    float ms = 0.f;
    PD_CHECK(cudaEventSynchronize(k.b));
    PD_CHECK(cudaEventElapsedTime(&ms, k.a, k.b));
    if (k.cls >= n_classes || (worker >= 0 && k.worker != worker)) continue;
    out9[3 * k.cls + 0] += 1.0;
    out9[3 * k.cls + 1] += ms;
    out9[3 * k.cls + 2] += k.flops;
  }
  return 0;
}

int pd_rt_layer_timing(pd_runtime* rt, uint64_t* ts, int cap) {
  if (!rt) return set_error(PD_ERR_INVALID, "pd_rt_layer_timing: null runtime");
  rt->ltiming = ts != nullptr && cap > 0;
  rt->ts = ts;
  rt->ts_cap = rt->ltiming ? cap : 0;
  rt->lt_used = 0;
  drop_graph(rt);  // the next run (re)captures with or without the stamps
  return 0;
}

int pd_rt_layer_stats(pd_runtime* rt, int worker, int n_layers, double* out) {
  if (!rt || !out || n_layers < 1) return set_error(PD_ERR_INVALID, "pd_rt_layer_stats: bad argument");
  std::vector<double> cnt(2 * n_layers, 0.0);
  for (int i = 0; i < 2 * n_layers; ++i) out[i] = 0.0;
  PD_CHECK(cudaSetDevice(rt->device));
  std::vector<uint64_t> h(2 * rt->lt_used);
  if (!h.empty()) PD_CHECK(cudaMemcpy(h.data(), rt->ts, h.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < rt->lt_used; ++i) {
    const auto& x = rt->lt[i];
    if (x.worker != worker || x.layer < 0 || x.layer >= n_layers) continue;
    out[2 * x.layer + x.dir] += (double)(h[2 * i + 1] - h[2 * i]) * 1e-6;  // ns -> ms
    cnt[2 * x.layer + x.dir] += 1.0;
  }
  for (int i = 0; i < 2 * n_layers; ++i)
    if (cnt[i] > 0) out[i] /= cnt[i];
  return 0;
}

int pd_rt_launch_count(pd_runtime* rt, int64_t* out) {
  if (!rt || !out) return set_error(PD_ERR_INVALID, "pd_rt_launch_count: null argument");
  *out = rt->launches;
  return 0;
}

int pd_rt_destroy(pd_runtime* rt) {
  if (!rt) return 0;
  cudaSetDevice(rt->device);
  drop_graph(rt);
  if (rt->graph_stream) cudaStreamDestroy(rt->graph_stream);
  for (auto& kv : rt->stages) {
    cudaStreamSynchronize(kv.second.stream);
    cudaStreamDestroy(kv.second.stream);
    cudaEventDestroy(kv.second.ev_done);
    if (kv.second.rstream) {
      cudaStreamSynchronize(kv.second.rstream);
      cudaStreamDestroy(kv.second.rstream);
      cudaEventDestroy(kv.second.ev_red);
      for (auto e : kv.second.ev_layer) cudaEventDestroy(e);
      for (auto e : kv.second.ev_upd) cudaEventDestroy(e);
    }
  }
  for (auto e : rt->ev_start) cudaEventDestroy(e);
  for (auto e : rt->ev_end) cudaEventDestroy(e);
  for (auto& k : rt->kt) {
    cudaEventDestroy(k.a);
    cudaEventDestroy(k.b);
  }
  if (rt->ev0) cudaEventDestroy(rt->ev0);
  if (rt->shared) {
    cudaStreamSynchronize(rt->shared);
    cudaStreamDestroy(rt->shared);
  }
  delete rt;
  return 0;
}

}  // extern "C"

extern "C" int64_t pd_layer_save_bytes(const pd_layer* layer, int batch) {
  if (!layer || batch < 1) return 0;
  return tlayout(*layer, batch).save_bytes;
}

extern "C" int64_t pd_layer_work_bytes(const pd_layer* layer, int batch) {
  if (!layer || batch < 1) return 0;
  return tlayout(*layer, batch).work_bytes;
}

extern "C" int64_t pd_layer_scratch_floats(const pd_layer* layer, int batch) {
  if (!layer || batch < 1) return 0;
  const pd_layer& y = *layer;
  if (y.kind == PD_LAYER_EMBED) return (int64_t)(y.c_in + y.h) * y.c_out;
  if (y.kind == PD_LAYER_BLOCK || y.kind == PD_LAYER_HEAD) {
    const int64_t T = (int64_t)batch * y.h;
    const int64_t D = y.c_in;
    int64_t need = (int64_t)pd::ln_bwd_blocks(T) * 2 * D;
    const int64_t widest = y.kind == PD_LAYER_BLOCK ? (3 * D > y.ffn ? 3 * D : y.ffn) : 0;
    for (int64_t c : {D, widest}) {
      if (c <= 0) continue;
      const int64_t cs = (int64_t)pd::colsum_blocks(T, (int)c) * c;
      need = cs > need ? cs : need;
    }
    return need;
  }
  if (y.kind != PD_LAYER_CONV3) return 0;
  const int M = y.im2col ? 64 : 9 * y.c_in;
  const int64_t pix = (int64_t)batch * y.h * y.w;
  int splits = 1, per = 0;
  pd::splitk_plan(M, y.c_out, (int)pix, &splits, &per);
  const int64_t wpart = (int64_t)splits * M * y.c_out;
  const int64_t bpart = (int64_t)pd::colsum_blocks(pix, y.c_out) * y.c_out;
  return wpart > bpart ? wpart : bpart;
}
