/*
 * pd_b200.h - C ABI of libpd_b200.so, the B200-native executor behind
 * paper_1806_03377_b200.run(), the drop-in for pipesim.run().
 *
 * The reference (pipesim, pure Python) has no FFI: its hot-path boundary is the
 * Python call  pipesim.run(cfg, ctx, schedule=None) -> SimResult
 * (/root/reference/pkg/src/pipesim/simulator.py:401-411).  That call is kept
 * verbatim in Python (paper_1806_03377_b200/executor.py); this header is the
 * thin layer under it.  Each entry point below names the reference routine
 * whose work it takes over.
 *
 * Conventions
 *   - Plain pointers and sizes only; device memory is allocated by the caller
 *     (PyTorch) and never freed here.  Streams are passed as void* (cudaStream_t).
 *   - Every function returns 0 on success.  PD_ERR_INVALID maps to the
 *     reference's ValidationError, PD_ERR_TIMEOUT / PD_ERR_DEADLOCK to its
 *     SimulationError ("deadlock: worker w (stage s, ...)" simulator.py:350-357),
 *     PD_ERR_CUDA to a RuntimeError.  pd_last_error() holds the message.
 *   - One host thread per process (one process per GPU), as the reference's
 *     engine is single-threaded.
 */
#ifndef PD_B200_H
#define PD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PD_ABI_VERSION 1

enum pd_status { PD_OK = 0, PD_ERR_INVALID = 1, PD_ERR_CUDA = 2, PD_ERR_TIMEOUT = 3, PD_ERR_DEADLOCK = 4 };
enum pd_dtype { PD_F32 = 0, PD_BF16 = 1 };
enum pd_epi_kind {
  PD_EPI_STORE = 0, PD_EPI_LOSS = 1, PD_EPI_MASK = 2, PD_EPI_SGD = 3, PD_EPI_GRADF32 = 4,
  PD_EPI_GELU = 5,      /* z = acc + bias -> aux; out = gelu_tanh(z)        (A, B K-major) */
  PD_EPI_GELU_BWD = 6,  /* out = acc * gelu_tanh'(mask)                     (A K-major, B MN-major) */
  PD_EPI_RESID = 7      /* out = acc + bias + mask (residual stream)        (A, B K-major) */
};

/* ------------------------------------------------------------------ library */
int pd_abi_version(void);
/* Last error message of the calling thread (empty string if none). */
const char* pd_last_error(void);
int pd_device_sm_count(int device, int* out);

/* ------------------------------------------------------------------ kernels
 * One linear-layer pass as a GEMM with a fused epilogue; replaces the per-stage
 * numeric step of semantics._step (semantics.py:119-144) generalised to an MLP:
 *   C[M,N] = sum_k A(m,k) B(n,k);  A(m,k) = A[m*lda+k] (a_mn=0) or A[k*lda+m] (a_mn=1).
 * dtype PD_BF16 runs the tcgen05/TMEM/TMA kernel, PD_F32 the SIMT FFMA kernel. */
typedef struct pd_epilogue {
  int kind;             /* pd_epi_kind */
  void* out;            /* activation dtype (fp32 for GRADF32) */
  int64_t ldo;
  const float* bias;    /* STORE/LOSS: per-column bias or NULL */
  int relu;             /* STORE */
  const void* mask;     /* MASK: layer input X; out = acc * (X > 0) */
  int64_t ldm;
  const float* target;  /* LOSS: fp32 targets */
  int64_t ldt;
  float scale;          /* LOSS: out = (acc+bias-target)*scale, loss += 0.5*scale*sum(d^2) */
  float* loss;          /* LOSS: fp32 accumulator */
  float* master;        /* SGD: fp32 latest weights, master -= lr*acc, out = cast(master) */
  int64_t ldw;
  float lr;
  void* aux;            /* GELU: pre-activation output, ld = ldo */
} pd_epilogue;

int pd_gemm(int dtype, const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N,
            int K, const pd_epilogue* ep, void* stream);
/* Bias gradient + SGD: b_master[j] -= lr * sum_r dz[r*ld+j];  b_out[j] = b_master[j]. */
int pd_bias_sgd(int dtype, const void* dz, int rows, int cols, int64_t ld, float* b_master, float* b_out, float lr,
                void* stream);
/* master[i] -= lr*grad[i]; out[i] = cast(master[i]). */
int pd_sgd_update(int dtype, float* master, const float* grad, void* out, int64_t n, float lr, void* stream);
/* Replicated-stage allreduce fused with SGD, over peer memory: every replica reads all n_rep
 * gradient buffers (its own and the peers' mapped ones, summed in replica order so all
 * replicas compute bit-identical weights), then master -= lr*sum; out = cast(master). */
int pd_allreduce_sgd(int dtype, const float* const* grads, int n_rep, float* master, void* out, int64_t n, float lr,
                     void* stream);
/* out[j] = sum_r dz[r*ld+j] (bias gradient of a replicated stage). */
int pd_bias_grad(int dtype, const void* dz, int rows, int cols, int64_t ld, float* out, void* stream);
/* out[i] = cast(src[i]) (fp32 -> dtype). */
int pd_cast(int dtype, const float* src, void* out, int64_t n, void* stream);

/* ------------------------------------------------------------------ convolutional stages
 * VGG-style stages (configs[2]): 3x3 / stride 1 / pad 1 convolutions over NHWC bf16
 * activations with weights stored tap-major, Wt[9*c_in][c_out] (row = (r*3+s)*c_in + c), as
 * implicit GEMMs on the tcgen05 kernel whose activation operand is loaded by TMA im2col
 * (the zero-filled halo is the padding; no im2col matrix is written).
 *   PD_CONV_FWD  : act = X [n,h,w,c_in],  other = Wt;  ep STORE  -> out Y [n,h,w,c_out] (+bias, ReLU)
 *   PD_CONV_DGRAD: act = dY [n,h,w,c_out], other = Wt; ep MASK   -> out dX [n,h,w,c_in] * (X > 0)
 *   PD_CONV_WGRAD: act = X, other = dY;  ep GRADF32 -> out = split-K partials [splits][9*c_in][c_out]
 *                  (ldo = c_out; splits from pd_splitk_plan(9*c_in, c_out, n*h*w)), summed by pd_reduce_sgd
 *   PD_GEMM_WGRAD_SPLITK: act = cols [n*h*w, c_in] (the im2col'ed first layer), other = dY;
 *                  partials [splits][c_in][c_out] (pd_splitk_plan(c_in, c_out, n*h*w))
 * These replace the reference's per-stage numeric step (semantics.py:119-144) for conv layers. */
enum pd_conv_pass { PD_CONV_FWD = 0, PD_CONV_DGRAD = 1, PD_CONV_WGRAD = 2, PD_GEMM_WGRAD_SPLITK = 3 };
int pd_conv3x3(int pass, const void* act, const void* other, int n, int h, int w, int c_in, int c_out,
               const pd_epilogue* ep, void* stream);
int pd_splitk_plan(int M, int N, int K, int* splits);
/* 2x2/stride-2 max pool over NHWC bf16; argmax[n,h/2,w/2,c] = window index (dh*2+dw), first max wins. */
int pd_maxpool2(const void* x, void* y, uint8_t* argmax, int n, int h, int w, int c, void* stream);
int pd_maxpool2_bwd(const void* dy, const uint8_t* argmax, void* dx, int n, int h, int w, int c, void* stream);
/* First-layer im2col: cols[pix][(r*3+s)*c + ch] for k < 9c, zero up to kpad. */
int pd_im2col3(const void* x, void* cols, int n, int h, int w, int c, int kpad, void* stream);
/* g[i] = sum_{s<splits} part[s*stride+i] (fixed order); grad ? grad[i]=g : (master[i]-=lr*g; out[i]=cast(master[i])). */
int pd_reduce_sgd(int dtype, const float* part, int splits, int64_t stride, int64_t n, float* grad, float* master,
                  void* out, float lr, void* stream);
/* Bias gradient of a tall [rows, c] bf16 gradient (conv layers): two-pass column sum through
 * part[pd_colsum_blocks(rows,c) * c], then grad or SGD as pd_reduce_sgd. */
int pd_colsum_blocks(int64_t rows, int c);
int pd_bias_grad_tall(const void* dz, int64_t rows, int c, float* part, float* grad, float* master, float* out,
                      float lr, void* stream);
/* Softmax cross-entropy over fp32 logits [b, v] (row pitch ldz), int32 labels:
 * loss += mean_r (logsumexp_r - z[r,label_r]);  dz = (softmax - onehot) / b (bf16). */
int pd_softmax_ce(const float* logits, int64_t ldz, const int* labels, int b, int v, void* dz, int64_t ldd,
                  float* loss, void* stream);

/* ------------------------------------------------------------------ P2P transport
 * Replaces _Engine._send (simulator.py:284-292): payloads are stored by the
 * producing GEMM epilogue straight into the consumer's inbox slot (a peer-mapped
 * pointer when the consumer is on another GPU); these flags order them.
 * signal: system-scope release store of `value`; wait: acquire-poll until *flag >= value. */
int pd_flag_signal(int* flag, int value, void* stream);
/* SM-issued 16-byte-vector copy (dst may be a peer-mapped inbox): the store half of a hand-off. */
int pd_copy(void* dst, const void* src, int64_t bytes, void* stream);
int pd_flag_wait(const int* flag, int value, int* err_word, void* stream);
/* Copy-engine device->device (or peer-mapped) copy: the comparison leg of the P2P microbench. */
int pd_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* CUDA IPC so a peer process can map an inbox: handle is 64 opaque bytes naming the whole
 * allocation that contains dev_ptr; *offset_out is dev_ptr's byte offset inside it. */
int pd_ipc_get_handle(const void* dev_ptr, void* handle_out64, int64_t* offset_out);
int pd_ipc_open(const void* handle64, void** dev_ptr_out);
int pd_ipc_close(void* dev_ptr);
int pd_enable_peer_access(int peer_device);

/* ------------------------------------------------------------------ executor
 * Replaces _Engine.__init__/run/_try_start/_on_done (simulator.py:150-357) for the
 * workers (stage replicas) hosted by this process: executes a compiled 1F1B-RR program.
 *
 * Every inbox is owned by its receiving worker, together with its flags:
 *   ready[slot]  written by the producer after its epilogue stored the payload (peer store)
 *   ack[slot]    written by the receiver once the slot's backward no longer needs it
 * Producers in another process poll the receiver's ack before overwriting a slot, and
 * release-signal its ready after writing; in-process neighbours use CUDA events instead. */
typedef struct pd_stage_desc {
  int worker;               /* Schedule.worker_id(stage, replica) */
  int stage;                /* global stage index (0-based, plan order) */
  int replica;
  int rep;                  /* replication of this stage */
  int first_worker;         /* worker id of replica 0 of this stage */
  int n_layers;
  const int64_t* dims;      /* n_layers+1 widths: in of layer 0 .. out of layer n-1 */
  int batch;                /* minibatch size */
  int dtype;                /* pd_dtype of weights/activations */
  int is_first, is_last;
  int relu_last;            /* ReLU after the stage's last layer (all but the model output) */
  int ring_depth;           /* weight-version ring slots */
  int init_slot;            /* slot of version 0: refreshed from the masters at every run start */
  int act_depth;            /* activation-stash slots (in-flight minibatches) */
  int in_depth;             /* activation inbox slots (stage > 0) */
  int grad_depth;           /* gradient inbox slots (stage < n-1) */
  int n_data_blocks;
  int remote_prev;          /* some producer of my activation inbox lives in another process */
  int remote_next;          /* some producer of my gradient inbox lives in another process */
  float lr;
  /* per layer l: */
  float* const* w_master;   /* [n_layers]            fp32 [out,in] latest weights */
  float* const* b_master;   /* [n_layers]            fp32 [out] */
  void* const* w_ring;      /* [n_layers*ring_depth] dtype [out,in], index l*ring_depth+slot */
  float* const* b_ring;     /* [n_layers*ring_depth] fp32 [out] */
  void* const* act;         /* [(n_layers-1)*act_depth] dtype [batch, dims[l+1]], index l*act_depth+slot */
  void* const* act_in;      /* stage>0: [in_depth] dtype [batch, dims[0]]; stage 0: data blocks */
  void* const* grad_in;     /* stage<n-1: [grad_depth] dtype [batch, dims[n]] */
  void* const* dz_last;     /* last stage: [act_depth] dtype [batch, dims[n]] */
  const float* const* target; /* last stage: [n_data_blocks] fp32 [batch, dims[n]] */
  float* loss;              /* last stage: fp32 [num_minibatches+1] */
  void* tmp[2];             /* dtype [batch, max dim] gradient ping-pong */
  int* act_ready;           /* [in_depth]   my inbox flags */
  int* act_ack;             /* [in_depth] */
  int* grad_ready;          /* [grad_depth] */
  int* grad_ack;            /* [grad_depth] */
  /* replicated stages (rep > 1): this replica's round-parity gradient buffers and flags */
  float* const* red_grad;   /* [n_layers*2] fp32 [out,in] */
  float* const* red_bgrad;  /* [n_layers*2] fp32 [out] */
  int* red_ready;           /* last round whose gradients are complete here */
  int* red_done;            /* last round whose reduction has finished reading every replica */
  int* err_word;            /* device int, set non-zero by a timed-out flag wait */
  /* Layered stages (VGG-style conv / classifier stages).  layers == NULL: the MLP stage above
   * (Linear + ReLU per layer, MSE at the model output).  Otherwise n_layers descriptors; the
   * per-layer arrays above keep their meaning with
   *   weights  LINEAR [c_out, c_in];  CONV3 Wt [9*c_in, c_out] (im2col layer: [64, c_out]);
   *   act[l]   the layer's (pooled) output, [batch, out_features(l)] in NHWC order;
   *   tmp[2]   [batch, max pre-pool features] (forward pre-pool scratch / gradient ping-pong). */
  const struct pd_layer* layers;
  int loss_kind;            /* last stage: PD_LOSS_MSE (target = fp32 [batch, out]) or PD_LOSS_CE
                               (target = int32 labels [batch], logits below) */
  float* logits;            /* PD_LOSS_CE: fp32 [batch, classes] */
  float* part;              /* fp32 scratch for split-K partials and column-sum blocks (size from
                               pd_layer_scratch_floats) */
  int* sync;                /* 16 zeroed int32: self-resetting counters of single-launch reductions ([0])
                               and of the fused hand-off GEMMs ([8] forward, [9] backward) */
  /* Fused bias gradient (bf16 MLP stages with rep 1 and every width % 32 == 0): the GEMM that
   * writes a layer's output gradient dZ also writes fp32 column-sum partials [ceil(batch/32)][width]
   * of it, and the layer's wgrad+SGD GEMM applies the bias update from them (no separate bias
   * pass over dZ).  bpart[l], l < n_layers-1: partials of the inner layers' dZ (from this stage's
   * dgrad); grad_bpart[grad_depth]: one per gradient-inbox slot (written by the next stage's dgrad,
   * peer-mapped across processes); dz_bpart[act_depth]: the loss gradient's (last stage). */
  int fused_bias;
  float* const* bpart;
  float* const* grad_bpart;
  float* const* dz_bpart;
  /* Replicated stages: per-layer round flags of the sharded reduction (runtime.cu
   * issue_layer_reduce): red_lready[l] = last round whose layer-l gradient is complete here,
   * red_lupd[l] = last round whose layer-l shard this replica has reduced and applied. */
  int* red_lready;          /* [n_layers] */
  int* red_lupd;            /* [n_layers] */
} pd_stage_desc;

enum pd_layer_kind { PD_LAYER_LINEAR = 0, PD_LAYER_CONV3 = 1, PD_LAYER_EMBED = 2, PD_LAYER_BLOCK = 3, PD_LAYER_HEAD = 4 };
enum pd_loss_kind { PD_LOSS_MSE = 0, PD_LOSS_CE = 1 };

/* Transformer layers (GPT-2, configs[3]); T = batch * seq tokens, d = c_in:
 *   EMBED  c_in = padded vocab Vp, c_out = d, h = seq.  input int32 tokens [T];
 *          weights [wte Vp x d | wpe seq x d]; no biases.
 *   BLOCK  pre-LN transformer block, c_in = c_out = d, h = seq, w = heads (head dim 64), ffn.
 *          weights [Wqkv 3d x d | Wo d x d | W1 ffn x d | W2 d x ffn] ([out, in] each);
 *          biases  [bqkv 3d | bo d | b1 ffn | b2 d | ln1 gamma,beta 2d | ln2 gamma,beta 2d].
 *   HEAD   final LayerNorm + LM head + softmax cross-entropy over `vocab` of c_out = Vp logits;
 *          c_in = d, h = seq; weights [W Vp x d]; biases [lnf gamma,beta 2d]; the stage's target
 *          blocks are int32 next-token labels [T], dz_last holds dlogits [T, Vp], logits fp32 [T, Vp].
 * save[act_depth]: per in-flight minibatch tensors the backward needs (pd_layer_save_bytes);
 * work: per-stage backward scratch shared by the stage's layers (pd_layer_work_bytes). */
typedef struct pd_layer {
  int kind;                 /* pd_layer_kind */
  int relu;                 /* ReLU after the layer */
  int pool;                 /* CONV3: 2x2/2 max pool after the ReLU */
  int im2col;               /* CONV3 with c_in < 64 (the image layer): explicit im2col to 64 columns */
  int h, w;                 /* CONV3: input (= pre-pool output) spatial size; transformer: seq, heads */
  int c_in, c_out;          /* channels (CONV3) or features (LINEAR); see above for transformer kinds */
  uint8_t* const* argmax;   /* pool: [act_depth] uint8 [batch, h/2, w/2, c_out] */
  void* const* cols;        /* im2col: [act_depth] dtype [batch*h*w, 64] */
  int ffn;                  /* BLOCK: hidden width */
  int vocab;                /* HEAD: valid vocabulary (<= c_out) */
  void* const* save;        /* transformer kinds: [act_depth] saved tensors */
  void* work;               /* transformer kinds: backward scratch */
} pd_layer;

/* fp32 elements the stage's `part` scratch needs for this layer (split-K partials of the weight
 * gradient, then the bias column-sum blocks; the larger of the two). */
int64_t pd_layer_scratch_floats(const pd_layer* layer, int batch);
/* Bytes of one `save` slot and of the `work` scratch of a transformer layer (0 for others). */
int64_t pd_layer_save_bytes(const pd_layer* layer, int batch);
int64_t pd_layer_work_bytes(const pd_layer* layer, int batch);
/* Transformer kernels (also used by the runtime): causal flash attention (head dim 64),
 * LayerNorm, embeddings, vocabulary-padded cross-entropy.  See csrc/attention.cu, transformer.cu. */
int pd_attention_fwd(const void* qkv, void* out, float* lse, int batch, int seq, int heads, void* stream);
int pd_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* dvec,
                     float* dq_acc, void* dqkv, int batch, int seq, int heads, void* stream);
int pd_layernorm_fwd(const void* x, const float* gb, void* y, float* mean, float* rstd, int64_t rows, int d,
                     void* stream);
int pd_layernorm_bwd_blocks(int64_t rows);
int pd_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* gb,
                     const void* dres, void* dx, float* part, int64_t rows, int d, void* stream);
int pd_embedding_fwd(const int* tok, const void* wte, const void* wpe, void* x, int64_t tokens, int seq, int d,
                     void* stream);
int pd_embedding_bwd(const int* tok, const void* dx, float* gte, float* gpe, int64_t tokens, int seq, int d,
                     void* stream);
int pd_softmax_ce_vocab(const float* logits, int64_t ldz, const int* labels, int64_t rows, int v, int vpad, void* dz,
                        int64_t ldd, float* loss, void* stream);

/* What any worker (in this process or a peer-mapped one in another) exposes to the others. */
typedef struct pd_worker_view {
  int worker;
  int remote;               /* 1: pointers below are peer mappings of another process's memory */
  int in_depth, grad_depth, n_layers;
  void* const* act_in;      /* [in_depth] */
  void* const* grad_in;     /* [grad_depth] */
  int* act_ready; int* act_ack; int* grad_ready; int* grad_ack;
  float* const* red_grad;   /* [n_layers*2] */
  float* const* red_bgrad;  /* [n_layers*2] */
  int* red_ready; int* red_done;
  int fused_bias;           /* the worker consumes bias partials (pd_stage_desc.fused_bias) */
  float* const* grad_bpart; /* [grad_depth]: partials of its gradient-inbox slots */
  /* replicated stages: the replica's fp32 masters (all-gather source) and per-layer round flags */
  float* const* w_master;   /* [n_layers] */
  float* const* b_master;   /* [n_layers] */
  int* red_lready; int* red_lupd;  /* [n_layers] each */
} pd_worker_view;

/* Program item: PD_ITEM_WIDTH int32 fields, see program.py:compile_program. */
#define PD_ITEM_WIDTH 20
enum pd_item_field {
  PD_IT_OP = 0,        /* 0 forward, 1 backward, 2 reduce (replicated stage: sum replicas, SGD, commit) */
  PD_IT_STAGE = 1,
  PD_IT_MB = 2,        /* 1-based minibatch id */
  PD_IT_WORKER = 3,
  PD_IT_VERSION = 4,   /* weight version read (ledger value) */
  PD_IT_WSLOT = 5,     /* ring slot holding that version */
  PD_IT_WNEW = 6,      /* ring slot receiving the committed version (-1: none) */
  PD_IT_ACT = 7,       /* activation-stash slot of this minibatch */
  PD_IT_XSLOT = 8,     /* inbox slot of the stage input (stage 0: data block) */
  PD_IT_GSLOT = 9,     /* backward: gradient inbox slot (-1 at the last stage) */
  PD_IT_OUT = 10,      /* forward: slot in dst's activation inbox; backward: slot in dst's gradient inbox */
  PD_IT_BLOCK = 11,    /* data / target block */
  PD_IT_DEP = 12,      /* in-process producer item (index), -1 */
  PD_IT_WAR = 13,      /* in-process item that must finish before PD_IT_OUT is overwritten, -1 */
  PD_IT_RWAIT = 14,    /* cross-process: my inbox ready value to wait for (0 = none) */
  PD_IT_AWAIT = 15,    /* cross-process: dst's ack value to wait for before writing PD_IT_OUT (0 = none) */
  PD_IT_DST = 16,      /* worker receiving PD_IT_OUT (-1) */
  PD_IT_SRC = 17,      /* worker that produced this item's input (-1) */
  PD_IT_ROUND = 18     /* replicated stage: allreduce round of this backward / reduce (0 otherwise) */
};

typedef struct pd_runtime pd_runtime;
typedef struct pd_record { int32_t item; int32_t pad; double t_start_ms; double t_end_ms; } pd_record;

int pd_rt_create(int device, pd_runtime** out);
int pd_rt_add_stage(pd_runtime* rt, const pd_stage_desc* desc);
/* Register the view of every worker of the plan (hosted here or peer-mapped). */
int pd_rt_add_view(pd_runtime* rt, const pd_worker_view* view);
int pd_rt_load_program(pd_runtime* rt, const int32_t* items, int n_items);
/* Enqueue the whole program behind `stream` (everything joins back onto it).
 * trace=1 records per-item device timestamps (pd_rt_records). */
int pd_rt_run(pd_runtime* rt, void* stream, int trace);
int pd_rt_records(pd_runtime* rt, pd_record* out, int cap, int* n_out);
/* Device pass records of traced runs (replaces the reference's ledger.record at pass start,
 * simulator.py:256-264, and its trace, :266-282, with what the device observed).
 * rec: caller-owned device int64 [(1 + cap) * PD_REC_WIDTH]; row 0 holds the run's start
 * %globaltimer (ns, comparable across the GPUs of a node), row 1 + i the record of program
 * item i: PD_REC_T0 / PD_REC_T1 %globaltimer at the pass's start / end, PD_REC_VER0 / PD_REC_VER1
 * the version tag of the weight ring slot the pass reads at its start / end, PD_REC_BYTES payload
 * bytes stored into another process's inbox (counted by the storing kernel), PD_REC_COMMIT the
 * version the pass committed (-1: none).  tags: caller-owned device int32 [64 * hosted workers],
 * the version held by each ring slot (written in stream order after the committing kernels).
 * NULL rec switches the records off. */
#define PD_REC_WIDTH 8
/* Row 0: [0] run-start %globaltimer, [1] bytes the replicated stages' sharded reductions read from
 * other replicas' memory during the run (counted by the reduction kernels). */
enum pd_rec_field { PD_REC_T0 = 0, PD_REC_T1 = 1, PD_REC_VER0 = 2, PD_REC_VER1 = 3, PD_REC_BYTES = 4,
                    PD_REC_COMMIT = 5 };
int pd_rt_set_records(pd_runtime* rt, int64_t* rec, int cap, int32_t* tags);
/* The (cg, bn) tile configuration the tcgen05 GEMM dispatch picks for a problem: cg 1 = one CTA
 * per 128 x bn tile, 2 = a CTA pair per 256 x bn tile (tests pin the bench's instantiations). */
int pd_gemm_pick(int M, int N, int K, int a_mn, int b_mn, int kind, int* cg, int* bn);
/* serial=1: every hosted stage issues on one stream in program order (single-GPU mode;
 * the per-item dependencies are then satisfied by stream order). */
int pd_rt_set_serial(pd_runtime* rt, int on);
/* graph=1: single-process programs are captured into a CUDA graph on the next run and
 * replayed afterwards (runs with tracing, kernel timing or cross-process flags launch directly). */
int pd_rt_set_graph(pd_runtime* rt, int on);
/* Per-kernel CUDA-event timing on the launching stage stream (resets the counters).
 * stats: n_classes (<= 8) classes x {launches, total ms, algorithmic flops}; classes are
 * 0 forward GEMM, 1 dgrad GEMM, 2 wgrad(+SGD) GEMM, 3 attention, 4 LayerNorm, 5 loss,
 * 6 update/reduction (bias sums, split-K / allreduce + SGD), 7 other (pool, im2col, embedding, cast). */
int pd_rt_kernel_timing(pd_runtime* rt, int on);
int pd_rt_kernel_stats(pd_runtime* rt, int worker, double* out, int n_classes);  /* worker -1: all */
/* Per-layer timing (the layer profiler): %globaltimer stamps around every layer's forward and
 * backward on the stage stream, into the caller's device buffer ts[2*cap] (NULL: off); works in
 * graph replay.  stats = average ms per pass, out[2*l] forward, out[2*l+1] backward. */
int pd_rt_layer_timing(pd_runtime* rt, uint64_t* ts, int cap);
int pd_rt_layer_stats(pd_runtime* rt, int worker, int n_layers, double* out);
/* Kernels of this library launched by the runtime since creation. */
int pd_rt_launch_count(pd_runtime* rt, int64_t* out);
int pd_rt_destroy(pd_runtime* rt);

#ifdef __cplusplus
}
#endif
#endif /* PD_B200_H */
