// Internal declarations shared by the CUDA translation units of libpd_b200.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pd_b200.h"
#include "epilogue.cuh"

namespace pd {

// Records the message for pd_last_error() and returns `code`.
int set_error(int code, const char* fmt, ...);

int gemm_bf16_tc(const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N,
                 int K, int kind, const EpiArgs& ep, cudaStream_t st);
int gemm_simt(int dtype, const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N,
              int K, int kind, const EpiArgs& ep, cudaStream_t st);

// Dispatch: bf16 -> tcgen05, fp32 -> SIMT.
int gemm(int dtype, const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N, int K,
         int kind, const EpiArgs& ep, cudaStream_t st);

// Implicit-GEMM 3x3 convolution passes (PD_CONV_*), and the split-K plan they share.
int conv3x3_tc(int pass, const void* act, const void* other, int n, int H, int W, int cin, int cout, int kind,
               const EpiArgs& ep, cudaStream_t st);
int splitk_plan(int M, int N, int K, int* splits, int* kb_per);
int maxpool_fwd(const void* x, void* y, uint8_t* arg, int n, int H, int W, int C, cudaStream_t st);
int maxpool_bwd(const void* dy, const uint8_t* arg, void* dx, int n, int H, int W, int C, cudaStream_t st);
int im2col3(const void* x, void* cols, int n, int H, int W, int C, int kpad, cudaStream_t st);
int reduce_sgd(int out_dtype, const float* part, int S, int64_t stride, int64_t n, float* grad, float* master,
               void* out, float lr, cudaStream_t st);
int colsum_blocks(int64_t rows, int C);
// counter != nullptr: single launch, the last block reduces and applies (self-resetting int).
int bias_grad_tall(const void* dz, int64_t rows, int C, float* part, float* grad, float* master, float* out, float lr,
                   cudaStream_t st, int* counter = nullptr);
int softmax_ce(const float* logits, int64_t ldz, const int* labels, int B, int V, void* dz, int64_t ldd, float* loss,
               cudaStream_t st);

int attn_fwd(const void* qkv, void* out, float* lse, int B, int S, int H, cudaStream_t st);
int attn_fwd_tc(const void* qkv, void* out, float* lse, int B, int S, int H, cudaStream_t st);
int attn_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* Dv, float* dq_acc, void* dqkv, int B,
                int S, int H, cudaStream_t st);
int attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* Dv, float* dq_acc,
             void* dqkv, int B, int S, int H, cudaStream_t st);
int ln_fwd(const void* x, const float* gb, void* y, float* mean, float* rstd, int64_t T, int D, cudaStream_t st);
int ln_bwd_blocks(int64_t T);
// counter != nullptr: the last block sums the gamma/beta partials and applies SGD to master/out.
int ln_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* gb, const void* dres,
           void* dx, float* part, int64_t T, int D, cudaStream_t st, int* counter = nullptr, float* master = nullptr,
           float* out = nullptr, float lr = 0.f);
int embed_fwd(const int* tok, const void* wte, const void* wpe, void* x, int64_t T, int S, int D, cudaStream_t st);
int embed_bwd(const int* tok, const void* dx, float* gte, float* gpe, int64_t T, int S, int D, cudaStream_t st);
int softmax_ce_v(const float* logits, int64_t ldz, const int* labels, int64_t rows, int V, int Vp, void* dz,
                 int64_t ldd, float* loss, cudaStream_t st);

int bias_sgd(int dtype, const void* dz, int rows, int cols, int64_t ld, float* b_master, float* b_out, float lr,
             cudaStream_t st);
int sgd_update(int dtype, float* master, const float* grad, void* out, int64_t n, float lr, cudaStream_t st);
int allreduce_sgd(int dtype, const float* const* grads, int n_rep, float* master, void* out, int64_t n, float lr,
                  cudaStream_t st);
int bias_grad(int dtype, const void* dz, int rows, int cols, int64_t ld, float* out, cudaStream_t st);
// Sharded replica reduction (kernels.cu): reduce-scatter + SGD of this replica's shard, then the
// all-gather of the other owners' updated master shards.  peer_bytes: nullable byte counter.
int64_t shard_size(int64_t n, int R);
int shard_rs_sgd(int dtype, const float* const* grads, int R, int self, float* master, void* out, int64_t n, float lr,
                 unsigned long long* peer_bytes, cudaStream_t st);
int shard_ag(int dtype, const float* const* masters, int R, int self, float* master, void* out, int64_t n,
             unsigned long long* peer_bytes, cudaStream_t st);
int cast_f32(int dtype, const float* src, void* out, int64_t n, cudaStream_t st);
int flag_signal(int* flag, int value, cudaStream_t st);
int timestamp(uint64_t* p, cudaStream_t st);  // *p = %globaltimer (ns) when the stream reaches it
int rec_begin(int64_t* rec, const int* tag, cudaStream_t st);
int rec_end(int64_t* rec, const int* tag, int* commit_tag, int commit_v, int64_t host_bytes, cudaStream_t st);
int set_tags(int* tags, int n, int slot, int v, cudaStream_t st);  // tags[slot] = v, others -1
int flag_wait(const int* flag, int value, int* err_word, cudaStream_t st);

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while its
// stream predecessor drains; it must call griddep_wait() (ptx.cuh) before reading earlier results.
// PD_PDL=1 in the environment enables programmatic dependent launch (default off, kernels.cu).
bool pdl_enabled();

// Kernel timing (pd_rt_kernel_timing): the runtime records a start event, then sets g_pre_launch to
// it; the first kernel launch of the timed call re-records it right before cudaLaunchKernelEx, so
// the measured interval excludes the host's launch preparation (tensor-map encoding etc.), which
// would otherwise be counted whenever the GPU is ahead of the host.
extern thread_local cudaEvent_t g_pre_launch;
inline void mark_pre_launch(cudaStream_t st) {
  if (g_pre_launch) {
    cudaEventRecord(g_pre_launch, st);
    g_pre_launch = nullptr;
  }
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  mark_pre_launch(st);
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

inline EpiArgs to_epi(const pd_epilogue& e) {
  EpiArgs a{};
  a.out = e.out; a.ldo = e.ldo; a.bias = e.bias; a.relu = e.relu; a.mask = e.mask; a.ldm = e.ldm;
  a.target = e.target; a.ldt = e.ldt; a.scale = e.scale; a.loss = e.loss; a.master = e.master;
  a.ldw = e.ldw; a.lr = e.lr; a.aux = e.aux;
  return a;
}

}  // namespace pd
