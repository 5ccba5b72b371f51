// Elementwise / reduction kernels, cross-GPU flags, error state and the C ABI wrappers
// for single kernels (include/pd_b200.h).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>

#include "pd_internal.h"
#include "ptx.cuh"

namespace pd {

thread_local cudaEvent_t g_pre_launch = nullptr;  // pd_internal.h: kernel-timing start event

static thread_local char g_err[1024] = {0};

// Programmatic dependent launch is opt-in (PD_PDL=1): with several stage streams replayed from
// one CUDA graph it measured slower (GPT-2: 290 vs 294 seq/s) and one run in five hung, so the
// default launches fully serialized kernels.  The kernels keep their griddepcontrol.wait, which
// returns at once for a normally launched grid.
bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PD_PDL");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int gemm(int dtype, const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N, int K,
         int kind, const EpiArgs& ep, cudaStream_t st) {
  if (dtype == PD_BF16) return gemm_bf16_tc(A, a_mn, lda, B, b_mn, ldb, M, N, K, kind, ep, st);
  if (dtype == PD_F32) return gemm_simt(PD_F32, A, a_mn, lda, B, b_mn, ldb, M, N, K, kind, ep, st);
  return set_error(PD_ERR_INVALID, "unknown dtype %d", dtype);
}

// ---------------------------------------------------------------- bias gradient + SGD
// Block = 32 columns x 16 row groups; coalesced across the 32 lanes of each row.
template <typename T>
__global__ void __launch_bounds__(512)
    k_bias_sgd(const T* __restrict__ dz, int rows, int cols, int64_t ld, float* __restrict__ bm,
               float* __restrict__ bo, float lr) {
  __shared__ float part[16][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < cols)
    for (int r = grp; r < rows; r += 16) s += to_f<T>(dz[(int64_t)r * ld + c]);
  part[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int g = 0; g < 16; ++g) t += part[g][lane];
    const float b = bm[c] - lr * t;
    bm[c] = b;
    bo[c] = b;
  }
}

// bf16 with cols % 64 == 0: block = 64 columns; 8 lanes x 16 B cover a row segment, 64 row lanes,
// four independent 16-byte loads in flight per thread (a [2048 x 8192] gradient: 128 blocks).
__global__ void __launch_bounds__(512)
    k_bias_sgd_v(const __nv_bfloat16* __restrict__ dz, int rows, int64_t ld, float* __restrict__ bm,
                 float* __restrict__ bo, float lr) {
  __shared__ float part[64][65];
  const int cl = threadIdx.x & 7, rl = threadIdx.x >> 3;  // column lane (8 cols), row lane (0..63)
  const int64_t c0 = blockIdx.x * 64 + cl * 8;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int r = rl;
  for (; r + 192 < rows; r += 256) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const uint4*>(dz + (int64_t)(r + 64 * u) * ld + c0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float a, b;
        unpack_bf16x2(w[j], a, b);
        acc[2 * j] += a;
        acc[2 * j + 1] += b;
      }
    }
  }
  for (; r < rows; r += 64) {
    const uint4 v = *reinterpret_cast<const uint4*>(dz + (int64_t)r * ld + c0);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float a, b;
      unpack_bf16x2(w[j], a, b);
      acc[2 * j] += a;
      acc[2 * j + 1] += b;
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) part[rl][cl * 8 + j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 64) {
    float t = 0.f;
    for (int g = 0; g < 64; ++g) t += part[g][threadIdx.x];
    const int64_t c = blockIdx.x * 64 + threadIdx.x;
    const float b = bm[c] - lr * t;
    bm[c] = b;
    bo[c] = b;
  }
}

int bias_sgd(int dtype, const void* dz, int rows, int cols, int64_t ld, float* b_master, float* b_out, float lr,
             cudaStream_t st) {
  if (dtype == PD_BF16 && cols % 64 == 0 && ld % 8 == 0 && (reinterpret_cast<uintptr_t>(dz) & 15) == 0) {
    k_bias_sgd_v<<<cols / 64, 512, 0, st>>>(static_cast<const __nv_bfloat16*>(dz), rows, ld, b_master, b_out, lr);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "bias_sgd: %s", cudaGetErrorString(e));
  }
  dim3 grid((cols + 31) / 32);
  if (dtype == PD_BF16)
    k_bias_sgd<__nv_bfloat16><<<grid, 512, 0, st>>>(static_cast<const __nv_bfloat16*>(dz), rows, cols, ld,
                                                     b_master, b_out, lr);
  else
    k_bias_sgd<float><<<grid, 512, 0, st>>>(static_cast<const float*>(dz), rows, cols, ld, b_master, b_out, lr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "bias_sgd: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------- SGD on a flat buffer
template <typename T>
__global__ void k_sgd(float* __restrict__ m, const float* __restrict__ g, T* __restrict__ o, int64_t n, float lr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float w = m[i] - lr * g[i];
    m[i] = w;
    o[i] = from_f<T>(w);
  }
}

int sgd_update(int dtype, float* master, const float* grad, void* out, int64_t n, float lr, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * 8;
  if (dtype == PD_BF16)
    k_sgd<__nv_bfloat16><<<grid, 256, 0, st>>>(master, grad, static_cast<__nv_bfloat16*>(out), n, lr);
  else
    k_sgd<float><<<grid, 256, 0, st>>>(master, grad, static_cast<float*>(out), n, lr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "sgd_update: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------- replicated stages
constexpr int PD_MAX_REP = 16;
struct GradPtrs { const float* p[PD_MAX_REP]; };

// Sum of every replica's gradient (peer-mapped loads over NVLink for the remote ones), fused
// with the SGD step.  Fixed summation order r = 0..R-1 -> every replica gets identical weights.
template <typename T>
__global__ void __launch_bounds__(256)
    k_allreduce_sgd(GradPtrs g, int R, float* __restrict__ m, T* __restrict__ o, int64_t n, float lr) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 s = reinterpret_cast<const float4*>(g.p[0])[i];
    for (int r = 1; r < R; ++r) {
      const float4 t = reinterpret_cast<const float4*>(g.p[r])[i];
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    float4 w = reinterpret_cast<float4*>(m)[i];
    w.x -= lr * s.x; w.y -= lr * s.y; w.z -= lr * s.z; w.w -= lr * s.w;
    reinterpret_cast<float4*>(m)[i] = w;
    o[4 * i] = from_f<T>(w.x); o[4 * i + 1] = from_f<T>(w.y);
    o[4 * i + 2] = from_f<T>(w.z); o[4 * i + 3] = from_f<T>(w.w);
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < R; ++r) s += g.p[r][i];
    const float w = m[i] - lr * s;
    m[i] = w;
    o[i] = from_f<T>(w);
  }
}

int allreduce_sgd(int dtype, const float* const* grads, int n_rep, float* master, void* out, int64_t n, float lr,
                  cudaStream_t st) {
  if (n_rep < 1 || n_rep > PD_MAX_REP) return set_error(PD_ERR_INVALID, "allreduce_sgd: %d replicas", n_rep);
  GradPtrs g{};
  for (int r = 0; r < n_rep; ++r) g.p[r] = grads[r];
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dtype == PD_BF16)
    k_allreduce_sgd<__nv_bfloat16><<<sms * 8, 256, 0, st>>>(g, n_rep, master, static_cast<__nv_bfloat16*>(out), n, lr);
  else
    k_allreduce_sgd<float><<<sms * 8, 256, 0, st>>>(g, n_rep, master, static_cast<float*>(out), n, lr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "allreduce_sgd: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------- sharded replica reduction
// A replicated stage's round-k update as reduce-scatter + all-gather over peer memory, issued per
// layer as soon as every replica's layer gradient exists (runtime.cu issue_layer_reduce), so it
// runs under the remaining backward.  Replica `self` owns the shard [self*shard, (self+1)*shard):
//   step 1 (k_shard_rs_sgd): sum the R replicas' fp32 gradients of its shard in replica order
//          0..R-1, master -= lr * sum, ring (new version) = cast(master);
//   step 2 (k_shard_ag): copy every other owner's updated master shard, ring = cast.
// Every element is summed once, by its owner, in a fixed order, so all replicas end bit-identical
// (the same arithmetic as k_allreduce_sgd, which every replica ran over the whole tensor).
// Peer traffic per replica and round: (R-1)/R of the gradient in step 1 plus (R-1)/R of the
// master in step 2 = 2 (R-1)/R x 4 B per parameter (k_allreduce_sgd read (R-1) x 4 B).
// peer_bytes (nullable) accumulates the bytes each kernel loaded from other replicas' memory.
__device__ __forceinline__ void add_peer_bytes(unsigned long long* ctr, unsigned long long v) {
  if (!ctr) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr, v);
}

template <typename T>
__global__ void __launch_bounds__(256)
    k_shard_rs_sgd(GradPtrs g, int R, int self, float* __restrict__ m, T* __restrict__ o, int64_t lo, int64_t hi,
                   float lr, unsigned long long* peer_bytes) {
  unsigned long long nb = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t lo4 = lo / 4, hi4 = hi / 4;  // lo is a multiple of 4
  for (int64_t i = lo4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi4; i += stride) {
    float4 s = reinterpret_cast<const float4*>(g.p[0])[i];
    for (int r = 1; r < R; ++r) {
      const float4 t = reinterpret_cast<const float4*>(g.p[r])[i];
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    nb += (unsigned long long)(R - 1) * 16;
    float4 w = reinterpret_cast<float4*>(m)[i];
    w.x -= lr * s.x; w.y -= lr * s.y; w.z -= lr * s.z; w.w -= lr * s.w;
    reinterpret_cast<float4*>(m)[i] = w;
    o[4 * i] = from_f<T>(w.x); o[4 * i + 1] = from_f<T>(w.y);
    o[4 * i + 2] = from_f<T>(w.z); o[4 * i + 3] = from_f<T>(w.w);
  }
  for (int64_t i = 4 * hi4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += stride) {
    float s = 0.f;
    for (int r = 0; r < R; ++r) s += g.p[r][i];
    nb += (unsigned long long)(R - 1) * 4;
    const float w = m[i] - lr * s;
    m[i] = w;
    o[i] = from_f<T>(w);
  }
  add_peer_bytes(peer_bytes, nb);
}

template <typename T>
__global__ void __launch_bounds__(256)
    k_shard_ag(GradPtrs masters, int self, float* __restrict__ m, T* __restrict__ o, int64_t n, int64_t shard,
               unsigned long long* peer_bytes) {
  unsigned long long nb = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n / 4;  // shard is a multiple of 4, so a float4 never straddles two owners
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const int q = (int)((4 * i) / shard);
    if (q == self) continue;
    const float4 w = reinterpret_cast<const float4*>(masters.p[q])[i];
    nb += 16;
    reinterpret_cast<float4*>(m)[i] = w;
    o[4 * i] = from_f<T>(w.x); o[4 * i + 1] = from_f<T>(w.y);
    o[4 * i + 2] = from_f<T>(w.z); o[4 * i + 3] = from_f<T>(w.w);
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int q = (int)(i / shard);
    if (q == self) continue;
    const float w = masters.p[q][i];
    nb += 4;
    m[i] = w;
    o[i] = from_f<T>(w);
  }
  add_peer_bytes(peer_bytes, nb);
}

int64_t shard_size(int64_t n, int R) { return ((n + R - 1) / R + 3) / 4 * 4; }

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

int shard_rs_sgd(int dtype, const float* const* grads, int R, int self, float* master, void* out, int64_t n, float lr,
                 unsigned long long* peer_bytes, cudaStream_t st) {
  if (R < 2 || R > PD_MAX_REP || self < 0 || self >= R) return set_error(PD_ERR_INVALID, "shard_rs_sgd: %d/%d", self, R);
  GradPtrs g{};
  for (int r = 0; r < R; ++r) g.p[r] = grads[r];
  const int64_t sh = shard_size(n, R);
  const int64_t lo = std::min<int64_t>(n, self * sh), hi = std::min<int64_t>(n, lo + sh);
  if (hi <= lo) return 0;
  const int grid = (int)std::min<int64_t>((int64_t)sm_count() * 4, ((hi - lo) / 4 + 255) / 256 + 1);
  if (dtype == PD_BF16)
    k_shard_rs_sgd<__nv_bfloat16><<<grid, 256, 0, st>>>(g, R, self, master, static_cast<__nv_bfloat16*>(out), lo, hi,
                                                         lr, peer_bytes);
  else
    k_shard_rs_sgd<float><<<grid, 256, 0, st>>>(g, R, self, master, static_cast<float*>(out), lo, hi, lr, peer_bytes);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "shard_rs_sgd: %s", cudaGetErrorString(e));
}

int shard_ag(int dtype, const float* const* masters, int R, int self, float* master, void* out, int64_t n,
             unsigned long long* peer_bytes, cudaStream_t st) {
  if (R < 2 || R > PD_MAX_REP || self < 0 || self >= R) return set_error(PD_ERR_INVALID, "shard_ag: %d/%d", self, R);
  GradPtrs g{};
  for (int r = 0; r < R; ++r) g.p[r] = masters[r];
  const int64_t sh = shard_size(n, R);
  const int grid = (int)std::min<int64_t>((int64_t)sm_count() * 4, (n / 4 + 255) / 256 + 1);
  if (dtype == PD_BF16)
    k_shard_ag<__nv_bfloat16><<<grid, 256, 0, st>>>(g, self, master, static_cast<__nv_bfloat16*>(out), n, sh, peer_bytes);
  else
    k_shard_ag<float><<<grid, 256, 0, st>>>(g, self, master, static_cast<float*>(out), n, sh, peer_bytes);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "shard_ag: %s", cudaGetErrorString(e));
}

template <typename T>
__global__ void __launch_bounds__(512)
    k_bias_grad(const T* __restrict__ dz, int rows, int cols, int64_t ld, float* __restrict__ out) {
  __shared__ float part[16][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < cols)
    for (int r = grp; r < rows; r += 16) s += to_f<T>(dz[(int64_t)r * ld + c]);
  part[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) t += part[q][lane];
    out[c] = t;
  }
}

int bias_grad(int dtype, const void* dz, int rows, int cols, int64_t ld, float* out, cudaStream_t st) {
  dim3 grid((cols + 31) / 32);
  if (dtype == PD_BF16)
    k_bias_grad<__nv_bfloat16><<<grid, 512, 0, st>>>(static_cast<const __nv_bfloat16*>(dz), rows, cols, ld, out);
  else
    k_bias_grad<float><<<grid, 512, 0, st>>>(static_cast<const float*>(dz), rows, cols, ld, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "bias_grad: %s", cudaGetErrorString(e));
}

template <typename T>
__global__ void k_cast(const float* __restrict__ src, T* __restrict__ o, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = from_f<T>(src[i]);
}

int cast_f32(int dtype, const float* src, void* out, int64_t n, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dtype == PD_BF16)
    k_cast<__nv_bfloat16><<<sms * 8, 256, 0, st>>>(src, static_cast<__nv_bfloat16*>(out), n);
  else
    k_cast<float><<<sms * 8, 256, 0, st>>>(src, static_cast<float*>(out), n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "cast: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------- payload copy (P2P microbench)
__global__ void __launch_bounds__(256) k_copy16(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int copy_bytes(void* dst, const void* src, int64_t bytes, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | (uintptr_t)bytes) & 15)
    return set_error(PD_ERR_INVALID, "copy: 16-byte alignment required");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n16 = bytes / 16;
  const int64_t want = (n16 + 255) / 256;
  const int grid = (int)(want < sms * 4 ? (want > 0 ? want : 1) : sms * 4);
  k_copy16<<<grid, 256, 0, st>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "copy: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------- flags
__global__ void k_flag_signal(int* flag, int v) {
  __threadfence_system();
  st_release_sys(flag, v);
}

// Bounded spin: ~10 s at %globaltimer resolution, then report through err_word so the host
// raises SimulationError instead of hanging the GPU.  Flag values grow monotonically modulo 2^32
// (epoch * 65536 + minibatch, runtime.cu flag_val), so "reached" is a wrap-safe signed difference.
__global__ void k_flag_wait(const int* flag, int v, int* err) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (flag_before(ld_acquire_sys(const_cast<volatile int*>(flag)), v)) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 10ull * 1000 * 1000 * 1000) {
      if (err) atomicExch(err, v);
      break;
    }
    __nanosleep(200);
  }
}

__global__ void k_timestamp(uint64_t* p) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *p = t;
}

// Device pass records (traced runs): each program item gets two one-thread kernels on its
// worker's stream, bracketing the item's kernels.  Record layout (int64 x PD_REC_WIDTH):
//   [0] %globaltimer at the start, [1] at the end (ns);
//   [2] version tag of the weight ring slot the pass reads (wslot) when it starts,
//   [3] the same tag when it ends (differs only if the slot was overwritten under the pass);
//   [4] payload bytes stored into another process's inbox (counted by the storing kernel),
//   [5] version committed (tag written into slot wnew), -1 if none.
// Ring-slot tags are written only here, in stream order after the committing kernels, so a tag
// names the version the slot holds for every later kernel of the same worker.
__global__ void k_rec_begin(int64_t* rec, const int* tag) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  rec[0] = (int64_t)t;
  rec[2] = tag ? *tag : -1;
  rec[4] = 0;
  rec[5] = -1;
}
__global__ void k_rec_end(int64_t* rec, const int* tag, int* commit_tag, int commit_v, int64_t host_bytes) {
  rec[3] = tag ? *tag : -1;
  if (commit_tag) {
    *commit_tag = commit_v;
    rec[5] = commit_v;
  }
  if (host_bytes) rec[4] += host_bytes;
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  rec[1] = (int64_t)t;
}
int rec_begin(int64_t* rec, const int* tag, cudaStream_t st) {
  k_rec_begin<<<1, 1, 0, st>>>(rec, tag);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "rec_begin: %s", cudaGetErrorString(e));
}
int rec_end(int64_t* rec, const int* tag, int* commit_tag, int commit_v, int64_t host_bytes, cudaStream_t st) {
  k_rec_end<<<1, 1, 0, st>>>(rec, tag, commit_tag, commit_v, host_bytes);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "rec_end: %s", cudaGetErrorString(e));
}
__global__ void k_set_tags(int* tags, int n, int slot, int v) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) tags[i] = i == slot ? v : -1;
}
int set_tags(int* tags, int n, int slot, int v, cudaStream_t st) {
  k_set_tags<<<1, 64, 0, st>>>(tags, n, slot, v);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "set_tags: %s", cudaGetErrorString(e));
}

int timestamp(uint64_t* p, cudaStream_t st) {
  k_timestamp<<<1, 1, 0, st>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "timestamp: %s", cudaGetErrorString(e));
}

int flag_signal(int* flag, int value, cudaStream_t st) {
  k_flag_signal<<<1, 1, 0, st>>>(flag, value);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "flag_signal: %s", cudaGetErrorString(e));
}
int flag_wait(const int* flag, int value, int* err_word, cudaStream_t st) {
  k_flag_wait<<<1, 1, 0, st>>>(flag, value, err_word);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "flag_wait: %s", cudaGetErrorString(e));
}

}  // namespace pd

// ==================================================================== C ABI
using namespace pd;

extern "C" {

int pd_abi_version(void) { return PD_ABI_VERSION; }
const char* pd_last_error(void) { return g_err; }

int pd_device_sm_count(int device, int* out) {
  cudaError_t e = cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device);
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "sm count: %s", cudaGetErrorString(e));
}

int pd_gemm(int dtype, const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N,
            int K, const pd_epilogue* ep, void* stream) {
  if (!ep) return set_error(PD_ERR_INVALID, "pd_gemm: null epilogue");
  return gemm(dtype, A, a_mn, lda, B, b_mn, ldb, M, N, K, ep->kind, to_epi(*ep), static_cast<cudaStream_t>(stream));
}

int pd_bias_sgd(int dtype, const void* dz, int rows, int cols, int64_t ld, float* b_master, float* b_out, float lr,
                void* stream) {
  return bias_sgd(dtype, dz, rows, cols, ld, b_master, b_out, lr, static_cast<cudaStream_t>(stream));
}

int pd_sgd_update(int dtype, float* master, const float* grad, void* out, int64_t n, float lr, void* stream) {
  return sgd_update(dtype, master, grad, out, n, lr, static_cast<cudaStream_t>(stream));
}

int pd_allreduce_sgd(int dtype, const float* const* grads, int n_rep, float* master, void* out, int64_t n, float lr,
                     void* stream) {
  return allreduce_sgd(dtype, grads, n_rep, master, out, n, lr, static_cast<cudaStream_t>(stream));
}
int pd_bias_grad(int dtype, const void* dz, int rows, int cols, int64_t ld, float* out, void* stream) {
  return bias_grad(dtype, dz, rows, cols, ld, out, static_cast<cudaStream_t>(stream));
}

int pd_cast(int dtype, const float* src, void* out, int64_t n, void* stream) {
  return cast_f32(dtype, src, out, n, static_cast<cudaStream_t>(stream));
}

int pd_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  return copy_bytes(dst, src, bytes, static_cast<cudaStream_t>(stream));
}

int pd_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "memcpy: %s", cudaGetErrorString(e));
}

int pd_flag_signal(int* flag, int value, void* stream) {
  return flag_signal(flag, value, static_cast<cudaStream_t>(stream));
}
int pd_flag_wait(const int* flag, int value, int* err_word, void* stream) {
  return flag_wait(flag, value, err_word, static_cast<cudaStream_t>(stream));
}

int pd_ipc_get_handle(const void* dev_ptr, void* handle_out64, int64_t* offset_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return set_error(PD_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  memcpy(handle_out64, &h, sizeof(h));
  if (offset_out) {
    // the handle names the allocation, not the pointer: report where dev_ptr sits inside it
    using range_fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static range_fn fn = nullptr;
    if (!fn) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        return set_error(PD_ERR_CUDA, "cuMemGetAddressRange unavailable");
      fn = reinterpret_cast<range_fn>(p);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
      return set_error(PD_ERR_CUDA, "cuMemGetAddressRange failed");
    *offset_out = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  }
  return 0;
}
int pd_ipc_open(const void* handle64, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
}
int pd_ipc_close(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
}
int pd_enable_peer_access(int peer_device) {
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); return 0; }
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "enable peer access: %s", cudaGetErrorString(e));
}

}  // extern "C"
