// Non-GEMM kernels of the GPT-2 stages (BASELINE configs[3]): LayerNorm
// forward / backward (the backward fused with the residual-stream gradient add and the
// gamma/beta column sums), token + position embedding gather / scatter-add, and the
// vocabulary-padded softmax cross-entropy.  One warp per row, 16-byte vector accesses; the
// column-sum partials go through the fixed-order reduction of layers.cu (reduce_sgd).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "pd_internal.h"
#include "ptx.cuh"

namespace pd {

namespace {

int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int status(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

constexpr int LN_WARPS = 8;
constexpr int LN_MAXV = 8;  // up to 8 x 256 = 2048 features per row (NV = D / 256 is a template parameter)

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) unpack_bf16x2(w[j], v[2 * j], v[2 * j + 1]);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&v)[8]) {
  *reinterpret_cast<uint4*>(p) = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                                            pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
}

// y = (x - mean) * rstd * gamma + beta ; gamma/beta = gb[0:D], gb[D:2D] (fp32)
// o[j] = o[j] * gamma[j] + beta[j] for 8 consecutive columns (two 16-byte loads each)
__device__ __forceinline__ void ln_affine8(const float* __restrict__ g, const float* __restrict__ b, float (&o)[8]) {
  const float4 g0 = reinterpret_cast<const float4*>(g)[0], g1 = reinterpret_cast<const float4*>(g)[1];
  const float4 b0 = reinterpret_cast<const float4*>(b)[0], b1 = reinterpret_cast<const float4*>(b)[1];
  const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
  const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = fmaf(o[j], gg[j], bb[j]);
}

template <int NV>
__global__ void __launch_bounds__(LN_WARPS * 32) k_ln_fwd(const __nv_bfloat16* __restrict__ x, const float* __restrict__ gb,
                                                          __nv_bfloat16* __restrict__ y, float* __restrict__ mean,
                                                          float* __restrict__ rstd, int64_t T, int D, float eps) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)LN_WARPS + (threadIdx.x >> 5);
  if (row >= T) return;
  constexpr int nv = NV;
  float v[NV][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (i < nv) {
      load8(x + row * D + i * 256 + lane * 8, v[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[i][j];
    }
  s = warp_sum(s);
  const float mu = s / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (i < nv)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = v[i][j] - mu;
        q += d * d;
      }
  q = warp_sum(q);
  const float rs = rsqrtf(q / D + eps);
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (i < nv) {
      const int c = i * 256 + lane * 8;
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (v[i][j] - mu) * rs;
      ln_affine8(gb + c, gb + D + c, o);
      store8(y + row * D + c, o);
    }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// dx = dres + rstd * (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat));  part[block] += (dy*xhat, dy)
template <int NV>
__global__ void __launch_bounds__(LN_WARPS * 32) k_ln_bwd(const __nv_bfloat16* __restrict__ dy,
                                                          const __nv_bfloat16* __restrict__ x,
                                                          const float* __restrict__ mean, const float* __restrict__ rstd,
                                                          const float* __restrict__ gb,
                                                          const __nv_bfloat16* __restrict__ dres,
                                                          __nv_bfloat16* __restrict__ dx, float* __restrict__ part,
                                                          int64_t T, int D, int64_t rows_per_block, int* counter,
                                                          float* master, float* mout, float lr) {
  griddep_wait();
  extern __shared__ float red[];  // [LN_WARPS][2*D]
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nv = NV;
  float pg[NV][8], pb[NV][8];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) pg[i][j] = pb[i][j] = 0.f;
  const int64_t r0 = blockIdx.x * rows_per_block;
  const int64_t r1 = r0 + rows_per_block < T ? r0 + rows_per_block : T;
  for (int64_t row = r0 + warp; row < r1; row += LN_WARPS) {
    const float mu = mean[row], rs = rstd[row];
    float g[NV][8], xh[NV][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (i < nv) {
        const int c = i * 256 + lane * 8;
        float dv[8], xv[8];
        load8(dy + row * D + c, dv);
        load8(x + row * D + c, xv);
#pragma unroll
        const float4 ga = reinterpret_cast<const float4*>(gb + c)[0], gc = reinterpret_cast<const float4*>(gb + c)[1];
        const float gm[8] = {ga.x, ga.y, ga.z, ga.w, gc.x, gc.y, gc.z, gc.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xh[i][j] = (xv[j] - mu) * rs;
          g[i][j] = dv[j] * gm[j];
          s1 += g[i][j];
          s2 += g[i][j] * xh[i][j];
          pg[i][j] += dv[j] * xh[i][j];
          pb[i][j] += dv[j];
        }
      }
    s1 = warp_sum(s1) / D;
    s2 = warp_sum(s2) / D;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (i < nv) {
        const int c = i * 256 + lane * 8;
        float o[8], r[8];
        if (dres) load8(dres + row * D + c, r);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rs * (g[i][j] - s1 - xh[i][j] * s2) + (dres ? r[j] : 0.f);
        store8(dx + row * D + c, o);
      }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (i < nv)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = i * 256 + lane * 8 + j;
        red[warp * 2 * D + c] = pg[i][j];
        red[warp * 2 * D + D + c] = pb[i][j];
      }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * D; c += LN_WARPS * 32) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < LN_WARPS; ++w) s += red[w * 2 * D + c];
    if (counter) atomicAdd(part + c, s);  // fused mode: part[0..2D) is a zeroed accumulator
    else part[blockIdx.x * 2 * (int64_t)D + c] = s;
  }
  if (!counter) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int c = threadIdx.x; c < 2 * D; c += LN_WARPS * 32) {
    const float g = __ldcg(part + c);
    const float w = master[c] - lr * g;
    master[c] = w;
    mout[c] = w;
  }
  if (threadIdx.x == 0) *counter = 0;
}

// x[t] = wte[tok[t]] + wpe[t % S]
__global__ void __launch_bounds__(256) k_embed_fwd(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ wte,
                                                   const __nv_bfloat16* __restrict__ wpe, __nv_bfloat16* __restrict__ x,
                                                   int64_t T, int S, int D) {
  griddep_wait();
  const int D8 = D / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T * D8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / D8;
    const int c = (int)(i % D8) * 8;
    float a[8], b[8];
    load8(wte + (int64_t)tok[t] * D + c, a);
    load8(wpe + (t % S) * D + c, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += b[j];
    store8(x + t * D + c, a);
  }
}

// gte[tok[t]] += dx[t]; gpe[t % S] += dx[t]   (fp32 atomics into zeroed gradient buffers)
__global__ void __launch_bounds__(256) k_embed_bwd(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ dx,
                                                   float* __restrict__ gte, float* __restrict__ gpe, int64_t T, int S,
                                                   int D) {
  const int D8 = D / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T * D8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / D8;
    const int c = (int)(i % D8) * 8;
    float g[8];
    load8(dx + t * D + c, g);
    float* a = gte + (int64_t)tok[t] * D + c;
    float* b = gpe + (t % S) * D + c;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      atomicAdd(a + j, g[j]);
      atomicAdd(b + j, g[j]);
    }
  }
}

// Softmax cross-entropy over the first V of Vp fp32 logit columns; columns >= V get dz = 0.
// One block per row, two passes over the row: an online (max, sum-exp) pass with 16-byte loads,
// then the gradient pass (softmax - onehot) / rows written as bf16.
__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mx = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mx)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mx));
  m = mx;
}

__global__ void __launch_bounds__(512) k_softmax_ce_v(const float* __restrict__ z, int64_t ldz,
                                                      const int* __restrict__ labels, int V, int Vp, float inv_n,
                                                      __nv_bfloat16* __restrict__ dz, int64_t ldd,
                                                      float* __restrict__ loss) {
  griddep_wait();
  __shared__ float shm[32], shs[32];
  const int64_t r = blockIdx.x;
  const float* row = z + r * ldz;
  const int nw = blockDim.x >> 5;
  const int V4 = V / 4;
  float m = -INFINITY, s = 0.f;
  for (int j = threadIdx.x; j < V4; j += blockDim.x) {
    const float4 x = reinterpret_cast<const float4*>(row)[j];
    const float mx = fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w));
    if (mx > m) {
      s = (m == -INFINITY ? 0.f : s * __expf(m - mx));
      m = mx;
    }
    s += __expf(x.x - m) + __expf(x.y - m) + __expf(x.z - m) + __expf(x.w - m);
  }
  for (int j = V4 * 4 + threadIdx.x; j < V; j += blockDim.x) online_merge(m, s, row[j], 1.f);
#pragma unroll
  for (int o = 16; o; o >>= 1) online_merge(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) {
    shm[threadIdx.x >> 5] = m;
    shs[threadIdx.x >> 5] = s;
  }
  __syncthreads();
  m = shm[0];
  s = shs[0];
  for (int w = 1; w < nw; ++w) online_merge(m, s, shm[w], shs[w]);
  const int lab = labels[r];
  const float inv_s = 1.f / s;
  __nv_bfloat16* drow = dz + r * ldd;
  const int Vp4 = Vp / 4;
  for (int j = threadIdx.x; j < Vp4; j += blockDim.x) {
    const float4 x = reinterpret_cast<const float4*>(row)[j];
    const float xv[4] = {x.x, x.y, x.z, x.w};
    float g[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = 4 * j + e;
      const float p = c < V ? __expf(xv[e] - m) * inv_s : 0.f;
      g[e] = (p - (c == lab ? 1.f : 0.f)) * inv_n;
    }
    *reinterpret_cast<uint2*>(drow + 4 * j) = make_uint2(pack_bf16x2(g[0], g[1]), pack_bf16x2(g[2], g[3]));
  }
  if (threadIdx.x == 0) atomicAdd(loss, inv_n * (m + __logf(s) - row[lab]));
}

}  // namespace

int ln_fwd(const void* x, const float* gb, void* y, float* mean, float* rstd, int64_t T, int D, cudaStream_t st) {
  if (D % 256 || D > 256 * LN_MAXV) return set_error(PD_ERR_INVALID, "layernorm: D %% 256 == 0, D <= 2048");
  const unsigned g = (unsigned)((T + LN_WARPS - 1) / LN_WARPS);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto Y = static_cast<__nv_bfloat16*>(y);
  switch (D / 256) {
    case 1: launch_pdl(k_ln_fwd<1>, dim3(g), dim3(LN_WARPS * 32), 0, st, X, gb, Y, mean, rstd, T, D, 1e-5f); break;
    case 2: launch_pdl(k_ln_fwd<2>, dim3(g), dim3(LN_WARPS * 32), 0, st, X, gb, Y, mean, rstd, T, D, 1e-5f); break;
    case 4: launch_pdl(k_ln_fwd<4>, dim3(g), dim3(LN_WARPS * 32), 0, st, X, gb, Y, mean, rstd, T, D, 1e-5f); break;
    case 8: launch_pdl(k_ln_fwd<8>, dim3(g), dim3(LN_WARPS * 32), 0, st, X, gb, Y, mean, rstd, T, D, 1e-5f); break;
    default: return set_error(PD_ERR_INVALID, "layernorm: D/256 must be 1, 2, 4 or 8");
  }
  return status("ln_fwd");
}

int ln_bwd_blocks(int64_t T) {
  int64_t b = (T + 31) / 32;
  const int64_t cap = (int64_t)sms() * 2;
  return (int)(b < 1 ? 1 : (b < cap ? b : cap));
}

int ln_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* gb, const void* dres,
           void* dx, float* part, int64_t T, int D, cudaStream_t st, int* counter, float* master, float* out,
           float lr) {
  if (D % 256 || D > 256 * LN_MAXV) return set_error(PD_ERR_INVALID, "layernorm: D %% 256 == 0, D <= 2048");
  const int blocks = ln_bwd_blocks(T);
  const int64_t per = (T + blocks - 1) / blocks;
  const size_t smem = (size_t)LN_WARPS * 2 * D * sizeof(float);
  if (counter) {
    cudaError_t e = cudaMemsetAsync(part, 0, sizeof(float) * 2 * D, st);
    if (e != cudaSuccess) return set_error(PD_ERR_CUDA, "ln_bwd accumulator: %s", cudaGetErrorString(e));
  }
  auto launch = [&](auto kern) -> int {
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return set_error(PD_ERR_CUDA, "ln_bwd: shared memory attribute");
    launch_pdl(kern, dim3(blocks), dim3(LN_WARPS * 32), smem, st, static_cast<const __nv_bfloat16*>(dy),
                                              static_cast<const __nv_bfloat16*>(x), mean, rstd, gb,
                                              static_cast<const __nv_bfloat16*>(dres), static_cast<__nv_bfloat16*>(dx),
                                              part, T, D, per, counter, master, out, lr);
    return status("ln_bwd");
  };
  switch (D / 256) {
    case 1: return launch(k_ln_bwd<1>);
    case 2: return launch(k_ln_bwd<2>);
    case 4: return launch(k_ln_bwd<4>);
    case 8: return launch(k_ln_bwd<8>);
  }
  return set_error(PD_ERR_INVALID, "layernorm: D/256 must be 1, 2, 4 or 8");
}

int embed_fwd(const int* tok, const void* wte, const void* wpe, void* x, int64_t T, int S, int D, cudaStream_t st) {
  if (D % 8) return set_error(PD_ERR_INVALID, "embedding: D %% 8 == 0");
  launch_pdl(k_embed_fwd, dim3(sms() * 8), dim3(256), 0, st, tok, static_cast<const __nv_bfloat16*>(wte),
                                        static_cast<const __nv_bfloat16*>(wpe), static_cast<__nv_bfloat16*>(x), T, S, D);
  return status("embed_fwd");
}

int embed_bwd(const int* tok, const void* dx, float* gte, float* gpe, int64_t T, int S, int D, cudaStream_t st) {
  if (D % 8) return set_error(PD_ERR_INVALID, "embedding: D %% 8 == 0");
  k_embed_bwd<<<sms() * 8, 256, 0, st>>>(tok, static_cast<const __nv_bfloat16*>(dx), gte, gpe, T, S, D);
  return status("embed_bwd");
}

int softmax_ce_v(const float* logits, int64_t ldz, const int* labels, int64_t rows, int V, int Vp, void* dz,
                 int64_t ldd, float* loss, cudaStream_t st) {
  if (rows < 1 || V < 1 || Vp < V || Vp % 4 || ldz % 4 || ldd % 4)
    return set_error(PD_ERR_INVALID, "softmax_ce: bad shape (Vp and row pitches must be multiples of 4)");
  launch_pdl(k_softmax_ce_v, dim3((unsigned)rows), dim3(512), 0, st, logits, ldz, labels, V, Vp, 1.f / (float)rows,
                                                 static_cast<__nv_bfloat16*>(dz), ldd, loss);
  return status("softmax_ce_v");
}

}  // namespace pd

extern "C" {

int pd_layernorm_fwd(const void* x, const float* gb, void* y, float* mean, float* rstd, int64_t rows, int d,
                     void* stream) {
  return pd::ln_fwd(x, gb, y, mean, rstd, rows, d, static_cast<cudaStream_t>(stream));
}
int pd_layernorm_bwd_blocks(int64_t rows) { return pd::ln_bwd_blocks(rows); }
int pd_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* gb,
                     const void* dres, void* dx, float* part, int64_t rows, int d, void* stream) {
  return pd::ln_bwd(dy, x, mean, rstd, gb, dres, dx, part, rows, d, static_cast<cudaStream_t>(stream));
}
int pd_embedding_fwd(const int* tok, const void* wte, const void* wpe, void* x, int64_t tokens, int seq, int d,
                     void* stream) {
  return pd::embed_fwd(tok, wte, wpe, x, tokens, seq, d, static_cast<cudaStream_t>(stream));
}
int pd_embedding_bwd(const int* tok, const void* dx, float* gte, float* gpe, int64_t tokens, int seq, int d,
                     void* stream) {
  return pd::embed_bwd(tok, dx, gte, gpe, tokens, seq, d, static_cast<cudaStream_t>(stream));
}
int pd_softmax_ce_vocab(const float* logits, int64_t ldz, const int* labels, int64_t rows, int v, int vpad, void* dz,
                        int64_t ldd, float* loss, void* stream) {
  return pd::softmax_ce_v(logits, ldz, labels, rows, v, vpad, dz, ldd, loss, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
