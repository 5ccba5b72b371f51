// Attention host entry points and the backward's pre/post passes.
//
// The forward and backward main kernels are the tcgen05/TMEM flash-attention kernels of
// attention_tc.cu.  Layout: qkv [T, 3*D] bf16 with T = b*S + s and head h at columns h*64 (q),
// D + h*64 (k), 2D + h*64 (v); out [T, D]; lse [B, H, S] fp32 (log2 domain, scores pre-scaled by
// softmax_scale*log2(e)).  Backward = D_i = rowsum(dO*O) preprocess (also zeroes the fp32 dQ
// accumulator), the key-tile-major main kernel (dK, dV in TMEM; dQ tiles TMA-reduce-added into
// dq_acc), then a cast kernel writing dQ*scale into the q slice of dqkv.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "pd_internal.h"
#include "ptx.cuh"

namespace pd {

namespace {

constexpr int HD = 64;  // head dim

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void __launch_bounds__(256) k_attn_bwd_pre(const __nv_bfloat16* __restrict__ o,
                                                      const __nv_bfloat16* __restrict__ dout, float* __restrict__ Dv,
                                                      float* __restrict__ dq_acc, int Bsz, int S, int H) {
  griddep_wait();
  const int D = H * HD;
  const int64_t rows = (int64_t)Bsz * S * H;  // one (token, head) per 8 threads
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = gid >> 3;
  const int c = (int)(gid & 7);
  if (r >= rows) return;
  const int64_t t = r / H;
  const int h = (int)(r % H);
  const uint4 a = *reinterpret_cast<const uint4*>(o + t * D + h * HD + c * 8);
  const uint4 g = *reinterpret_cast<const uint4*>(dout + t * D + h * HD + c * 8);
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(g2[i]);
    s += x.x * y.x + x.y * y.y;
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  float4* z = reinterpret_cast<float4*>(dq_acc + t * D + h * HD + c * 8);
  z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c == 0) {
    const int64_t bb = t / S, ss = t % S;
    Dv[(bb * H + h) * S + ss] = s;
  }
}

__global__ void __launch_bounds__(256) k_attn_dq_cast(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                                                      int64_t T, int D, float scale) {
  griddep_wait();
  const int64_t n4 = T * D / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(dq_acc)[i];
    const int64_t e = i * 4;
    const int64_t t = e / D, c = e % D;
    uint2 o;
    o.x = pack2(v.x * scale, v.y * scale);
    o.y = pack2(v.z * scale, v.w * scale);
    *reinterpret_cast<uint2*>(dqkv + t * 3 * (int64_t)D + c) = o;
  }
}

int status(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace

int attn_fwd(const void* qkv, void* out, float* lse, int B, int S, int H, cudaStream_t st) {
  return attn_fwd_tc(qkv, out, lse, B, S, H, st);
}

int attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* Dv, float* dq_acc,
             void* dqkv, int B, int S, int H, cudaStream_t st) {
  if (S % 128 || B < 1 || H < 1) return set_error(PD_ERR_INVALID, "attention: S %% 128 == 0 required");
  const float scale = 1.0f / sqrtf((float)HD);
  const int64_t rows = (int64_t)B * S * H;
  launch_pdl(k_attn_bwd_pre, dim3((unsigned)((rows * 8 + 255) / 256)), dim3(256), 0, st, 
      static_cast<const __nv_bfloat16*>(out), static_cast<const __nv_bfloat16*>(dout), Dv, dq_acc, B, S, H);
  int rc = status("attn_bwd_pre");
  if (rc) return rc;
  rc = attn_bwd_tc(qkv, dout, lse, Dv, dq_acc, dqkv, B, S, H, st);
  if (rc) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  launch_pdl(k_attn_dq_cast, dim3(sms * 8), dim3(256), 0, st, dq_acc, static_cast<__nv_bfloat16*>(dqkv), (int64_t)B * S, H * HD, scale);
  return status("attn_dq_cast");
}

}  // namespace pd

extern "C" {

int pd_attention_fwd(const void* qkv, void* out, float* lse, int batch, int seq, int heads, void* stream) {
  return pd::attn_fwd(qkv, out, lse, batch, seq, heads, static_cast<cudaStream_t>(stream));
}

int pd_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* dvec,
                     float* dq_acc, void* dqkv, int batch, int seq, int heads, void* stream) {
  return pd::attn_bwd(qkv, out, dout, lse, dvec, dq_acc, dqkv, batch, seq, heads, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
