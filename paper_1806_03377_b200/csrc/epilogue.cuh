// GEMM epilogues shared by the tcgen05 and the SIMT GEMM.
//
// Every stage GEMM of the pipeline ends in one of these, so no separate
// elementwise pass touches HBM for bias/ReLU, the ReLU-backward mask, the MSE
// loss gradient or the SGD weight update:
//   EPI_STORE : out = act(acc + bias)                          (forward, K1)
//   EPI_LOSS  : d = acc + bias - target; out = d*scale;
//               loss += 0.5*scale*sum(d^2)                     (last layer fwd + MSE bwd)
//   EPI_MASK  : out = acc * (mask > 0)                         (dgrad + ReLU bwd, K2)
//   EPI_SGD   : master -= lr*acc; out = cast(master)           (wgrad + SGD, K3; writes the
//                                                               new weight version's ring slot)
//   EPI_GRADF32: out(fp32) = acc                                (wgrad for replicated stages,
//                                                               allreduced before the update)
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace pd {

//   EPI_GELU   : z = acc + bias; aux = z; out = gelu(z)        (transformer FC1, tanh GELU)
//   EPI_GELU_BWD: out = acc * gelu'(mask)                       (FC2 dgrad, mask = saved z)
//   EPI_RESID  : out = acc + bias + mask                        (projection + residual stream)
enum EpiKind : int {
  EPI_STORE = 0, EPI_LOSS = 1, EPI_MASK = 2, EPI_SGD = 3, EPI_GRADF32 = 4,
  EPI_GELU = 5, EPI_GELU_BWD = 6, EPI_RESID = 7,
  EPI_SGD_STREAM = 8  // internal: EPI_SGD for short K on the tcgen05 path (deeper master prefetch)
};

struct EpiArgs {
  void* out;            // activation dtype (fp32 for EPI_GRADF32)
  int64_t ldo;
  const float* bias;    // STORE / LOSS, per output column, nullable
  int relu;             // STORE
  const void* mask;     // MASK: the layer input X, activation dtype
  int64_t ldm;
  const float* target;  // LOSS
  int64_t ldt;
  float scale;          // LOSS: dL/dZ scale (1/B)
  float* loss;          // LOSS: accumulates 0.5*scale*sum(d^2)
  float* master;        // SGD: fp32 latest weights [M, N]
  int64_t ldw;
  float lr;             // SGD
  void* aux;            // GELU: pre-activation output (activation dtype, ld = ldo)
  int accumulate;       // GRADF32: red.add into out (zeroed by the caller) instead of storing;
                        // split-K partials then all land in one buffer (runtime-internal)
  // Fused cross-process hand-off (runtime-internal, tcgen05 path): when sig_flag is set, every
  // CTA fences its epilogue stores at system scope and bumps sig_counter; the last CTA resets the
  // counter and st.release.sys's sig_value into sig_flag (the receiver's inbox flag).
  int* sig_flag;
  int sig_value;
  int* sig_counter;
  unsigned long long* sig_bytes;  // nullable: payload bytes stored by the hand-off GEMM (traced runs)
  // Fused bias gradient (tcgen05 path, runtime-internal).  Producer side (EPI_MASK / EPI_LOSS, the
  // kernels that write a layer's output gradient dZ): when colsum is set, every epilogue warp also
  // writes the column sums of its 32 stored (bf16-rounded) rows, colsum[(row / 32) * ldc + col],
  // one plain store per (row block, column): the partials are complete and deterministic, no
  // atomics.  Consumer side (EPI_SGD, the wgrad of that layer): bpart = those partials ([nrb][ldc],
  // summed in row-block order), bmaster -= lr * sum; bring (the new version's bias) = bmaster.
  float* colsum;
  int64_t ldc;
  const float* bpart;
  int nrb;
  float* bmaster;
  float* bring;
  int group;            // SGD rasterisation band height in tiles (set by the launcher; 0 = default 16)
  int b_stream;         // set by the launcher: B operand loads carry an evict-first L2 policy
  int tma_out;          // set by the launcher: GRADF32 stores its fp32 blocks with TMA (map in tmW)
};

// GPT-2's tanh GELU and its derivative.  tanh on the SFU (tanh.approx.f32, max relative error
// ~2^-11): the accurate tanhf is ~20 instructions per element and made the FC1 forward (33.5 M GELUs
// per 8 x 1024-token minibatch) and the FC2 dgrad 63-89 % slower than the plain GEMM; the results
// are rounded to bf16 (2^-9) right after, so the approximation is below the storage rounding.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_f(float x) {
  const float u = x * fmaf(0.0356774081f, x * x, 0.7978845608028654f);  // sqrt(2/pi) (x + 0.044715 x^3)
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_fast(u), hx);
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float x2 = x * x;
  const float t = tanh_fast(x * fmaf(0.0356774081f, x2, 0.7978845608028654f));
  // 0.5 (1 + t) + 0.5 x (1 - t^2) sqrt(2/pi) (1 + 3 * 0.044715 x^2)
  return fmaf(0.5f * x * fmaf(-t, t, 1.f), fmaf(0.1070322243f, x2, 0.7978845608028654f), fmaf(0.5f, t, 0.5f));
}

// Operand sources of the tcgen05 GEMM (gemm.cu).  SRC_2D: both operands are 2-D row-major
// matrices.  The three implicit-GEMM 3x3/stride-1/pad-1 convolution passes (NHWC activations,
// weights stored tap-major as Wt[9*Cin][Cout]) load their activation operand with TMA im2col:
//   SRC_CONV_FWD  : Y[pix,Cout]   = sum_{tap,c} X(pix+tap)[c] * Wt[tap*Cin+c][Cout]
//   SRC_CONV_DGRAD: dX[pix,Cin]   = sum_{tap,k} dY(pix+flip(tap))[k] * Wt[(8-tap)*Cin+c][k]
//   SRC_CONV_WGRAD: dWt[tap*Cin+c][Cout] = sum_pix X(pix+tap)[c] * dY[pix][Cout]   (split-K)
enum GemmSrc : int { SRC_2D = 0, SRC_CONV_FWD = 1, SRC_CONV_DGRAD = 2, SRC_CONV_WGRAD = 3 };

struct ConvArgs {
  int H, W;          // spatial size of the im2col'ed activation (input == output size)
  int C;             // its channels (multiple of 64)
  int brows;         // DGRAD: weight rows per tap (= Cin)
  int kb_per;        // k-blocks per K split
  int splits;        // K splits (>= 1); split s writes out + s*split_stride (EPI_GRADF32)
  int64_t split_stride;
};

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// Per-element epilogue: returns the loss contribution (EPI_LOSS) or 0.
template <int KIND, typename T>
__device__ __forceinline__ float epi_elem(const EpiArgs& ep, int64_t r, int64_t c, float v) {
  if constexpr (KIND == EPI_STORE) {
    float x = v + (ep.bias ? ep.bias[c] : 0.f);
    if (ep.relu) x = fmaxf(x, 0.f);
    static_cast<T*>(ep.out)[r * ep.ldo + c] = from_f<T>(x);
    return 0.f;
  } else if constexpr (KIND == EPI_LOSS) {
    float d = v + (ep.bias ? ep.bias[c] : 0.f) - ep.target[r * ep.ldt + c];
    static_cast<T*>(ep.out)[r * ep.ldo + c] = from_f<T>(d * ep.scale);
    return d * d;
  } else if constexpr (KIND == EPI_MASK) {
    float m = to_f<T>(static_cast<const T*>(ep.mask)[r * ep.ldm + c]);
    static_cast<T*>(ep.out)[r * ep.ldo + c] = from_f<T>(m > 0.f ? v : 0.f);
    return 0.f;
  } else if constexpr (KIND == EPI_GELU) {
    const float z = v + (ep.bias ? ep.bias[c] : 0.f);
    static_cast<T*>(ep.aux)[r * ep.ldo + c] = from_f<T>(z);
    static_cast<T*>(ep.out)[r * ep.ldo + c] = from_f<T>(gelu_f(to_f<T>(from_f<T>(z))));
    return 0.f;
  } else if constexpr (KIND == EPI_GELU_BWD) {
    const float z = to_f<T>(static_cast<const T*>(ep.mask)[r * ep.ldm + c]);
    static_cast<T*>(ep.out)[r * ep.ldo + c] = from_f<T>(v * gelu_grad_f(z));
    return 0.f;
  } else if constexpr (KIND == EPI_RESID) {
    const float x = v + (ep.bias ? ep.bias[c] : 0.f) + to_f<T>(static_cast<const T*>(ep.mask)[r * ep.ldm + c]);
    static_cast<T*>(ep.out)[r * ep.ldo + c] = from_f<T>(x);
    return 0.f;
  } else if constexpr (KIND == EPI_SGD) {
    float w = ep.master[r * ep.ldw + c] - ep.lr * v;
    ep.master[r * ep.ldw + c] = w;
    static_cast<T*>(ep.out)[r * ep.ldo + c] = from_f<T>(w);
    return 0.f;
  } else {
    static_cast<float*>(ep.out)[r * ep.ldo + c] = v + (ep.bias ? ep.bias[c] : 0.f);
    return 0.f;
  }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void unpack_bf16x2(uint32_t u, float& a, float& b) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
  a = __low2float(h);
  b = __high2float(h);
}

// ---------------------------------------------------------------------------------------
// Chunked tcgen05 epilogue with one-chunk-ahead prefetch of the per-element global input
// (fp32 master for SGD, bf16 mask for dgrad, fp32 target for the loss), so the HBM latency
// of chunk c+1 overlaps the math/stores of chunk c.
// STORE / GELU also prefetch the next chunk's 32 bias values (loaded at use they put a global-load
// latency on every chunk's critical path: ncu showed the FC1 GELU epilogue stalled on long
// scoreboard at the bias add, tensor pipe 41 %).  RESID / LOSS keep the load at use: with their
// prefetched residual / target the extra 2 x 32 registers spill.
template <int KIND> struct Aux { };
template <> struct Aux<EPI_STORE> { float4 b[8]; };
template <> struct Aux<EPI_GELU> { float4 b[8]; };
template <> struct Aux<EPI_SGD> { float4 m[8]; };
template <> struct Aux<EPI_MASK> { uint4 m[4]; };
template <> struct Aux<EPI_LOSS> { float4 t[8]; };
template <> struct Aux<EPI_GELU_BWD> { uint4 m[4]; };
template <> struct Aux<EPI_RESID> { uint4 m[4]; };

template <int KIND>
__device__ __forceinline__ void aux_load(const EpiArgs& ep, int64_t r, int64_t c0, Aux<KIND>& a) {
  if constexpr (KIND == EPI_SGD) {
    const float4* w4 = reinterpret_cast<const float4*>(ep.master + r * ep.ldw + c0);
#pragma unroll
    for (int i = 0; i < 8; ++i) a.m[i] = w4[i];
  } else if constexpr (KIND == EPI_MASK || KIND == EPI_GELU_BWD || KIND == EPI_RESID) {
    const uint4* m4 =
        reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.mask) + r * ep.ldm + c0);
#pragma unroll
    for (int i = 0; i < 4; ++i) a.m[i] = m4[i];
  } else if constexpr (KIND == EPI_LOSS) {
    const float4* t4 = reinterpret_cast<const float4*>(ep.target + r * ep.ldt + c0);
#pragma unroll
    for (int i = 0; i < 8; ++i) a.t[i] = t4[i];
  } else if constexpr (KIND == EPI_STORE || KIND == EPI_GELU) {
    if (ep.bias) {
      const float4* b4 = reinterpret_cast<const float4*>(ep.bias + c0);
#pragma unroll
      for (int i = 0; i < 8; ++i) a.b[i] = __ldg(b4 + i);
    }
  }
}

__device__ __forceinline__ void store32_bf16(void* out, int64_t ld, int64_t r, int64_t c0, const float (&v)[32]) {
  uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + r * ld + c0);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    o[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                      pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
}

// Full 32-column chunk (c0 + 32 <= N); returns the loss contribution.
template <int KIND>
__device__ __forceinline__ float apply_chunk(const EpiArgs& ep, int64_t r, int64_t c0, float (&v)[32],
                                             const Aux<KIND>& a) {
  float lsum = 0.f;
  if constexpr (KIND == EPI_STORE) {
    if (ep.bias) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 b = a.b[i];
        v[4 * i] += b.x; v[4 * i + 1] += b.y; v[4 * i + 2] += b.z; v[4 * i + 3] += b.w;
      }
    }
    if (ep.relu) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
    }
    store32_bf16(ep.out, ep.ldo, r, c0, v);
  } else if constexpr (KIND == EPI_LOSS) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 b = ep.bias ? __ldg(reinterpret_cast<const float4*>(ep.bias + c0) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * i] += b.x - a.t[i].x; v[4 * i + 1] += b.y - a.t[i].y;
      v[4 * i + 2] += b.z - a.t[i].z; v[4 * i + 3] += b.w - a.t[i].w;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) { lsum += v[i] * v[i]; v[i] *= ep.scale; }
    store32_bf16(ep.out, ep.ldo, r, c0, v);
  } else if constexpr (KIND == EPI_MASK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t mw[4] = {a.m[i].x, a.m[i].y, a.m[i].z, a.m[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x0, x1;
        unpack_bf16x2(mw[j], x0, x1);
        if (!(x0 > 0.f)) v[8 * i + 2 * j] = 0.f;
        if (!(x1 > 0.f)) v[8 * i + 2 * j + 1] = 0.f;
      }
    }
    store32_bf16(ep.out, ep.ldo, r, c0, v);
  } else if constexpr (KIND == EPI_GELU) {
    if (ep.bias) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 b = a.b[i];
        v[4 * i] += b.x; v[4 * i + 1] += b.y; v[4 * i + 2] += b.z; v[4 * i + 3] += b.w;
      }
    }
    store32_bf16(ep.aux, ep.ldo, r, c0, v);
    // the stored (bf16) pre-activation is what the backward sees: apply GELU to the rounded value
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = gelu_f(__bfloat162float(__float2bfloat16_rn(v[i])));
    store32_bf16(ep.out, ep.ldo, r, c0, v);
  } else if constexpr (KIND == EPI_GELU_BWD || KIND == EPI_RESID) {
    float bb[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) bb[i] = 0.f;
    if (KIND == EPI_RESID && ep.bias) {
      const float4* b4 = reinterpret_cast<const float4*>(ep.bias + c0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 b = __ldg(b4 + i);
        bb[4 * i] = b.x; bb[4 * i + 1] = b.y; bb[4 * i + 2] = b.z; bb[4 * i + 3] = b.w;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t mw[4] = {a.m[i].x, a.m[i].y, a.m[i].z, a.m[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x0, x1;
        unpack_bf16x2(mw[j], x0, x1);
        const int k = 8 * i + 2 * j;
        if constexpr (KIND == EPI_GELU_BWD) {
          v[k] *= gelu_grad_f(x0);
          v[k + 1] *= gelu_grad_f(x1);
        } else {
          v[k] += bb[k] + x0;
          v[k + 1] += bb[k + 1] + x1;
        }
      }
    }
    store32_bf16(ep.out, ep.ldo, r, c0, v);
  } else if constexpr (KIND == EPI_SGD) {
    float4* w4 = reinterpret_cast<float4*>(ep.master + r * ep.ldw + c0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 w = a.m[i];
      w.x -= ep.lr * v[4 * i]; w.y -= ep.lr * v[4 * i + 1];
      w.z -= ep.lr * v[4 * i + 2]; w.w -= ep.lr * v[4 * i + 3];
      w4[i] = w;
      v[4 * i] = w.x; v[4 * i + 1] = w.y; v[4 * i + 2] = w.z; v[4 * i + 3] = w.w;
    }
    store32_bf16(ep.out, ep.ldo, r, c0, v);
  } else {
    float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + r * ep.ldo + c0);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  }
  return lsum;
}

// Column sums of a warp's 32 x 32 block (lane = row, v[j] = column j): a butterfly transpose-
// reduction (31 shuffles) that leaves the sum of column `lane` in the return value.
__device__ __forceinline__ float warp_colsum32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const bool upper = lane & k;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const float send = upper ? v[i] : v[i + k];
      const float keep = upper ? v[i + k] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  return v[0];
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

}  // namespace pd
