// Non-GEMM layer kernels of the convolutional / classification stages:
// max-pool forward/backward, first-layer im2col, tall column sums (conv bias gradients), the
// split-K reduction fused with SGD, and softmax cross-entropy.  All HBM-bound: 16-byte vector
// accesses, grids sized in multiples of the SM count, deterministic fixed-order reductions (so
// the replicas of a replicated stage compute bit-identical weights).
#include <cuda_runtime.h>

#include "pd_internal.h"
#include "ptx.cuh"

namespace pd {

namespace {

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int grid_for(int64_t work, int threads) {
  const int64_t want = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 8;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

// ---------------------------------------------------------------- 2x2 / stride-2 max pool (NHWC)
// out[n,p,q,c] = max over the window (dh, dw) in scan order (0,0),(0,1),(1,0),(1,1), first
// maximum wins; arg[n,p,q,c] = dh*2+dw.  8 channels (16 bytes) per thread.
__global__ void __launch_bounds__(256) k_maxpool_fwd(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                                     uint8_t* __restrict__ arg, int n, int H, int W, int C) {
  griddep_wait();
  const int Ho = H / 2, Wo = W / 2, C8 = C / 8;
  const int64_t total = (int64_t)n * Ho * Wo * C8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % C8);
    int64_t r = i / C8;
    const int q = (int)(r % Wo);
    r /= Wo;
    const int p = (int)(r % Ho);
    const int b = (int)(r / Ho);
    const __nv_bfloat16* base = x + (((int64_t)b * H + 2 * p) * W + 2 * q) * C + c8 * 8;
    float best[8];
    uint8_t idx[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 v = *reinterpret_cast<const uint4*>(base + ((k >> 1) * (int64_t)W + (k & 1)) * C);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float a, bb;
        unpack_bf16x2(w[j], a, bb);
        if (k == 0 || a > best[2 * j]) { best[2 * j] = a; idx[2 * j] = (uint8_t)k; }
        if (k == 0 || bb > best[2 * j + 1]) { best[2 * j + 1] = bb; idx[2 * j + 1] = (uint8_t)k; }
      }
    }
    const int64_t o = i * 8;
    *reinterpret_cast<uint4*>(y + o) = make_uint4(pack_bf16x2(best[0], best[1]), pack_bf16x2(best[2], best[3]),
                                                  pack_bf16x2(best[4], best[5]), pack_bf16x2(best[6], best[7]));
    uint2 a8;
    a8.x = idx[0] | (idx[1] << 8) | (idx[2] << 16) | ((uint32_t)idx[3] << 24);
    a8.y = idx[4] | (idx[5] << 8) | (idx[6] << 16) | ((uint32_t)idx[7] << 24);
    *reinterpret_cast<uint2*>(arg + o) = a8;
  }
}

// dx[window position k] = (arg == k) ? dy : 0  (every input element written exactly once)
__global__ void __launch_bounds__(256) k_maxpool_bwd(const __nv_bfloat16* __restrict__ dy, const uint8_t* __restrict__ arg,
                                                     __nv_bfloat16* __restrict__ dx, int n, int H, int W, int C) {
  griddep_wait();
  const int Ho = H / 2, Wo = W / 2, C8 = C / 8;
  const int64_t total = (int64_t)n * Ho * Wo * C8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % C8);
    int64_t r = i / C8;
    const int q = (int)(r % Wo);
    r /= Wo;
    const int p = (int)(r % Ho);
    const int b = (int)(r / Ho);
    const uint4 g = *reinterpret_cast<const uint4*>(dy + i * 8);
    const uint2 a8 = *reinterpret_cast<const uint2*>(arg + i * 8);
    const uint16_t* gh = reinterpret_cast<const uint16_t*>(&g);
    const uint8_t* ab = reinterpret_cast<const uint8_t*>(&a8);
    __nv_bfloat16* base = dx + (((int64_t)b * H + 2 * p) * W + 2 * q) * C + c8 * 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint16_t o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = ab[j] == k ? gh[j] : (uint16_t)0;
      *reinterpret_cast<uint4*>(base + ((k >> 1) * (int64_t)W + (k & 1)) * C) = *reinterpret_cast<const uint4*>(o);
    }
  }
}

int maxpool_fwd(const void* x, void* y, uint8_t* arg, int n, int H, int W, int C, cudaStream_t st) {
  if (C % 8 || H % 2 || W % 2) return set_error(PD_ERR_INVALID, "maxpool: C %% 8 and even H, W required");
  const int64_t total = (int64_t)n * (H / 2) * (W / 2) * (C / 8);
  launch_pdl(k_maxpool_fwd, dim3(grid_for(total, 256)), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(x),
                                                      static_cast<__nv_bfloat16*>(y), arg, n, H, W, C);
  return launch_status("maxpool_fwd");
}

int maxpool_bwd(const void* dy, const uint8_t* arg, void* dx, int n, int H, int W, int C, cudaStream_t st) {
  if (C % 8 || H % 2 || W % 2) return set_error(PD_ERR_INVALID, "maxpool: C %% 8 and even H, W required");
  const int64_t total = (int64_t)n * (H / 2) * (W / 2) * (C / 8);
  launch_pdl(k_maxpool_bwd, dim3(grid_for(total, 256)), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(dy), arg,
                                                      static_cast<__nv_bfloat16*>(dx), n, H, W, C);
  return launch_status("maxpool_bwd");
}

// ---------------------------------------------------------------- first-layer im2col
// cols[pix, k] for k = (r*3+s)*C + c < 9C: x[n, p+r-1, q+s-1, c] (0 outside); k >= 9C: 0.
// Only the first convolution (C = 3 image channels) uses it: its 27-wide K would waste a
// 64-channel im2col TMA box; every other layer reads im2col tiles straight from the activation.
// One thread per output pixel: gathers its 9*C inputs (C <= 7) and writes the 128-byte cols row
// with eight 16-byte stores (the output stream is what bounds this kernel).
// CC > 0: channel count known at compile time (VGG's RGB input, C = 3), so the 27 taps unroll and
// the packed row stays in registers; CC = 0: runtime C (the packing index is dynamic).
template <int CC>
__global__ void __launch_bounds__(256) k_im2col3(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ cols,
                                                 int n, int H, int W, int C_rt, int kpad) {
  griddep_wait();
  const int C = CC > 0 ? CC : C_rt;
  const int64_t pixels = (int64_t)n * H * W;
  for (int64_t pix = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pix < pixels;
       pix += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(pix % W), p = (int)((pix / W) % H);
    const int64_t b = pix / ((int64_t)H * W);
    uint32_t w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) w[i] = 0;
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      const int hh = p + tap / 3 - 1, ww = q + tap % 3 - 1;
      const bool ok = hh >= 0 && hh < H && ww >= 0 && ww < W;
      const __nv_bfloat16* src = x + ((b * H + hh) * W + ww) * C;
      if constexpr (CC > 0) {
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          const int k = tap * CC + c;
          const uint16_t v = ok ? __bfloat16_as_ushort(src[c]) : (uint16_t)0;
          w[k >> 1] |= (uint32_t)v << ((k & 1) * 16);
        }
      } else {
        for (int c = 0; c < C; ++c) {
          const int k = tap * C + c;
          const uint16_t v = ok ? __bfloat16_as_ushort(src[c]) : (uint16_t)0;
          w[k >> 1] |= (uint32_t)v << ((k & 1) * 16);
        }
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(cols + pix * kpad);
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
  }
}

int im2col3(const void* x, void* cols, int n, int H, int W, int C, int kpad, cudaStream_t st) {
  if (9 * C > kpad || kpad != 64) return set_error(PD_ERR_INVALID, "im2col: kpad must be 64 and >= 9*C (%d)", kpad);
  const int64_t total = (int64_t)n * H * W;
  if (C == 3)
    launch_pdl(k_im2col3<3>, dim3(grid_for(total, 256)), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(x),
               static_cast<__nv_bfloat16*>(cols), n, H, W, C, kpad);
  else
    launch_pdl(k_im2col3<0>, dim3(grid_for(total, 256)), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(x),
               static_cast<__nv_bfloat16*>(cols), n, H, W, C, kpad);
  return launch_status("im2col3");
}

// ---------------------------------------------------------------- column sums (bias gradients)
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Block b sums rows [b*rows_per, ...) of a [rows, C] bf16 matrix into part[b][C] (fp32); narrow
// rows: each thread owns 8 columns (one 16-byte vector) and a strided set of rows; wide rows
// (C/8 > 128): each thread owns column groups and walks the block's rows.  With a counter, the
// last block to finish (threadfence + atomic ticket) sums the partials in block order and applies
// the update itself (grad, or SGD into master/out), so the whole bias gradient is one launch;
// the counter resets itself for the next launch on the stream.
constexpr int CS_THREADS = 256;
__device__ __forceinline__ void finish_update(const float* part, int S, int C, float* grad, float* master, float* out,
                                              float lr) {
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float g = 0.f;
    for (int b = 0; b < S; ++b) g += __ldcg(part + (int64_t)b * C + c);
    if (grad) {
      grad[c] = g;
    } else {
      const float w = master[c] - lr * g;
      master[c] = w;
      out[c] = w;
    }
  }
}

// acc[0..8) += the 8 bf16 of v
__device__ __forceinline__ void acc_bf16x8(float (&acc)[8], const uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float a, b;
    unpack_bf16x2(w[j], a, b);
    acc[2 * j] += a;
    acc[2 * j + 1] += b;
  }
}

// Sum rows r, r+step, ... < r1 of column group cg (8 bf16) into acc, four 16-byte loads in flight.
__device__ __forceinline__ void colsum_rows(const __nv_bfloat16* __restrict__ x, int C, int cg, int64_t r, int64_t r1,
                                            int64_t step, float (&acc)[8]) {
  for (; r + 3 * step < r1; r += 4 * step) {
    const uint4 v0 = *reinterpret_cast<const uint4*>(x + r * C + cg * 8);
    const uint4 v1 = *reinterpret_cast<const uint4*>(x + (r + step) * C + cg * 8);
    const uint4 v2 = *reinterpret_cast<const uint4*>(x + (r + 2 * step) * C + cg * 8);
    const uint4 v3 = *reinterpret_cast<const uint4*>(x + (r + 3 * step) * C + cg * 8);
    acc_bf16x8(acc, v0);
    acc_bf16x8(acc, v1);
    acc_bf16x8(acc, v2);
    acc_bf16x8(acc, v3);
  }
  for (; r < r1; r += step) acc_bf16x8(acc, *reinterpret_cast<const uint4*>(x + r * C + cg * 8));
}

__global__ void __launch_bounds__(CS_THREADS) k_colsum_part(const __nv_bfloat16* __restrict__ x, int64_t rows, int C,
                                                            int64_t rows_per, float* __restrict__ part, int* counter,
                                                            float* grad, float* master, float* out, float lr) {
  griddep_wait();
  extern __shared__ float red[];  // narrow rows: [CS_THREADS / (C/8)][C]
  __shared__ bool last;
  const int C8 = C / 8;
  const int64_t r0 = blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < rows ? r0 + rows_per : rows;
  if (C8 > CS_THREADS / 2) {
    for (int cg = threadIdx.x; cg < C8; cg += CS_THREADS) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      colsum_rows(x, C, cg, r0, r1, 1, acc);
      if (counter) {  // fused mode: accumulate straight into the zeroed part[0..C)
        red_add_v4(part + cg * 8, acc[0], acc[1], acc[2], acc[3]);
        red_add_v4(part + cg * 8 + 4, acc[4], acc[5], acc[6], acc[7]);
      } else {
        float4* dst = reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * C + cg * 8);
        dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      }
    }
  } else {
    const int lanes = CS_THREADS / C8;  // row lanes per block
    const int cg = threadIdx.x % C8, rl = threadIdx.x / C8;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (rl < lanes) colsum_rows(x, C, cg, r0 + rl, r1, lanes, acc);
    if (rl < lanes)
#pragma unroll
      for (int j = 0; j < 8; ++j) red[rl * C + cg * 8 + j] = acc[j];
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += CS_THREADS) {
      float s = 0.f;
      for (int l = 0; l < lanes; ++l) s += red[l * C + c];
      if (counter) atomicAdd(part + c, s);
      else part[(int64_t)blockIdx.x * C + c] = s;
    }
  }
  if (!counter) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  finish_update(part, 1, C, grad, master, out, lr);  // part[0..C) holds the column sums
  if (threadIdx.x == 0) *counter = 0;
}

// Pass 2 (shared with split-K): g[i] = sum_s part[s*stride + i] in order s = 0..S-1, then
//   grad != null : grad[i] = g            (replicated stage: allreduced before the update)
//   otherwise    : master[i] -= lr*g; out[i] = cast(master[i])   (SGD into the new ring slot)
template <typename T>
__global__ void __launch_bounds__(256) k_reduce_sgd(const float* __restrict__ part, int S, int64_t stride, int64_t n,
                                                    float* __restrict__ grad, float* __restrict__ master,
                                                    T* __restrict__ out, float lr) {
  griddep_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float g = 0.f;
    for (int s = 0; s < S; ++s) g += part[s * stride + i];
    if (grad) {
      grad[i] = g;
    } else {
      const float w = master[i] - lr * g;
      master[i] = w;
      out[i] = from_f<T>(w);
    }
  }
}

int reduce_sgd(int out_dtype, const float* part, int S, int64_t stride, int64_t n, float* grad, float* master,
               void* out, float lr, cudaStream_t st) {
  if (S < 1 || n < 1) return set_error(PD_ERR_INVALID, "reduce_sgd: empty");
  if (!grad && (!master || !out)) return set_error(PD_ERR_INVALID, "reduce_sgd: need grad or master+out");
  const int g = grid_for(n, 256);
  if (out_dtype == PD_BF16)
    launch_pdl(k_reduce_sgd<__nv_bfloat16>, dim3(g), dim3(256), 0, st, part, S, stride, n, grad, master, static_cast<__nv_bfloat16*>(out), lr);
  else
    launch_pdl(k_reduce_sgd<float>, dim3(g), dim3(256), 0, st, part, S, stride, n, grad, master, static_cast<float*>(out), lr);
  return launch_status("reduce_sgd");
}

// One wave of blocks (at least 16 rows each): enough parallelism to stream the matrix at HBM
// rate, few enough partials that the fixed-order final sum stays cheap.
int colsum_blocks(int64_t rows, int C) {
  (void)C;
  int64_t b = (rows + 15) / 16;
  const int64_t cap = (int64_t)sm_count() * 2;
  return (int)(b < 1 ? 1 : (b < cap ? b : cap));
}

// Bias gradient of a [rows, C] bf16 gradient; part must hold colsum_blocks(rows, C) * C floats.
int bias_grad_tall(const void* dz, int64_t rows, int C, float* part, float* grad, float* master, float* out, float lr,
                   cudaStream_t st, int* counter) {
  if (C % 8) return set_error(PD_ERR_INVALID, "bias_grad_tall: C %% 8 == 0");
  const int blocks = colsum_blocks(rows, C);
  const int64_t per = (rows + blocks - 1) / blocks;
  const int lanes = CS_THREADS / (C / 8);
  const size_t smem = C / 8 > CS_THREADS / 2 ? 0 : (size_t)(lanes > 0 ? lanes : 1) * C * sizeof(float);
  if (counter) {
    cudaError_t e = cudaMemsetAsync(part, 0, sizeof(float) * C, st);
    if (e != cudaSuccess) return set_error(PD_ERR_CUDA, "colsum accumulator: %s", cudaGetErrorString(e));
  }
  launch_pdl(k_colsum_part, dim3(blocks), dim3(CS_THREADS), smem, st, static_cast<const __nv_bfloat16*>(dz), rows, C, per, part, counter,
                                                  grad, master, out, lr);
  int rc = launch_status("colsum_part");
  if (rc || counter) return rc;
  return reduce_sgd(PD_F32, part, blocks, C, C, grad, master, out, lr, st);
}

// ---------------------------------------------------------------- softmax cross-entropy
// One block per row of fp32 logits [B, V]: loss += (1/B) * (logsumexp - z[label]);
// dz[r, j] = (softmax_j - [j == label]) / B  in the activation dtype.
__global__ void __launch_bounds__(256) k_softmax_ce(const float* __restrict__ z, int64_t ldz, const int* __restrict__ labels,
                                                    int V, float inv_b, __nv_bfloat16* __restrict__ dz, int64_t ldd,
                                                    float* __restrict__ loss) {
  __shared__ float sh[32];
  const int r = blockIdx.x;
  const float* row = z + r * ldz;
  float m = -INFINITY;
  for (int j = threadIdx.x; j < V; j += blockDim.x) m = fmaxf(m, row[j]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  m = sh[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, sh[w]);
  __syncthreads();
  float s = 0.f;
  for (int j = threadIdx.x; j < V; j += blockDim.x) s += __expf(row[j] - m);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  s = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
  const int lab = labels[r];
  const float inv_s = 1.f / s;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const float p = __expf(row[j] - m) * inv_s;
    dz[r * ldd + j] = __float2bfloat16_rn((p - (j == lab ? 1.f : 0.f)) * inv_b);
  }
  if (threadIdx.x == 0) atomicAdd(loss, inv_b * (m + __logf(s) - row[lab]));
}

int softmax_ce(const float* logits, int64_t ldz, const int* labels, int B, int V, void* dz, int64_t ldd, float* loss,
               cudaStream_t st) {
  if (B < 1 || V < 1) return set_error(PD_ERR_INVALID, "softmax_ce: empty");
  k_softmax_ce<<<B, 256, 0, st>>>(logits, ldz, labels, V, 1.f / (float)B, static_cast<__nv_bfloat16*>(dz), ldd, loss);
  return launch_status("softmax_ce");
}

}  // namespace pd

// ==================================================================== C ABI
using namespace pd;

extern "C" {

int pd_conv3x3(int pass, const void* act, const void* other, int n, int h, int w, int c_in, int c_out,
               const pd_epilogue* ep, void* stream) {
  if (!ep) return set_error(PD_ERR_INVALID, "pd_conv3x3: null epilogue");
  return conv3x3_tc(pass, act, other, n, h, w, c_in, c_out, ep->kind, to_epi(*ep), static_cast<cudaStream_t>(stream));
}

int pd_splitk_plan(int M, int N, int K, int* splits) {
  if (!splits || M < 1 || N < 1 || K < 1) return set_error(PD_ERR_INVALID, "pd_splitk_plan: bad arguments");
  int per = 0;
  return splitk_plan(M, N, K, splits, &per);
}

int pd_maxpool2(const void* x, void* y, uint8_t* argmax, int n, int h, int w, int c, void* stream) {
  return maxpool_fwd(x, y, argmax, n, h, w, c, static_cast<cudaStream_t>(stream));
}

int pd_maxpool2_bwd(const void* dy, const uint8_t* argmax, void* dx, int n, int h, int w, int c, void* stream) {
  return maxpool_bwd(dy, argmax, dx, n, h, w, c, static_cast<cudaStream_t>(stream));
}

int pd_im2col3(const void* x, void* cols, int n, int h, int w, int c, int kpad, void* stream) {
  return im2col3(x, cols, n, h, w, c, kpad, static_cast<cudaStream_t>(stream));
}

int pd_reduce_sgd(int dtype, const float* part, int splits, int64_t stride, int64_t n, float* grad, float* master,
                  void* out, float lr, void* stream) {
  return reduce_sgd(dtype, part, splits, stride, n, grad, master, out, lr, static_cast<cudaStream_t>(stream));
}

int pd_colsum_blocks(int64_t rows, int c) { return colsum_blocks(rows, c); }

int pd_bias_grad_tall(const void* dz, int64_t rows, int c, float* part, float* grad, float* master, float* out,
                      float lr, void* stream) {
  return bias_grad_tall(dz, rows, c, part, grad, master, out, lr, static_cast<cudaStream_t>(stream));
}

int pd_softmax_ce(const float* logits, int64_t ldz, const int* labels, int b, int v, void* dz, int64_t ldd,
                  float* loss, void* stream) {
  return softmax_ce(logits, ldz, labels, b, v, dz, ldd, loss, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
