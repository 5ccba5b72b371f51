// Causal multi-head attention for the transformer stages, FlashAttention-2
// style: the score matrix never leaves the SM.  head_dim 64, bf16 operands, fp32 accumulation,
// mma.sync m16n8k16 tensor-core fragments fed by ldmatrix from XOR-swizzled shared memory,
// cp.async double buffering.  (A tcgen05/TMEM version is the follow-up; the linear layers, which
// carry ~90 % of GPT-2's FLOPs, already run on the tcgen05 GEMM.)
//
// Layout: qkv [T, 3*D] bf16 with T = b*S + s and head h at columns h*64 (q), D + h*64 (k),
// 2D + h*64 (v); out [T, D]; lse [B, H, S] fp32 (log2 domain, scores pre-scaled by
// softmax_scale*log2(e)).  Backward: D_i = rowsum(dO*O) preprocess, key-tile-major main kernel
// (dK, dV accumulated in registers, dQ via fp32 atomics into dq_acc [T, D]), then a cast kernel
// writing dQ*scale into the q slice of dqkv.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "pd_internal.h"

namespace pd {

namespace {

constexpr int HD = 64;     // head dim
constexpr int BM = 64;     // query rows per tile
constexpr int BN = 64;     // key rows per tile
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of (row, 16-byte chunk) in a [rows][64] bf16 tile with XOR swizzle
__device__ __forceinline__ int swz(int row, int chunk) { return row * 128 + ((chunk ^ (row & 7)) << 4); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Load a 64 x 64 bf16 tile (rows of `ld` elements in global) into swizzled smem; 128 threads.
__device__ __forceinline__ void load_tile(uint8_t* s, const __nv_bfloat16* g, int64_t ld, int rows_valid) {
  const int t = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = t + i * THREADS;  // 0..511 = 64 rows x 8 chunks
    const int row = idx >> 3, ch = idx & 7;
    uint8_t* dst = s + swz(row, ch);
    if (row < rows_valid) cp_async16(dst, g + row * ld + ch * 8);
    else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_addr(p)));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// A fragments (16 rows x 64 cols, 4 k-steps) of a row-major swizzled tile at row r0.
__device__ __forceinline__ void load_a_frags(uint32_t (&a)[4][4], const uint8_t* s, int r0) {
  const int lane = threadIdx.x & 31;
  const int row = r0 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) ldsm_x4(a[ks], s + swz(row, ks * 2 + (lane >> 4)));
}

// B fragments for n-tiles (n0, n0+8) and k-step ks from a tile stored [n][k] (non-trans):
// returns b[0..1] for n-tile n0 and b[2..3] for n0+8.
__device__ __forceinline__ void load_b_nk(uint32_t (&b)[4], const uint8_t* s, int n0, int ks) {
  const int lane = threadIdx.x & 31;
  const int row = n0 + (lane & 7) + (lane >> 4) * 8;
  ldsm_x4(b, s + swz(row, ks * 2 + ((lane >> 3) & 1)));
}
// B fragments for n-tiles (n0, n0+8) and k-step ks from a tile stored [k][n] (trans).
__device__ __forceinline__ void load_b_kn(uint32_t (&b)[4], const uint8_t* s, int n0, int ks) {
  const int lane = threadIdx.x & 31;
  const int row = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
  ldsm_x4_t(b, s + swz(row, (n0 >> 3) + (lane >> 4)));
}
// A fragments (16 m-rows at m0 x 16 k at k-step ks) from a tile stored [k][m] (trans).
__device__ __forceinline__ void load_a_km(uint32_t (&a)[4], const uint8_t* s, int m0, int ks) {
  const int lane = threadIdx.x & 31;
  const int row = ks * 16 + (lane & 7) + (lane >> 4) * 8;
  ldsm_x4_t(a, s + swz(row, (m0 >> 3) + ((lane >> 3) & 1)));
}

// ================================================================ forward
__global__ void __launch_bounds__(THREADS) k_attn_fwd(const __nv_bfloat16* __restrict__ qkv,
                                                      __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                                                      int S, int H, float scale_log2) {
  __shared__ __align__(128) uint8_t sQ[BM * 128];
  __shared__ __align__(128) uint8_t sK[2][BN * 128];
  __shared__ __align__(128) uint8_t sV[2][BN * 128];
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int D = H * HD;
  const int64_t ld = 3 * (int64_t)D;
  const __nv_bfloat16* base = qkv + (int64_t)b * S * ld;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qt * BM;
  load_tile(sQ, base + (int64_t)q0 * ld + h * HD, ld, S - q0);
  cp_async_commit();
  const int n_kt = qt + 1;  // causal: key tiles 0..qt (BM == BN)
  auto load_kv = [&](int kt, int buf) {
    const int k0 = kt * BN;
    load_tile(sK[buf], base + (int64_t)k0 * ld + D + h * HD, ld, S - k0);
    load_tile(sV[buf], base + (int64_t)k0 * ld + 2 * D + h * HD, ld, S - k0);
    cp_async_commit();
  };
  load_kv(0, 0);
  cp_async_wait<1>();
  __syncthreads();
  uint32_t qa[4][4];
  load_a_frags(qa, sQ, warp * 16);
  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const int qrow0 = q0 + warp * 16 + (lane >> 2);  // this thread's rows: qrow0, qrow0 + 8
  for (int kt = 0; kt < n_kt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < n_kt) {
      load_kv(kt + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bb[4];
        load_b_nk(bb, sK[buf], np * 16, ks);
        mma16816(s[2 * np], qa[ks], bb[0], bb[1]);
        mma16816(s[2 * np + 1], qa[ks], bb[2], bb[3]);
      }
    }
    // scale, causal mask on the diagonal tile, online softmax (log2 domain)
    const int k0 = kt * BN;
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + nt * 8 + (lane & 3) * 2 + (e & 1);
        const int qr = qrow0 + (e >> 1) * 8;
        float v = s[nt][e] * scale_log2;
        if (key > qr || key >= S) v = -INFINITY;
        s[nt][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) corr[r] = m_r[r] == -INFINITY ? 0.f : exp2f(m_r[r] - mx[r]);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(s[nt][e] - mx[e >> 1]);
        s[nt][e] = p;
        rs[e >> 1] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      l_r[r] = l_r[r] * corr[r] + rs[r];
      m_r[r] = mx[r];
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      o[nt][0] *= corr[0]; o[nt][1] *= corr[0];
      o[nt][2] *= corr[1]; o[nt][3] *= corr[1];
    }
    // O += P V  (P from the score accumulators, re-packed as A fragments)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t pa[4];
      pa[0] = pack2(s[2 * ks][0], s[2 * ks][1]);
      pa[1] = pack2(s[2 * ks][2], s[2 * ks][3]);
      pa[2] = pack2(s[2 * ks + 1][0], s[2 * ks + 1][1]);
      pa[3] = pack2(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bb[4];
        load_b_kn(bb, sV[buf], np * 16, ks);
        mma16816(o[2 * np], pa, bb[0], bb[1]);
        mma16816(o[2 * np + 1], pa, bb[2], bb[3]);
      }
    }
    __syncthreads();  // buffer `buf` is reloaded two iterations later
  }
  // normalise, write O and the row log-sum-exp
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  const float inv[2] = {1.f / l_r[0], 1.f / l_r[1]};
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qr = qrow0 + r * 8;
    if (qr >= S) continue;
    __nv_bfloat16* orow = out + ((int64_t)b * S + qr) * D + h * HD;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int c = nt * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(orow + c) = pack2(o[nt][2 * r] * inv[r], o[nt][2 * r + 1] * inv[r]);
    }
    if ((lane & 3) == 0) lse[((int64_t)b * H + h) * S + qr] = m_r[r] + log2f(l_r[r]);
  }
}

// ================================================================ backward
// D[b,h,s] = sum_d dO * O ; dq_acc zeroed.
__global__ void __launch_bounds__(256) k_attn_bwd_pre(const __nv_bfloat16* __restrict__ o,
                                                      const __nv_bfloat16* __restrict__ dout, float* __restrict__ Dv,
                                                      float* __restrict__ dq_acc, int Bsz, int S, int H) {
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

__global__ void __launch_bounds__(THREADS) k_attn_bwd(const __nv_bfloat16* __restrict__ qkv,
                                                      const __nv_bfloat16* __restrict__ dout,
                                                      const float* __restrict__ lse, const float* __restrict__ Dv,
                                                      __nv_bfloat16* __restrict__ dqkv, float* __restrict__ dq_acc,
                                                      int S, int H, float scale_log2, float scale) {
  extern __shared__ __align__(128) uint8_t smem_bwd[];
  uint8_t* sK = smem_bwd;
  uint8_t* sV = sK + BN * 128;
  uint8_t(*sQ)[BM * 128] = reinterpret_cast<uint8_t(*)[BM * 128]>(sV + BN * 128);
  uint8_t(*sdO)[BM * 128] = reinterpret_cast<uint8_t(*)[BM * 128]>(sV + BN * 128 + 2 * BM * 128);
  uint8_t* sdS = sV + BN * 128 + 4 * BM * 128;  // dS^T [key][query]
  float(*sL)[BM] = reinterpret_cast<float(*)[BM]>(sdS + BN * 128);
  float(*sD)[BM] = reinterpret_cast<float(*)[BM]>(sdS + BN * 128 + 2 * BM * 4);
  const int kt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int D = H * HD;
  const int64_t ld = 3 * (int64_t)D;
  const __nv_bfloat16* base = qkv + (int64_t)b * S * ld;
  const __nv_bfloat16* dbase = dout + (int64_t)b * S * D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k0 = kt * BN;
  load_tile(sK, base + (int64_t)k0 * ld + D + h * HD, ld, S - k0);
  load_tile(sV, base + (int64_t)k0 * ld + 2 * D + h * HD, ld, S - k0);
  cp_async_commit();
  const int n_qt = (S + BM - 1) / BM;
  auto load_q = [&](int qt, int buf) {
    const int q0 = qt * BM;
    load_tile(sQ[buf], base + (int64_t)q0 * ld + h * HD, ld, S - q0);
    load_tile(sdO[buf], dbase + (int64_t)q0 * D + h * HD, D, S - q0);
    if (threadIdx.x < BM) {
      const int q = q0 + threadIdx.x;
      sL[buf][threadIdx.x] = q < S ? lse[((int64_t)b * H + h) * S + q] : 0.f;
      sD[buf][threadIdx.x] = q < S ? Dv[((int64_t)b * H + h) * S + q] : 0.f;
    }
    cp_async_commit();
  };
  load_q(kt, 0);  // causal: query tiles kt..n_qt-1
  cp_async_wait<1>();
  __syncthreads();
  uint32_t ka[4][4], va[4][4];
  load_a_frags(ka, sK, warp * 16);
  load_a_frags(va, sV, warp * 16);
  float dk[8][4], dv[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int krow0 = k0 + warp * 16 + (lane >> 2);  // this thread's keys: krow0, krow0 + 8
  for (int qt = kt; qt < n_qt; ++qt) {
    const int buf = (qt - kt) & 1;
    if (qt + 1 < n_qt) {
      load_q(qt + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int q0 = qt * BM;
    // S^T = K Q^T (16 keys x 64 queries per warp)
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bb[4];
        load_b_nk(bb, sQ[buf], np * 16, ks);
        mma16816(st[2 * np], ka[ks], bb[0], bb[1]);
        mma16816(st[2 * np + 1], ka[ks], bb[2], bb[3]);
        uint32_t dd[4];
        load_b_nk(dd, sdO[buf], np * 16, ks);  // dP^T = V dO^T
        mma16816(dpt[2 * np], va[ks], dd[0], dd[1]);
        mma16816(dpt[2 * np + 1], va[ks], dd[2], dd[3]);
      }
    // P^T = exp2(S^T * scale_log2 - lse[q]) (0 above the causal diagonal); dS^T = P^T (dP^T - D[q])
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + (lane & 3) * 2 + (e & 1);
        const int q = q0 + ql;
        const int key = krow0 + (e >> 1) * 8;
        float p = exp2f(st[nt][e] * scale_log2 - sL[buf][ql]);
        if (key > q || q >= S || key >= S) p = 0.f;
        st[nt][e] = p;
        dpt[nt][e] = p * (dpt[nt][e] - sD[buf][ql]);
      }
    // dV += P^T dO ; dK += dS^T Q   (k = query)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t pa[4], sa[4];
      pa[0] = pack2(st[2 * ks][0], st[2 * ks][1]);
      pa[1] = pack2(st[2 * ks][2], st[2 * ks][3]);
      pa[2] = pack2(st[2 * ks + 1][0], st[2 * ks + 1][1]);
      pa[3] = pack2(st[2 * ks + 1][2], st[2 * ks + 1][3]);
      sa[0] = pack2(dpt[2 * ks][0], dpt[2 * ks][1]);
      sa[1] = pack2(dpt[2 * ks][2], dpt[2 * ks][3]);
      sa[2] = pack2(dpt[2 * ks + 1][0], dpt[2 * ks + 1][1]);
      sa[3] = pack2(dpt[2 * ks + 1][2], dpt[2 * ks + 1][3]);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bb[4];
        load_b_kn(bb, sdO[buf], np * 16, ks);
        mma16816(dv[2 * np], pa, bb[0], bb[1]);
        mma16816(dv[2 * np + 1], pa, bb[2], bb[3]);
        uint32_t qq[4];
        load_b_kn(qq, sQ[buf], np * 16, ks);
        mma16816(dk[2 * np], sa, qq[0], qq[1]);
        mma16816(dk[2 * np + 1], sa, qq[2], qq[3]);
      }
      // stash dS^T (bf16) for the dQ product: rows = this warp's keys
      const int r0 = warp * 16 + (lane >> 2);
      const int c0 = ks * 16 + (lane & 3) * 2;  // query column of sa[0]
      *reinterpret_cast<uint32_t*>(sdS + swz(r0, c0 >> 3) + (c0 & 7) * 2) = sa[0];
      *reinterpret_cast<uint32_t*>(sdS + swz(r0 + 8, c0 >> 3) + (c0 & 7) * 2) = sa[1];
      *reinterpret_cast<uint32_t*>(sdS + swz(r0, (c0 + 8) >> 3) + ((c0 + 8) & 7) * 2) = sa[2];
      *reinterpret_cast<uint32_t*>(sdS + swz(r0 + 8, (c0 + 8) >> 3) + ((c0 + 8) & 7) * 2) = sa[3];
    }
    __syncthreads();
    // dQ[q, :] += dS[q, keys] K[keys, :]  (warp: 16 queries x 64 dims, all 64 keys of the tile)
    {
      float dq[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t aa[4];
        load_a_km(aa, sdS, warp * 16, ks);
#pragma unroll
        for (int np = 0; np < 4; ++np) {
          uint32_t bb[4];
          load_b_kn(bb, sK, np * 16, ks);
          mma16816(dq[2 * np], aa, bb[0], bb[1]);
          mma16816(dq[2 * np + 1], aa, bb[2], bb[3]);
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = q0 + warp * 16 + (lane >> 2) + r * 8;
        if (q >= S) continue;
        float* drow = dq_acc + ((int64_t)b * S + q) * D + h * HD;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const int c = nt * 8 + (lane & 3) * 2;
          atomicAdd(drow + c, dq[nt][2 * r]);
          atomicAdd(drow + c + 1, dq[nt][2 * r + 1]);
        }
      }
    }
    __syncthreads();  // sdS and buffer `buf` are rewritten next iteration
  }
  // write dK (scaled) and dV into the k / v slices of dqkv
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = krow0 + r * 8;
    if (key >= S) continue;
    __nv_bfloat16* row = dqkv + ((int64_t)b * S + key) * ld;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int c = nt * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(row + D + h * HD + c) = pack2(dk[nt][2 * r] * scale, dk[nt][2 * r + 1] * scale);
      *reinterpret_cast<uint32_t*>(row + 2 * D + h * HD + c) = pack2(dv[nt][2 * r], dv[nt][2 * r + 1]);
    }
  }
}

__global__ void __launch_bounds__(256) k_attn_dq_cast(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                                                      int64_t T, int D, float scale) {
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
  if (S % 64 || B < 1 || H < 1) return set_error(PD_ERR_INVALID, "attention: S %% 64 == 0 required");
  const float scale = 1.0f / sqrtf((float)HD);
  dim3 grid((S + BM - 1) / BM, H, B);
  k_attn_fwd<<<grid, THREADS, 0, st>>>(static_cast<const __nv_bfloat16*>(qkv), static_cast<__nv_bfloat16*>(out), lse,
                                       S, H, scale * 1.4426950408889634f);
  return status("attn_fwd");
}

int attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* Dv, float* dq_acc,
             void* dqkv, int B, int S, int H, cudaStream_t st) {
  if (S % 64 || B < 1 || H < 1) return set_error(PD_ERR_INVALID, "attention: S %% 64 == 0 required");
  const float scale = 1.0f / sqrtf((float)HD);
  const int64_t rows = (int64_t)B * S * H;
  k_attn_bwd_pre<<<(unsigned)((rows * 8 + 255) / 256), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(out), static_cast<const __nv_bfloat16*>(dout), Dv, dq_acc, B, S, H);
  int rc = status("attn_bwd_pre");
  if (rc) return rc;
  dim3 grid((S + BN - 1) / BN, H, B);
  constexpr int kSmem = 2 * BN * 128 + 4 * BM * 128 + BN * 128 + 4 * BM * 4;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess)
      return set_error(PD_ERR_CUDA, "attn_bwd: cannot set %d B of shared memory", kSmem);
    attr = true;
  }
  k_attn_bwd<<<grid, THREADS, kSmem, st>>>(static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(dout),
                                       lse, Dv, static_cast<__nv_bfloat16*>(dqkv), dq_acc, S, H,
                                       scale * 1.4426950408889634f, scale);
  rc = status("attn_bwd");
  if (rc) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_attn_dq_cast<<<sms * 8, 256, 0, st>>>(dq_acc, static_cast<__nv_bfloat16*>(dqkv), (int64_t)B * S, H * HD, scale);
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
