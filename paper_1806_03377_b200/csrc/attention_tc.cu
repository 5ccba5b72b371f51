// Causal flash attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), head_dim 64.
//
// Forward, one CTA per (128-query tile, head, sequence), two CTAs per SM:
//   warp 0  TMA producer: Q tile once, then K_j / V_j tiles (128 keys x 64 dims, 128B swizzle)
//   warp 1  MMA issuer (one elected thread) + TMEM owner:
//             S_j = Q K_j^T       tcgen05.mma M=128 N=128 K=64   -> TMEM cols [0,128)
//             O  += P_j V_j       tcgen05.mma M=128 N=64  K=128  -> TMEM cols [128,192)
//   warps 2-5  softmax, one thread per query row (its TMEM lane): tcgen05.ld the S row, online
//             max / exp2 / sum in fp32, rescale the O row in TMEM (tcgen05.ld/st) when the max
//             moved, write P (bf16) into shared memory in the K-major SW128 layout the PV MMA
//             reads, then signal the MMA warp.  At the end O/l is written to HBM and the row's
//             log-sum-exp (log2 domain) is kept for the backward.
// S_{j+1} is issued before PV_j so the next tile's scores are ready as soon as the softmax
// warps finish writing P_j; the second CTA on the SM overlaps its MMAs with this CTA's softmax.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "epilogue.cuh"
#include "pd_internal.h"
#include "ptx.cuh"

namespace pd {

namespace {

constexpr int TQ = 128;     // queries per tile (TMEM lanes)
constexpr int TK = 128;     // keys per tile
constexpr int HDIM = 64;    // head dim = one 128-byte swizzle row
constexpr int FWD_THREADS = 192;
constexpr int TILE_BYTES = 128 * 128;  // 128 rows x 64 bf16

struct FwdSmem {
  static constexpr int Q = 0;
  static constexpr int K = Q + TILE_BYTES;
  static constexpr int V = K + TILE_BYTES;
  static constexpr int P = V + TILE_BYTES;          // two K-major atoms: keys 0..63, 64..127
  static constexpr int BAR = P + 2 * TILE_BYTES;
  static constexpr int TOTAL = BAR + 256 + 1024;    // barriers + TMEM slot + alignment slack
};

PD_DEVICE void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
PD_DEVICE void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
PD_DEVICE void tmem_st_32x32b_x32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 2^x on the SFU (ex2.approx, flush-to-zero): x <= 0 here, so no range handling is needed.
PD_DEVICE float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr float RESCALE_LOG2 = 8.f;  // forward: rescale O only when the running max grows by > 2^8

// Row max over 64 S values (raw scores); MASK: only columns base+i <= lim count.  The unmasked form
// keeps four independent chains (3-input FMNMX).
template <bool MASK>
PD_DEVICE float row_max64(const uint32_t (&sr)[64], int base, int lim, float mx) {
  if constexpr (MASK) {
#pragma unroll
    for (int i = 0; i < 64; ++i)
      if (base + i <= lim) mx = fmaxf(mx, __uint_as_float(sr[i]));
    return mx;
  } else {
    float a = mx, b = -INFINITY, c = -INFINITY, d = -INFINITY;
#pragma unroll
    for (int i = 0; i < 64; i += 8) {
      a = fmaxf(a, fmaxf(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])));
      b = fmaxf(b, fmaxf(__uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3])));
      c = fmaxf(c, fmaxf(__uint_as_float(sr[i + 4]), __uint_as_float(sr[i + 5])));
      d = fmaxf(d, fmaxf(__uint_as_float(sr[i + 6]), __uint_as_float(sr[i + 7])));
    }
    return fmaxf(fmaxf(a, b), fmaxf(c, d));
  }
}

// p = exp2(s*scale + neg) for 64 scores -> 32 packed bf16 pairs; returns the fp32 sum.  The
// unmasked form computes s*scale + neg two at a time (FFMA2) and sums with FADD2.
template <bool MASK>
PD_DEVICE float exp_pack64(const uint32_t (&sr)[64], int base, int lim, float scale, float neg, uint32_t (&pk)[32]) {
  if constexpr (MASK) {
    float rs = 0.f;
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
      float p0 = fast_exp2(fmaf(__uint_as_float(sr[i]), scale, neg));
      float p1 = fast_exp2(fmaf(__uint_as_float(sr[i + 1]), scale, neg));
      if (base + i > lim) p0 = 0.f;
      if (base + i + 1 > lim) p1 = 0.f;
      rs += p0 + p1;
      pk[i / 2] = pack_bf16x2(p0, p1);
    }
    return rs;
  } else {
    const float2 sc = make_float2(scale, scale), ng = make_float2(neg, neg);
    float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0;
#pragma unroll
    for (int i = 0; i < 64; i += 4) {
      const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])), sc, ng);
      const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3])), sc, ng);
      const float2 p0 = make_float2(fast_exp2(x0.x), fast_exp2(x0.y));
      const float2 p1 = make_float2(fast_exp2(x1.x), fast_exp2(x1.y));
      acc0 = __fadd2_rn(acc0, p0);
      acc1 = __fadd2_rn(acc1, p1);
      pk[i / 2] = pack_bf16x2(p0.x, p0.y);
      pk[i / 2 + 1] = pack_bf16x2(p1.x, p1.y);
    }
    const float2 t = __fadd2_rn(acc0, acc1);
    return t.x + t.y;
  }
}

// 2^x for two values on the FMA pipe (no MUFU): x = r + f with r = rint(x) (the 1.5*2^23 add puts
// r in the low mantissa bits) and f in [-1/2, 1/2]; 2^f by a degree-3 minimax polynomial (max
// relative error 7.5e-5, far below the bf16 rounding of P), 2^r by adding r << 23 to the exponent
// field.  x is clamped at -126 so the exponent add cannot wrap (2^-126 ~ 0 after bf16 / the sum).
PD_DEVICE float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 r = __fadd2_rn(x, magic);
  const float2 ri = __fadd2_rn(r, make_float2(-12582912.f, -12582912.f));  // rint(x), exact
  const float2 f = __ffma2_rn(ri, make_float2(-1.f, -1.f), x);                 // x - rint(x), exact
  float2 p = __ffma2_rn(f, make_float2(0.05517134442925453f, 0.05517134442925453f),
                        make_float2(0.24261033535003662f, 0.24261033535003662f));
  p = __ffma2_rn(p, f, make_float2(0.6932609677314758f, 0.6932609677314758f));
  p = __ffma2_rn(p, f, make_float2(0.9999281167984009f, 0.9999281167984009f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(r.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(r.y) << 23)));
}

// p = exp2(s*scale + neg) for 32 scores sr[0..31] -> 16 packed bf16 pairs (pk[i] = keys 2i, 2i+1,
// the column layout of a bf16 A operand in TMEM); returns the fp32 sum.  MASK: only columns
// base+i <= lim are kept.  POLY8 of every 8 pairs are computed on the FMA pipe (exp2_poly2) instead
// of the MUFU, whose 16 results / clock / SM bound the forward when every exp goes to it.
template <bool MASK, int POLY8>
PD_DEVICE float exp_pack32(const uint32_t* sr, int base, int lim, float scale, float neg, uint32_t (&pk)[16]) {
  const float2 sc = make_float2(scale, scale), ng = make_float2(neg, neg);
  float2 acc0 = make_float2(0.f, 0.f), acc1 = acc0;
#pragma unroll
  for (int i = 0; i < 32; i += 4) {
    const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])), sc, ng);
    const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3])), sc, ng);
    float2 p0 = ((i / 2) % 8) >= 8 - POLY8 ? exp2_poly2(x0) : make_float2(fast_exp2(x0.x), fast_exp2(x0.y));
    float2 p1 = ((i / 2 + 1) % 8) >= 8 - POLY8 ? exp2_poly2(x1) : make_float2(fast_exp2(x1.x), fast_exp2(x1.y));
    if constexpr (MASK) {
      if (base + i > lim) p0.x = 0.f;
      if (base + i + 1 > lim) p0.y = 0.f;
      if (base + i + 2 > lim) p1.x = 0.f;
      if (base + i + 3 > lim) p1.y = 0.f;
    }
    acc0 = __fadd2_rn(acc0, p0);
    acc1 = __fadd2_rn(acc1, p1);
    pk[i / 2] = pack_bf16x2(p0.x, p0.y);
    pk[i / 2 + 1] = pack_bf16x2(p1.x, p1.y);
  }
  const float2 t = __fadd2_rn(acc0, acc1);
  return t.x + t.y;
}

// Byte offset of (row, 16-byte chunk) of a 128B-swizzled tile (the TMA / UMMA SW128 pattern).
PD_DEVICE uint32_t sw128(int row, int chunk) { return row * 128 + ((chunk ^ (row & 7)) << 4); }

__global__ void __launch_bounds__(FWD_THREADS, 2)
    k_attn_fwd_tc(const __grid_constant__ CUtensorMap tm_qkv, __nv_bfloat16* __restrict__ out,
                  float* __restrict__ lse, int S, int H, float scale_log2) {
  griddep_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align_1k(smem_raw);
  uint8_t* sQ = smem + FwdSmem::Q;
  uint8_t* sK = smem + FwdSmem::K;
  uint8_t* sV = smem + FwdSmem::V;
  uint8_t* sP = smem + FwdSmem::P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + FwdSmem::BAR);
  uint64_t* full_q = bar + 0;
  uint64_t* full_k = bar + 1;
  uint64_t* full_v = bar + 2;
  uint64_t* empty_k = bar + 3;
  uint64_t* empty_v = bar + 4;
  uint64_t* s_full = bar + 5;
  uint64_t* p_ready = bar + 6;
  uint64_t* o_done = bar + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);

  const int n_qt = S / TQ;
  const int qt = n_qt - 1 - (int)blockIdx.x;  // heaviest (longest causal row) tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int D = H * HDIM;
  const int n_kt = qt + 1;
  const int row0 = b * S;  // token row of this sequence in qkv
  const int warp = warp_id();

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tm_qkv);
    mbar_init(full_q, 1);
    mbar_init(full_k, 1);
    mbar_init(full_v, 1);
    mbar_init(empty_k, 1);
    mbar_init(empty_v, 1);
    mbar_init(s_full, 1);
    mbar_init(p_ready, 4);
    mbar_init(o_done, 1);
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 1) tmem_alloc<256, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;

  if (warp == 0) {
    // ---------------- TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(full_q, TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, full_q, h * HDIM, row0 + qt * TQ);
      for (int j = 0; j < n_kt; ++j) {
        mbar_wait(empty_k, (j & 1) ^ 1);
        mbar_arrive_expect_tx(full_k, TILE_BYTES);
        tma_load_2d(sK, &tm_qkv, full_k, D + h * HDIM, row0 + j * TK);
        mbar_wait(empty_v, (j & 1) ^ 1);
        mbar_arrive_expect_tx(full_v, TILE_BYTES);
        tma_load_2d(sV, &tm_qkv, full_v, 2 * D + h * HDIM, row0 + j * TK);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(TQ, TK, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(TQ, HDIM, false, true);
      const uint32_t q_addr = smem_u32(sQ), k_addr = smem_u32(sK), v_addr = smem_u32(sV), p_addr = smem_u32(sP);
      auto issue_s = [&]() {
#pragma unroll
        for (int k = 0; k < HDIM / 16; ++k)
          umma_bf16(tS, make_sw128_desc(q_addr + k * 32, 16, 1024), make_sw128_desc(k_addr + k * 32, 16, 1024),
                    idesc_s, k != 0);
        umma_commit(s_full);
        umma_commit(empty_k);
      };
      mbar_wait(full_q, 0);
      mbar_wait(full_k, 0);
      tc_fence_after();
      issue_s();
      for (int j = 0; j < n_kt; ++j) {
        mbar_wait(p_ready, j & 1);  // S_j consumed, P_j in smem, O rescaled
        tc_fence_after();
        if (j + 1 < n_kt) {
          mbar_wait(full_k, (j + 1) & 1);
          tc_fence_after();
          issue_s();
        }
        mbar_wait(full_v, j & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < TK / 16; ++k) {
          // A = P (K-major over keys, 64-key atoms 16 KB apart); B = V (MN-major, +16 key rows = 2 KB)
          const uint64_t ad = make_sw128_desc(p_addr + (k >> 2) * TILE_BYTES + (k & 3) * 32, 16, 1024);
          const uint64_t bd = make_sw128_desc(v_addr + k * 2048, 8192, 1024);
          umma_bf16(tO, ad, bd, idesc_o, (j | k) != 0);
        }
        umma_commit(o_done);
        umma_commit(empty_v);
      }
    }
  } else {
    // ---------------- softmax: thread = query row (TMEM lane 32*(warp%4) + lane)
    const int quad = warp & 3;
    const int r = 32 * quad + lane_id();
    const int q = qt * TQ + r;  // query position in the sequence
    const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kt; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      const bool diag = j == qt;
      // two passes over the S row in TMEM, 64 columns (two loads, one wait) at a time, so the
      // softmax warps stay within the register budget of two CTAs per SM.  Only the diagonal tile
      // carries the causal mask (keys j*TK + i > q); the others run the unmasked, packed path.
      const int lim = diag ? q - j * TK : TK;
      float mx = -INFINITY;
#pragma unroll 1
      for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t sr[64];
        tmem_ld_32x32b_x32_nowait(tS + lane_base + h2 * 64, *reinterpret_cast<uint32_t(*)[32]>(sr));
        tmem_ld_32x32b_x32_nowait(tS + lane_base + h2 * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
        tmem_wait_ld();
        mx = diag ? row_max64<true>(sr, h2 * 64, lim, mx) : row_max64<false>(sr, 0, 0, mx);
      }
      const float m_new = fmaxf(m, mx * scale_log2);  // scale > 0: max commutes with it
      if (j > 0) mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} finished: O final for j-1, P free
      tc_fence_after();
      // Lazy rescaling: keep the stale running max (exponents up to 2^RESCALE_LOG2, exact in fp32
      // and bf16 range) unless some row of the warp moved by more than that; then the warp
      // rescales its O rows in TMEM and l.  m only has to be consistent between O, l and lse.
      if (j == 0) {
        m = m_new;
      } else if (__any_sync(0xffffffffu, m_new > m + RESCALE_LOG2)) {
        const float alpha = fast_exp2(m - m_new);
#pragma unroll
        for (int c = 0; c < HDIM / 32; ++c) {
          float o[32];
          tmem_ld_32x32b_x32(tO + lane_base + c * 32, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= alpha;
          tmem_st_32x32b_x32(tO + lane_base + c * 32, o);
        }
        l *= alpha;
        m = m_new;
      }
      // P = exp2(s*scale - m) -> bf16 -> smem (K-major SW128; 64-key atom h2)
      float rs = 0.f;
      const float neg = -m;
#pragma unroll 1
      for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t sr[64];
        tmem_ld_32x32b_x32_nowait(tS + lane_base + h2 * 64, *reinterpret_cast<uint32_t(*)[32]>(sr));
        tmem_ld_32x32b_x32_nowait(tS + lane_base + h2 * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
        tmem_wait_ld();
        uint32_t pk[32];
        rs += diag ? exp_pack64<true>(sr, h2 * 64, lim, scale_log2, neg, pk)
                   : exp_pack64<false>(sr, 0, 0, scale_log2, neg, pk);
        uint8_t* atom = sP + h2 * TILE_BYTES;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<uint4*>(atom + sw128(r, u)) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
      l += rs;
      fence_proxy_async_shared();  // P (generic-proxy stores) -> visible to the tensor core
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(p_ready);
    }
    mbar_wait(o_done, (n_kt - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = out + ((int64_t)row0 + q) * D + h * HDIM;
#pragma unroll
    for (int c = 0; c < HDIM / 32; ++c) {
      float o[32];
      tmem_ld_32x32b_x32(tO + lane_base + c * 32, o);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] *= inv;
      store32_bf16(orow, 0, 0, c * 32, o);
    }
    lse[((int64_t)b * H + h) * S + q] = m + log2f(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256, 1>(tmem);
  }
}

// ================================================================ forward, S decoupled from P
// One CTA per (128-query tile, head, sequence), two CTAs per SM, 256 TMEM columns each:
//   S [0,128) fp32 scores, O [128,192) fp32 output, P [192,256) bf16 probabilities (key pairs).
// The softmax warps pull the whole S row into registers (four 32-column loads, one wait) and
// release S at once (s_free), so S_{j+1} = Q K_{j+1}^T runs on the tensor core while they compute
// exp2 of tile j.  P_j goes to TMEM (tcgen05.st) and O += P_j V_j reads it as the A operand
// straight from TMEM (the TS form), so P never touches shared memory.  K and V stream through a
// two-stage ring.  Numerics are those of k_attn_fwd_tc (same max, exp2, lazy rescale, bf16 P).
#if PD_ATTN_TRACE
// Diagnostic build only (tools/build_variant.sh ... -DPD_ATTN_TRACE=1): %globaltimer stamps of the
// forward's per-tile events for the first CTAs, read back with pd_attn_trace().
constexpr int TR_CTAS = 2048, TR_EV = 64;
__device__ unsigned long long g_attn_trace[TR_CTAS][TR_EV];
PD_DEVICE void tr_stamp(int slot) {
  const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (cta < TR_CTAS && slot < TR_EV) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_attn_trace[cta][slot] = t;
    if (slot == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_attn_trace[cta][TR_EV - 1] = smid;
    }
  }
}
#define TR(slot) tr_stamp(slot)
#else
#define TR(slot) ((void)0)
#endif
constexpr int FWD2_STAGES = 2;
struct Fwd2Smem {
  static constexpr int Q = 0;
  static constexpr int K = Q + TILE_BYTES;                     // [FWD2_STAGES]
  static constexpr int V = K + FWD2_STAGES * TILE_BYTES;       // [FWD2_STAGES]
  static constexpr int BAR = V + FWD2_STAGES * TILE_BYTES;
  static constexpr int TOTAL = BAR + 256 + 1024;
};

template <int POLY8>
__global__ void __launch_bounds__(FWD_THREADS, 2)
    k_attn_fwd_tc2(const __grid_constant__ CUtensorMap tm_qkv, __nv_bfloat16* __restrict__ out,
                   float* __restrict__ lse, int S, int H, float scale_log2) {
  griddep_wait();
  if (threadIdx.x == 64) TR(0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align_1k(smem_raw);
  uint8_t* sQ = smem + Fwd2Smem::Q;
  uint8_t* sK = smem + Fwd2Smem::K;
  uint8_t* sV = smem + Fwd2Smem::V;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Fwd2Smem::BAR);
  uint64_t* full_q = bar + 0;
  uint64_t* full_k = bar + 1;                    // [FWD2_STAGES]
  uint64_t* full_v = full_k + FWD2_STAGES;       // [FWD2_STAGES]
  uint64_t* empty_k = full_v + FWD2_STAGES;      // [FWD2_STAGES]
  uint64_t* empty_v = empty_k + FWD2_STAGES;     // [FWD2_STAGES]
  uint64_t* s_full = empty_v + FWD2_STAGES;
  uint64_t* s_free = s_full + 1;
  uint64_t* p_ready = s_full + 2;
  uint64_t* o_done = s_full + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 4);

  const int n_qt = S / TQ;
  // grid (H, B, tiles): the tile index varies slowest, so the block scheduler hands out every
  // (head, sequence)'s longest causal row first and the light diagonal tiles last (LPT order)
  const int qt = n_qt - 1 - (int)blockIdx.z;
  const int h = blockIdx.x, b = blockIdx.y;
  const int D = H * HDIM;
  const int n_kt = qt + 1;
  const int row0 = b * S;
  const int warp = warp_id();

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tm_qkv);
    mbar_init(full_q, 1);
    for (int i = 0; i < FWD2_STAGES; ++i) {
      mbar_init(&full_k[i], 1);
      mbar_init(&full_v[i], 1);
      mbar_init(&empty_k[i], 1);
      mbar_init(&empty_v[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(p_ready, 4);
    mbar_init(o_done, 1);
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 1) tmem_alloc<256, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128, tP = tmem + 192;

  if (warp == 0) {
    // ---------------- TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(full_q, TILE_BYTES);
      tma_load_2d(sQ, &tm_qkv, full_q, h * HDIM, row0 + qt * TQ);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j % FWD2_STAGES;
        const uint32_t ph = ((j / FWD2_STAGES) & 1) ^ 1;
        mbar_wait(&empty_k[st], ph);
        mbar_arrive_expect_tx(&full_k[st], TILE_BYTES);
        tma_load_2d(sK + st * TILE_BYTES, &tm_qkv, &full_k[st], D + h * HDIM, row0 + j * TK);
        mbar_wait(&empty_v[st], ph);
        mbar_arrive_expect_tx(&full_v[st], TILE_BYTES);
        tma_load_2d(sV + st * TILE_BYTES, &tm_qkv, &full_v[st], 2 * D + h * HDIM, row0 + j * TK);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(TQ, TK, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(TQ, HDIM, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_s = [&](int j) {
        const int st = j % FWD2_STAGES;
        const uint32_t k_addr = smem_u32(sK + st * TILE_BYTES);
        mbar_wait(&full_k[st], (j / FWD2_STAGES) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < HDIM / 16; ++k)
          umma_bf16(tS, make_sw128_desc(q_addr + k * 32, 16, 1024), make_sw128_desc(k_addr + k * 32, 16, 1024),
                    idesc_s, k != 0);
        umma_commit(s_full);
        umma_commit(&empty_k[st]);
      };
      mbar_wait(full_q, 0);
      issue_s(0);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j % FWD2_STAGES;
        mbar_wait(s_free, j & 1);  // S_j is in the softmax warps' registers
        tc_fence_after();
        if (j + 1 < n_kt) issue_s(j + 1);
        mbar_wait(p_ready, j & 1);  // P_j in TMEM, O rescaled
        mbar_wait(&full_v[st], (j / FWD2_STAGES) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + st * TILE_BYTES);
#pragma unroll
        for (int k = 0; k < TK / 16; ++k)  // A = P from TMEM (8 columns = 16 keys), B = V (MN-major)
          umma_bf16_ts(tO, tP + k * 8, make_sw128_desc(v_addr + k * 2048, 8192, 1024), idesc_o, (j | k) != 0);
        umma_commit(o_done);
        umma_commit(&empty_v[st]);
      }
    }
  } else {
    // ---------------- softmax: thread = query row (TMEM lane 32*(warp%4) + lane)
    const int quad = warp & 3;
    const int r = 32 * quad + lane_id();
    const int q = qt * TQ + r;
    const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
    float m = -INFINITY, l = 0.f;
    if (threadIdx.x == 64) TR(1);
    for (int j = 0; j < n_kt; ++j) {
      mbar_wait(s_full, j & 1);
      if (threadIdx.x == 64) TR(2 + 4 * j);
      tc_fence_after();
      uint32_t sr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tmem_ld_32x32b_x32_nowait(tS + lane_base + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32 * c));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(s_free);  // the tensor core may write S_{j+1} now
      const bool diag = j == qt;
      const int lim = diag ? q - j * TK : TK;
      float mx;
      if (diag) {
        mx = row_max64<true>(*reinterpret_cast<const uint32_t(*)[64]>(sr), 0, lim, -INFINITY);
        mx = row_max64<true>(*reinterpret_cast<const uint32_t(*)[64]>(sr + 64), 64, lim, mx);
      } else {
        mx = row_max64<false>(*reinterpret_cast<const uint32_t(*)[64]>(sr), 0, 0, -INFINITY);
        mx = row_max64<false>(*reinterpret_cast<const uint32_t(*)[64]>(sr + 64), 0, 0, mx);
      }
      const float m_new = fmaxf(m, mx * scale_log2);
      // lazy rescale decision; O itself is rescaled below, once PV_{j-1} has finished with it
      float alpha = 1.f;
      const bool rescale = j > 0 && __any_sync(0xffffffffu, m_new > m + RESCALE_LOG2);
      if (j == 0 || rescale) {
        alpha = fast_exp2(m - m_new);
        m = m_new;
      }
      // P_j = exp2(s*scale - m) -> packed bf16 pairs in registers (independent of PV_{j-1})
      float rs = 0.f;
      const float neg = -m;
      uint32_t pk[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        rs += diag ? exp_pack32<true, POLY8>(sr + 32 * c, 32 * c, lim, scale_log2, neg, pk[c])
                   : exp_pack32<false, POLY8>(sr + 32 * c, 0, 0, scale_log2, neg, pk[c]);
      if (threadIdx.x == 64) TR(3 + 4 * j);
      if (j > 0) mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} done: O final for j-1, P free
      if (threadIdx.x == 64) TR(4 + 4 * j);
      tc_fence_after();
      if (rescale) {
#pragma unroll
        for (int c = 0; c < HDIM / 16; ++c) {
          uint32_t o[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7]),
                "=r"(o[8]), "=r"(o[9]), "=r"(o[10]), "=r"(o[11]), "=r"(o[12]), "=r"(o[13]), "=r"(o[14]), "=r"(o[15])
              : "r"(tO + lane_base + c * 16)
              : "memory");
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st_32x32b_x16(tO + lane_base + c * 16, o);
        }
      }
      l = l * alpha + rs;
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st_32x32b_x16(tP + lane_base + c * 16, pk[c]);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(p_ready);
      if (threadIdx.x == 64) TR(5 + 4 * j);
    }
    mbar_wait(o_done, (n_kt - 1) & 1);
    if (threadIdx.x == 64) TR(40);
    tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = out + ((int64_t)row0 + q) * D + h * HDIM;
#pragma unroll
    for (int c = 0; c < HDIM / 32; ++c) {
      float o[32];
      tmem_ld_32x32b_x32(tO + lane_base + c * 32, o);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] *= inv;
      store32_bf16(orow, 0, 0, c * 32, o);
    }
    lse[((int64_t)b * H + h) * S + q] = m + log2f(l);
    if (threadIdx.x == 64) TR(41);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256, 1>(tmem);
  }
}

// ================================================================ backward
// One CTA per (128-key tile, head, sequence), looping over the query tiles at or after the
// diagonal.  TMEM columns: S^T [0,128), dP^T [128,256), dV [256,320), dK [320,384), dQ [384,448),
// P^T (bf16 pairs) [448,512).
//   MMA warp:   S^T = K Q^T, dP^T = V dO^T (M = keys, N = queries, K = 64)
//               dV += P^T dO, dK += dS^T Q  (M = keys, N = 64, K = queries)
//               dQ  = dS K                  (M = queries, N = 64, K = keys; A = dS^T read MN-major)
//   warps 2-9:  thread = TMEM lane, two warps per lane quadrant splitting the 128 query columns (and
//               the 64 dQ / dK / dV columns) so two compute warps per SM sub-partition hide each
//               other's latency: P^T = exp2(S^T*scale - lse) -> bf16 into TMEM cols [448,512)
//               (the A operand of dV += P^T dO, read straight from TMEM), dS^T = P^T (dP^T - D)
//               -> bf16 into shared memory (K-major over queries; A of dK, MN-major A of dQ), and
//               the previous tile's dQ out of TMEM into the fp32 dq_acc by TMA reduce-add.
//   Q / dO / lse / D stream through a 3-stage ring; S^T / dP^T of tile n+1 are issued once the
//   compute warps hold tile n in registers (sdp_free).
constexpr int BWD_THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 compute (two per TMEM lane quadrant)
PD_DEVICE void named_sync_compute() { asm volatile("bar.sync 1, 256;" ::: "memory"); }  // the 8 compute warps

// One 32-query chunk of a key row: P^T = exp2(S^T*scale - lse), dS^T = P^T (dP^T - D) -> bf16 pairs.
// lse: the query rows' log-sum-exp (log2 domain).  MASK (diagonal tile only): queries q0+i < key are causal-masked.  The unmasked
// form runs two elements per FFMA2 / FMUL2.
template <bool MASK>
PD_DEVICE void bwd_chunk32(const uint32_t (&svr)[32], const uint32_t (&dpr)[32], const float* lse_row, const float* Dd,
                           int q0, int key, float scale, uint32_t (&pk)[16], uint32_t (&dk)[16]) {
  const float* sv = reinterpret_cast<const float*>(svr);
  const float* dp = reinterpret_cast<const float*>(dpr);
  const float4* L4 = reinterpret_cast<const float4*>(lse_row);
  const float4* D4 = reinterpret_cast<const float4*>(Dd);
  const float2 sc = make_float2(scale, scale), m1 = make_float2(-1.f, -1.f);
#pragma unroll
  for (int i = 0; i < 32; i += 4) {
    const float4 lv = L4[i / 4], dv = D4[i / 4];
    const float2 x0 = __ffma2_rn(make_float2(sv[i], sv[i + 1]), sc, make_float2(-lv.x, -lv.y));
    const float2 x1 = __ffma2_rn(make_float2(sv[i + 2], sv[i + 3]), sc, make_float2(-lv.z, -lv.w));
    float2 p0 = make_float2(fast_exp2(x0.x), fast_exp2(x0.y));
    float2 p1 = make_float2(fast_exp2(x1.x), fast_exp2(x1.y));
    if constexpr (MASK) {
      if (q0 + i < key) p0.x = 0.f;
      if (q0 + i + 1 < key) p0.y = 0.f;
      if (q0 + i + 2 < key) p1.x = 0.f;
      if (q0 + i + 3 < key) p1.y = 0.f;
    }
    const float2 t0 = __ffma2_rn(make_float2(dv.x, dv.y), m1, make_float2(dp[i], dp[i + 1]));  // dP - D
    const float2 t1 = __ffma2_rn(make_float2(dv.z, dv.w), m1, make_float2(dp[i + 2], dp[i + 3]));
    const float2 d0 = __fmul2_rn(p0, t0), d1 = __fmul2_rn(p1, t1);
    pk[i / 2] = pack_bf16x2(p0.x, p0.y);
    pk[i / 2 + 1] = pack_bf16x2(p1.x, p1.y);
    dk[i / 2] = pack_bf16x2(d0.x, d0.y);
    dk[i / 2 + 1] = pack_bf16x2(d1.x, d1.y);
  }
}
constexpr int BWD_STAGES = 2;  // Q / dO / lse / D ring (the K / V double buffer takes the third stage's smem)
struct BwdSmem {
  static constexpr int K = 0;                                   // [2] (this item's, the next item's)
  static constexpr int V = K + 2 * TILE_BYTES;                  // [2]
  static constexpr int Q = V + 2 * TILE_BYTES;                  // [BWD_STAGES]
  static constexpr int DO = Q + BWD_STAGES * TILE_BYTES;        // [BWD_STAGES]
  static constexpr int DS = DO + BWD_STAGES * TILE_BYTES;       // dS^T: two K-major atoms over queries
  static constexpr int LD = DS + 2 * TILE_BYTES;                // lse/D: [stage][2][128] floats
  static constexpr int DQ = LD + BWD_STAGES * 2 * 128 * 4;      // dQ staging [128][64] fp32 (TMA reduce-add)
  static constexpr int BAR = DQ + 128 * 64 * 4;
  static constexpr int TOTAL = BAR + 256 + 1024;
};
static_assert(BwdSmem::TOTAL <= 227 * 1024, "attention bwd smem");

// Work item of the persistent backward: one (key tile, head, sequence).  Items are numbered key tile
// slowest, so item order is longest-first (key tile kt has n_t - kt query tiles); CTA c of P takes
// items c, 2P-1-c, 2P+c, 4P-1-c, ... (a boustrophedon over the longest-first list), which balances
// the per-CTA sums of query tiles to within one tile of the mean (8 x 1024 tokens, 16 heads: 32 vs 31.1).
struct BwdItem {
  int kt, h, b, N;
};
PD_DEVICE bool bwd_item(int r, int n_items, int H, int B, int n_t, BwdItem& it) {
  const int P = (int)gridDim.x, c = (int)blockIdx.x;
  const int idx = r * P + ((r & 1) ? P - 1 - c : c);
  if (idx >= n_items) return false;
  it.kt = idx / (H * B);
  const int hb = idx - it.kt * (H * B);
  it.h = hb % H;
  it.b = hb / H;
  it.N = n_t - it.kt;
  return true;
}

// Persistent causal attention backward: one CTA per SM loops over its work items.  Per item the
// K / V tiles are loaded once (double-buffered, so the next item's arrive during this one) and the
// query tiles kt .. n_t-1 stream through the Q / dO / lse / D ring.  TMEM columns: S^T [0,128),
// dP^T [128,256), dV [256,320), dK [320,384), dQ [384,448), P^T (bf16 pairs) [448,512).
//   MMA warp:   S^T = K Q^T, dP^T = V dO^T (M = keys, N = queries, K = 64)
//               dV += P^T dO (P^T from TMEM), dK += dS^T Q (M = keys, N = 64, K = queries)
//               dQ  = dS K (M = queries, N = 64, K = keys; A = dS^T read MN-major)
//   warps 2-9:  thread = TMEM lane, two warps per lane quadrant splitting the 128 query columns (and
//               the 64 dQ / dK / dV columns): P^T = exp2(S^T*scale - lse) -> bf16 into TMEM, dS^T =
//               P^T (dP^T - D) -> bf16 into shared memory, the previous tile's dQ out of TMEM into the
//               fp32 dq_acc by TMA reduce-add, and at an item boundary the finished item's dK / dV.
// S^T / dP^T of the next tile (also across an item boundary) are issued as soon as the compute warps
// hold the current tile in registers (sdp_free), so the previous item's dQ flush and dK / dV
// read-out run under the next item's first S^T / dP^T MMAs: there is no per-item prologue or tail.
__global__ void __launch_bounds__(BWD_THREADS, 1)
    k_attn_bwd_tc(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                  const __grid_constant__ CUtensorMap tm_dq,
                  const float* __restrict__ lse, const float* __restrict__ Dv, __nv_bfloat16* __restrict__ dqkv,
                  float* __restrict__ dq_acc, int S, int H, int B, float scale_log2, float scale) {
  griddep_wait();
  if (threadIdx.x == 64) TR(0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align_1k(smem_raw);
  uint8_t* sK = smem + BwdSmem::K;
  uint8_t* sV = smem + BwdSmem::V;
  uint8_t* sQ = smem + BwdSmem::Q;
  uint8_t* sdO = smem + BwdSmem::DO;
  uint8_t* sdS = smem + BwdSmem::DS;
  float* sLD = reinterpret_cast<float*>(smem + BwdSmem::LD);
  float* sDQ = reinterpret_cast<float*>(smem + BwdSmem::DQ);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + BwdSmem::BAR);
  uint64_t* full_kv = bar + 0;                   // [2]
  uint64_t* empty_kv = full_kv + 2;              // [2]
  uint64_t* full_qdo = empty_kv + 2;             // [BWD_STAGES]
  uint64_t* empty_qdo = full_qdo + BWD_STAGES;   // [BWD_STAGES]
  uint64_t* sdp_full = empty_qdo + BWD_STAGES;
  uint64_t* pds_ready = sdp_full + 1;
  uint64_t* dq_full = sdp_full + 2;
  uint64_t* sdp_free = sdp_full + 3;  // compute warps have read S^T / dP^T of the current tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sdp_full + 4);

  const int n_t = S / TK;
  const int n_items = n_t * H * B;
  const int D = H * HDIM;
  const int warp = warp_id();

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    for (int i = 0; i < 2; ++i) { mbar_init(&full_kv[i], 1); mbar_init(&empty_kv[i], 1); }
    for (int i = 0; i < BWD_STAGES; ++i) { mbar_init(&full_qdo[i], 1); mbar_init(&empty_qdo[i], 1); }
    mbar_init(sdp_full, 1);
    mbar_init(pds_ready, 8);
    mbar_init(dq_full, 1);
    mbar_init(sdp_free, 8);
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 1) tmem_alloc<512, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tdV = tmem + 256, tdK = tmem + 320, tdQ = tmem + 384;
  const uint32_t tPt = tmem + 448;  // P^T as bf16 pairs (64 columns), the A operand of dV

  if (warp == 0) {
    // ---------------- TMA producer: per item K / V (double-buffered), then the query tiles
    if (elect_one()) {
      BwdItem it;
      int g = 0, ic = 0;
      for (int r = 0; r * (int)gridDim.x < n_items; ++r) {
        if (!bwd_item(r, n_items, H, B, n_t, it)) continue;
        const int kb = ic & 1, row0 = it.b * S;
        mbar_wait(&empty_kv[kb], ((ic >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&full_kv[kb], 2 * TILE_BYTES);
        tma_load_2d(sK + kb * TILE_BYTES, &tm_qkv, &full_kv[kb], D + it.h * HDIM, row0 + it.kt * TK);
        tma_load_2d(sV + kb * TILE_BYTES, &tm_qkv, &full_kv[kb], 2 * D + it.h * HDIM, row0 + it.kt * TK);
        for (int n = 0; n < it.N; ++n, ++g) {
          const int st = g % BWD_STAGES, qt = it.kt + n;
          mbar_wait(&empty_qdo[st], ((g / BWD_STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full_qdo[st], 2 * TILE_BYTES + 2 * TQ * 4);
          tma_load_2d(sQ + st * TILE_BYTES, &tm_qkv, &full_qdo[st], it.h * HDIM, row0 + qt * TQ);
          tma_load_2d(sdO + st * TILE_BYTES, &tm_do, &full_qdo[st], it.h * HDIM, row0 + qt * TQ);
          // this query tile's log-sum-exp and D rows ride along with Q / dO (stage buffers)
          const int64_t lrow = ((int64_t)it.b * H + it.h) * S + qt * TQ;
          bulk_load_1d(sLD + st * 256, lse + lrow, TQ * 4, &full_qdo[st]);
          bulk_load_1d(sLD + st * 256 + 128, Dv + lrow, TQ * 4, &full_qdo[st]);
        }
        ++ic;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_sq = make_idesc_bf16(TK, TQ, false, false);      // S^T, dP^T
      constexpr uint32_t idesc_kv = make_idesc_bf16(TK, HDIM, false, true);     // dV, dK
      constexpr uint32_t idesc_q = make_idesc_bf16(TQ, HDIM, true, true);       // dQ (A = dS^T MN-major)
      const uint32_t ds_addr = smem_u32(sdS);
      auto issue_sdp = [&](int g, int kb) {
        const int st = g % BWD_STAGES;
        const uint32_t k_addr = smem_u32(sK + kb * TILE_BYTES), v_addr = smem_u32(sV + kb * TILE_BYTES);
        const uint32_t q_addr = smem_u32(sQ + st * TILE_BYTES), do_addr = smem_u32(sdO + st * TILE_BYTES);
        mbar_wait(&full_qdo[st], (g / BWD_STAGES) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < HDIM / 16; ++k) {
          umma_bf16(tS, make_sw128_desc(k_addr + k * 32, 16, 1024), make_sw128_desc(q_addr + k * 32, 16, 1024),
                    idesc_sq, k != 0);
          umma_bf16(tP, make_sw128_desc(v_addr + k * 32, 16, 1024), make_sw128_desc(do_addr + k * 32, 16, 1024),
                    idesc_sq, k != 0);
        }
        umma_commit(sdp_full);
      };
      BwdItem it, nx;
      int r = 0;
      auto fetch = [&](BwdItem& x) {  // next item of this CTA (false: none left)
        for (; r * (int)gridDim.x < n_items; ++r)
          if (bwd_item(r, n_items, H, B, n_t, x)) { ++r; return true; }
        return false;
      };
      bool have = fetch(it);
      int g = 0, ic = 0;
      if (have) {
        mbar_wait(&full_kv[0], 0);
        issue_sdp(0, 0);
      }
      while (have) {
        const int kb = ic & 1;
        const bool more = fetch(nx);
        const uint32_t k_addr = smem_u32(sK + kb * TILE_BYTES);
        for (int n = 0; n < it.N; ++n, ++g) {
          const int st = g % BWD_STAGES;
          const uint32_t q_addr = smem_u32(sQ + st * TILE_BYTES), do_addr = smem_u32(sdO + st * TILE_BYTES);
          mbar_wait(sdp_free, g & 1);  // S^T / dP^T of g are in the compute warps' registers
          if (n + 1 < it.N) {
            issue_sdp(g + 1, kb);
          } else if (more) {  // the next item's first tile, on the other K / V buffer
            mbar_wait(&full_kv[kb ^ 1], ((ic + 1) >> 1) & 1);
            issue_sdp(g + 1, kb ^ 1);
          }
          mbar_wait(pds_ready, g & 1);  // P^T / dS^T of g in place, dQ of g-1 (and the last item's dK / dV) read
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < TQ / 16; ++k) {
            const uint32_t a_off = (k >> 2) * TILE_BYTES + (k & 3) * 32;  // K-major over queries
            // dV += P^T dO with P^T in TMEM (8 columns = 16 bf16 queries per step)
            umma_bf16_ts(tdV, tPt + k * 8, make_sw128_desc(do_addr + k * 2048, 8192, 1024), idesc_kv, (n | k) != 0);
            umma_bf16(tdK, make_sw128_desc(ds_addr + a_off, 16, 1024), make_sw128_desc(q_addr + k * 2048, 8192, 1024),
                      idesc_kv, (n | k) != 0);
          }
#pragma unroll
          for (int k = 0; k < TK / 16; ++k)  // K = keys: dS^T rows (+2 KB per 16), query atoms 16 KB apart
            umma_bf16(tdQ, make_sw128_desc(ds_addr + k * 2048, TILE_BYTES, 1024),
                      make_sw128_desc(k_addr + k * 2048, 8192, 1024), idesc_q, k != 0);
          umma_commit(dq_full);
          umma_commit(&empty_qdo[st]);
        }
        umma_commit(&empty_kv[kb]);
        it = nx;
        have = more;
        ++ic;
      }
    }
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;         // warps 2-5: query columns 0..63, warps 6-9: 64..127
    const int r = 32 * quad + lane_id();      // TMEM lane: key row (S^T, dP^T, dK, dV) / query row (dQ)
    const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
    const int t = threadIdx.x - 64;           // 0..255 within the compute warps
    // dQ rows of a query tile: TMEM -> staging smem (two [128][32] fp32 halves, 128B-swizzled,
    // conflict-free) -> one TMA reduce-add per half of the 128 x 32 fp32 box into dq_acc.
    // dQ rows of a query tile: TMEM -> staging smem (two [128][32] fp32 halves, 128B-swizzled,
    // conflict-free) -> one TMA reduce-add per half of the 128 x 32 fp32 box into dq_acc.  Staging
    // and issue are split so the tile's dS^T / P^T stores share one proxy fence with the staging.
    auto stage_dq = [&]() {
      uint32_t v0[32];
      tmem_ld_32x32b_x32_nowait(tdQ + lane_base + half * 32, v0);
      tmem_wait_ld();
      if (t == 0) bulk_wait_read0();  // the previous reduce has finished reading the staging
      named_sync_compute();
      uint8_t* sth = reinterpret_cast<uint8_t*>(sDQ) + half * 128 * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(sth + sw128(r, c)) = make_uint4(v0[4 * c], v0[4 * c + 1], v0[4 * c + 2], v0[4 * c + 3]);
    };
    auto issue_dq = [&](int h, int trow) {  // after the staging stores + fence.proxy.async of every warp
      named_sync_compute();
      if (t == 0) {
        uint8_t* st0 = reinterpret_cast<uint8_t*>(sDQ);
        tma_reduce_add_2d(&tm_dq, st0, h * HDIM, trow);
        tma_reduce_add_2d(&tm_dq, st0 + 128 * 128, h * HDIM + 32, trow);
        bulk_commit();
      }
    };
    // dK (scaled) and dV rows of this thread's key of a finished item into the k / v slices of dqkv
    auto store_dkv = [&](const BwdItem& x) {
      __nv_bfloat16* row = dqkv + ((int64_t)x.b * S + x.kt * TK + r) * 3 * D;
      const int c = half;  // this warp's 32 of the 64 head dims
      float v[32];
      tmem_ld_32x32b_x32(tdK + lane_base + c * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= scale;
      store32_bf16(row + D + x.h * HDIM, 0, 0, c * 32, v);
      tmem_ld_32x32b_x32(tdV + lane_base + c * 32, v);
      store32_bf16(row + 2 * D + x.h * HDIM, 0, 0, c * 32, v);
    };
    BwdItem it, prev;
    int pend_h = 0, pend_row = 0;  // the previous tile's dQ destination (head, token row)
    int g = 0;
    for (int rr = 0; rr * (int)gridDim.x < n_items; ++rr) {
      if (!bwd_item(rr, n_items, H, B, n_t, it)) continue;
      const int key = it.kt * TK + r;
      for (int n = 0; n < it.N; ++n, ++g) {
        const int qt = it.kt + n;
        const int par = g % BWD_STAGES;  // stage of this query tile's Q / dO / lse / D buffers
        const float* sL = sLD + par * 256;  // this query tile's lse (log2 domain), then D
        const float* sDd = sL + 128;
        mbar_wait(sdp_full, g & 1);  // implies the stage's TMA (incl. lse / D) has landed
        if (threadIdx.x == 64 && g < 9) TR(1 + 4 * g);
        tc_fence_after();
        const bool diag = n == 0;
        uint32_t pk[2][16], dk[2][16];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {  // this warp's two 32-query chunks
          const int c = 2 * half + cc;
          uint32_t svr[32], dpr[32];
          tmem_ld_32x32b_x32_nowait(tS + lane_base + c * 32, svr);
          tmem_ld_32x32b_x32_nowait(tP + lane_base + c * 32, dpr);
          tmem_wait_ld();
          if (diag) bwd_chunk32<true>(svr, dpr, sL + c * 32, sDd + c * 32, qt * TQ + c * 32, key, scale_log2, pk[cc], dk[cc]);
          else bwd_chunk32<false>(svr, dpr, sL + c * 32, sDd + c * 32, 0, 0, scale_log2, pk[cc], dk[cc]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(sdp_free);  // the tensor core may overwrite S^T / dP^T now
        if (threadIdx.x == 64 && g < 9) TR(2 + 4 * g);
        if (g > 0) {  // dV / dK / dQ of g-1 are done: P / dS smem is free, flush dQ of g-1
          mbar_wait(dq_full, (g - 1) & 1);
          if (threadIdx.x == 64 && g < 9) TR(3 + 4 * g);
          tc_fence_after();
          stage_dq();
        }
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = 2 * half + cc;
          const int atom = (c >> 1) * TILE_BYTES;
          const int chunk0 = (c & 1) * 4;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<uint4*>(sdS + atom + sw128(r, chunk0 + u)) =
                make_uint4(dk[cc][4 * u], dk[cc][4 * u + 1], dk[cc][4 * u + 2], dk[cc][4 * u + 3]);
          tmem_st_32x32b_x16(tPt + lane_base + c * 16, pk[cc]);
        }
        // g-1 was the previous item's last tile: its dK / dV are final (dq_full above), read them
        // out before pds_ready lets this item's first dV / dK MMAs overwrite the accumulators
        if (diag && g > 0) store_dkv(prev);
        tmem_wait_st();
        fence_proxy_async_shared();
        if (g > 0) issue_dq(pend_h, pend_row);
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(pds_ready);
        if (threadIdx.x == 64 && g < 9) TR(4 + 4 * g);
        pend_h = it.h;
        pend_row = it.b * S + qt * TQ;
      }
      prev = it;
    }
    if (g > 0) {
      mbar_wait(dq_full, (g - 1) & 1);
      tc_fence_after();
      stage_dq();
      fence_proxy_async_shared();
      issue_dq(pend_h, pend_row);
      store_dkv(prev);
    }
    if (t == 0) bulk_wait_all0();  // the last reduce-add has completed before the CTA exits
    if (threadIdx.x == 64) TR(41);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D map over a row-major bf16 [rows, cols] matrix, 64 x 128 boxes, 128B swizzle.
int map_rows(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols) {
  auto fn = encode_tiled();
  if (!fn) return set_error(PD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : set_error(PD_ERR_CUDA, "attention tensor map (%d)", (int)r);
}

}  // namespace

int attn_fwd_tc(const void* qkv, void* out, float* lse, int B, int S, int H, cudaStream_t st) {
  if (S % TQ || B < 1 || H < 1) return set_error(PD_ERR_INVALID, "attention: seq %% 128 == 0 required");
  CUtensorMap tm;
  const int rc = map_rows(&tm, qkv, (int64_t)B * S, 3ll * H * HDIM);
  if (rc) return rc;
  static int v1 = -1, poly = -1;  // PD_ATTN_FWD_V1=1: the round-1 kernel; PD_ATTN_POLY: FMA-pipe exp2 pairs of 8
  if (v1 < 0) {
    const char* e = getenv("PD_ATTN_FWD_V1");
    v1 = e && atoi(e) ? 1 : 0;
    const char* p = getenv("PD_ATTN_POLY");
    poly = p ? atoi(p) : 0;  // MUFU only: the FMA-pipe split measured no faster
  }
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_attn_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem::TOTAL) != cudaSuccess ||
        cudaFuncSetAttribute(k_attn_fwd_tc2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Smem::TOTAL) != cudaSuccess ||
        cudaFuncSetAttribute(k_attn_fwd_tc2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Smem::TOTAL) != cudaSuccess ||
        cudaFuncSetAttribute(k_attn_fwd_tc2<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Smem::TOTAL) != cudaSuccess ||
        cudaFuncSetAttribute(k_attn_fwd_tc2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Smem::TOTAL) != cudaSuccess)
      return set_error(PD_ERR_CUDA, "attention fwd: shared memory attribute");
    attr = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)HDIM);
  auto* __restrict__ o = static_cast<__nv_bfloat16*>(out);
  if (v1) {
    launch_pdl(k_attn_fwd_tc, dim3(S / TQ, H, B), dim3(FWD_THREADS), FwdSmem::TOTAL, st, tm, o, lse, S, H, scale_log2);
  } else {
    const dim3 grid(H, B, S / TQ);
    if (poly == 2) launch_pdl(k_attn_fwd_tc2<2>, grid, dim3(FWD_THREADS), Fwd2Smem::TOTAL, st, tm, o, lse, S, H, scale_log2);
    else if (poly == 3) launch_pdl(k_attn_fwd_tc2<3>, grid, dim3(FWD_THREADS), Fwd2Smem::TOTAL, st, tm, o, lse, S, H, scale_log2);
    else if (poly == 4) launch_pdl(k_attn_fwd_tc2<4>, grid, dim3(FWD_THREADS), Fwd2Smem::TOTAL, st, tm, o, lse, S, H, scale_log2);
    else launch_pdl(k_attn_fwd_tc2<0>, grid, dim3(FWD_THREADS), Fwd2Smem::TOTAL, st, tm, o, lse, S, H, scale_log2);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "attention fwd: %s", cudaGetErrorString(e));
}

int attn_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* Dv, float* dq_acc, void* dqkv, int B,
                int S, int H, cudaStream_t st) {
  if (S % TQ || B < 1 || H < 1) return set_error(PD_ERR_INVALID, "attention: seq %% 128 == 0 required");
  CUtensorMap tq, tdo, tdq;
  int rc = map_rows(&tq, qkv, (int64_t)B * S, 3ll * H * HDIM);
  if (rc) return rc;
  rc = map_rows(&tdo, dout, (int64_t)B * S, (int64_t)H * HDIM);
  if (rc) return rc;
  {
    auto fn = encode_tiled();
    cuuint64_t dims[2] = {(cuuint64_t)H * HDIM, (cuuint64_t)B * S};
    cuuint64_t strides[1] = {(cuuint64_t)H * HDIM * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t es[2] = {1, 1};
    if (fn(&tdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq_acc, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return set_error(PD_ERR_CUDA, "attention bwd: dQ tensor map");
  }
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_attn_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdSmem::TOTAL) != cudaSuccess)
      return set_error(PD_ERR_CUDA, "attention bwd: shared memory attribute");
    attr = true;
  }
  const float scale = 1.0f / sqrtf((float)HDIM);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int items = (S / TK) * H * B;
  launch_pdl(k_attn_bwd_tc, dim3(items < sms ? items : sms), dim3(BWD_THREADS), BwdSmem::TOTAL, st,
      tq, tdo, tdq, lse, Dv, static_cast<__nv_bfloat16*>(dqkv), dq_acc, S, H, B, scale * 1.4426950408889634f, scale);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_error(PD_ERR_CUDA, "attention bwd: %s", cudaGetErrorString(e));
}

}  // namespace pd

#if PD_ATTN_TRACE
extern "C" int pd_attn_trace(unsigned long long* host, int n) {
  const size_t bytes = sizeof(unsigned long long) * (size_t)(n < pd::TR_CTAS ? n : pd::TR_CTAS) * pd::TR_EV;
  return cudaMemcpyFromSymbol(host, pd::g_attn_trace, bytes) == cudaSuccess ? 0 : 1;
}
extern "C" int pd_attn_trace_clear() {
  static unsigned long long zero[pd::TR_CTAS][pd::TR_EV];
  return cudaMemcpyToSymbol(pd::g_attn_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : 1;
}
#endif
