// Stage GEMMs for the pipeline runtime.
//
//   C[M,N] = sum_k A(m,k) * B(n,k)   followed by one fused epilogue (epilogue.cuh)
//
// A operand "K-major": A(m,k) = A[m*lda + k]; "MN-major": A(m,k) = A[k*lda + m] (same for B).
// With X=[batch,in], W=[out,in], dZ=[batch,out] (all row-major) the three passes of a
// linear layer are:
//   forward  Y  = X W^T : A=X  (K-major), B=W (K-major),  M=batch, N=out, K=in
//   dgrad    dX = dZ W  : A=dZ (K-major), B=W (MN-major), M=batch, N=in,  K=out
//   wgrad    dW = dZ^T X: A=dZ (MN-major),B=X (MN-major), M=out,   N=in,  K=batch
// so no operand is ever transposed in HBM: the tcgen05 smem descriptors take both majors.
//
// bf16 path: persistent, warp-specialised tcgen05 kernel. TMA (128B swizzle) fills a
// STAGES-deep smem ring; one elected thread issues tcgen05.mma (M=128, N=BN, K=16)
// into a double-buffered TMEM accumulator; eight epilogue warps (two per TMEM lane
// quadrant) drain TMEM with tcgen05.ld while the next tile's MMAs run, prefetching the
// next 32-column chunk's global operand (master weights / mask / targets) one chunk ahead.
// The tile width is picked per problem (256 or 224) to avoid a partial last wave.
// fp32 path (the 4-stage MLP-1024 fp32 config): SIMT FFMA GEMM with the same epilogues
// (tcgen05 has no IEEE-fp32 kind; tf32 would not meet the fp32 tolerance).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "epilogue.cuh"
#include "ptx.cuh"
#include "pd_internal.h"

namespace pd {

// ============================================================== tcgen05 bf16 GEMM
constexpr int TC_BM = 128;
constexpr int TC_BK = 64;           // 64 bf16 = 128 B = one swizzle row
constexpr int TC_EPI_WARPS = 8;     // two warps per TMEM lane quadrant, each owning half the columns
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;  // warp0 TMA, warp1 MMA (+TMEM alloc), warps 2.. epilogue
// wgrad + SGD comes in two flavours: EPI_SGD (long K: MMA-bound, one fp32 master block in flight
// per epilogue warp so the smem goes to operand stages) and EPI_SGD_STREAM (K <= 256, e.g. the
// VGG classifier at batch 32: the master read-modify-write is the whole kernel, four blocks in
// flight per warp = a whole tile's master prefetched while its MMAs run).
__host__ __device__ constexpr bool is_sgd(int kind) { return kind == EPI_SGD || kind == EPI_SGD_STREAM; }
#ifndef PD_SGD_BUFS
#define PD_SGD_BUFS 1
#endif
__host__ __device__ constexpr int sgd_bufs(int kind) { return kind == EPI_SGD_STREAM ? 4 : PD_SGD_BUFS; }
constexpr int SGD_STREAM_MAX_K = 256;
constexpr int TC_ACC_STRIDE = 256;  // TMEM columns between the two accumulator buffers

// fp32-output epilogues (SGD update of the fp32 master, raw fp32 gradient) stage each warp's
// 32x32 accumulator block through shared memory so global traffic is row-contiguous per warp.
__host__ __device__ constexpr bool transposed_epilogue(int kind) { return is_sgd(kind) || kind == EPI_GRADF32; }
constexpr int TC_STG_FLOATS = 32 * 33;  // per epilogue warp, padded against bank conflicts
// GRADF32 per-warp staging: the padded transpose block, or (plain fp32 output) a 1 KB-aligned 4 KB
// 128B-swizzled block for a TMA store
constexpr int TC_STG_WARP_BYTES = 5120;

// CG = CTA group: 1 -> one SM computes a 128 x BN tile; 2 -> a CTA pair (cluster of 2) computes
// 256 x BN with tcgen05 cta_group::2: each CTA stages its 128 rows of A and BN/2 rows of B, the
// leader issues the M=256 MMA, and each CTA's TMEM receives its own 128 accumulator rows.  The
// pair halves the per-SM operand traffic from L2 and lets each CTA keep more pipeline stages.
template <int CG, int BN, bool B_MN, int KIND = EPI_STORE>
struct TcCfg {
  static constexpr int B_ROWS = BN / CG;  // B rows (N extent) staged by each CTA
  // MN-major B tiles are loaded as whole 64-wide swizzle atoms
  static constexpr int BNL = B_MN ? ((B_ROWS + 63) / 64) * 64 : B_ROWS;
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BNL * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // SGD: per epilogue warp sgd_bufs(KIND) TMA-fed 32x32 fp32 master blocks (4 KB each, 128B-
  // swizzled).  Long K wants one (2048x8192x8192 wgrad+SGD 246 / 252 / 271 / 294 us with 1 / 2 / 3
  // / 4: the smem is worth more as operand stages, 6 / 5 / 4 / 3); short K wants four (see is_sgd);
  // GRADF32: per warp a padded 32x33 transpose block.
  static constexpr int STG_BYTES = is_sgd(KIND) ? TC_EPI_WARPS * sgd_bufs(KIND) * 4096
                                 : (KIND == EPI_GRADF32 ? TC_EPI_WARPS * TC_STG_WARP_BYTES : 0);
  static constexpr int PIPE_BUDGET = 227 * 1024 - 2048 - STG_BYTES;  // all of the 227 KB opt-in smem
  static constexpr int STAGES = PIPE_BUDGET / STAGE_BYTES > 8 ? 8 : PIPE_BUDGET / STAGE_BYTES;
  static constexpr int TMEM_COLS = 512;
  static constexpr int BAR_BYTES = 1024;  // mbarriers + TMEM slot, keeps the epilogue region 1 KB aligned
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + BAR_BYTES + STG_BYTES;
  static_assert(BN % 32 == 0 && BN % (16 * CG) == 0 && BN <= 256, "BN");
  // MN-major B is staged as whole 64-wide swizzle atoms; a partial last atom (BN=224: 112 rows per
  // CTA = 64 + 48) is loaded in full and the MMA reads only its first B_ROWS % 64 columns
  static_assert(!B_MN || B_ROWS % 16 == 0, "MN-major B rows per CTA");
};

template <int CG, int BN, bool A_MN, bool B_MN, int KIND, int SRC = SRC_2D, bool SIG = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmW, int M, int N, int K, EpiArgs ep, ConvArgs cv) {
  using C = TcCfg<CG, BN, B_MN, KIND>;
  constexpr int UM = TC_BM * CG;  // tile rows per unit (CTA or CTA pair)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align_1k(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tmem_full = empty + C::STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  uint64_t* epi_bar = tmem_empty + 4;  // SGD: two per epilogue warp (master block loaded)
  uint8_t* epi_smem = smem + C::STAGES * C::STAGE_BYTES + C::BAR_BYTES;

  const int warp = warp_id();
  const uint32_t cta = CG == 2 ? cluster_ctarank() : 0;  // rank inside the pair
  const bool leader = cta == 0;
  const int unit = blockIdx.x / CG, units = gridDim.x / CG;
  const int num_m = (M + UM - 1) / UM;
  const int num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int num_kb = (K + TC_BK - 1) / TC_BK;
  // split-K: work unit u covers tile u % tiles over k-blocks [kb_lo(u), kb_hi(u))
  const int work = tiles * cv.splits;
  auto kb_lo = [&](int u) { return (u / tiles) * cv.kb_per; };
  auto kb_hi = [&](int u) { const int e = (u / tiles + 1) * cv.kb_per; return e < num_kb ? e : num_kb; };
  const int HW = cv.H * cv.W;
  // bounding-box coordinate of output pixel `pix` for the im2col loads (lower corner -1, -1)
  auto pix_coord = [&](int pix, int& w, int& h, int& n) {
    n = pix / HW;
    const int rem = pix - n * HW;
    h = rem / cv.W;
    w = rem - h * cv.W - 1;
    h -= 1;
  };
  // Rasterisation.  Forward/dgrad stream a large B (the weights) through L2, so co-resident
  // tiles share B (m fastest).  The wgrad+SGD operands (dZ, X) are L2-resident and its cost is
  // the fp32 master read-modify-write, so co-resident tiles walk along the rows (n fastest) and
  // HBM sees long contiguous row runs instead of 1 KB pieces 32 KB apart.
  constexpr bool kNFast = transposed_epilogue(KIND);
  // SGD: grouped rasterisation - bands of kGroup tile rows walked column by column, so the
  // co-resident tiles touch ~kGroup A blocks and ~units/kGroup B blocks (a compact operand
  // working set that survives the streamed master traffic in L2)
  constexpr bool kGrouped = is_sgd(KIND);
  const int kGroup = kGrouped ? (ep.group > 0 ? ep.group : 16) : 0;
  constexpr int NBUF = sgd_bufs(KIND);  // SGD: fp32 master blocks in flight per epilogue warp
  auto tile_m = [&](int t) {
    if constexpr (kGrouped) {
      const int band = t / (kGroup * num_n), in = t - band * kGroup * num_n;
      const int rows = num_m - band * kGroup < kGroup ? num_m - band * kGroup : kGroup;
      return band * kGroup + in % rows;
    }
    return kNFast ? t / num_n : t % num_m;
  };
  auto tile_n = [&](int t) {
    if constexpr (kGrouped) {
      const int band = t / (kGroup * num_n), in = t - band * kGroup * num_n;
      const int rows = num_m - band * kGroup < kGroup ? num_m - band * kGroup : kGroup;
      return in / rows;
    }
    return kNFast ? t % num_n : t / num_m;
  };

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if constexpr (is_sgd(KIND)) tma_prefetch_desc(&tmW);
    // full: leader's arrive.expect_tx (+ the peer's remote arrive for a pair); empty: one MMA commit;
    // tmem_empty: one arrival per epilogue warp of every CTA of the unit
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], CG); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tmem_full[a], 1); mbar_init(&tmem_empty[a], CG * TC_EPI_WARPS); }
    if constexpr (is_sgd(KIND))
      for (int i = 0; i < NBUF * TC_EPI_WARPS; ++i) mbar_init(&epi_bar[i], 1);
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS, CG>(tmem_slot);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();    // operands / epilogue inputs may come from the previous kernel on the stream
  griddep_launch();  // the next kernel may start its prologue as our CTAs retire

  if (warp == 0) {
    // ---------------- TMA producer (every CTA loads its own halves)
    if (elect_one()) {
      const uint64_t keep = l2_policy_evict_last();
      // a B operand far larger than L2's share (the MLP-8192 weights: 128 MB, read by the few
      // co-resident M tiles of its column and never again) streams with evict-first, so it does not
      // push the re-read A operand (dZ / X: every column tile reads it) out between waves
      const uint64_t b_pol = ep.b_stream ? l2_policy_evict_first() : keep;
      int stage = 0;
      uint32_t phase = 0;
      for (int u = unit; u < work; u += units) {
        const int t = u % tiles;
        const int m0 = tile_m(t) * UM + TC_BM * cta;
        const int n0 = tile_n(t) * BN + C::B_ROWS * cta;
        int aw = 0, ah = 0, an = 0;
        if constexpr (SRC == SRC_CONV_FWD || SRC == SRC_CONV_DGRAD) pix_coord(m0, aw, ah, an);
        const int kb_end = kb_hi(u);
        for (int kb = kb_lo(u); kb < kb_end; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], CG * C::STAGE_BYTES);
          else mbar_arrive_cluster_relaxed(&full[stage], 0);
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          const int k0 = kb * TC_BK;
          auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1, uint64_t pol) {
            // operands are re-read by many tiles: keep them in L2 ahead of streamed epilogue data
            if constexpr (CG == 2) tma_load_2d_2sm(dst, map, &full[stage], c0, c1, pol);
            else tma_load_2d_hint(dst, map, &full[stage], c0, c1, pol);
          };
          if constexpr (SRC == SRC_CONV_FWD || SRC == SRC_CONV_DGRAD) {
            // 128 output pixels x 64 channels of tap `tap` (dgrad reads dY at the flipped offset)
            const int tap = k0 / cv.C, c0 = k0 - tap * cv.C;
            if constexpr (CG == 2)
              tma_load_im2col_4d_2sm(a_dst, &tmA, &full[stage], c0, aw, ah, an, (uint16_t)(tap % 3), (uint16_t)(tap / 3));
            else
              tma_load_im2col_4d(a_dst, &tmA, &full[stage], c0, aw, ah, an, (uint16_t)(tap % 3), (uint16_t)(tap / 3));
            if constexpr (SRC == SRC_CONV_DGRAD) {
              load(b_dst, &tmB, c0, (8 - tap) * cv.brows + n0, keep);  // Wt rows of the mirrored tap
            } else {
#pragma unroll
              for (int i = 0; i < C::BNL / 64; ++i) load(b_dst + i * 8192, &tmB, n0 + 64 * i, k0, keep);
            }
          } else if constexpr (SRC == SRC_CONV_WGRAD) {
            // A(m = tap*C + c, k = pixel): two 64-channel x 64-pixel im2col atoms (MN-major)
            int pw, ph, pn;
            pix_coord(k0, pw, ph, pn);
#pragma unroll
            for (int i = 0; i < TC_BM / 64; ++i) {
              const int mm = m0 + 64 * i;
              int tap = mm / cv.C;
              tap = tap < 8 ? tap : 8;  // rows past 9*C are clipped by the epilogue
              const int c0 = mm - tap * cv.C < cv.C ? mm - tap * cv.C : 0;
              if constexpr (CG == 2)
                tma_load_im2col_4d_2sm(a_dst + i * 8192, &tmA, &full[stage], c0, pw, ph, pn, (uint16_t)(tap % 3),
                                       (uint16_t)(tap / 3));
              else
                tma_load_im2col_4d(a_dst + i * 8192, &tmA, &full[stage], c0, pw, ph, pn, (uint16_t)(tap % 3),
                                   (uint16_t)(tap / 3));
            }
#pragma unroll
            for (int i = 0; i < C::BNL / 64; ++i) load(b_dst + i * 8192, &tmB, n0 + 64 * i, k0, keep);
          } else {
            if constexpr (A_MN) {
#pragma unroll
              for (int i = 0; i < TC_BM / 64; ++i) load(a_dst + i * 8192, &tmA, m0 + 64 * i, k0, keep);
            } else {
              load(a_dst, &tmA, k0, m0, keep);
            }
            if constexpr (B_MN) {
#pragma unroll
              for (int i = 0; i < C::BNL / 64; ++i) load(b_dst + i * 8192, &tmB, n0 + 64 * i, k0, b_pol);
            } else {
              load(b_dst, &tmB, k0, n0, b_pol);
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (single thread of the leader CTA)
    if (leader && elect_one()) {
      constexpr uint32_t idesc = make_idesc_bf16(UM, BN, A_MN, B_MN);
      // K-major SW128: 8-row core groups 1024 B apart (SBO); +32 B per K=16 step.
      // MN-major SW128: 64-element MN atoms of 64 K-rows are 8 KB apart (LBO), 8-K-row
      // groups 1024 B apart (SBO); +2048 B per K=16 step.
      constexpr uint32_t A_LBO = A_MN ? 8192 : 16, A_SBO = 1024, A_KSTEP = A_MN ? 2048 : 32;
      constexpr uint32_t B_LBO = B_MN ? 8192 : 16, B_SBO = 1024, B_KSTEP = B_MN ? 2048 : 32;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = unit; u < work; u += units) {
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * TC_ACC_STRIDE;
        const int kb_begin = kb_lo(u), kb_end = kb_hi(u);
        for (int kb = kb_begin; kb < kb_end; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            uint64_t ad = make_sw128_desc(a_addr + k * A_KSTEP, A_LBO, A_SBO);
            uint64_t bd = make_sw128_desc(b_addr + k * B_KSTEP, B_LBO, B_SBO);
            if constexpr (CG == 2) umma_bf16_2sm(d, ad, bd, idesc, (kb != kb_begin) | (k != 0));
            else umma_bf16(d, ad, bd, idesc, (kb != kb_begin) | (k != 0));
          }
          if constexpr (CG == 2) umma_commit_2sm_mc(&empty[stage]); else umma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (CG == 2) umma_commit_2sm_mc(&tmem_full[acc]); else umma_commit(&tmem_full[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if constexpr (is_sgd(KIND)) {
    // ---------------- wgrad + SGD epilogue.  Each warp owns 32 accumulator rows (its TMEM lane
    // quadrant) and half of the tile's 32-column chunks.  The fp32 master block of a chunk
    // (32x32, 4 KB) is TMA-loaded into a 128B-swizzled smem buffer ahead of use (NBUF
    // deep, the first issued before the tile's accumulator is ready), updated in place
    // (w = m - lr*acc), TMA-stored back, and the bf16 version copy is written from registers.
    // HBM sees only bulk, fully coalesced master traffic.
    const int q = warp & 3;
    const int half = (warp - 2) / 4;
    constexpr int NC = BN / 32;
    const int c_begin = half ? (NC + 1) / 2 : 0;
    const int c_end = half ? NC : (NC + 1) / 2;
    const int e = warp - 2;
    uint8_t* buf0 = epi_smem + e * NBUF * 4096;
    uint64_t* bars = epi_bar + NBUF * e;
    const int lane = lane_id();
    uint32_t bar_phase = 0;  // bit b: parity of buffer b's next load
    // the master stream (read once, written once) must not evict the L2-resident operands
    const uint64_t stream_pol = l2_policy_evict_first();
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = unit; u < work; u += units) {
      const int t = u % tiles;
      const int m0 = tile_m(t) * UM + TC_BM * cta;
      const int n0 = tile_n(t) * BN;
      const int row0 = m0 + 32 * q;
      const int nck = c_end - c_begin;
      // fused bias SGD (rows of this warp, once per row: the tile of column 0, first half):
      // b -= lr * sum of the producer's per-row-block column sums, written as the new version
      if (ep.bpart && tile_n(t) == 0 && half == 0 && row0 + lane < M) {
        const int64_t rr = row0 + lane;
        float g = 0.f;
#pragma unroll 8
        for (int rb = 0; rb < ep.nrb; ++rb) g += ep.bpart[(int64_t)rb * ep.ldc + rr];
        const float b = ep.bmaster[rr] - ep.lr * g;
        ep.bmaster[rr] = b;
        ep.bring[rr] = b;
      }
      // prefetch the first two master blocks of this tile while its MMAs are still running
      if (lane == 0) {
        bulk_wait_read0();  // previous tile's stores have finished reading both buffers
        for (int i = 0; i < NBUF && i < nck; ++i) {
          mbar_arrive_expect_tx(&bars[i], 4096);
          tma_load_2d_hint(buf0 + i * 4096, &tmW, &bars[i], n0 + (c_begin + i) * 32, row0, stream_pol);
        }
      }
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int i = 0; i < nck; ++i) {
        const int c = c_begin + i, b = i % NBUF;
        float v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * TC_ACC_STRIDE + c * 32, v);
        mbar_wait(&bars[b], (bar_phase >> b) & 1);
        bar_phase ^= 1u << b;
        // row `lane` of the block: 16-byte chunk j sits at position j ^ (lane & 7) (SWIZZLE_128B)
        float4* row = reinterpret_cast<float4*>(buf0 + b * 4096 + lane * 128);
        uint32_t packed[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 m = row[j ^ (lane & 7)];
          m.x -= ep.lr * v[4 * j];
          m.y -= ep.lr * v[4 * j + 1];
          m.z -= ep.lr * v[4 * j + 2];
          m.w -= ep.lr * v[4 * j + 3];
          row[j ^ (lane & 7)] = m;
          packed[2 * j] = pack_bf16x2(m.x, m.y);
          packed[2 * j + 1] = pack_bf16x2(m.z, m.w);
        }
        const int64_t r = row0 + lane, col0 = n0 + c * 32;
        if (r < M) {
          if (col0 + 32 <= N) {
            uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + r * ep.ldo + col0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              st_stream_v4(o + j, make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]),
                           stream_pol);  // the version copy is next read many kernels later
          } else {
            for (int j = 0; j < 32 && col0 + j < N; ++j) {
              float a, bb;
              unpack_bf16x2(packed[j / 2], a, bb);
              static_cast<__nv_bfloat16*>(ep.out)[r * ep.ldo + col0 + j] = __float2bfloat16_rn(j & 1 ? bb : a);
            }
          }
        }
        fence_proxy_async_shared();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d_hint(&tmW, buf0 + b * 4096, col0, row0, stream_pol);  // TMA clips rows/cols outside [M, N)
          bulk_commit();
          if (i + NBUF < nck) {
            bulk_wait_read0();  // this buffer's store has read the smem block
            mbar_arrive_expect_tx(&bars[b], 4096);
            tma_load_2d_hint(buf0 + b * 4096, &tmW, &bars[b], n0 + (c + NBUF) * 32, row0, stream_pol);
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster_relaxed(&tmem_empty[acc], 0); else mbar_arrive(&tmem_empty[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait_all0();
  } else if constexpr (transposed_epilogue(KIND)) {
    // ---------------- fp32 epilogue: TMEM -> regs -> smem (transpose within the warp) -> lanes
    // along columns, so each warp reads/writes whole 128-byte rows of the fp32 master.
    const int q = warp & 3;
    const int half = (warp - 2) / 4;
    constexpr int NC = BN / 32;
    const int c_begin = half ? (NC + 1) / 2 : 0;
    const int c_end = half ? NC : (NC + 1) / 2;
    float* stg = reinterpret_cast<float*>(epi_smem + (warp - 2) * (is_sgd(KIND) ? TC_STG_FLOATS * 4 : TC_STG_WARP_BYTES));
    const int lane = lane_id();
    const uint64_t stream = l2_policy_evict_first();  // master / ring are touched once per GEMM
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = unit; u < work; u += units) {
      const int t = u % tiles;
      const int m0 = tile_m(t) * UM + TC_BM * cta;
      const int n0 = tile_n(t) * BN;
      const int64_t row0 = m0 + 32 * q;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      if constexpr (KIND == EPI_GRADF32) {
        if (ep.tma_out) {
          // plain fp32 output (the GPT-2 head's logits, replicated-stage gradients): each lane's row
          // of a 32x32 block -> swizzled smem -> one asynchronous TMA store per block (the output map
          // clips rows / columns past M / N), instead of 32 row stores per block from the transpose
          uint8_t* blk = reinterpret_cast<uint8_t*>(stg);
#pragma unroll 1
          for (int c = c_begin; c < c_end; ++c) {
            float v[32];
            tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * TC_ACC_STRIDE + c * 32, v);
            const int64_t col0 = n0 + c * 32;
            if (ep.bias && col0 < N) {
              const float* bp = ep.bias + col0;
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += col0 + j < N ? __ldg(bp + j) : 0.f;
            }
            if (lane == 0) bulk_wait_read0();  // the previous block's store has read the buffer
            __syncwarp();
            float4* row = reinterpret_cast<float4*>(blk + lane * 128);
#pragma unroll
            for (int j = 0; j < 8; ++j) row[j ^ (lane & 7)] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0 && col0 < N && row0 < M) {
              tma_store_2d_hint(&tmW, blk, (int)col0, (int)row0, stream);
              bulk_commit();
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster_relaxed(&tmem_empty[acc], 0); else mbar_arrive(&tmem_empty[acc]);
          }
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
          continue;
        }
      }
      // Two 32-column chunks per step: 64 independent 128-byte master loads in flight per warp
      // (the epilogue is HBM-latency bound, it has to keep up with the next tile's MMAs).
#pragma unroll 1
      for (int c = c_begin; c < c_end; c += 2) {
        const bool two = c + 1 < c_end;
        const int64_t colA = n0 + c * 32 + lane, colB = colA + 32;
        const bool okA = colA < N, okB = two && colB < N;
        const int rows = M - row0 < 32 ? (int)(M - row0) : 32;
        float mA[32], mB[32];
        if constexpr (is_sgd(KIND)) {
          const float* pa = ep.master + row0 * ep.ldw + colA;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            mA[i] = (okA && i < rows) ? ld_stream_f32(pa, stream) : 0.f;
            mB[i] = (okB && i < rows) ? ld_stream_f32(pa + 32, stream) : 0.f;
            pa += ep.ldw;
          }
        }
        auto process = [&](int cc, int64_t col, bool col_ok, const float (&m)[32]) {
          float v[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * TC_ACC_STRIDE + cc * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = v[j];
          __syncwarp();
          if (col_ok) {
            if constexpr (is_sgd(KIND)) {
              float* pm = ep.master + row0 * ep.ldw + col;
              __nv_bfloat16* po = static_cast<__nv_bfloat16*>(ep.out) + row0 * ep.ldo + col;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                if (i < rows) {
                  const float w = m[i] - ep.lr * stg[i * 33 + lane];
                  st_stream_f32(pm, w, stream);
                  st_stream_b16(po, __bfloat16_as_ushort(__float2bfloat16_rn(w)), stream);
                }
                pm += ep.ldw;
                po += ep.ldo;
              }
            } else {
              // fp32 result (+ per-column bias: logits); split-K partial s goes to out + s*split_stride
              float* po = static_cast<float*>(ep.out) + (u / tiles) * cv.split_stride + row0 * ep.ldo + col;
              const float bcol = ep.bias ? ep.bias[col] : 0.f;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                if (i < rows) {
                  if (ep.accumulate) atomicAdd(po, stg[i * 33 + lane] + bcol);
                  else *po = stg[i * 33 + lane] + bcol;
                }
                po += ep.ldo;
              }
            }
          }
          __syncwarp();
        };
        process(c, colA, okA, mA);
        if (two) process(c + 1, colB, okB, mB);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster_relaxed(&tmem_empty[acc], 0); else mbar_arrive(&tmem_empty[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if constexpr (KIND == EPI_GRADF32)
      if (lane == 0) bulk_wait_all0();  // TMA-store path: the last blocks' stores completed
  } else {
    // ---------------- epilogue warps: TMEM -> registers -> fused epilogue -> HBM
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int half = (warp - 2) / 4;        // which half of the tile's 32-column chunks
    constexpr int NC = BN / 32;
    const int c_begin = half ? (NC + 1) / 2 : 0;
    const int c_end = half ? NC : (NC + 1) / 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    float lsum = 0.f;
    uint32_t stored = 0;  // SIG: payload bytes this lane stored into the peer inbox
    for (int u = unit; u < work; u += units) {
      const int t = u % tiles;
      const int m0 = tile_m(t) * UM + TC_BM * cta;
      const int n0 = tile_n(t) * BN;
      const int64_t r = m0 + 32 * q + lane_id();
      const bool row_ok = r < M;
      Aux<KIND> cur, nxt;
      if (row_ok && c_begin < c_end && n0 + c_begin * 32 + 32 <= N) aux_load<KIND>(ep, r, n0 + c_begin * 32, cur);
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = c_begin; c < c_end; ++c) {
        const int64_t c0 = n0 + c * 32;
        if (row_ok && c + 1 < c_end && c0 + 64 <= N) aux_load<KIND>(ep, r, c0 + 32, nxt);
        float v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * TC_ACC_STRIDE + c * 32, v);
        if (row_ok) {
          if (c0 + 32 <= N) {
            lsum += apply_chunk<KIND>(ep, r, c0, v, cur);
            if constexpr (SIG) stored += 32 * sizeof(__nv_bfloat16);
          } else {
            for (int j = 0; j < 32; ++j)
              if (c0 + j < N) {
                lsum += epi_elem<KIND, __nv_bfloat16>(ep, r, c0 + j, v[j]);
                if constexpr (SIG) stored += sizeof(__nv_bfloat16);
              }
          }
        }
        if constexpr (KIND == EPI_MASK || KIND == EPI_LOSS) {
          // fused bias gradient: column sums of the 32 stored rows (bf16-rounded, as the
          // consumer's stand-alone column sum would read them); the host enables it only for
          // N % 32 == 0, so a chunk is either full or (the tail of a last, partial tile) wholly
          // past N, where it must not write: c0 + lane would land in the next row block's columns
          if (ep.colsum && c0 < N) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = row_ok ? __bfloat162float(__float2bfloat16_rn(v[j])) : 0.f;
            const float cs = warp_colsum32(v);
            const int64_t rb = (m0 + 32 * q) / 32;
            if (m0 + 32 * q < M) {
              ep.colsum[rb * ep.ldc + c0 + lane_id()] = cs;
              if constexpr (SIG) stored += sizeof(float);
            }
          }
        }
        cur = nxt;
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster_relaxed(&tmem_empty[acc], 0); else mbar_arrive(&tmem_empty[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if constexpr (KIND == EPI_LOSS) {
      lsum = warp_sum(lsum);
      if (lane_id() == 0 && lsum != 0.f) atomicAdd(ep.loss, 0.5f * ep.scale * lsum);
    }
    if constexpr (SIG) {
      stored = __reduce_add_sync(0xffffffffu, stored);
      if (lane_id() == 0 && ep.sig_bytes && stored) atomicAdd(ep.sig_bytes, (unsigned long long)stored);
    }
  }
  // SIG (a compile-time variant, so kernels without a hand-off carry none of this code: a runtime
  // branch here measurably slowed the red.add-heavy split-K wgrad epilogues)
  if constexpr (SIG) __threadfence_system();  // this thread's payload stores, before the CTA's arrival
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS, CG>(tmem_base);
  }
  if (SIG && threadIdx.x == 0) {
    // fused hand-off: the last CTA to finish publishes the payload to the peer's inbox flag
    __threadfence_system();
    if (atomicAdd(ep.sig_counter, 1) == (int)gridDim.x - 1) {
      *ep.sig_counter = 0;
      __threadfence();
      st_release_sys(ep.sig_flag, ep.sig_value);
    }
  }
}

// ============================================================== SIMT GEMM (fp32 / bf16)
constexpr int SM_BM = 32, SM_BN = 32, SM_BK = 32;

template <typename T, int KIND>
__global__ void __launch_bounds__(256)
    k_gemm_simt(const T* __restrict__ A, int a_mn, int64_t lda, const T* __restrict__ B, int b_mn,
                int64_t ldb, int M, int N, int K, EpiArgs ep) {
  __shared__ float sA[SM_BK][SM_BM + 1];
  __shared__ float sB[SM_BK][SM_BN + 1];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * SM_BM, n0 = blockIdx.x * SM_BN;
  const int tr = tid / 16, tc = tid % 16;  // 16x16 threads, 2x2 outputs each
  float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  for (int k0 = 0; k0 < K; k0 += SM_BK) {
    for (int i = tid; i < SM_BM * SM_BK; i += 256) {
      int mm, kk;
      if (a_mn) { kk = i / SM_BM; mm = i % SM_BM; } else { mm = i / SM_BK; kk = i % SM_BK; }
      const int m = m0 + mm, k = k0 + kk;
      float x = 0.f;
      if (m < M && k < K) x = to_f<T>(a_mn ? A[(int64_t)k * lda + m] : A[(int64_t)m * lda + k]);
      sA[kk][mm] = x;
    }
    for (int i = tid; i < SM_BN * SM_BK; i += 256) {
      int nn, kk;
      if (b_mn) { kk = i / SM_BN; nn = i % SM_BN; } else { nn = i / SM_BK; kk = i % SM_BK; }
      const int n = n0 + nn, k = k0 + kk;
      float x = 0.f;
      if (n < N && k < K) x = to_f<T>(b_mn ? B[(int64_t)k * ldb + n] : B[(int64_t)n * ldb + k]);
      sB[kk][nn] = x;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < SM_BK; ++kk) {
      const float a0 = sA[kk][tr], a1 = sA[kk][tr + 16];
      const float b0 = sB[kk][tc], b1 = sB[kk][tc + 16];
      acc[0][0] = fmaf(a0, b0, acc[0][0]);
      acc[0][1] = fmaf(a0, b1, acc[0][1]);
      acc[1][0] = fmaf(a1, b0, acc[1][0]);
      acc[1][1] = fmaf(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
  float lsum = 0.f;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = m0 + tr + 16 * i, n = n0 + tc + 16 * j;
      if (m < M && n < N) lsum += epi_elem<KIND, T>(ep, m, n, acc[i][j]);
    }
  if constexpr (KIND == EPI_LOSS) {
    lsum = warp_sum(lsum);
    if ((tid & 31) == 0 && lsum != 0.f) atomicAdd(ep.loss, 0.5f * ep.scale * lsum);
  }
}

// ============================================================== host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows, row pitch ld elements.
static int make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer, bool fp32 = false) {
  auto fn = encode_fn();
  if (!fn) return set_error(PD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * (fp32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// 4-D im2col map over an NHWC bf16 activation [n, H, W, C] for 3x3 / stride 1 / pad 1: bounding
// box corners (-1, -1) .. (-1, -1) relative to the extent, 64 channels (128 B, swizzled) per pixel,
// `pixels` pixels per load.
static PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col_fn() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  });
  return fn;
}

static int make_im2col_map(CUtensorMap* map, const void* ptr, int n, int H, int W, int C, int pixels) {
  auto fn = encode_im2col_fn();
  if (!fn) return set_error(PD_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  int lower[2] = {-1, -1}, upper[2] = {-1, -1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, lower, upper, 64,
                  (cuuint32_t)pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PD_ERR_CUDA, "cuTensorMapEncodeIm2col failed (%d)", (int)r);
  // Drivers up to 13.1 mis-handle im2col maps over tensors smaller than 128 KiB unless this
  // descriptor bit is cleared (the same workaround CUTLASS applies).
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && (int64_t)n * H * W * C * 2 < 131072) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return 0;
}

template <int CG, int BN, bool A_MN, bool B_MN, int KIND, int SRC = SRC_2D>
static int launch_tc(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K, const EpiArgs& ep,
                     cudaStream_t st, ConvArgs cv = ConvArgs{}) {
  using C = TcCfg<CG, BN, B_MN, KIND>;
  CUtensorMap ta, tb;
  int rc;
  if (cv.splits < 1) {  // no split-K
    cv.splits = 1;
    cv.kb_per = (K + TC_BK - 1) / TC_BK;
  }
  if (SRC == SRC_CONV_FWD || SRC == SRC_CONV_DGRAD) rc = make_im2col_map(&ta, A, M / (cv.H * cv.W), cv.H, cv.W, cv.C, TC_BM);
  else if (SRC == SRC_CONV_WGRAD) rc = make_im2col_map(&ta, A, K / (cv.H * cv.W), cv.H, cv.W, cv.C, 64);
  else if (A_MN) rc = make_map(&ta, A, (uint64_t)M, (uint64_t)K, lda, 64, 64);
  else rc = make_map(&ta, A, (uint64_t)K, (uint64_t)M, lda, 64, TC_BM);
  if (rc) return rc;
  if (SRC == SRC_CONV_DGRAD) rc = make_map(&tb, B, (uint64_t)cv.C, 9ull * cv.brows, ldb, 64, C::B_ROWS);
  else if (B_MN) rc = make_map(&tb, B, (uint64_t)N, (uint64_t)K, ldb, 64, 64);
  else rc = make_map(&tb, B, (uint64_t)K, (uint64_t)N, ldb, 64, C::B_ROWS);
  if (rc) return rc;
  CUtensorMap tw;
  memset(&tw, 0, sizeof(tw));
  if (is_sgd(KIND)) {
    if ((ep.ldw % 4) || (reinterpret_cast<uintptr_t>(ep.master) % 16))
      return set_error(PD_ERR_INVALID, "gemm: SGD master must be 16-byte aligned with ld %% 4 == 0");
    rc = make_map(&tw, ep.master, (uint64_t)N, (uint64_t)M, ep.ldw, 32, 32, true);
    if (rc) return rc;
  }
  // plain fp32 output (no split-K, no red.add): asynchronous TMA stores of 32 x 32 blocks
  bool tma_out = false;
  if (KIND == EPI_GRADF32 && !ep.accumulate && cv.splits == 1 && !(ep.ldo % 4) &&
      !(reinterpret_cast<uintptr_t>(ep.out) % 16)) {
    static int off = -1;  // PD_F32_TMA_STORE=0: the row-store path (A/B runs)
    if (off < 0) {
      const char* e = getenv("PD_F32_TMA_STORE");
      off = e && atoi(e) == 0 ? 1 : 0;
    }
    if (!off) {
      rc = make_map(&tw, ep.out, (uint64_t)N, (uint64_t)M, ep.ldo, 32, 32, true);
      if (rc) return rc;
      tma_out = true;
    }
  }
  EpiArgs epl = ep;
  epl.tma_out = tma_out ? 1 : 0;
  {
    // B operand streamed with evict-first when it is far larger than its reuse window in L2
    // (PD_B_STREAM=0/1 forces it off/on for A/B runs)
    static int force = -2;
    if (force == -2) {
      const char* e = getenv("PD_B_STREAM");
      force = e ? atoi(e) : -1;
    }
    // measured on the MLP-8192 layer (tools/gpu_dram_ab.sh): forward (K-major W) DRAM reads 243 -> 194 MB
    // and 180 -> 175 us; the dgrad (MN-major W) reads grew (310 -> 330 MB), so it keeps evict-last
    const bool big = SRC == SRC_2D && !is_sgd(KIND) && !B_MN && (int64_t)N * K * 2 >= (64ll << 20);
    epl.b_stream = force >= 0 ? force : (big ? 1 : 0);
  }
  if constexpr (is_sgd(KIND)) {
    static int group = -1;  // PD_SGD_GROUP: tile rows per rasterisation band (A/B experiments)
    if (group < 0) {
      const char* e = getenv("PD_SGD_GROUP");
      group = e ? atoi(e) : 16;  // measured: 8 / 12 / 16 / 24 / 32 -> 241 / 240 / 237 / 238 / 238 us (8192^2 x 2048)
    }
    epl.group = group;
  }
  auto kern = k_gemm_tc<CG, BN, A_MN, B_MN, KIND, SRC, false>;
  static bool attr_set[2] = {false, false};  // per instantiation (plain / hand-off variant)
  int var = 0;
  if (ep.sig_flag) {
    // the fused hand-off exists for the payload-producing epilogues only (MLP forward / dgrad)
    if constexpr ((KIND == EPI_STORE || KIND == EPI_MASK) && SRC == SRC_2D) {
      kern = k_gemm_tc<CG, BN, A_MN, B_MN, KIND, SRC, true>;
      var = 1;
    } else {
      return set_error(PD_ERR_INVALID, "gemm: fused hand-off is not available for epilogue kind %d", KIND);
    }
  }
  if (!attr_set[var]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) != cudaSuccess)
      return set_error(PD_ERR_CUDA, "cudaFuncSetAttribute(smem=%d) failed", C::SMEM_BYTES);
    attr_set[var] = true;
  }
  const int units = ((M + TC_BM * CG - 1) / (TC_BM * CG)) * ((N + BN - 1) / BN) * cv.splits;
  const int max_units = num_sms() / CG;
  const int grid = CG * (units < max_units ? units : max_units);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  mark_pre_launch(st);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tw, M, N, K, epl, cv);
  if (e != cudaSuccess) return set_error(PD_ERR_CUDA, "tcgen05 gemm launch: %s", cudaGetErrorString(e));
  return 0;
}

// CTA group and tile width: minimise (waves x tile time).  E.g. 2048x8192 with a K-major B:
// CTA pairs with BN=224 give 296 pair-tiles = 4.00 waves over 74 pairs, where BN=256 leaves a
// 46 %-full last wave.  PD_GEMM_CG=1|2 forces the CTA group (benchmarks / A-B tests).
static int g_force_cg = -1;
static void pick_cfg(int M, int N, bool b_mn, int* cg, int* bn) {
  if (g_force_cg < 0) {
    const char* e = getenv("PD_GEMM_CG");
    g_force_cg = e ? atoi(e) : 0;
  }
  const int sms = num_sms();
  long best = -1;
  *cg = 1;
  *bn = 256;
  for (int c = 1; c <= 2; ++c) {
    if (g_force_cg && c != g_force_cg) continue;
    if (c == 2 && M <= TC_BM) continue;  // a single 128-row tile gains nothing from a pair
    for (int b : {256, 224, 192, 128}) {
      // waves x (tile width + ~24 columns of fixed per-tile cost: prologue, operand re-reads);
      // a pair is ~2.5 % faster per tile than two single CTAs (halved B traffic per SM).  An MN-major
      // B is staged in whole 64-column swizzle atoms, so 224 / 192-wide pair tiles load as much as a
      // 256-wide one, and narrow tiles re-read the A operand once per extra column tile: measured on
      // the MLP-8192 dgrad (2048 x 8192, whole bench step on one box) 256 / 224 / 128-wide tiles gave
      // 193.5k / 190.9k / 188.7k samples/s.  So MN-major B tiles are 256 or 128 wide, with a larger
      // fixed cost.
      if (b_mn && (b == 224 || b == 192)) continue;
      const int fixed = b_mn ? 64 : 24;
      const long units = (long)((M + TC_BM * c - 1) / (TC_BM * c)) * ((N + b - 1) / b);
      const long slots = sms / c;
      const long cost = ((units + slots - 1) / slots) * (b + fixed) * (c == 2 ? 2 : 1) * 1000 / (c == 2 ? 2050 : 1000);
      if (best < 0 || cost < best) { best = cost; *cg = c; *bn = b; }
    }
  }
}

// The tile configuration of one problem (also reported by pd_gemm_pick for the tests).
static void choose_cfg(int M, int N, bool a_mn, bool b_mn, int kind, int* cg, int* bn) {
  if (!a_mn && !b_mn && (kind == EPI_STORE || kind == EPI_LOSS)) {
    static int force = -1;  // PD_FWD_BN=256|224|192|128: tile width of the K-major forward (A/B runs)
    if (force < 0) {
      const char* e = getenv("PD_FWD_BN");
      force = e ? atoi(e) : 0;
    }
    if (force == 256 || force == 224 || force == 192 || force == 128) {
      *cg = M > TC_BM ? 2 : 1;
      *bn = force;
      return;
    }
  }
  if (!a_mn && b_mn && kind == EPI_MASK) {
    static int force = -1;  // PD_DGRAD_BN=256|224|192|128: tile width of the MN-major-B dgrad (A/B runs)
    if (force < 0) {
      const char* e = getenv("PD_DGRAD_BN");
      force = e ? atoi(e) : 0;
    }
    if (force == 256 || force == 224 || force == 192 || force == 128) {
      *cg = M > TC_BM ? 2 : 1;
      *bn = force;
      return;
    }
  }
  if (!a_mn && b_mn && kind == EPI_STORE && N <= 128) {
    // narrow outputs (the im2col'ed first convolution, c_out = 64): a 256-wide tile would be 3/4 padding
    *cg = 1;
    *bn = N <= 64 ? 64 : 128;
    return;
  }
  if (is_sgd(kind) && b_mn) {
    // wgrad + SGD on small weight matrices: 256 x 128 pair tiles double the tile count (e.g. a
    // 1024 x 1024 weight: 32 instead of 16 pair tiles); large ones keep 256-wide tiles, whose
    // operand traffic per flop is lower (measured: 8192^2 0.27 ms vs 0.31 ms with 128-wide tiles)
    const long units256 = (long)((M + 255) / 256) * ((N + 255) / 256);
    if (M > TC_BM && units256 <= 16) {
      *cg = 2;
      *bn = 128;
      return;
    }
  }
  pick_cfg(M, N, b_mn, cg, bn);
}

template <bool A_MN, bool B_MN, int KIND>
static int launch_bn(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K, const EpiArgs& ep,
                     cudaStream_t st) {
  int cg, bn;
  choose_cfg(M, N, A_MN, B_MN, KIND, &cg, &bn);
  if constexpr (!A_MN && B_MN && KIND == EPI_STORE) {
    if (bn == 64) return launch_tc<1, 64, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
  }
  if (cg == 2) {
    if (bn == 224) return launch_tc<2, 224, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
    if (bn == 192) return launch_tc<2, 192, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
    if (bn == 128) return launch_tc<2, 128, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
    return launch_tc<2, 256, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
  }
  if (bn == 224) return launch_tc<1, 224, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
  if (bn == 192) return launch_tc<1, 192, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
  if (bn == 128) return launch_tc<1, 128, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
  return launch_tc<1, 256, A_MN, B_MN, KIND>(A, lda, B, ldb, M, N, K, ep, st);
}

template <bool A_MN, bool B_MN>
static int dispatch_kind(int kind, const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
                         const EpiArgs& ep, cudaStream_t st) {
  switch (kind) {
    case EPI_STORE: return launch_bn<A_MN, B_MN, EPI_STORE>(A, lda, B, ldb, M, N, K, ep, st);
    case EPI_LOSS: return launch_bn<A_MN, B_MN, EPI_LOSS>(A, lda, B, ldb, M, N, K, ep, st);
    case EPI_MASK: return launch_bn<A_MN, B_MN, EPI_MASK>(A, lda, B, ldb, M, N, K, ep, st);
    case EPI_SGD:
      if constexpr (A_MN && B_MN)
        if (K <= SGD_STREAM_MAX_K) return launch_bn<A_MN, B_MN, EPI_SGD_STREAM>(A, lda, B, ldb, M, N, K, ep, st);
      return launch_bn<A_MN, B_MN, EPI_SGD>(A, lda, B, ldb, M, N, K, ep, st);
    case EPI_GRADF32: return launch_bn<A_MN, B_MN, EPI_GRADF32>(A, lda, B, ldb, M, N, K, ep, st);
    case EPI_GELU:
      if constexpr (!A_MN && !B_MN) return launch_bn<A_MN, B_MN, EPI_GELU>(A, lda, B, ldb, M, N, K, ep, st);
      break;
    case EPI_RESID:
      if constexpr (!A_MN && !B_MN) return launch_bn<A_MN, B_MN, EPI_RESID>(A, lda, B, ldb, M, N, K, ep, st);
      break;
    case EPI_GELU_BWD:
      if constexpr (!A_MN && B_MN) return launch_bn<A_MN, B_MN, EPI_GELU_BWD>(A, lda, B, ldb, M, N, K, ep, st);
      break;
    default:
      return set_error(PD_ERR_INVALID, "unknown epilogue kind %d", kind);
  }
  return set_error(PD_ERR_INVALID, "epilogue kind %d is not instantiated for operand majors (%d, %d)", kind,
                   (int)A_MN, (int)B_MN);
}

// ============================================================== 3x3 convolution passes
// Implicit GEMM on the same tcgen05 kernel; the activation operand comes from TMA im2col loads
// (zero-filled halo = padding), so no im2col matrix is ever materialised in HBM.
static int conv_bn(int N) { return N >= 256 ? 256 : (N >= 128 ? 128 : 64); }

// Split count minimising (waves of (tile, split) units) x (k-blocks per unit) x the k-block time
// (128 x bn x 64 MACs per SM at ~10 TFLOP/s), plus each split's fp32 partial (M x N x 4 B written,
// then read by the reduce, at ~6 TB/s); cg = 2 counts CTA-pair tiles of 256 rows on sms / 2 pairs.
// E.g. 4608 x 512 x 6272 (VGG 14x14, 72 tiles): 2 splits = 1 wave x 49 k-blocks, where a
// two-wave rule's 5 splits give 3 waves x 20 k-blocks and 2.5x the partial traffic.
static int wave_splits(int M, int N, int num_kb, int cg, int max_s) {
  const int bn = conv_bn(N);
  const int tiles = ((M + TC_BM * cg - 1) / (TC_BM * cg)) * ((N + bn - 1) / bn);
  const int slots = num_sms() / cg;
  const double kb_ns = 128.0 * bn * TC_BK * 2.0 / 1.0e4;
  const double part_ns = 8.0 * (double)M * (double)N / 6000.0;
  int s = 1;
  double best = -1.0;
  for (int c = 1; c <= max_s; ++c) {
    const int per_c = (num_kb + c - 1) / c;
    if ((num_kb + per_c - 1) / per_c != c) continue;  // c splits would leave an empty one
    const long waves = ((long)tiles * c + slots - 1) / slots;
    const double cost = (double)waves * per_c * kb_ns + c * part_ns;
    if (best < 0.0 || cost < best) { best = cost; s = c; }
  }
  return s;
}

int splitk_plan(int M, int N, int K, int* splits, int* kb_per) {
  const int bn = conv_bn(N);
  const int tiles = ((M + TC_BM - 1) / TC_BM) * ((N + bn - 1) / bn);
  const int num_kb = (K + TC_BK - 1) / TC_BK;
  const int cap = num_kb / 4 > 1 ? num_kb / 4 : 1;  // at least 4 k-blocks per split
  const int sms = num_sms();
  static int old = -1;  // PD_SPLITK_OLD=1: the round-1 rule (about two waves of units), for A/B runs
  if (old < 0) {
    const char* e = getenv("PD_SPLITK_OLD");
    old = e && atoi(e) == 1 ? 1 : 0;
  }
  int s;
  if (old) {
    s = (2 * sms + tiles - 1) / tiles;
    s = s < 1 ? 1 : (s > cap ? cap : s);
  } else {
    s = wave_splits(M, N, num_kb, 1, cap < 4 * sms ? cap : 4 * sms);
  }
  const int per = (num_kb + s - 1) / s;
  *kb_per = per;
  *splits = (num_kb + per - 1) / per;  // no empty split
  return 0;
}

template <int BN>
static int conv_launch(int pass, const void* act, const void* other, int n, int H, int W, int cin, int cout,
                       int kind, const EpiArgs& ep, cudaStream_t st) {
  const int pix = n * H * W;
  ConvArgs cv{};
  cv.H = H;
  cv.W = W;
  // CTA-pair (cta_group::2) tiles: each CTA of the pair stages half of the weight tile, halving the
  // per-SM weight traffic from L2 (VGG-16 7-1 step on one box: 7.8k -> 8.1k images/s; conv fwd / dgrad
  // classes 77 -> 73 / 75 -> 69 us).  PD_CONV_CG=1 keeps single-CTA tiles (A/B runs).
  static int pair = -1;
  if (pair < 0) {
    const char* e = getenv("PD_CONV_CG");
    pair = e && atoi(e) == 1 ? 0 : 1;
  }
  if (pass == PD_CONV_FWD) {
    if (kind != EPI_STORE) return set_error(PD_ERR_INVALID, "conv fwd: STORE epilogue only");
    cv.C = cin;
    if (pair && pix >= 2 * TC_BM)
      return launch_tc<2, BN, false, true, EPI_STORE, SRC_CONV_FWD>(act, cin, other, cout, pix, cout, 9 * cin, ep, st, cv);
    return launch_tc<1, BN, false, true, EPI_STORE, SRC_CONV_FWD>(act, cin, other, cout, pix, cout, 9 * cin, ep, st,
                                                                  cv);
  }
  if (pass == PD_CONV_DGRAD) {
    if (kind != EPI_MASK) return set_error(PD_ERR_INVALID, "conv dgrad: MASK epilogue only");
    cv.C = cout;
    cv.brows = cin;
    if (pair && pix >= 2 * TC_BM)
      return launch_tc<2, BN, false, false, EPI_MASK, SRC_CONV_DGRAD>(act, cout, other, cout, pix, cin, 9 * cout, ep, st, cv);
    return launch_tc<1, BN, false, false, EPI_MASK, SRC_CONV_DGRAD>(act, cout, other, cout, pix, cin, 9 * cout, ep,
                                                                   st, cv);
  }
  if (kind != EPI_GRADF32) return set_error(PD_ERR_INVALID, "conv wgrad: GRADF32 epilogue only");
  const int M = pass == PD_CONV_WGRAD ? 9 * cin : cin;
  splitk_plan(M, cout, pix, &cv.splits, &cv.kb_per);
  cv.split_stride = ep.accumulate ? 0 : (int64_t)M * ep.ldo;  // accumulate: every split adds into one buffer
  if (pass == PD_CONV_WGRAD) {
    cv.C = cin;
    // CTA pairs (each CTA stages half of the dY tile).  Accumulating into one gradient (the
    // runtime's path: splits red.add), they use their own split plan capped at the single-CTA
    // count; with per-split partials (pd_conv3x3 callers size and reduce pd_splitk_plan's count)
    // they keep that count.  VGG-16 step: 7 986-8 006 -> 8 051-8 071 images/s with the single-CTA
    // plan's splits.  PD_CONV_WGRAD_CG=1: single CTAs.
    static int wpair = -1;
    if (wpair < 0) {
      const char* e = getenv("PD_CONV_WGRAD_CG");
      wpair = e && atoi(e) == 1 ? 0 : 1;
    }
    if (wpair && M > TC_BM) {
      const int num_kb = (pix + TC_BK - 1) / TC_BK;
      const int s = ep.accumulate ? wave_splits(M, cout, num_kb, 2, cv.splits) : cv.splits;
      cv.kb_per = (num_kb + s - 1) / s;
      cv.splits = (num_kb + cv.kb_per - 1) / cv.kb_per;
      return launch_tc<2, BN, true, true, EPI_GRADF32, SRC_CONV_WGRAD>(act, cin, other, cout, M, cout, pix, ep, st, cv);
    }
    return launch_tc<1, BN, true, true, EPI_GRADF32, SRC_CONV_WGRAD>(act, cin, other, cout, M, cout, pix, ep, st, cv);
  }
  // PD_GEMM_WGRAD_SPLITK: plain dW^T[cin, cout] = X^T dY over `pix` rows (im2col'ed first layer)
  return launch_tc<1, BN, true, true, EPI_GRADF32, SRC_2D>(act, cin, other, cout, M, cout, pix, ep, st, cv);
}

int conv3x3_tc(int pass, const void* act, const void* other, int n, int H, int W, int cin, int cout, int kind,
               const EpiArgs& ep, cudaStream_t st) {
  if (n < 1 || H < 1 || W < 1 || cin < 1 || cout < 1) return set_error(PD_ERR_INVALID, "conv: empty shape");
  if (pass != PD_GEMM_WGRAD_SPLITK && (cin % 64 || cout % 64))
    return set_error(PD_ERR_INVALID, "conv: channels must be multiples of 64 (got %d -> %d)", cin, cout);
  if (pass == PD_GEMM_WGRAD_SPLITK && (cin % 8 || cout % 64))
    return set_error(PD_ERR_INVALID, "split-K wgrad: cin %% 8, cout %% 64 required");
  if ((int64_t)n * H * W >= (1ll << 31) / 64) return set_error(PD_ERR_INVALID, "conv: too many pixels");
  if ((reinterpret_cast<uintptr_t>(act) | reinterpret_cast<uintptr_t>(other) | reinterpret_cast<uintptr_t>(ep.out)) & 15)
    return set_error(PD_ERR_INVALID, "conv: 16-byte aligned operands required");
  const int N = (pass == PD_CONV_DGRAD) ? cin : cout;
  switch (conv_bn(N)) {
    case 64: return conv_launch<64>(pass, act, other, n, H, W, cin, cout, kind, ep, st);
    case 128: return conv_launch<128>(pass, act, other, n, H, W, cin, cout, kind, ep, st);
    default: return conv_launch<256>(pass, act, other, n, H, W, cin, cout, kind, ep, st);
  }
}

int gemm_bf16_tc(const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N,
                 int K, int kind, const EpiArgs& ep, cudaStream_t st) {
  if (M <= 0 || N <= 0 || K <= 0) return set_error(PD_ERR_INVALID, "gemm: empty shape %dx%dx%d", M, N, K);
  if ((lda % 8) || (ldb % 8) || (reinterpret_cast<uintptr_t>(A) % 16) || (reinterpret_cast<uintptr_t>(B) % 16))
    return set_error(PD_ERR_INVALID, "gemm: operands must be 16-byte aligned with ld %% 8 == 0");
  if ((kind != EPI_GRADF32 && (ep.ldo % 8)) || (reinterpret_cast<uintptr_t>(ep.out) % 16))
    return set_error(PD_ERR_INVALID, "gemm: output must be 16-byte aligned with ld %% 8 == 0");
  if (!a_mn && !b_mn) return dispatch_kind<false, false>(kind, A, lda, B, ldb, M, N, K, ep, st);
  if (!a_mn && b_mn) return dispatch_kind<false, true>(kind, A, lda, B, ldb, M, N, K, ep, st);
  if (a_mn && !b_mn) return dispatch_kind<true, false>(kind, A, lda, B, ldb, M, N, K, ep, st);
  return dispatch_kind<true, true>(kind, A, lda, B, ldb, M, N, K, ep, st);
}

template <typename T>
static int simt(const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N, int K,
                int kind, const EpiArgs& ep, cudaStream_t st) {
  dim3 grid((N + SM_BN - 1) / SM_BN, (M + SM_BM - 1) / SM_BM);
  const T* a = static_cast<const T*>(A);
  const T* b = static_cast<const T*>(B);
  switch (kind) {
    case EPI_STORE: k_gemm_simt<T, EPI_STORE><<<grid, 256, 0, st>>>(a, a_mn, lda, b, b_mn, ldb, M, N, K, ep); break;
    case EPI_LOSS: k_gemm_simt<T, EPI_LOSS><<<grid, 256, 0, st>>>(a, a_mn, lda, b, b_mn, ldb, M, N, K, ep); break;
    case EPI_MASK: k_gemm_simt<T, EPI_MASK><<<grid, 256, 0, st>>>(a, a_mn, lda, b, b_mn, ldb, M, N, K, ep); break;
    case EPI_SGD: k_gemm_simt<T, EPI_SGD><<<grid, 256, 0, st>>>(a, a_mn, lda, b, b_mn, ldb, M, N, K, ep); break;
    case EPI_GRADF32: k_gemm_simt<T, EPI_GRADF32><<<grid, 256, 0, st>>>(a, a_mn, lda, b, b_mn, ldb, M, N, K, ep); break;
    case EPI_GELU: k_gemm_simt<T, EPI_GELU><<<grid, 256, 0, st>>>(a, a_mn, lda, b, b_mn, ldb, M, N, K, ep); break;
    case EPI_GELU_BWD: k_gemm_simt<T, EPI_GELU_BWD><<<grid, 256, 0, st>>>(a, a_mn, lda, b, b_mn, ldb, M, N, K, ep); break;
    case EPI_RESID: k_gemm_simt<T, EPI_RESID><<<grid, 256, 0, st>>>(a, a_mn, lda, b, b_mn, ldb, M, N, K, ep); break;
    default: return set_error(PD_ERR_INVALID, "unknown epilogue kind %d", kind);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(PD_ERR_CUDA, "simt gemm launch: %s", cudaGetErrorString(e));
  return 0;
}

int gemm_simt(int dtype, const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, int M, int N,
              int K, int kind, const EpiArgs& ep, cudaStream_t st) {
  if (M <= 0 || N <= 0 || K <= 0) return set_error(PD_ERR_INVALID, "gemm: empty shape %dx%dx%d", M, N, K);
  if (ep.sig_flag) return set_error(PD_ERR_INVALID, "gemm: fused hand-off needs the tcgen05 path");
  if (dtype == PD_F32) return simt<float>(A, a_mn, lda, B, b_mn, ldb, M, N, K, kind, ep, st);
  if (dtype == PD_BF16) return simt<__nv_bfloat16>(A, a_mn, lda, B, b_mn, ldb, M, N, K, kind, ep, st);
  return set_error(PD_ERR_INVALID, "unknown dtype %d", dtype);
}

}  // namespace pd

extern "C" int pd_gemm_pick(int M, int N, int K, int a_mn, int b_mn, int kind, int* cg, int* bn) {
  if (!cg || !bn || M <= 0 || N <= 0 || K <= 0) return pd::set_error(PD_ERR_INVALID, "pd_gemm_pick: bad argument");
  pd::choose_cfg(M, N, a_mn != 0, b_mn != 0, kind, cg, bn);
  return 0;
}
