// (2) Global similarity heat map as an implicit GEMM on tcgen05 tensor cores.
//
// Reference: glr/matching.py:140-167 (similarity_heatmap, im2col branch
// :145-156): heat[u,v,n] = sum over the P x P x 4C window of the product of
// the binary edge stack at position (u,v) and at exemplar anchor n. The
// reference runs this as an OpenBLAS sgemm on an explicit im2col copy; here
// the im2col is never materialised:
//
//   * The edge stack holds the binary maps as (H, W, Ce) elements with
//     Ce = e*4C ("e-row expanded": channel p*4C+k of pixel (r,c) holds
//     map_k(r+p, c)), each element an E2M1 (fp4) 1.0 or 0.0 packed two per
//     byte, so a pixel is Cb = Ce/2 bytes. For a fixed output row u and slab
//     s, the K-run of position v is the contiguous byte range
//     stack[u+s*e][v .. v+P-1][*] of length L = P*Cb, and consecutive v are
//     Cb bytes apart. A 3-D TMA map with dims {L, ow, H} and strides
//     {Cb, W*Cb} therefore addresses the overlapping im2col rows directly;
//     one TMA box = 128 positions x 128 bytes (256 K-elements).
//   * The exemplar operand B (Npad x Kp bytes, K-major, zero-padded) is
//     gathered once per refresh from the same stack (exemplar_pack_kernel).
//   * tcgen05.mma kind::mxf4 (block-scaled fp4, f32 accumulate) with every
//     UE8M0 scale factor = 2^0: products of 0/1 are exact and the f32 sums
//     are exact integers (max 4*C*P^2 < 2^24). fp4 halves the operand bytes
//     per multiply-add of the u8 formulation (this kernel is bound by the
//     L2 -> shared-memory operand stream) and runs at twice the i8 rate.
//     Accumulators live in TMEM (2 x 128 lanes x 224 columns), the constant
//     scale factors in the remaining 64 columns.
//   * Output: exemplar-major u16 heat[n][u*ow+v] (flat index = the
//     reference's row-major slice index, matching.py:177-178), rows padded
//     to a multiple of 8 entries (glr_heat_stride) for 16-byte loads.
//
// Persistent, warp-specialised kernel (one CTA per SM), launched as CTA pairs
// (cta_group::2): the pair works on two adjacent 128-position tiles of the
// same 224-exemplar tile, each CTA loads its own A box and half of the B box.
//   warp 0 (one lane)  TMA producer, 7-stage smem ring (full/empty mbarriers;
//                      a stage is refilled once the pair's MMAs released it);
//   warp 1 (one lane)  pair leader: tcgen05.mma.cta_group::2 into one of two
//                      TMEM accumulators;
//   warp 2             owns the 512-column TMEM allocation;
//   warps 4..          epilogue, 4 lane quadrants x EG column groups (EG = 4,
//                      or 7 for tiles of one or two k-blocks): also write the
//                      constant scale factors at start-up; tcgen05.ld -> u16
//                      stores (dense map) or candidate-list appends (fused
//                      top-K), then release the accumulator, so tile i's
//                      epilogue overlaps tile i+1's MMAs (tmem_full/tmem_empty).
#include <cstdio>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "internal.cuh"

namespace glr {

// Candidate floor of the fused path: the sampled pre-pass aims at this many
// pool-sizes of positions above the floor (measured 8 / 4 / 2: C2 92.2 / 91.0 /
// 90.4 ms of fused matching per solve, C5 34.4 / 33.4 / 33.0 ms per pass, no
// exemplar handed to the dense path at any of them; 4 keeps a 4x margin
// against a sample that overestimates the count).
#ifndef GLR_HEAT_WANT_POOLS
#define GLR_HEAT_WANT_POOLS 4
#endif

namespace heat {
constexpr int BM = 128;      // positions per CTA tile (the pair's UMMA M = 256)
constexpr int BN = 224;      // exemplars per pair tile (UMMA N)
constexpr int BNH = BN / 2;  // exemplar rows of B held by each CTA of the pair
constexpr int BK = 128;      // bytes of K per stage (one 128B swizzle row = 256 fp4)
constexpr int UK = 32;       // bytes of K per tcgen05.mma kind::mxf4 (64 fp4)
constexpr int STAGES = 7;
constexpr int ACC = 2;       // TMEM accumulators (2 x 224 columns)
// Epilogue warps: 4 lane quadrants x EG column groups (warps 4 ..), the kernel
// is a template on EG. Four groups (chunks 0-1 | 2-3 | 4-5 | 6, 96 registers
// per thread) by default; seven (one 32-column chunk per warp, 64 registers)
// where a tile is one or two k-blocks and the epilogue IS the kernel (C5:
// fused heat + top-K 42.8 / 36.7 / 34.3 ms with 3 / 4 / 7 groups; C2: 93.3 /
// 92.6 / 93.8 ms per solve).
constexpr int threads_for(int eg) { return 128 + 128 * eg; }
constexpr int A_BYTES = BM * BK;
constexpr int B_BYTES = BNH * BK;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t SFA_COL = 448;  // 32 columns of scale factors for A
constexpr uint32_t SFB_COL = 480;  // 32 columns of scale factors for B
}  // namespace heat

struct HeatGeom {
  int H, W, C4, P, e, Ce, Cb, S, L, kchunks, Kp, oh, ow;
};

static HeatGeom heat_geom(int H, int W, int C, int P, int e) {
  HeatGeom g;
  g.H = H;
  g.W = W;
  g.C4 = 4 * C;
  g.P = P;
  g.e = e;
  g.Ce = e * 4 * C;
  g.Cb = g.Ce / 2;
  g.S = (int)cdiv(P, e);
  g.L = P * g.Cb;
  g.kchunks = (int)cdiv(g.L, heat::BK);
  g.Kp = g.S * g.kchunks * heat::BK;
  g.oh = H - P + 1;
  g.ow = W - P + 1;
  return g;
}

struct HeatParams {
  // oh: output rows the kernel covers; row i is image row u = i * u_step + u0
  // (u_step > 1: a row-sampled map for the candidate floor, see glr_heat_topk)
  int oh, ow, Mpad, n_max, m_tiles_per_row, S, kchunks, e, u_step, u0;
  const int32_t* n_dev;
  uint16_t* heat;
  // candidate mode (cand != nullptr): instead of the dense u16 map, append
  // (score << 32) | position for every score >= thr[n] to cand[n][0 .. cap)
  const uint16_t* thr;
  uint32_t* cnt;
  uint64_t* cand;
  int cap;
};

template <int EPI_GROUPS>
__global__ void __launch_bounds__(heat::threads_for(EPI_GROUPS), 1)
    heat_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, HeatParams p) {
  using namespace heat;
  constexpr int EPI_WARPS = 4 * EPI_GROUPS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC);

  const int N = p.n_dev ? min(*p.n_dev, p.n_max) : p.n_max;
  const int n_tiles = (N + BN - 1) / BN;
  // pair tiles (two m tiles, one n tile), n fastest: pairs share A tiles in L2
  const int total = p.oh * (p.m_tiles_per_row / 2) * n_tiles;
  const int num_k = p.S * p.kchunks;
  const int rank = (int)cluster_ctarank();
  const bool leader = rank == 0;
  const int cl = blockIdx.x >> 1, n_cl = gridDim.x >> 1;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: its expect_tx; both CTAs' TMA bytes land here
      mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast to both CTAs)
    }
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);   // the leader's MMA commit (multicast)
      mbar_init(&tempty[a], 2 * EPI_WARPS);  // leader: one arrive per epilogue warp, both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 2) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp >= 4 && warp < 8) {
    // every scale-factor byte = UE8M0 127 = 2^0, whatever the layout the MMA reads
    uint32_t ones[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) ones[j] = 0x7F7F7F7Fu;
    const uint32_t lanes = (uint32_t)((warp - 4) * 32) << 16;
    tmem_st_32x32b_x32(tmem + lanes + SFA_COL, ones);
    tmem_st_32x32b_x32(tmem + lanes + SFB_COL, ones);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' scale factors written before the leader's first MMA
  tc_fence_after();

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): own A tile + own half of the B tile ----
      int it = 0;
      for (int t = cl; t < total; t += n_cl) {
        const int n0 = (t % n_tiles) * BN;
        const int m_tile = 2 * (t / n_tiles) + rank;
        const int u = (m_tile / p.m_tiles_per_row) * p.u_step + p.u0;
        const int v0 = (m_tile % p.m_tiles_per_row) * BM;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          if (it >= STAGES) mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * STAGE_BYTES);
          const uint32_t fb = cluster_addr(&full[s], 0);
          const int slab = kb / p.kchunks;
          const int kc = kb - slab * p.kchunks;
          tma_load_3d_pair(sA + s * A_BYTES, &tmA, fb, kc * BK, v0, u + slab * p.e);
          tma_load_2d_pair(sB + s * B_BYTES, &tmB, fb, kb * BK, n0 + rank * BNH);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---- MMA issuer (pair leader): 256 x 224 x 64 fp4 per instruction ----
      constexpr uint32_t idesc = idesc_mxf4(2 * BM, BN);
      int it = 0, lt = 0;
      for (int t = cl; t < total; t += n_cl, ++lt) {
        const int acc = lt & 1, use = lt >> 1;
        if (use > 0) mbar_wait_cluster(&tempty[acc], (use - 1) & 1);  // both epilogues drained it
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = smem_desc_k_sw128(sA + s * A_BYTES);
          const uint64_t bd = smem_desc_k_sw128(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)  // +32 bytes inside the 128B swizzle atom
            umma_mxf4_pair(d, ad + (uint64_t)((k * UK) >> 4), bd + (uint64_t)((k * UK) >> 4),
                           idesc, (kb | k) != 0, tmem + SFA_COL, tmem + SFB_COL);
          umma_commit_pair_mc(&empty[s], 0x3);  // frees stage s in both CTAs
        }
        umma_commit_pair_mc(&tfull[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue (both CTAs): own 128 TMEM lanes -> u16 exemplar-major rows ----
    const int ew = warp & 3;           // TMEM lanes 32*ew .. 32*ew+31 (warp id % 4)
    const int grp = (warp - 4) >> 2;  // column group: 32-column chunks [c_lo, c_hi)
    constexpr int NCH = BN / 32;
    const int c_lo = (NCH * grp + EPI_GROUPS - 1) / EPI_GROUPS;
    const int c_hi = (NCH * (grp + 1) + EPI_GROUPS - 1) / EPI_GROUPS;
    const uint32_t te_leader[ACC] = {cluster_addr(&tempty[0], 0), cluster_addr(&tempty[1], 0)};
    int lt = 0;
    for (int t = cl; t < total; t += n_cl, ++lt) {
      const int acc = lt & 1, use = lt >> 1;
      const int n0 = (t % n_tiles) * BN;
      const int m_tile = 2 * (t / n_tiles) + rank;
      const int ui = m_tile / p.m_tiles_per_row;  // output row (sample row index)
      const int u = ui * p.u_step + p.u0;         // image row
      const int v = (m_tile % p.m_tiles_per_row) * BM + ew * 32 + lane;
      // candidate mode: this warp's exemplar floors, loaded before the wait
      // (a global load per chunk after it was the kernel's top stall)
      constexpr int MAXC = (NCH + EPI_GROUPS - 1) / EPI_GROUPS;
      int tl_c[MAXC];
      if (p.cand) {
#pragma unroll
        for (int k = 0; k < MAXC; ++k) {
          const int n = n0 + (c_lo + k) * 32 + lane;
          tl_c[k] = (c_lo + k < c_hi && n < N) ? (int)p.thr[n] : 0x10000;
        }
      }
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const bool v_ok = v < p.ow;
      GLR_DCHECK(ui < p.oh && u < p.oh * p.u_step + p.u0 && (int64_t)ui * p.ow < p.Mpad);
      uint16_t* out = p.heat + (size_t)ui * p.ow + v;
      if (p.cand) {
        // Candidate lists, two sweeps over this warp's chunks so the slot
        // reservations (one returning atomic per chunk, ~700 cycles) overlap
        // the next chunks' work instead of sitting on each chunk's critical
        // path (C5: ~3 hits per 32 x 32 chunk, the epilogue is the kernel).
        // Sweep A per chunk: lane-local hit bits (float compares, the floors
        // broadcast from the lane that owns the column), col_mask = their
        // 32 x 32 bit transpose across the warp (five butterfly stages instead
        // of a ballot per column; lane j: the lanes that hit column j), and
        // ONE warp-wide atomic reserving every hit column's slots (lane j for
        // column j). Sweep B re-reads the chunk from TMEM and appends.
        const uint32_t pos = (uint32_t)(u * p.ow + v);
        const unsigned lt = (1u << lane) - 1u;
        const uint32_t trow = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * BN);
        unsigned hits_c[MAXC], cmask_c[MAXC];
        uint32_t base_c[MAXC];
#pragma unroll
        for (int k = 0; k < MAXC; ++k) {
          hits_c[k] = 0;
          cmask_c[k] = 0;
          base_c[k] = 0;
          const int c = c_lo + k;
          if (c >= c_hi) continue;  // warp-uniform
          uint32_t r[32];
          tmem_ld_32x32b_x32(trow + (uint32_t)(c * 32), r);
          tmem_ld_wait();
          const float tlf = (float)tl_c[k];
          unsigned my_hits = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            my_hits |= (unsigned)(__uint_as_float(r[j]) >= __shfl_sync(0xffffffffu, tlf, j)) << j;
          if (!v_ok) my_hits = 0;
          if (!__any_sync(0xffffffffu, my_hits != 0)) continue;
          unsigned col_mask = my_hits;
#pragma unroll
          for (int sft = 16; sft >= 1; sft >>= 1) {
            const unsigned M = sft == 16 ? 0x0000FFFFu : sft == 8 ? 0x00FF00FFu
                             : sft == 4 ? 0x0F0F0F0Fu : sft == 2 ? 0x33333333u : 0x55555555u;
            const unsigned y = __shfl_xor_sync(0xffffffffu, col_mask, sft);
            col_mask = (lane & sft) ? ((col_mask & ~M) | ((y & ~M) >> sft))
                                    : ((col_mask & M) | ((y & M) << sft));
          }
          hits_c[k] = my_hits;
          cmask_c[k] = col_mask;
          if (col_mask)
            base_c[k] = atomicAdd(&p.cnt[n0 + c * 32 + lane], (uint32_t)__popc(col_mask));
        }
#pragma unroll
        for (int k = 0; k < MAXC; ++k) {
          const int c = c_lo + k;
          if (c >= c_hi) continue;  // warp-uniform
          const unsigned any_cols = __ballot_sync(0xffffffffu, cmask_c[k] != 0);
          if (!any_cols) continue;
          uint32_t r[32];
          tmem_ld_32x32b_x32(trow + (uint32_t)(c * 32), r);
          tmem_ld_wait();
          const int nb = n0 + c * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (!((any_cols >> j) & 1u)) continue;  // warp-uniform
            const unsigned m = __shfl_sync(0xffffffffu, cmask_c[k], j);
            const uint32_t b = __shfl_sync(0xffffffffu, base_c[k], j) + __popc(m & lt);
            if (((hits_c[k] >> j) & 1u) && b < (uint32_t)p.cap) {
              const int sc = (int)__float2uint_rn(__uint_as_float(r[j]));
              p.cand[(size_t)(nb + j) * p.cap + b] = ((uint64_t)sc << 32) | pos;
            }
          }
        }
      } else {
#pragma unroll 1
        for (int c = c_lo; c < c_hi; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * BN + c * 32), r);
          tmem_ld_wait();
          const int nb = n0 + c * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = nb + j;
            // streaming (evict-first) stores: the 8.5 GB map must not push the
            // reused A/B operand tiles out of L2
            if (v_ok && n < N)
              __stcs(reinterpret_cast<unsigned short*>(out + (size_t)n * p.Mpad),
                     (unsigned short)__float2uint_rn(__uint_as_float(r[j])));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(te_leader[acc]);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still use its smem / TMEM
  if (warp == 2) tmem_dealloc_pair<TMEM_COLS>(tmem);
}

// B operand (bytes): bmat[n][s*kchunks*BK + k'] = stack[r_n + s*e][c_n + k'/Cb][k' % Cb]
// for k' < L, zero for the K padding, for the padded exemplars and past row H.
__global__ void exemplar_pack_kernel(const uint8_t* __restrict__ stack, HeatGeom g,
                                     const int32_t* __restrict__ anchors, int n_max,
                                     const int32_t* n_dev, int n_pad, uint8_t* __restrict__ bmat) {
  const int N = n_dev ? min(*n_dev, n_max) : n_max;
  const int row_bytes = g.Kp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n_pad * row_bytes;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / row_bytes);
    const int k = (int)(i - (int64_t)n * row_bytes);
    const int slab = k / (g.kchunks * heat::BK);
    const int kk = k - slab * g.kchunks * heat::BK;
    uint8_t val = 0;
    if (n < N && kk < g.L) {
      const int cb = kk % g.Cb;
      // the byte's two expanded channels 2cb, 2cb+1 (same row: 4C is even) hold
      // map row (anchor row + slab*e + 2cb / 4C); rows at or past P belong to
      // no patch and stay zero
      if (slab * g.e + (2 * cb) / g.C4 < g.P) {
        const int r = anchors[2 * n] + slab * g.e;
        const int c = anchors[2 * n + 1] + kk / g.Cb;
        val = stack[((size_t)r * g.W + c) * g.Cb + cb];
      }
    }
    bmat[i] = val;
  }
}

// thr[n] = |E_n| / 4: a quarter of the exemplar's self-score (the number of
// 1.0 nibbles of its packed operand row = the maximum of its heat row)
__global__ void exemplar_thr_kernel(const uint8_t* __restrict__ bmat, int Kp, int n_max,
                                    uint16_t* __restrict__ thr) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n_max) return;
  const uint32_t* row = reinterpret_cast<const uint32_t*>(bmat + (size_t)w * Kp);
  int cnt = 0;
  for (int i = lane; i < Kp / 4; i += 32) {
    const uint32_t v = row[i];
#pragma unroll
    for (int k = 0; k < 8; ++k) cnt += ((v >> (4 * k)) & 0xFu) == kFp4One;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) thr[w] = (uint16_t)(cnt >> 2);
}

// Sampled candidate floor: thr[n] = T_n, the largest score with at least
// `want` entries >= T_n among the exemplar's row-sampled heat scores (want ~
// 8 pool x the sampled fraction of the positions; 0 when the sample is
// smaller than `want`). Unlike the quarter-self-score floor it may go below
// |E_n| / 4, which the pool does reach on mixed images (C1, C3). So the
// fused epilogue records a few pool-sizes of candidates per exemplar whatever
// the score distribution. One CTA per exemplar, shared-memory histogram of
// the top score range. Exactness does not depend on it: an exemplar whose
// cut falls below its floor (or whose list overflows) goes to the dense path.
__global__ void __launch_bounds__(256) sample_thr_kernel(const uint16_t* __restrict__ hs,
                                                         int64_t mpad, int ns, int n_max,
                                                         int bins, int want,
                                                         uint16_t* __restrict__ thr) {
  extern __shared__ int hist_s[];
  __shared__ int s_T;
  const int n = blockIdx.x;
  if (n >= n_max) return;
  const int lo = 0;
  for (int b = threadIdx.x; b < bins; b += blockDim.x) hist_s[b] = 0;
  if (threadIdx.x == 0) s_T = lo;
  __syncthreads();
  const uint16_t* row = hs + (size_t)n * mpad;  // 16-byte aligned (mpad % 8 == 0)
  const uint4* rv = reinterpret_cast<const uint4*>(row);
  for (int i = threadIdx.x; i < ns / 8; i += blockDim.x) {
    const uint4 q = rv[i];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int v = min((int)((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu), bins - 1);
      if (v > lo) atomicAdd(&hist_s[v], 1);
    }
  }
  for (int i = (ns / 8) * 8 + threadIdx.x; i < ns; i += blockDim.x) {
    const int v = min((int)row[i], bins - 1);
    if (v > lo) atomicAdd(&hist_s[v], 1);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int running = 0;
    for (int top = bins - 1; top > lo; top -= 32) {
      const int b = top - lane;
      const int c = b > lo ? hist_s[b] : 0;
      int incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, b > lo && running + incl >= want);
      if (hit) {
        if (lane == 0) s_T = top - (__ffs(hit) - 1);
        break;
      }
      running += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) thr[n] = (uint16_t)s_T;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

}  // namespace glr

using namespace glr;

extern "C" int glr_heat_expand_factor(int C, int P) {
  // Smallest padded K (then the smallest expansion) among e in [1, max(P,8)]
  // whose pixel stride e*4C/2 bytes is a multiple of 16 (TMA stride rule);
  // e = 8 always qualifies. Expanded rows at or past P are zero in B.
  int best_e = -1;
  int64_t best_k = 0;
  for (int e = 1; e <= (P > 8 ? P : 8); ++e) {
    if ((4 * C * e) % 32 != 0) continue;
    HeatGeom g = heat_geom(P, P, C, P, e);
    if (best_e < 0 || g.Kp < best_k) {
      best_e = e;
      best_k = g.Kp;
    }
  }
  return best_e;
}

extern "C" int64_t glr_heat_stride(int H, int W, int P) {
  return cdiv((int64_t)(H - P + 1) * (W - P + 1), 8) * 8;
}

extern "C" size_t glr_heat_workspace(int C, int P, int n_max) {
  int e = glr_heat_expand_factor(C, P);
  if (e < 1) return 0;
  HeatGeom g = heat_geom(P, P, C, P, e);
  size_t n_pad = (size_t)cdiv(n_max, heat::BN) * heat::BN;
  return n_pad * (size_t)g.Kp + 256;
}

// pack B (+ thresholds in candidate mode) and launch the GEMM; shared by
// glr_heat_map (dense map) and glr_heat_topk (candidate lists)
// sampled rows of the candidate floor's pre-pass (u_step > 1): the map
// covers image rows u0, u0 + u_step, ... (oh_eff of them, row stride mpad)
struct HeatRows {
  int oh_eff = -1, u_step = 1, u0 = 0;
  int64_t mpad = -1;
  bool pack = true;
};

template <int EG>
static int launch_heat(const CUtensorMap& tmA, const CUtensorMap& tmB, const HeatParams& hp,
                       int64_t pairs, cudaStream_t st) {
  {
    const int s = ensure_smem_attr((const void*)heat_gemm_kernel<EG>, heat::SMEM_BYTES);
    if (s) return s;
  }
  const int sms = device_sms();
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(heat::threads_for(EG));
  cfg.dynamicSmemBytes = heat::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent: one CTA per SM, in clusters of two -- as many clusters as can
  // be co-resident (the GPCs need not split into pairs evenly)
  // (per device: the occupancy query depends on the device's GPC layout)
  struct Q {
    cudaLaunchConfig_t* cfg;
    int sms;
  } q{&cfg, sms};
  const int max_clusters = cached_per_device(
      (const void*)heat_gemm_kernel<EG>,
      [](void* ctx) -> int {
        Q* qq = static_cast<Q*>(ctx);
        qq->cfg->gridDim = dim3(2 * (qq->sms / 2));
        int mc = 0;
        if (cudaOccupancyMaxActiveClusters(&mc, heat_gemm_kernel<EG>, qq->cfg) != cudaSuccess ||
            mc < 1)
          mc = qq->sms / 2;
        cudaGetLastError();
        return mc;
      },
      &q);
  cfg.gridDim = dim3(2 * (unsigned)std::min<int64_t>(pairs, max_clusters));
  GLR_CUDA(cudaLaunchKernelEx(&cfg, heat_gemm_kernel<EG>, tmA, tmB, hp));
  return GLR_OK;
}

static int run_heat(const uint8_t* stack_d, int H, int W, int P, const HeatGeom& g,
                    const int32_t* anchors_d, int n_max, const int32_t* n_dev_d,
                    uint16_t* heat_d, uint8_t* bmat, uint16_t* thr_d, uint32_t* cnt_d,
                    uint64_t* cand_d, int cap, cudaStream_t st, HeatRows rows = HeatRows()) {
  const int n_pad = (int)cdiv(n_max, heat::BN) * heat::BN;
  auto encode = get_encode_fn();
  GLR_REQUIRE(encode != nullptr, GLR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (rows.pack) {
    int64_t total = (int64_t)n_pad * g.Kp;
    int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
    exemplar_pack_kernel<<<blocks, 256, 0, st>>>(stack_d, g, anchors_d, n_max, n_dev_d, n_pad,
                                                 bmat);
    GLR_CUDA(cudaGetLastError());
  }
  if (cand_d) GLR_CUDA(cudaMemsetAsync(cnt_d, 0, (size_t)n_max * sizeof(uint32_t), st));

  CUtensorMap tmA, tmB;
  {
    cuuint64_t dims[3] = {(cuuint64_t)g.L, (cuuint64_t)g.ow, (cuuint64_t)H};
    cuuint64_t strides[2] = {(cuuint64_t)g.Cb, (cuuint64_t)W * g.Cb};
    cuuint32_t box[3] = {heat::BK, heat::BM, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)stack_d, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GLR_REQUIRE(r == CUDA_SUCCESS, GLR_ERR_CUDA, "cuTensorMapEncodeTiled(A) failed: %d", (int)r);
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)g.Kp, (cuuint64_t)n_pad};
    cuuint64_t strides[1] = {(cuuint64_t)g.Kp};
    cuuint32_t box[2] = {heat::BK, heat::BNH};  // each CTA of a pair loads its half
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)bmat, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GLR_REQUIRE(r == CUDA_SUCCESS, GLR_ERR_CUDA, "cuTensorMapEncodeTiled(B) failed: %d", (int)r);
  }

  HeatParams hp;
  hp.oh = rows.oh_eff >= 0 ? rows.oh_eff : g.oh;
  hp.ow = g.ow;
  hp.u_step = rows.u_step;
  hp.u0 = rows.u0;
  hp.Mpad = (int)(rows.mpad >= 0 ? rows.mpad : glr_heat_stride(H, W, P));
  hp.n_max = n_max;
  hp.m_tiles_per_row = (int)cdiv(g.ow, 2 * heat::BM) * 2;  // even: tiles go in pairs
  hp.S = g.S;
  hp.kchunks = g.kchunks;
  hp.e = g.e;
  hp.n_dev = n_dev_d;
  hp.heat = heat_d;
  hp.thr = thr_d;
  hp.cnt = cnt_d;
  hp.cand = cand_d;
  hp.cap = cap;
  const int64_t pairs = (int64_t)hp.oh * (hp.m_tiles_per_row / 2) * (n_pad / heat::BN);
  if (pairs == 0) return GLR_OK;  // pack only
  GLR_REQUIRE(pairs < (1ll << 31), GLR_ERR_UNSUPPORTED, "heat_map: too many tiles");
  if (g.S * g.kchunks <= 2) return launch_heat<7>(tmA, tmB, hp, pairs, st);
  return launch_heat<4>(tmA, tmB, hp, pairs, st);
}

extern "C" int glr_heat_map(const uint8_t* stack_d, int H, int W, int C, int P, int expand,
                            const int32_t* anchors_d, int n_max, const int32_t* n_dev_d,
                            uint16_t* heat_d, void* ws_d, size_t ws_bytes, void* stream) {
  GLR_REQUIRE(P >= 1 && P <= H && P <= W && C >= 1, GLR_ERR_INVALID,
              "heat_map: bad shape H=%d W=%d C=%d P=%d", H, W, C, P);
  GLR_REQUIRE(expand >= 1 && expand <= (P > 8 ? P : 8) && (4 * C * expand) % 32 == 0,
              GLR_ERR_INVALID,
              "heat_map: expand factor %d invalid for C=%d", expand, C);
  if (n_max <= 0) return GLR_OK;
  HeatGeom g = heat_geom(H, W, C, P, expand);
  GLR_REQUIRE(4 * C * P * P <= 65535, GLR_ERR_UNSUPPORTED,
              "heat_map: max score %d does not fit u16", 4 * C * P * P);
  const int n_pad = (int)cdiv(n_max, heat::BN) * heat::BN;
  GLR_REQUIRE(ws_bytes >= (size_t)n_pad * g.Kp, GLR_ERR_WORKSPACE,
              "heat_map: workspace %zu < %zu", ws_bytes, (size_t)n_pad * g.Kp);
  return run_heat(stack_d, H, W, P, g, anchors_d, n_max, n_dev_d, heat_d,
                  reinterpret_cast<uint8_t*>(ws_d), nullptr, nullptr, nullptr, 0,
                  reinterpret_cast<cudaStream_t>(stream));
}

// workspace of glr_heat_topk: packed B | thresholds | counts | candidate lists
static size_t heat_topk_layout(int C, int P, int n_max, int cap, size_t off[4]) {
  int e = glr_heat_expand_factor(C, P);
  HeatGeom g = heat_geom(P, P, C, P, e < 1 ? 1 : e);
  const size_t n_pad = (size_t)cdiv(std::max(n_max, 1), heat::BN) * heat::BN;
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  off[0] = 0;
  off[1] = al(off[0] + n_pad * (size_t)g.Kp);
  off[2] = al(off[1] + n_pad * sizeof(uint16_t));
  off[3] = al(off[2] + n_pad * sizeof(uint32_t));
  return off[3] + (size_t)std::max(n_max, 1) * cap * sizeof(uint64_t) + 256;
}

extern "C" size_t glr_heat_topk_workspace(int C, int P, int n_max, int cap) {
  size_t off[4];
  return heat_topk_layout(C, P, n_max, cap, off);
}

extern "C" int glr_heat_topk(const uint8_t* stack_d, int H, int W, int C, int P, int expand,
                             const int32_t* anchors_d, int n_max, int K, int sep, int cap,
                             int32_t* positions_d, int32_t* padded_d, uint8_t* fallback_d,
                             void* ws_d, size_t ws_bytes, void* stream) {
  GLR_REQUIRE(P >= 1 && P <= H && P <= W && C >= 1, GLR_ERR_INVALID,
              "heat_topk: bad shape H=%d W=%d C=%d P=%d", H, W, C, P);
  GLR_REQUIRE(expand >= 1 && expand <= (P > 8 ? P : 8) && (4 * C * expand) % 32 == 0,
              GLR_ERR_INVALID, "heat_topk: expand factor %d invalid for C=%d", expand, C);
  GLR_REQUIRE(cap >= 1, GLR_ERR_INVALID, "heat_topk: cap %d", cap);
  if (n_max <= 0) return GLR_OK;
  HeatGeom g = heat_geom(H, W, C, P, expand);
  GLR_REQUIRE(4 * C * P * P <= 65535, GLR_ERR_UNSUPPORTED,
              "heat_topk: max score %d does not fit u16", 4 * C * P * P);
  size_t off[4];
  const size_t need = heat_topk_layout(C, P, n_max, cap, off);
  GLR_REQUIRE(ws_bytes >= need, GLR_ERR_WORKSPACE, "heat_topk: workspace %zu < %zu", ws_bytes,
              need);
  uint8_t* base = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(ws_d) + 255) & ~uintptr_t(255));
  GLR_REQUIRE(ws_bytes - (size_t)(base - reinterpret_cast<uint8_t*>(ws_d)) >= need - 256,
              GLR_ERR_WORKSPACE, "heat_topk: workspace alignment");
  uint8_t* bmat = base + off[0];
  uint16_t* thr = reinterpret_cast<uint16_t*>(base + off[1]);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(base + off[2]);
  uint64_t* cand = reinterpret_cast<uint64_t*>(base + off[3]);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // 1. pack B + sampled pre-pass: the dense map of every u_step-th output row
  //    (at most 16 rows, aliasing the candidate lists, which are written
  //    only later) -> per-exemplar floor thr[n] (sample_thr_kernel) over the
  //    |E_n| / 4 lower bound
  {
    const int64_t row_room = (int64_t)cap * 4;  // u16 entries per exemplar in the list region
    int oh_eff = (int)std::min<int64_t>(std::min(32, g.oh), row_room / g.ow);
    HeatRows rows;
    if (oh_eff >= 1) {
      rows.oh_eff = oh_eff;
      rows.u_step = g.oh / oh_eff;
      rows.u0 = rows.u_step / 2;
      rows.mpad = cdiv((int64_t)oh_eff * g.ow, 8) * 8;
      if (rows.mpad > row_room) rows.oh_eff = oh_eff = 0;
    }
    uint16_t* hs = reinterpret_cast<uint16_t*>(cand);
    if (oh_eff >= 1) {
      const int r = run_heat(stack_d, H, W, P, g, anchors_d, n_max, nullptr, hs, bmat, nullptr,
                             nullptr, nullptr, 0, st, rows);
      if (r != GLR_OK) return r;
    } else {
      HeatRows pk;
      pk.oh_eff = 0;  // pack only: no tiles
      const int r = run_heat(stack_d, H, W, P, g, anchors_d, n_max, nullptr, hs, bmat, nullptr,
                             nullptr, nullptr, 0, st, pk);
      if (r != GLR_OK) return r;
    }
    exemplar_thr_kernel<<<(unsigned)cdiv((int64_t)n_max * 32, 256), 256, 0, st>>>(bmat, g.Kp,
                                                                                  n_max, thr);
    GLR_CUDA(cudaGetLastError());
    if (oh_eff >= 1) {
      const int bins = 4 * C * P * P + 1;
      const int ns = oh_eff * g.ow;
      const int64_t M = (int64_t)g.oh * g.ow;
      const int pool = K * (2 * sep + 1) * (2 * sep + 1) + 1;
      // aim at a few pool-sizes above the floor: the integer scores tie heavily
      // at the cut, and a floor estimated too high sends the exemplar to the
      // dense fallback
      const int want = (int)std::max<int64_t>(1, (GLR_HEAT_WANT_POOLS * (int64_t)pool * ns + M - 1) / M);
      const int smem = bins * (int)sizeof(int);
      {
        const int s_ = ensure_smem_attr((const void*)sample_thr_kernel, smem);
        if (s_) return s_;
      }
      sample_thr_kernel<<<n_max, 256, smem, st>>>(hs, rows.mpad, ns, n_max, bins, want, thr);
      GLR_CUDA(cudaGetLastError());
    }
  }
  // 2. the candidate GEMM (no pack: B is in place) and the exact top-K on the lists
  HeatRows nopack;
  nopack.pack = false;
  const int r = run_heat(stack_d, H, W, P, g, anchors_d, n_max, nullptr, nullptr, bmat, thr, cnt,
                         cand, cap, st, nopack);
  if (r != GLR_OK) return r;
  return topk_cand_launch(cand, cnt, thr, cap, n_max, g.oh, g.ow, 4 * C * P * P, anchors_d, K,
                          sep, positions_d, padded_d, fallback_d, stream);
}
