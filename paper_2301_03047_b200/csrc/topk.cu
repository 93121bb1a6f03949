// (3) Exact tie-ordered top-K selection per exemplar + patch gather.
//
// Reference: glr/matching.py:170-231 (top_k_positions) and :240-252
// (global_match loop), glr/patches.py:43-54 (gather_group).
//
// Semantics reproduced exactly (integer decisions, no tolerance):
//   slot 0 = the exemplar's anchor; remaining slots walk positions in
//   (score desc, flat row-major index asc) order, skipping any position within
//   Chebyshev distance <= sep of an already-chosen one; if the walk runs out,
//   a second walk with sep = 0; missing slots repeat the anchor ("padded").
//
// One CTA per exemplar over its u16 heat-map row:
//   1. shared-memory histogram of the integer scores (only the top range
//      unless the cut falls below it);
//   2. the cut T = largest score with count(>= T) >= need, need = min(pool, M)
//      where pool = K(2 sep + 1)^2 + 1 (the reference's bound: the first pool
//      entries of the ordered walk always fill the group, matching.py:219-225);
//   3. one pass collecting A = {score > T} (all, < need entries) and the ties
//      B = {score == T}, of which the first need-|A| in index order are kept
//      — exactly the first `need` entries of the reference's ordered walk;
//   4. bitonic sort of A by (score desc, index asc) in shared memory;
//   5. one warp runs the greedy walk, 32 candidates per step: lanes test
//      their candidate against the chosen set in parallel, then accepted
//      candidates are committed in lane order with an in-warp re-check.
#include "common.cuh"
#include "internal.cuh"

namespace glr {

namespace topk {
constexpr int THREADS = 512;
constexpr int kSelB = 2048;  // tie-selection buckets / kept ties of the list path
constexpr int VEC = 8;  // u16 scores per 16-byte load
constexpr int MAX_BINS = 12288;
constexpr int RING_STAGES = 3;
constexpr int RING_BYTES = 16384;  // 32 bytes per thread per slice
}  // namespace topk

#ifdef GLR_TOPK_PHASES  // dev: per-phase cycles of topk_kernel (thread 0 of every CTA)
__device__ unsigned long long g_topk_phase[8];
#define TK_MARK(i)                                                        \
  do {                                                                    \
    if (threadIdx.x == 0) {                                               \
      const long long now_ = clock64();                                   \
      atomicAdd(&g_topk_phase[i], (unsigned long long)(now_ - tk_t0_));   \
      tk_t0_ = now_;                                                      \
    }                                                                     \
  } while (0)
extern "C" int glr_debug_topk_phases(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_topk_phase, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_topk_phase, z, sizeof(z));
  }
  return 0;
}
#else
#define TK_MARK(i)
#endif
#ifdef GLR_TOPK_STATS
__device__ unsigned int g_topk_stats[4];  // rows, fallbacks below L, sum / max of count(>= L)
__device__ unsigned int g_cand_stats[6];  // list path: rows, overflow, short, ties, sum / max count
#endif

struct TopkParams {
  const uint16_t* heat;
  int64_t stride;  // heat row stride (entries)
  int n_max;
  const int32_t* n_dev;
  int oh, ow;
  int64_t M;
  int bins;  // max_score + 1
  const int32_t* anchors;
  int K, sep, pool, a_cap;  // a_cap: power of two >= pool
  int b_cap;                // tie buffer: power of two >= max(pool, 4096)
  int32_t* positions;
  int32_t* padded;
  // optional per-exemplar scratch (n_max x scap): the first pass also records
  // every (score >= L, position) so the collection pass reads this list
  // instead of the row again
  uint64_t* scratch;
  int scap;
  // optional split (with the scratch): the row pass stops after collecting
  // A and the ties and stages them here (n_max x a_cap / b_cap / 2 counts);
  // topk_select_kernel sorts them and runs the greedy walk, so the
  // barrier-heavy sorts and the single-warp walk no longer hold up the
  // bandwidth-bound row stream
  uint64_t* stageA;
  int32_t* stageB;
  int32_t* stageN;
};

// Ascending bitonic sort of sz (a power of two >= 64) 64-bit keys in shared
// memory with the keys held in registers: thread t owns a[EPT t .. EPT t + EPT),
// so partner distances below EPT are register exchanges, those below 32 EPT
// warp shuffles, and only the rest go through shared memory (sz = 2048,
// EPT = 4: 10 of the 66 stages -- the plain version paid a block barrier for
// every stage and was ~27 % of the dense top-K kernel on C4).
template <class T, int EPT>
__device__ __forceinline__ void bitonic_regs(T* a, int sz) {
  const int tid = threadIdx.x, lane = tid & 31;
  const bool act = tid < sz / EPT;  // whole warps: sz / EPT is a multiple of 32
  const int i0 = tid * EPT;
  T x[EPT];
  if (act) {
#pragma unroll
    for (int q = 0; q < EPT; ++q) x[q] = a[i0 + q];
  }
  for (int k = 2; k <= sz; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < EPT) {
        if (act) {
#pragma unroll
          for (int jc = 1; jc < EPT; jc <<= 1) {  // compile-time distances: x[] stays in registers
            if (j != jc) continue;
#pragma unroll
            for (int q = 0; q < EPT; ++q) {
              if ((q & jc) == 0) {
                const int pq = q | jc;
                const bool up = ((i0 + q) & k) == 0;
                const T lo = x[q] < x[pq] ? x[q] : x[pq], hi = x[q] < x[pq] ? x[pq] : x[q];
                x[q] = up ? lo : hi;
                x[pq] = up ? hi : lo;
              }
            }
          }
        }
      } else if (j < 32 * EPT) {
        if (act) {
          const int lm = j / EPT;
          const bool lower = (lane & lm) == 0;
#pragma unroll
          for (int q = 0; q < EPT; ++q) {
            const T y = __shfl_xor_sync(0xffffffffu, x[q], lm);
            const bool up = ((i0 + q) & k) == 0;
            const bool keep_min = lower == up;
            x[q] = (x[q] < y) == keep_min ? x[q] : y;
          }
        }
      } else {
        if (act) {
#pragma unroll
          for (int q = 0; q < EPT; ++q) a[i0 + q] = x[q];
        }
        __syncthreads();
        if (act) {
#pragma unroll
          for (int q = 0; q < EPT; ++q) {
            const int i = i0 + q;
            const T y = a[i ^ j];
            const bool up = (i & k) == 0;
            const bool keep_min = ((i & j) == 0) == up;
            x[q] = (x[q] < y) == keep_min ? x[q] : y;
          }
        }
        __syncthreads();
      }
    }
  }
  if (act) {
#pragma unroll
    for (int q = 0; q < EPT; ++q) a[i0 + q] = x[q];
  }
  __syncthreads();
}

__device__ __forceinline__ int cheb(int r0, int c0, int r1, int c1) {
  return max(abs(r0 - r1), abs(c0 - c1));
}

// Steps 4-5, shared by both top-K kernels: bitonic sort of A (score desc,
// index asc), then the greedy walk over the first `need` entries of A ++ B.
__device__ __forceinline__ void topk_finish(const TopkParams& p, int n, int64_t M, int need,
                                            int cntA, uint64_t* sA, const int32_t* sB,
                                            int32_t* chosen) {
  using namespace topk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef GLR_TOPK_PHASES
  long long tk_t0_ = clock64();
#endif
  // 4. bitonic sort of A (padded to the next power of two >= cntA)
  int sz = 1;
  while (sz < cntA) sz <<= 1;
  for (int i = cntA + tid; i < sz; i += THREADS) sA[i] = ~0ull;
  __syncthreads();
  // keys are distinct (the position is part of the key; the padding sorts last
  // in any order), so every sorting network gives the same result
  const int ept = sz / THREADS;
  if (sz >= 64 && ept <= 8) {
    switch (ept) {
      case 0: case 1: bitonic_regs<uint64_t, 1>(sA, sz); break;
      case 2: bitonic_regs<uint64_t, 2>(sA, sz); break;
      case 4: bitonic_regs<uint64_t, 4>(sA, sz); break;
      default: bitonic_regs<uint64_t, 8>(sA, sz); break;
    }
  } else
  for (int k = 2; k <= sz; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < sz; i += THREADS) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = sA[i], y = sA[ixj];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            sA[i] = y;
            sA[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }

  TK_MARK(4);
  // 5. greedy walk (warp 0)
  if (warp == 0) {
    const int ar = p.anchors[2 * n], ac = p.anchors[2 * n + 1];
    if (lane == 0) {
      chosen[0] = ar;
      chosen[1] = ac;
    }
    __syncwarp();
    int nch = 1;
    const int L = need;
    const bool full_walk = (int64_t)need == M;  // the list is the whole ordered slice
    for (int pass = 0; pass < (full_walk ? 2 : 1) && nch < p.K; ++pass) {
      const int sep = pass == 0 ? p.sep : 0;
      for (int base = 0; base < L && nch < p.K; base += 32) {
        const int j = base + lane;
        int idx = -1;
        if (j < L) idx = j < cntA ? (int)(uint32_t)(sA[j] & 0xFFFFFFFFull) : sB[j - cntA];
        const int r = idx >= 0 ? idx / p.ow : 0;
        const int c = idx >= 0 ? idx - r * p.ow : 0;
        bool blocked = idx < 0;
        for (int t = 0; t < nch && !blocked; ++t)
          if (cheb(r, c, chosen[2 * t], chosen[2 * t + 1]) <= sep) blocked = true;
        unsigned mask = __ballot_sync(0xffffffffu, !blocked);
        while (mask && nch < p.K) {
          const int l0 = __ffs(mask) - 1;
          const int pr = __shfl_sync(0xffffffffu, r, l0);
          const int pc = __shfl_sync(0xffffffffu, c, l0);
          if (lane == 0) {
            chosen[2 * nch] = pr;
            chosen[2 * nch + 1] = pc;
          }
          ++nch;
          if (lane <= l0 || cheb(r, c, pr, pc) <= sep) blocked = true;
          mask = __ballot_sync(0xffffffffu, !blocked);
        }
        __syncwarp();
      }
    }
    __syncwarp();
    int32_t* out = p.positions + (size_t)n * p.K * 2;
    GLR_DCHECK(nch >= 1 && nch <= p.K);
    for (int t = lane; t < p.K; t += 32) {
      GLR_DCHECK(t >= nch || (chosen[2 * t] >= 0 && chosen[2 * t] < p.oh &&
                              chosen[2 * t + 1] >= 0 && chosen[2 * t + 1] < p.ow));
      out[2 * t] = t < nch ? chosen[2 * t] : ar;
      out[2 * t + 1] = t < nch ? chosen[2 * t + 1] : ac;
    }
    if (lane == 0) p.padded[n] = p.K - nch;
    TK_MARK(5);
  }
}

// cut score T over hist[lo .. bins): the largest T with count(>= T) >= need,
// and cntA = count(> T); found = false if count(>= lo) < need. Warp-wide.
__device__ __forceinline__ void topk_cut(const int32_t* hist, int bins, int lo, int need,
                                         int& T, int& cntA, bool& found) {
  const int lane = threadIdx.x & 31;
  int running = 0;
  T = 0;
  cntA = 0;
  found = false;
  for (int top = bins - 1; top >= lo && !found; top -= 32) {
    const int b = top - lane;
    const int c = b >= lo ? hist[b] : 0;
    int incl = c;  // inclusive prefix from the top (lane 0 = highest bin)
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, b >= lo && running + incl >= need);
    if (hit) {
      const int l = __ffs(hit) - 1;
      T = top - l;
      cntA = running + __shfl_sync(0xffffffffu, incl - c, l);
      found = true;
    }
    running += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// The same cut found by the whole CTA: every warp sums 32-bin chunks of the
// histogram (from the top down) into csum, warp 0 scans the chunk sums for
// the chunk where the running count reaches `need` and finishes inside it
// with topk_cut -- a handful of dependent steps instead of one per 32 bins
// (C4: 4097 bins, the cut ~50-100 chunks from the top, two searches per row).
// Called by all threads; res = {T, cntA, found} in shared memory, valid after
// the closing barrier.
__device__ __forceinline__ void topk_cut_block(const int32_t* hist, int bins, int lo, int need,
                                               int* csum, int* res) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nchunks = (bins - lo + 31) / 32;
  for (int c = warp; c < nchunks; c += nw) {
    const int b = bins - 1 - 32 * c - lane;
    const int v = __reduce_add_sync(0xffffffffu, b >= lo ? hist[b] : 0);
    if (lane == 0) csum[c] = v;
  }
  __syncthreads();
  if (warp == 0) {
    int running = 0, cstar = -1;
    for (int c0 = 0; c0 < nchunks && cstar < 0; c0 += 32) {
      const int v = c0 + lane < nchunks ? csum[c0 + lane] : 0;
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, running + incl >= need);
      if (hit) {
        const int l = __ffs(hit) - 1;
        cstar = c0 + l;
        running += __shfl_sync(0xffffffffu, incl - v, l);
      } else {
        running += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    int T = 0, cntA = 0;
    bool found = false;
    if (cstar >= 0) {  // the cut lies inside chunk cstar: `need - running` more from its top
      const int top = bins - 1 - 32 * cstar;
      topk_cut(hist, top + 1, max(lo, top - 31), need - running, T, cntA, found);
      cntA += running;
    }
    if (lane == 0) {
      res[0] = T;
      res[1] = cntA;
      res[2] = found ? 1 : 0;
    }
  }
  __syncthreads();
}

// ascending bitonic sort of n int32 in shared memory (padded with INT_MAX)
__device__ __forceinline__ void bitonic_i32(int32_t* a, int n) {
  int sz = 1;
  while (sz < n) sz <<= 1;
  for (int i = n + threadIdx.x; i < sz; i += blockDim.x) a[i] = 0x7fffffff;
  __syncthreads();
  const int ept = sz / (int)blockDim.x;
  if (sz >= 64 && ept <= 8 && blockDim.x == topk::THREADS) {
    switch (ept) {
      case 0: case 1: bitonic_regs<int32_t, 1>(a, sz); break;
      case 2: bitonic_regs<int32_t, 2>(a, sz); break;
      case 4: bitonic_regs<int32_t, 4>(a, sz); break;
      default: bitonic_regs<int32_t, 8>(a, sz); break;
    }
    return;
  }
  for (int k = 2; k <= sz; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < sz; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int32_t x = a[i], y = a[ixj];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(topk::THREADS, 3) topk_kernel(TopkParams p) {
  using namespace topk;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* sA = reinterpret_cast<uint64_t*>(smem);                   // a_cap
  int32_t* sB = reinterpret_cast<int32_t*>(sA + p.a_cap);              // b_cap
  // hist after max(A + B, the first pass's ring), which aliases A and B
  int32_t* hist = reinterpret_cast<int32_t*>(
      smem + max(p.a_cap * 8 + p.b_cap * 4, topk::RING_STAGES * topk::RING_BYTES));  // bins
  int32_t* chosen = hist + p.bins;                                     // 2*K
  __shared__ int warp_tot[32];
  __shared__ int s_csum[topk::MAX_BINS / 32], s_cut[3];
  __shared__ int s_total, s_T, s_cntA, s_baseB, s_na, s_nb, s_found, s_nl, s_next, s_floor_est;
  const int BCAP = p.b_cap;

  const int n = blockIdx.x;
  const int N = p.n_dev ? min(*p.n_dev, p.n_max) : p.n_max;
  if (n >= N) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint16_t* row = p.heat + (size_t)n * p.stride;
  const int64_t M = p.M;
  const int need = (int)(M < (int64_t)p.pool ? M : (int64_t)p.pool);
#ifdef GLR_TOPK_PHASES
  long long tk_t0_ = clock64();
#endif

  // 1. histogram of the scores >= L, L = a quarter of the anchor's own score
  //    (for a heat map the row maximum: |E_u ∩ E_n| <= |E_n|), so the bulk of
  //    low scores costs no shared-memory atomics. If fewer than `need`
  //    positions reach L (or the row is not a heat map), a second pass adds
  //    the bins below L -- the cut is exact either way.
  const int64_t aidx = (int64_t)p.anchors[2 * n] * p.ow + p.anchors[2 * n + 1];
  const int L0 = min((int)row[aidx] >> 2, p.bins - 1);
  // Sampled floor: 2048 evenly spaced 16-byte chunks (16 K scores) estimate
  // the score distribution above L0; the floor L is raised to the highest
  // score the sample puts about kFloorSafety x `need` positions above, so the
  // single pass records a few thousand entries whatever the row's
  // distribution (few channels: far more positions pass a quarter of the
  // self-score). If the row has fewer than `need` positions >= L after all,
  // the exact fallback below adds the lower bins (second read).
  for (int b = L0 + tid; b < p.bins; b += THREADS) hist[b] = 0;
  if (tid == 0) {
    s_T = L0;
    s_floor_est = 0;
  }
  __syncthreads();
  {
    constexpr int SPT = 4, kFloorSafety = 4;
    const int nchk = (int)((M + VEC - 1) / VEC);
    const int ns = THREADS * SPT;
    if (nchk > 4 * ns) {
      const uint4* rv = reinterpret_cast<const uint4*>(row);
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        const int si = u * THREADS + tid;
        const int ci = (int)(((int64_t)si * nchk) / ns);
        const uint4 v = rv[ci];
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const int val = min((int)((j & 1) ? wv[j >> 1] >> 16 : wv[j >> 1] & 0xFFFFu), p.bins - 1);
          if ((int64_t)ci * VEC + j < M && val >= L0) atomicAdd(&hist[val], 1);
        }
      }
      __syncthreads();
      {
        const int64_t want = ((int64_t)kFloorSafety * need * ns * VEC + M - 1) / M;
        topk_cut_block(hist, p.bins, L0, want > 1 ? (int)want : 1, s_csum, s_cut);
        if (tid == 0) {
          if (s_cut[2]) s_T = max(s_cut[0], L0);
          // the sample's estimate of how many positions share the floor's score
          s_floor_est = (int)min((int64_t)hist[s_T] * (M / ((int64_t)ns * VEC) + 1),
                                 (int64_t)0x7fffffff);
        }
      }
      __syncthreads();
      for (int b = L0 + tid; b < p.bins; b += THREADS) hist[b] = 0;
    }
  }
  __syncthreads();
  const int L = s_T;
  // floor-level scores: recorded like the rest while they are few (the cut can
  // then be served from the list even when it lands on the floor), counted
  // only when the sample says thousands of positions share that score
  const bool count_floor = s_floor_est > 8192;
  TK_MARK(0);
  __shared__ __align__(8) uint64_t s_full[topk::RING_STAGES], s_empty[topk::RING_STAGES];
  if (tid == 0) {
    for (int r = 0; r < RING_STAGES; ++r) {
      mbar_init(&s_full[r], 1);
      mbar_init(&s_empty[r], THREADS / 32);
    }
    fence_barrier_init();
    s_na = 0;
    s_nb = 0;
    s_nl = 0;
    s_next = 0;
  }
  __syncthreads();
  uint64_t* list = p.scratch ? p.scratch + (size_t)n * p.scap : nullptr;
  auto hist_pass = [&](int lo, int hi, bool record) {  // add the scores in [lo, hi)
    constexpr int U = 4;  // 16-byte loads in flight per thread
    // SWAR pre-test, 8 scores per 16-byte chunk: scores are < 2^14, so adding
    // 0x8000 - lo to each halfword sets its top bit iff score >= lo, with no
    // carry into the neighbour (padding entries past M may carry, which only
    // adds false positives the exact path filters). Only the rare chunks
    // holding a score >= lo take the per-element path; 32-bit indices
    // (M < 2^31), and the scores are pulled out of the registers by shifts.
    const uint32_t kadd = (0x8000u - (uint32_t)lo) * 0x10001u;
    const int Mi = (int)M;
    const int nch = (Mi + VEC - 1) / VEC;
    const uint4* rv = reinterpret_cast<const uint4*>(row);
    // warp tiles of 32 x U chunks handed out dynamically (one shared atomic
    // per tile, the next grab issued one tile ahead), so the warps of a CTA
    // reach the barrier after the pass together instead of waiting on the
    // slowest of a static split
    const int ntl = (nch + 32 * U - 1) / (32 * U);
    int wt = 0;
    if (lane == 0) wt = atomicAdd(&s_next, 1);
    wt = __shfl_sync(0xffffffffu, wt, 0);
    while (wt < ntl) {
      const int c0 = wt * 32 * U;
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int ci = c0 + u * 32 + lane;
        v[u] = ci < nch ? rv[ci] : make_uint4(0, 0, 0, 0);
      }
      int wn = 0;
      if (lane == 0) wn = atomicAdd(&s_next, 1);
      wt = __shfl_sync(0xffffffffu, wn, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t any = ((v[u].x + kadd) | (v[u].y + kadd) | (v[u].z + kadd) |
                              (v[u].w + kadd)) & 0x80008000u;
        if (!any) continue;
        const int base = (c0 + u * 32 + lane) * VEC;
        const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
        int val[VEC];
        unsigned hit = 0;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          val[j] = min((int)((j & 1) ? wv[j >> 1] >> 16 : wv[j >> 1] & 0xFFFFu), p.bins - 1);
          if (base + j < Mi && val[j] >= lo && val[j] < hi) hit |= 1u << j;
        }
        if (!hit) continue;
        int off = record ? atomicAdd(&s_nl, __popc(hit)) : 0;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          if (!((hit >> j) & 1u)) continue;
          atomicAdd(&hist[val[j]], 1);
          if (record) {
            if (off < p.scap) list[off] = ((uint64_t)val[j] << 32) | (uint32_t)(base + j);
            ++off;
          }
        }
      }
    }
  };
  // First pass fed by bulk TMA copies: thread 0 keeps RING_STAGES 16 KB
  // slices of the row in flight (cp.async.bulk into a shared-memory ring that
  // aliases the A/B buffers, completion on mbarriers), every thread tests its
  // 32 bytes of a slice from shared memory and the warps release the slice on
  // an `empty` mbarrier -- the loads cost no registers and no issue slots.
  auto ring_pass = [&](int lo) {
    const uint32_t kadd = (0x8000u - (uint32_t)lo) * 0x10001u;
    const int Mi = (int)M;
    const int64_t rbytes = (int64_t)p.stride * 2;  // padded row: multiple of 16 B
    const int nst = (int)((rbytes + RING_BYTES - 1) / RING_BYTES);
    uint8_t* ring = reinterpret_cast<uint8_t*>(sA);
    auto issue = [&](int j) {
      const int sl = j % RING_STAGES;
      const uint32_t bytes = (uint32_t)min((int64_t)RING_BYTES, rbytes - (int64_t)j * RING_BYTES);
      mbar_arrive_expect_tx(&s_full[sl], bytes);
      bulk_load(ring + sl * RING_BYTES,
                reinterpret_cast<const uint8_t*>(row) + (int64_t)j * RING_BYTES, bytes,
                &s_full[sl]);
    };
    if (tid == 0)
      for (int j = 0; j < min(RING_STAGES, nst); ++j) issue(j);
    // Scores equal to the floor are only COUNTED (in a register, one shared
    // atomic per warp at the end): on few-channel images tens of thousands of
    // positions share the floor's score, and taking each through the shared
    // histogram atomic, the list slot reservation and an 8-byte global store
    // was most of the kernel (C3: ~207 K of 255 K entries per row). The list
    // then holds the scores ABOVE the floor; if the cut lands on the floor
    // itself, the ties are collected in index order with early exit below.
    int floor_cnt = 0;
    for (int i = 0; i < nst; ++i) {
      const int sl = i % RING_STAGES;
      mbar_wait(&s_full[sl], (uint32_t)(i / RING_STAGES) & 1u);
      const uint4* sv4 = reinterpret_cast<const uint4*>(ring + sl * RING_BYTES);
#pragma unroll
      for (int u = 0; u < RING_BYTES / 16 / THREADS; ++u) {
        const int cl = u * THREADS + tid;
        const uint4 v = sv4[cl];
        const uint32_t any =
            ((v.x + kadd) | (v.y + kadd) | (v.z + kadd) | (v.w + kadd)) & 0x80008000u;
        if (!any) continue;
        const int base = (i * (RING_BYTES / 16) + cl) * VEC;
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
        int val[VEC];
        unsigned hit = 0;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          val[j] = min((int)((j & 1) ? wv[j >> 1] >> 16 : wv[j >> 1] & 0xFFFFu), p.bins - 1);
          const bool in = base + j < Mi;
          if (in && val[j] >= lo + (count_floor ? 1 : 0)) hit |= 1u << j;
          floor_cnt += count_floor && in && val[j] == lo;
        }
        if (!hit) continue;
        int off = atomicAdd(&s_nl, __popc(hit));
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          if (!((hit >> j) & 1u)) continue;
          atomicAdd(&hist[val[j]], 1);
          if (off < p.scap) list[off] = ((uint64_t)val[j] << 32) | (uint32_t)(base + j);
          ++off;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sl]);
      if (tid == 0 && i + RING_STAGES < nst) {  // refill this slot once every warp let go
        mbar_wait(&s_empty[sl], (uint32_t)(i / RING_STAGES) & 1u);
        issue(i + RING_STAGES);
      }
    }
    __syncwarp();
    floor_cnt = __reduce_add_sync(0xffffffffu, floor_cnt);
    if (lane == 0 && floor_cnt) atomicAdd(&hist[lo], floor_cnt);
  };
  if (list) {
    ring_pass(L);  // bulk-TMA-fed first pass (records the list)
  } else {
    hist_pass(L, p.bins, false);
  }
  __syncthreads();

  TK_MARK(1);
  // 2. cut score T: walk bins from the top down to `lo`, 32 at a time
  auto cut_search = [&](int lo) {  // block-wide
    topk_cut_block(hist, p.bins, lo, need, s_csum, s_cut);
    if (tid == 0) {
      s_T = s_cut[0];
      s_cntA = s_cut[1];
      s_found = s_cut[2];
    }
    __syncthreads();
  };
  cut_search(L);
#ifdef GLR_TOPK_STATS
  if (tid == 0) {
    atomicAdd(&g_topk_stats[0], 1u);
    if (!s_found) atomicAdd(&g_topk_stats[1], 1u);
    unsigned above = 0;
    for (int b = L; b < p.bins; ++b) above += hist[b];
    atomicAdd(&g_topk_stats[2], above);
    atomicMax(&g_topk_stats[3], above);
  }
#endif
  const bool first_pass_cut = s_found;
  if (!s_found) {
    // The bins below L. Score 0 is not histogrammed: on sparse edge maps most
    // of a row is zero (C3's phantom: ~200 K of 255 K positions, one shared
    // bin = serialised atomics); its count is M minus everything else.
    for (int b = tid; b < L; b += THREADS) hist[b] = 0;
    __syncthreads();
    if (tid == 0) {
      s_next = 0;
      s_total = 0;
    }
    __syncthreads();
    if (L > 1) hist_pass(1, L, false);
    __syncthreads();
    int part = 0;
    for (int b = 1 + tid; b < p.bins; b += THREADS) part += hist[b];
    part = __reduce_add_sync(0xffffffffu, part);
    if (lane == 0 && part) atomicAdd(&s_total, part);
    __syncthreads();
    if (tid == 0) hist[0] = (int)(M - (int64_t)s_total);
    __syncthreads();
    cut_search(0);
  }
  const int T = s_T, cntA = s_cntA, capB = need - cntA;
  TK_MARK(2);

  // 3. collect A = {score > T} (cntA < need entries) and the ties {score == T};
  //    unordered warp-aggregated appends when the ties fit the buffer (they are
  //    then sorted by index), else an ordered block-scan compaction.
  const bool list_ok = list && first_pass_cut && s_nl <= p.scap;
  bool ties_done = false;  // false: the split path at the end collects the ties (and A if needed)
  bool a_done = false;
  if (list_ok && T == L && count_floor) {
    // the cut is the floor: the list holds exactly A = {score > T}; the ties
    // come from the ordered prefix scan below
    const int c = s_nl;
    for (int i = tid; i < c; i += THREADS) {
      const uint64_t e = list[i];
      const int ia = atomicAdd(&s_na, 1);
      GLR_DCHECK(ia < p.a_cap && (int)(e >> 32) > T);
      sA[ia] = ((uint64_t)(65535 - (int)(e >> 32)) << 32) | (uint32_t)e;
    }
    a_done = true;
  } else if (list_ok && hist[T] <= BCAP) {
    ties_done = a_done = true;
    // the recorded list holds every score >= T (the floor's level too unless
    // it was only counted, and then T > L): no second row read
    const int c = s_nl;
    for (int i = tid; i < c; i += THREADS) {
      const uint64_t e = list[i];
      const int sc = (int)(e >> 32);
      const uint32_t pos = (uint32_t)e;
      if (sc > T)
        sA[atomicAdd(&s_na, 1)] = ((uint64_t)(65535 - sc) << 32) | pos;
      else if (sc == T)
        sB[atomicAdd(&s_nb, 1)] = (int32_t)pos;
    }
    __syncthreads();
    if (!p.stageA) bitonic_i32(sB, s_nb);
  } else if (hist[T] <= BCAP) {
    ties_done = a_done = true;
    constexpr int U = 4;  // 16-byte loads in flight per thread
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t tile = 0; tile < M; tile += (int64_t)THREADS * VEC * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t base = tile + ((int64_t)u * THREADS + tid) * VEC;
        v[u] = base < M ? *reinterpret_cast<const uint4*>(row + base) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t base = tile + ((int64_t)u * THREADS + tid) * VEC;
        const uint16_t* sv = reinterpret_cast<const uint16_t*>(&v[u]);
        // warp-uniform skip of chunks holding no candidate (the common case)
        bool any = false;
#pragma unroll
        for (int j = 0; j < VEC; ++j) any |= base + j < M && sv[j] >= T;
        if (!__any_sync(0xffffffffu, any)) continue;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const bool ok = base + j < M;
          const bool isA = ok && sv[j] > T, isB = ok && sv[j] == T;
          const unsigned mA = __ballot_sync(0xffffffffu, isA);
          const unsigned mB = __ballot_sync(0xffffffffu, isB);
          if (mA) {
            int off = 0;
            if (lane == __ffs(mA) - 1) off = atomicAdd(&s_na, __popc(mA));
            off = __shfl_sync(0xffffffffu, off, __ffs(mA) - 1);
            if (isA)
              sA[off + __popc(mA & lt)] =
                  ((uint64_t)(65535 - sv[j]) << 32) | (uint32_t)(base + j);
          }
          if (mB) {
            int off = 0;
            if (lane == __ffs(mB) - 1) off = atomicAdd(&s_nb, __popc(mB));
            off = __shfl_sync(0xffffffffu, off, __ffs(mB) - 1);
            if (isB) sB[off + __popc(mB & lt)] = (int32_t)(base + j);
          }
        }
      }
    }
    __syncthreads();
    // ties in index order
    if (!p.stageA) bitonic_i32(sB, s_nb);
  }
  if (!ties_done) {
    // The cut is the floor, or more ties than the buffer holds (few channels: tens of thousands of
    // positions share the cut score). Only the ties need index order, and
    // only the first capB of them: (a) A = {score > T} is collected unordered
    // (it is sorted below anyway) in one streaming pass with the SWAR pre-test
    // -- A is rare, so almost every 16-byte chunk is skipped; (b) the ties by
    // an ordered block-scan compaction that stops as soon as capB are found,
    // typically within the first tiles. (One ordered compaction of both used
    // to walk the whole row with two block barriers per 4096 scores: ~125 us
    // per C3 row.)
    __syncthreads();
    if (tid == 0) {
      s_baseB = 0;
      s_next = 0;
      if (!a_done) s_na = 0;
    }
    __syncthreads();
    if (cntA > 0 && !a_done) {
      constexpr int U = 4;
      const uint32_t kadd = (0x8000u - (uint32_t)(T + 1)) * 0x10001u;
      const int Mi = (int)M;
      const int nch = (Mi + VEC - 1) / VEC;
      const uint4* rv = reinterpret_cast<const uint4*>(row);
      const int ntl = (nch + 32 * U - 1) / (32 * U);
      int wt = 0;
      if (lane == 0) wt = atomicAdd(&s_next, 1);
      wt = __shfl_sync(0xffffffffu, wt, 0);
      while (wt < ntl) {
        const int c0 = wt * 32 * U;
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ci = c0 + u * 32 + lane;
          v[u] = ci < nch ? rv[ci] : make_uint4(0, 0, 0, 0);
        }
        int wn = 0;
        if (lane == 0) wn = atomicAdd(&s_next, 1);
        wt = __shfl_sync(0xffffffffu, wn, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t any = ((v[u].x + kadd) | (v[u].y + kadd) | (v[u].z + kadd) |
                                (v[u].w + kadd)) & 0x80008000u;
          if (!any) continue;
          const int base = (c0 + u * 32 + lane) * VEC;
          const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (int j = 0; j < VEC; ++j) {
            const int val = (int)((j & 1) ? wv[j >> 1] >> 16 : wv[j >> 1] & 0xFFFFu);
            if (base + j < Mi && val > T) {
              const int ia = atomicAdd(&s_na, 1);
              GLR_DCHECK(ia < p.a_cap && ia < cntA);
              sA[ia] = ((uint64_t)(65535 - val) << 32) | (uint32_t)(base + j);
            }
          }
        }
      }
    }
    for (int64_t tile = 0; tile < M; tile += (int64_t)THREADS * VEC) {
      if (s_baseB >= capB) break;  // block-uniform
      const int64_t base = tile + (int64_t)tid * VEC;
      uint16_t sc[VEC];
      int b = 0;
      if (base < M) {
        const uint4 v = *reinterpret_cast<const uint4*>(row + base);
        const uint16_t* sv = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          sc[j] = (base + j < M) ? sv[j] : 0xFFFF;
          b += sc[j] == T;
        }
      }
      int ib = s_baseB + block_excl_scan_1024(b, warp_tot, &s_total);
      if (b) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          if (sc[j] == T) {
            GLR_DCHECK(capB <= BCAP);
            if (ib < capB) sB[ib] = (int32_t)(base + j);
            ++ib;
          }
        }
      }
      __syncthreads();
      if (tid == 0) s_baseB += s_total;
      __syncthreads();
    }
  }

  if (p.stageA) {
    // hand A and the ties over to topk_select_kernel (ordered-compaction
    // path: the first capB ties in index order; otherwise all, unsorted)
    const int nb = ties_done ? s_nb : min(s_baseB, capB);
    uint64_t* ga = p.stageA + (size_t)n * p.a_cap;
    int32_t* gb = p.stageB + (size_t)n * BCAP;
    for (int i = tid; i < cntA; i += THREADS) ga[i] = sA[i];
    for (int i = tid; i < nb; i += THREADS) gb[i] = sB[i];
    if (tid == 0) {
      p.stageN[2 * n] = cntA;
      p.stageN[2 * n + 1] = nb;
    }
    return;
  }
  __syncthreads();
  TK_MARK(3);
  topk_finish(p, n, M, need, cntA, sA, sB, chosen);
}

// Second half of the split top-K: per exemplar, the staged A and ties ->
// ties sorted by index, A by (score desc, index asc), the greedy walk.
__global__ void __launch_bounds__(topk::THREADS, 3) topk_select_kernel(TopkParams p) {
  using namespace topk;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* sA = reinterpret_cast<uint64_t*>(smem);       // a_cap
  int32_t* sB = reinterpret_cast<int32_t*>(sA + p.a_cap);  // b_cap
  int32_t* chosen = sB + p.b_cap;                          // 2*K
  const int n = blockIdx.x;
  const int N = p.n_dev ? min(*p.n_dev, p.n_max) : p.n_max;
  if (n >= N) return;
  const int tid = threadIdx.x;
  const int64_t M = p.M;
  const int need = (int)(M < (int64_t)p.pool ? M : (int64_t)p.pool);
  const int cntA = p.stageN[2 * n], nb = p.stageN[2 * n + 1];
  const uint64_t* ga = p.stageA + (size_t)n * p.a_cap;
  const int32_t* gb = p.stageB + (size_t)n * p.b_cap;
  for (int i = tid; i < cntA; i += THREADS) sA[i] = ga[i];
  for (int i = tid; i < nb; i += THREADS) sB[i] = gb[i];
  __syncthreads();
  bitonic_i32(sB, nb);
  topk_finish(p, n, M, need, cntA, sA, sB, chosen);
}

// Top-K over the candidate lists the heat-map GEMM appends in its epilogue
// (heat_gemm.cu, `glr_heat_topk`): every position whose score reaches
// L_n = |E_n| / 4 (a quarter of the exemplar's self-score, the row maximum),
// as (score << 32) | position in arbitrary order. The cut T, A = {> T} and
// the ties are then exactly those of the full row whenever count(>= L_n) >=
// need; otherwise (or on list overflow, or > BCAP ties) the exemplar is
// flagged for the full-row path and its positions are left untouched.
struct TopkCandParams {
  TopkParams base;  // heat / n_dev unused
  const uint64_t* cand;
  const uint32_t* cnt;
  const uint16_t* thr;
  int cap;
  uint8_t* fallback;
  int b_cap;  // tie buffer of the list path: 16384 (ties at the cut are common on few channels)
};

__global__ void __launch_bounds__(topk::THREADS, 3) topk_cand_kernel(TopkCandParams q) {
  using namespace topk;
  const TopkParams& p = q.base;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* sA = reinterpret_cast<uint64_t*>(smem);  // a_cap
  int32_t* sB = reinterpret_cast<int32_t*>(sA + p.a_cap);  // q.b_cap
  int32_t* hist = sB + q.b_cap;                              // bins
  int32_t* chosen = hist + p.bins;                           // 2*K
  int32_t* bkt = chosen + 2 * p.K;                           // kSelB (tie selection)
  int32_t* kept = bkt + kSelB;                               // kSelB
  __shared__ int s_T, s_cntA, s_na, s_nb, s_found;
  const int n = blockIdx.x;
  if (n >= p.n_max) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t M = p.M;
  const int need = (int)(M < (int64_t)p.pool ? M : (int64_t)p.pool);
  const int c = (int)q.cnt[n];
  const int L = min((int)q.thr[n], p.bins - 1);
#ifdef GLR_TOPK_STATS
  if (tid == 0) {
    atomicAdd(&g_cand_stats[0], 1u);
    if (c > q.cap) atomicAdd(&g_cand_stats[1], 1u);
    if (c < need) atomicAdd(&g_cand_stats[2], 1u);
    atomicAdd(&g_cand_stats[4], (unsigned)c);
    atomicMax(&g_cand_stats[5], (unsigned)c);
  }
#endif
  if (c > q.cap || c < need) {  // block-uniform
    if (tid == 0) q.fallback[n] = 1;
    return;
  }
  for (int b = L + tid; b < p.bins; b += THREADS) hist[b] = 0;
  if (tid == 0) {
    s_na = 0;
    s_nb = 0;
  }
  __syncthreads();
  const uint64_t* list = q.cand + (size_t)n * q.cap;
  for (int i = tid; i < c; i += THREADS)
    atomicAdd(&hist[min((int)(list[i] >> 32), p.bins - 1)], 1);
  __syncthreads();
  __shared__ int s_csum[topk::MAX_BINS / 32], s_cut[3];
  topk_cut_block(hist, p.bins, L, need, s_csum, s_cut);
  if (tid == 0) {
    s_T = s_cut[0];
    s_cntA = s_cut[1];
    s_found = s_cut[2];
  }
  __syncthreads();
  const int T = s_T, cntA = s_cntA;
#ifdef GLR_TOPK_STATS
  if (tid == 0 && s_found && hist[T] > q.b_cap) atomicAdd(&g_cand_stats[3], 1u);
#endif
  if (!s_found || hist[T] > q.b_cap) {  // block-uniform
    if (tid == 0) q.fallback[n] = 1;
    return;
  }
  if (tid == 0) q.fallback[n] = 0;
  for (int i = tid; i < c; i += THREADS) {
    const uint64_t e = list[i];
    const int sc = (int)(e >> 32);
    const uint32_t pos = (uint32_t)e;
    if (sc > T)
      sA[atomicAdd(&s_na, 1)] = ((uint64_t)(65535 - sc) << 32) | pos;
    else if (sc == T)
      sB[atomicAdd(&s_nb, 1)] = (int32_t)pos;
  }
  __syncthreads();
  // Only the first capB = need - cntA ties in index order are used. With
  // few channels thousands of positions tie at the cut; instead of sorting
  // them all, a radix select on the high index bits keeps the buckets below
  // the one holding the capB-th smallest index plus that bucket, and only
  // those (<= kSelB) are sorted.
  const int capB = need - cntA;
  int nb = s_nb;
  int32_t* ties = sB;
  if (nb > kSelB && capB < kSelB) {
    int shift = 0;
    while (((M - 1) >> shift) >= kSelB) ++shift;
    for (int b = tid; b < kSelB; b += THREADS) bkt[b] = 0;
    __syncthreads();
    for (int i = tid; i < nb; i += THREADS) atomicAdd(&bkt[sB[i] >> shift], 1);
    __syncthreads();
    __shared__ int s_cut, s_kept;
    if (warp == 0) {  // first bucket where the running count reaches capB
      const int lane = tid & 31;
      int running = 0;
      for (int b0 = 0; b0 < kSelB; b0 += 32) {
        const int c = bkt[b0 + lane];
        int incl = c;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, running + incl >= capB);
        if (hit) {
          if (lane == 0) s_cut = b0 + __ffs(hit) - 1;
          break;
        }
        running += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) s_kept = 0;
    }
    __syncthreads();
    const int cut = s_cut;
    for (int i = tid; i < nb; i += THREADS) {
      const int v = sB[i];
      if ((v >> shift) <= cut) {
        const int k = atomicAdd(&s_kept, 1);
        if (k < kSelB) kept[k] = v;
      }
    }
    __syncthreads();
    if (s_kept <= kSelB) {  // block-uniform; else keep the full sort below
      nb = s_kept;
      ties = kept;
    }
  }
  bitonic_i32(ties, nb);
  topk_finish(p, n, M, need, cntA, sA, ties, chosen);
}

// gather_group (patches.py:43-54): groups[g][j][i], i = (dr*P + dc)*C + ch
__global__ void gather_kernel(const double* __restrict__ x, int H, int W, int C, int P,
                              const int32_t* __restrict__ pos, int G, int K,
                              double* __restrict__ groups) {
  const int m = P * P * C;
  const int64_t total = (int64_t)G * K * m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i / m;
    const int e = (int)(i - col * m);
    const int r = pos[2 * col] + e / (P * C);
    const int c = pos[2 * col + 1] + (e / C) % P;
    groups[i] = x[((int64_t)r * W + c) * C + (e % C)];
  }
}

static int topk_pool(int K, int sep) { return K * (2 * sep + 1) * (2 * sep + 1) + 1; }

static int pow2_at_least(int v) {
  int c = 1;
  while (c < v) c <<= 1;
  return c;
}

static size_t topk_smem(int pool, int bins, int K) {
  // sA | sB | hist | chosen; the first pass's bulk-copy ring aliases sA/sB
  const size_t ab =
      (size_t)pow2_at_least(pool) * 8 + (size_t)pow2_at_least(std::max(pool, 4096)) * 4;
  return std::max(ab, (size_t)topk::RING_STAGES * topk::RING_BYTES) + (size_t)bins * 4 +
         (size_t)K * 8 + 16;
}

}  // namespace glr

using namespace glr;

// optional: n_max x kTopkScratch (score, position) records (single row pass)
constexpr int kTopkScratch = 32768;
static void topk_caps(int K, int sep, int& a_cap, int& b_cap) {
  const int pool = topk_pool(K, sep);
  a_cap = pow2_at_least(pool);
  b_cap = pow2_at_least(std::max(pool, 4096));
}

extern "C" size_t glr_topk_workspace(int n_max, int K, int sep) {
  // scratch lists, then the split's staging (A keys, ties, two counts)
  int a_cap, b_cap;
  topk_caps(K, sep, a_cap, b_cap);
  const size_t nm = (size_t)std::max(n_max, 0);
  return nm * kTopkScratch * sizeof(uint64_t) +
         nm * ((size_t)a_cap * 8 + (size_t)b_cap * 4 + 8) + 1024;
}

#ifdef GLR_TOPK_STATS
extern "C" int glr_debug_topk_stats(unsigned int* out) {
  cudaMemcpyFromSymbol(out, g_topk_stats, sizeof(unsigned int) * 4);
  cudaMemcpyFromSymbol(out + 4, g_cand_stats, sizeof(unsigned int) * 6);
  return 0;
}
#endif

static int topk_params(int n_max, int oh, int ow, int max_score, const int32_t* anchors_d,
                       int K, int sep, int32_t* positions_d, int32_t* padded_d, TopkParams& p,
                       size_t& smem) {
  GLR_REQUIRE(K >= 1, GLR_ERR_INVALID, "group_size must be >= 1");
  GLR_REQUIRE(sep >= 0, GLR_ERR_INVALID, "min_separation must be >= 0");
  GLR_REQUIRE(oh >= 1 && ow >= 1, GLR_ERR_INVALID, "topk: empty slice");
  GLR_REQUIRE(max_score >= 0 && max_score < topk::MAX_BINS, GLR_ERR_UNSUPPORTED,
              "topk: max score %d above %d", max_score, topk::MAX_BINS - 1);
  const int64_t M = (int64_t)oh * ow;
  const int pool = (int)std::min<int64_t>(topk_pool(K, sep), M);
  const int bins = max_score + 1;
  smem = topk_smem(pool, bins, K);
  GLR_REQUIRE(smem <= 200 * 1024, GLR_ERR_UNSUPPORTED,
              "topk: K=%d sep=%d needs %zu bytes of shared memory", K, sep, smem);
  p.heat = nullptr;
  p.stride = cdiv(M, 8) * 8;
  p.n_max = n_max;
  p.n_dev = nullptr;
  p.oh = oh;
  p.ow = ow;
  p.M = M;
  p.bins = bins;
  p.anchors = anchors_d;
  p.K = K;
  p.sep = sep;
  p.pool = pool;
  p.a_cap = pow2_at_least(pool);
  p.b_cap = pow2_at_least(std::max(pool, 4096));
  p.positions = positions_d;
  p.padded = padded_d;
  p.scratch = nullptr;
  p.scap = 0;
  p.stageA = nullptr;
  p.stageB = nullptr;
  p.stageN = nullptr;
  return GLR_OK;
}

extern "C" int glr_topk(const uint16_t* heat_d, int n_max, const int32_t* n_dev_d, int oh, int ow,
                        int max_score, const int32_t* anchors_d, int K, int sep,
                        int32_t* positions_d, int32_t* padded_d, void* ws_d, size_t ws_bytes,
                        void* stream) {
  TopkParams p;
  size_t smem = 0;
  const int st = topk_params(n_max, oh, ow, max_score, anchors_d, K, sep, positions_d,
                             padded_d, p, smem);
  if (st != GLR_OK) return st;
  if (n_max <= 0) return GLR_OK;
  p.heat = heat_d;
  p.n_dev = n_dev_d;
  if (ws_d && ws_bytes >= glr_topk_workspace(n_max, K, sep)) {
    p.scratch = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(ws_d) + 255) & ~uintptr_t(255));
    p.scap = kTopkScratch;
#ifdef GLR_TOPK_SPLIT  // dev A/B, off: measured 2.44 vs 2.36 ms per C2 refresh (the row
                       // stream, not the per-CTA tail, bounds the kernel)
    int a_cap, b_cap;
    topk_caps(K, sep, a_cap, b_cap);
    uint8_t* st = reinterpret_cast<uint8_t*>(p.scratch + (size_t)n_max * kTopkScratch);
    p.stageA = reinterpret_cast<uint64_t*>(st);
    p.stageB = reinterpret_cast<int32_t*>(st + (size_t)n_max * a_cap * 8);
    p.stageN = reinterpret_cast<int32_t*>(st + (size_t)n_max * (a_cap * 8 + (size_t)b_cap * 4));
#endif
  }
  { const int s_ = ensure_smem_attr((const void*)topk_kernel, (int)smem); if (s_) return s_; }
  topk_kernel<<<n_max, topk::THREADS, smem, (cudaStream_t)stream>>>(p);
  if (p.stageA) {
    GLR_CUDA(cudaGetLastError());
    const size_t ssmem = (size_t)p.a_cap * 8 + (size_t)p.b_cap * 4 + (size_t)K * 8 + 16;
    { const int s_ = ensure_smem_attr((const void*)topk_select_kernel, (int)ssmem); if (s_) return s_; }
    topk_select_kernel<<<n_max, topk::THREADS, ssmem, (cudaStream_t)stream>>>(p);
  }
  return check_launch("topk_kernel");
}

namespace glr {
int topk_cand_launch(const uint64_t* cand_d, const uint32_t* cnt_d, const uint16_t* thr_d,
                     int cap, int n_max, int oh, int ow, int max_score,
                     const int32_t* anchors_d, int K, int sep, int32_t* positions_d,
                     int32_t* padded_d, uint8_t* fallback_d, void* stream) {
  TopkCandParams q;
  size_t smem = 0;
  const int st = topk_params(n_max, oh, ow, max_score, anchors_d, K, sep, positions_d,
                             padded_d, q.base, smem);
  if (st != GLR_OK) return st;
  if (n_max <= 0) return GLR_OK;
  q.cand = cand_d;
  q.cnt = cnt_d;
  q.thr = thr_d;
  q.cap = cap;
  q.fallback = fallback_d;
  // tie buffer: 16384 where thousands of positions tie at the cut (few
  // channels: a short score range), 4096 otherwise so that three CTAs share
  // an SM (C2: 121 KB -> 73 KB per CTA; the selection is latency-bound --
  // sorts, barriers, a single-warp walk -- and one resident CTA left the SM
  // idle most of the time); more ties than that go to the dense path
  q.b_cap = q.base.bins <= 2048 ? 16384 : 4096;
  // the list path has no bulk-copy ring: sA | sB (ties) | hist | chosen
  smem = (size_t)q.base.a_cap * 8 + (size_t)q.b_cap * 4 + (size_t)q.base.bins * 4 +
         (size_t)K * 8 + 2 * topk::kSelB * 4 + 16;
  GLR_REQUIRE(smem <= 200 * 1024, GLR_ERR_UNSUPPORTED, "topk_cand: %zu bytes of shared memory",
              smem);
  { const int s_ = ensure_smem_attr((const void*)topk_cand_kernel, (int)smem); if (s_) return s_; }
  topk_cand_kernel<<<n_max, topk::THREADS, smem, (cudaStream_t)stream>>>(q);
  return check_launch("topk_cand_kernel");
}
}  // namespace glr

extern "C" int glr_gather(const double* x_d, int H, int W, int C, int P, const int32_t* positions_d,
                          int G, int K, double* groups_d, void* stream) {
  GLR_REQUIRE(P >= 1 && P <= H && P <= W, GLR_ERR_INVALID, "gather: bad patch size");
  int64_t total = (int64_t)G * K * P * P * C;
  if (total == 0) return GLR_OK;
  int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 32);
  gather_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(x_d, H, W, C, P, positions_d, G, K,
                                                         groups_d);
  return check_launch("gather_kernel");
}
