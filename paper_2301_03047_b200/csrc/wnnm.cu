// (4) Batched WNNM and (5) deterministic aggregation.
//
// Reference: glr/lowrank.py:46-65 (wnnm_prox: thin SVD, sigma_hat =
// sqrt(max(s^2 - K sigma^2, 0)), w = c sqrt(K) sigma^2 / (sigma_hat + eps),
// U diag(max(s - w, 0)) V^T) and :68-87 (glr_regularize: shrink every group,
// scatter_group, divide by the count), glr/patches.py:57-70 (scatter_group).
//
// B200 formulation, fp64 throughout, three kernels per batch of groups so each
// runs at the occupancy its bottleneck wants:
//   gram_kernel   G = M^T M (K x K, K padded to 64), the group read straight
//                 from the image at its K positions with cp.async tiles
//                 (never materialised); upper-triangle blocks only.
//   eig_kernel    parallel cyclic Jacobi on G (32 disjoint rotations per
//                 round), optionally warm-started from the group's cached
//                 eigenvectors Vp (G <- Vp^T G Vp); s = sqrt(lambda), the WNNM
//                 shrinkage f, and Wm = V diag(f(s)/s) V^T (written in place).
//   apply_kernel  out = M Wm, since M V = U S makes M V diag(f(s)/s) V^T =
//                 U diag(f(s)) V^T; the denoised patches are scatter-added
//                 into an int64 fixed-point numerator with integer atomics
//                 (exact, order-independent: bitwise deterministic for any
//                 exemplar sharding), or written out for the explicit-group API.
#include "common.cuh"
#include "internal.cuh"

namespace glr {

namespace wn {
constexpr int KMAX = 64;
constexpr int LD = KMAX + 4;      // row stride of Wm in the apply kernel (== 4 mod 16)
constexpr int GLD = KMAX + 1;     // row stride of G in the eigen kernel (odd, see eig_mm64)
constexpr int VLD = KMAX + 1;     // row stride of V^T in the eigen kernel
constexpr int GROWS = 32;         // rows of M per Gram tile
constexpr int GRS = GROWS + 4;    // column stride of the Gram tiles (== 4 mod 16)
constexpr int GRAM_THREADS = 128; // four warps, 9 of the 36 upper-triangle 8x8 tiles each
constexpr int EIG_THREADS = 256;
constexpr int APPLY_THREADS = 256;
#ifdef GLR_EIG_MAXSWEEPS  // dev experiments only
constexpr int MAX_SWEEPS = GLR_EIG_MAXSWEEPS;
#else
constexpr int MAX_SWEEPS = 24;
#endif
constexpr int GSZ = KMAX * KMAX;  // doubles per group in the G / Wm / V buffers
// Jacobi rotation threshold: skip (p,q) once |g_pq| <= kRotTol sqrt(|g_pp g_qq|).
// With quadratic convergence the last sweep above this level leaves the
// off-diagonal far below it; measured: 1e-10 keeps WNNM within 1e-9 of
// LAPACK gesdd and every parity test bit-identical on positions, and saves
// a sweep in ~40 % of C2's iterations against 1e-12 (415.6 -> 403.0 ms per
// solve; 1e-9 would save another 7 ms at a wider edge-threshold margin).
#ifndef GLR_EIG_ROTTOL
#define GLR_EIG_ROTTOL 1e-10
#endif
constexpr double kRotTol = GLR_EIG_ROTTOL;
// First-order finish: the sweeps may stop once every pair between two kept
// components (both in the smooth part of the shrinkage, away from its kink)
// is below kFinishTol sqrt(|g_pp g_qq|); the residue E is then folded into
// Wm to first order (Daleckii-Krein: f(L + E) = f(L) + E o D + O(|E|^2 f''),
// D the divided differences of f(s)/s), which leaves a second-order error
// ~kFinishTol^2 relative (numpy model of the scheme: 6e-11 at 6e-5, 9e-9 at
// 5.5e-4 max relative residue; the strict 1e-10 test alone leaves ~1e-11).
// 3e-5 leaves ~1.5e-11, the level of the strict path; measured on C2: 1e-5
// 294.1, 3e-5 288.9, 1e-4 281.9 ms per solve, every parity test (bitwise
// refresh traces included) green at all three. 1e-4 (~2e-10) is not taken:
// at C2's size an error of 1e-10 in x already gives a ~2 % chance per refresh
// that one of the ~1e8 edge-threshold comparisons flips against the reference.
#ifndef GLR_EIG_FINISHTOL
#define GLR_EIG_FINISHTOL 3e-5
#endif
constexpr double kFinishTol = GLR_EIG_FINISHTOL;
// Zero-shrinkage exemption, gap rule: a pair of exempt indices (j, k) is
// left alone only while |g_jk| <= kZGapTol (KD - max(g_jj, g_kk)), KD the
// smallest diagonal entry of a kept index. The couplings inside the exempt
// block feed back into the kept-exempt entries at the rate |g_jk| / gap per
// sweep (rotating (i, k) refills g_ij with -sin(theta_ik) g_kj), so where the
// kept and the exempt eigenvalues are close (C4's late iterations: 38 of 64
// components kept, a continuous spectrum across the threshold) an
// undiagonalised exempt block turned the quadratic convergence into a slow
// linear one (8-9 sweeps from a warm start, measured); where the gap is wide
// (C3: one dominant component) every exempt pair is still skipped.
#ifndef GLR_EIG_ZGAPTOL
#define GLR_EIG_ZGAPTOL 1e-3
#endif
constexpr double kZGapTol = GLR_EIG_ZGAPTOL;
}  // namespace wn

// Element (r, j) of group g lives at src[cbase(g, j) + roff(r)]: for image
// groups roff(r) = (r / PC) * W*C + r % PC (patch row dr, then the contiguous
// (dc, ch) run of P*C values) and cbase = (row_j * W + col_j) * C; for
// explicit (G, K, m) groups roff(r) = r and cbase = (g*K + j) * m.
struct GroupSrc {
  const double* src;
  const int32_t* pos;  // image groups: (n, K, 2) top-left positions
  int W, C, PC;
  int H;               // image groups: image rows (bounds checks of the checked build)
  int64_t rs;
  int m, K;
  // rows 2q, 2q+1 of every column are 16 contiguous, 16-byte aligned bytes
  // (image groups: even C; explicit groups: even m): the tile fills then
  // move two rows per cp.async
  int vec2;
};

template <bool IMG>
__device__ __forceinline__ long long col_base(const GroupSrc& s, int g, int j) {
  if constexpr (IMG) {
    const int32_t* q = s.pos + ((size_t)g * s.K + j) * 2;
    GLR_DCHECK(q[0] >= 0 && q[1] >= 0 && q[0] + s.m / s.PC <= s.H && q[1] + s.PC / s.C <= s.W);
    return ((long long)q[0] * s.W + q[1]) * s.C;
  } else {
    return ((long long)g * s.K + j) * s.m;
  }
}

// Asynchronous coalesced fill of a column-major tile Tt[j * RS + rr] (rows
// r0 .. r0+R-1): warp w takes columns w, w+nwarps, ...; lanes run down
// consecutive rows (contiguous in the image within one patch row).
template <int NWARPS>
__device__ __forceinline__ void fill_tile(double* Tt, const GroupSrc& s, const long long* cbase,
                                          int r0, int R, int RS) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (s.vec2 && R == 32) {
    // 16 lanes x 2 rows down the tile, the two half-warps on alternating
    // columns: half the cp.async instructions and shared-memory wavefronts of
    // the 8-byte fill (ncu: the fill was a third of the Gram kernel's stall
    // samples beside an 80 % busy DMMA pipe)
    const int rr = 2 * (lane & 15), r = r0 + rr;
    const bool rok = r < s.m;  // m even: the pair is in or out together
    const int64_t off = rok ? (int64_t)(r / s.PC) * s.rs + (r % s.PC) : 0;
#pragma unroll 4
    for (int j = 2 * warp + (lane >> 4); j < wn::KMAX; j += 2 * NWARPS) {
      if (rok && j < s.K) {
        cp_async16(&Tt[j * RS + rr], s.src + cbase[j] + off);
      } else {
        Tt[j * RS + rr] = 0.0;
        Tt[j * RS + rr + 1] = 0.0;
      }
    }
    cp_async_commit();
    return;
  }
  for (int rr = lane; rr < R; rr += 32) {
    const int r = r0 + rr;
    const bool rok = r < s.m;
    const int64_t off = rok ? (int64_t)(r / s.PC) * s.rs + (r % s.PC) : 0;
#pragma unroll 4
    for (int j = warp; j < wn::KMAX; j += NWARPS) {
      if (rok && j < s.K)
        cp_async8(&Tt[j * RS + rr], s.src + cbase[j] + off);
      else
        Tt[j * RS + rr] = 0.0;
    }
  }
  cp_async_commit();
}

// ---------------------------------------------------------------------------
// fp64 tensor-core MMA (DMMA, mma.sync m8n8k4): D(8x8) += A(8x4) B(4x8).
// Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// d = {D[lane/4][2(lane%4)], D[lane/4][2(lane%4)+1]}. Each warp reuses its A
// and B fragments across a block of 8x8 tiles, so shared-memory traffic per
// FMA is ~10x lower than a scalar 4x4 register block (which was bound by the
// 128 B/clk shared pipe at half the FP64 rate).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// K1: Gram G = M^T M on DMMA (column-major 32-row tiles, column stride
// GRS = 36 == 4 mod 16 doubles: fragment loads hit 2 wavefronts). Four
// warps; warp w owns tile rows w and 7-w of the upper triangle (8-w + w+1 =
// 9 of the 36 8x8 tiles each: 36 DMMAs per k-step for the CTA, the same 9 on
// every warp's critical path; measured 1.36 -> ~1.0 ms on C2 against three
// warps on 32x32 super-blocks). The A fragment of tile row i equals the B
// fragment of tile column i (G = M^T M), so a warp loads only the column
// fragments w..7 each k-step.
template <int W>
__device__ __forceinline__ void gram_tile(double (&acc)[9][2], const double* Tc, uint32_t& mx) {
  using namespace wn;
#pragma unroll 2
  for (int k0 = 0; k0 < GROWS; k0 += 4) {
    double f[8];
#pragma unroll
    for (int c = W; c < 8; ++c) f[c] = Tc[8 * c * GRS + k0];
    if constexpr (W == 0) {  // warp 0's fragments cover the whole tile: max |M| (high
                             // words, on the integer pipe beside the DMMAs)
#pragma unroll
      for (int c = 0; c < 8; ++c) mx = max(mx, (uint32_t)__double2hiint(f[c]) & 0x7FFFFFFFu);
    }
#pragma unroll
    for (int c = W; c < 8; ++c) dmma(acc[c - W][0], acc[c - W][1], f[W], f[c]);
#pragma unroll
    for (int c = 7 - W; c < 8; ++c)
      dmma(acc[8 - W + c - (7 - W)][0], acc[8 - W + c - (7 - W)][1], f[7 - W], f[c]);
  }
}

// gram_tile over one half of the tile's 32 rows (KH = 0: rows 0-15, 1: 16-31),
// for the eigen kernel's fused Gram phase (8 warps: 4 tile-row owners x 2
// row halves).
template <int W, int KH>
__device__ __forceinline__ void gram_tile_half(double (&acc)[9][2], const double* Tc,
                                               uint32_t& mx) {
  using namespace wn;
#pragma unroll 2
  for (int k0 = 16 * KH; k0 < 16 * KH + 16; k0 += 4) {
    double f[8];
#pragma unroll
    for (int c = W; c < 8; ++c) f[c] = Tc[8 * c * GRS + k0];
    if constexpr (W == 0) {
#pragma unroll
      for (int c = 0; c < 8; ++c) mx = max(mx, (uint32_t)__double2hiint(f[c]) & 0x7FFFFFFFu);
    }
#pragma unroll
    for (int c = W; c < 8; ++c) dmma(acc[c - W][0], acc[c - W][1], f[W], f[c]);
#pragma unroll
    for (int c = 7 - W; c < 8; ++c)
      dmma(acc[8 - W + c - (7 - W)][0], acc[8 - W + c - (7 - W)][1], f[7 - W], f[c]);
  }
}

template <bool IMG>
__global__ void __launch_bounds__(wn::GRAM_THREADS)
    gram_kernel(GroupSrc s, int n, double* __restrict__ Gout, double* __restrict__ gmax) {
  using namespace wn;
  extern __shared__ __align__(16) double sm[];
  double* T = sm;  // 2 x KMAX x GRS
  __shared__ long long cbase[KMAX];
  const int g = blockIdx.x;
  if (g >= n) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < KMAX) cbase[tid] = tid < s.K ? col_base<IMG>(s, g, tid) : 0;
  __syncthreads();
  const int ar = lane >> 2, ak = lane & 3;
  // accumulators: row w -> cols w..7 (slots 0..7-w), row 7-w -> cols 7-w..7
  // (slots 8-w..8): 9 slots; slot q -> (row, col)
  double acc[9][2];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q][0] = acc[q][1] = 0.0;
  uint32_t mx = 0;
  const int ntiles = (s.m + GROWS - 1) / GROWS;
  fill_tile<4>(T, s, cbase, 0, GROWS, GRS);
  for (int tt = 0; tt < ntiles; ++tt) {
    if (tt + 1 < ntiles)
      fill_tile<4>(T + ((tt + 1) & 1) * KMAX * GRS, s, cbase, (tt + 1) * GROWS, GROWS, GRS);
    else
      cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* Tc = T + (tt & 1) * KMAX * GRS + ar * GRS + ak;
    switch (w) {  // warp-uniform: compile-time accumulator indices per warp
      case 0: gram_tile<0>(acc, Tc, mx); break;
      case 1: gram_tile<1>(acc, Tc, mx); break;
      case 2: gram_tile<2>(acc, Tc, mx); break;
      default: gram_tile<3>(acc, Tc, mx); break;
    }
    __syncthreads();
  }
  if (w == 0) {
    mx = __reduce_max_sync(0xffffffffu, mx);
    // an upper bound of max |M| with its binary exponent
    if (lane == 0 && gmax) gmax[g] = __hiloint2double((int)mx, -1);
  }
  double* Gg = Gout + (size_t)g * GSZ;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const int ti = q < 8 - w ? w : 7 - w;
    const int tj = q < 8 - w ? w + q : q - (8 - w) + 7 - w;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = 8 * ti + ar, j = 8 * tj + 2 * ak + e;
      Gg[i * KMAX + j] = acc[q][e];
      if (tj != ti) Gg[j * KMAX + i] = acc[q][e];
    }
  }
}
// ---------------------------------------------------------------------------
// K2: eigen-decomposition + shrinkage -> Wm (in place over G)

// Work done by the eigen step since the last reset: [0] groups, [1] 4x4
// block super-rounds (one line of the schedule: 16 quads x three rotation
// rounds, the G and V updates), [2] groups finished by the first-order
// correction (two extra 64^3 products). Read by glr_eig_work for the bench's
// roofline (the O(K^3) eigen work is data dependent).
__device__ unsigned long long g_eig_work[3];

#ifdef GLR_EIG_STATS
// dev statistics: groups per sweep count (cold [0, 32), warm [32, 64))
__device__ unsigned int g_eig_hist[64];
__device__ unsigned int g_rank_hist[65];  // groups by number of kept components
// warm groups, first pre-check: [0] groups, [1 + d] non-exempt pairs above 1e-(4+d) relative
__device__ unsigned long long g_res_hist[8];
#endif

struct EigArgs {
  double* G;  // n x 64 x 64: G in, Wm out
  int n, K;
  double sigma, c_weight, eps, uniform_weight;
  double* vcache;  // optional per-group eigenvector cache (n x 64 x 64)
  int warm;        // 0 cold, 1 start every group from vcache, 2 only where warm_flags[g]
  const uint8_t* warm_flags;
  double* wmax;  // optional per-group max |Wm| (the split-integer apply's scale)
  int* counter;  // dynamic group counter (zeroed before the launch)
  // fused Gram (image groups): G = M^T M is formed in shared memory from the
  // image instead of being read from G, and max |M| goes to gmax
  GroupSrc src;
  double* gmax;
};

// Block-Jacobi schedule. The 63 rounds of a parallel cyclic sweep pair i
// with i ^ r; grouped into the 21 lines {a, b, a^b} of a line spread of
// PG(5, 2), three consecutive rounds act inside the 16 cosets ("quads") of
// {0, a, b, a^b}, so one super-round = three rounds = one 4x4 block step:
// G <- Q^T G Q, V <- V Q with Q block-diagonal over the quads, one read and
// one write of G and V per three rounds. g0..g3 span a complement whose
// low four bits are bijective: quad B's representative xor_k(bit k of B) g_k
// lands in its own shared-memory bank. Generated and checked by
// tools/jacobi_schedule.py (tests/test_native_abi.py re-checks the table).
__constant__ unsigned char kJacobiSched[21][6] = {
    {1, 59, 2, 4, 8, 17},   {2, 53, 1, 4, 8, 18},   {4, 41, 1, 2, 8, 20},
    {8, 17, 1, 2, 4, 40},   {16, 34, 1, 2, 4, 8},   {32, 7, 1, 2, 8, 20},
    {3, 14, 1, 4, 18, 40},  {6, 28, 1, 2, 8, 36},   {12, 56, 1, 2, 4, 24},
    {24, 51, 1, 2, 4, 8},   {48, 37, 1, 2, 4, 8},   {35, 9, 1, 2, 4, 24},
    {5, 18, 1, 2, 8, 36},   {10, 36, 1, 2, 4, 24},  {20, 11, 1, 2, 4, 40},
    {40, 22, 1, 2, 4, 8},   {19, 44, 1, 2, 4, 8},   {38, 27, 1, 2, 4, 8},
    {15, 54, 1, 2, 4, 24},  {30, 47, 1, 2, 4, 8},   {60, 29, 1, 2, 4, 8},
};

// round r = i ^ j of pair (i, j) -> its line (super-round) in kJacobiSched
__constant__ unsigned char kRoundLine[64] = {
    255, 0,  1,  6,  2,  12, 7,  5,  3,  11, 13, 14, 8,  6,  6,  18, 4,  3,  12, 16, 14, 10,
    15,  12, 9,  3,  7,  17, 7,  20, 19, 14, 5,  20, 4,  11, 13, 10, 17, 5,  15, 2,  11, 9,
    16,  2,  13, 19, 10, 19, 4,  9,  8,  1,  18, 1,  8,  18, 0,  0,  20, 17, 15, 16};

// the four indices of quad B in super-round sr: t, t^a, t^b, t^a^b
__device__ __forceinline__ void jacobi_quad(int sr, int B, int e[4]) {
  const int a = kJacobiSched[sr][0], b = kJacobiSched[sr][1];
  int t = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if ((B >> k) & 1) t ^= kJacobiSched[sr][2 + k];
  e[0] = t;
  e[1] = t ^ a;
  e[2] = t ^ b;
  e[3] = t ^ a ^ b;
}

// Short-latency reciprocal / reciprocal square root for the Jacobi rotation
// parameters: hardware approximation + two Newton steps (quadratic: full
// double precision to ~1 ulp; inputs are positive and normal when used).
template <int NR = 2>
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < NR; ++i) y = fma(y, fma(-x, y, 1.0), y);
  return y;
}
template <int NR = 2>
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < NR; ++i) y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
  return y;
}

// (u, v) <- (c u - s v, s u + c v) in one fixed evaluation order, so the
// (A, B) and (B, A) blocks of G stay exact transposes of each other.
__device__ __forceinline__ void jrot(double c, double s, double& u, double& v) {
  const double nu = __fma_rn(c, u, -__dmul_rn(s, v));
  const double nv = __fma_rn(s, u, __dmul_rn(c, v));
  u = nu;
  v = nv;
}

// 64 x 64 x 64 fp64 product on DMMA for the eigen kernel; A(i, k) and B(k, j)
// are read through the accessors. The four k of one MMA are 8 apart (k = kb + 8 (lane%4),
// kb = 0..7, 32..39): with the ODD row strides of G and V^T a fragment load
// then touches every bank exactly twice whether k indexes the row or the
// column of the operand ((lane/4) S + 8 (lane%4) or 8 (lane%4) S + lane/4
// mod 16 with S odd) -- consecutive k gave 4-way conflicts on the V^T reads
// (ncu: 4x the ideal wavefronts, the products were ~45 % of the kernel's
// shared-memory traffic on a one-sweep iteration).
// Warp w owns a 16 x 32 block of D: row tiles 2 (w / 2), 2 (w / 2) + 1 and
// column tiles 4 (w % 2) .. + 3, so a k-step loads 2 A and 4 B fragments for
// its 8 DMMAs (one A and 8 B fragments with a 8 x 64 strip per warp: a third
// more shared-memory wavefronts for the same math). Slot t of d = (row tile
// t / 4, column tile t % 4); mm64_row / mm64_col give an element's indices.
__device__ __forceinline__ int mm64_row(int warp, int t, int ar) {
  return 16 * (warp >> 1) + 8 * (t >> 2) + ar;
}
__device__ __forceinline__ int mm64_col(int warp, int t, int ak) {  // + e for the second value
  return 8 * (4 * (warp & 1) + (t & 3)) + 2 * ak;
}
template <class FA, class FB>
__device__ __forceinline__ void eig_mm64(FA A, FB B, double (&d)[8][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ar = lane >> 2, ak = lane & 3;
  const int r0 = 16 * (w >> 1), c0 = 32 * (w & 1);
#pragma unroll
  for (int t = 0; t < 8; ++t) d[t][0] = d[t][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < wn::KMAX / 4; ++kk) {
    const int k = (kk & 7) + 32 * (kk >> 3) + 8 * ak;
    const double fa0 = A(r0 + ar, k), fa1 = A(r0 + 8 + ar, k);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double fb = B(k, c0 + 8 * c + ar);
      dmma(d[c][0], d[c][1], fa0, fb);
      dmma(d[4 + c][0], d[4 + c][1], fa1, fb);
    }
  }
}

// True when the WNNM shrinkage maps EVERY eigenvalue <= lam to zero:
// r(lam) = max(s - w(s), 0) / s with s = sqrt(lam) (lowrank.py:58-64) is
// nondecreasing in lam (s grows, w = c sqrt(K) sigma^2 / (sigma_hat + eps)
// shrinks), so r(lam) == 0 covers everything below it.
__device__ __forceinline__ bool shrinks_to_zero(const EigArgs& a, double lam) {
  const double s = sqrt(fmax(lam, 0.0));
  double w;
  if (a.uniform_weight >= 0.0) {
    w = a.uniform_weight;
  } else {
    const double sig_hat = sqrt(fmax(s * s - a.K * a.sigma * a.sigma, 0.0));
    w = a.c_weight * sqrt((double)a.K) * a.sigma * a.sigma / (sig_hat + a.eps);
  }
  return s - w <= 0.0;
}

// f(s)/s of the WNNM shrinkage at eigenvalue lam (lowrank.py:58-64) and its
// derivative in lam (0 where the ratio is clamped to zero).
__device__ __forceinline__ double shrink_ratio(const EigArgs& a, double lam) {
  const double s = sqrt(fmax(lam, 0.0));
  double w;
  if (a.uniform_weight >= 0.0) {
    w = a.uniform_weight;
  } else {
    const double sig_hat = sqrt(fmax(s * s - a.K * a.sigma * a.sigma, 0.0));
    w = a.c_weight * sqrt((double)a.K) * a.sigma * a.sigma / (sig_hat + a.eps);
  }
  const double f = fmax(s - w, 0.0);
  return s > 0.0 ? f / s : 0.0;
}
__device__ __forceinline__ double shrink_ratio_deriv(const EigArgs& a, double lam) {
  const double s = sqrt(fmax(lam, 0.0));
  if (s == 0.0) return 0.0;
  if (a.uniform_weight >= 0.0) {
    const double w = a.uniform_weight;
    return s - w <= 0.0 ? 0.0 : w / (2.0 * s * s * s);
  }
  const double b = a.c_weight * sqrt((double)a.K) * a.sigma * a.sigma;
  const double sh = sqrt(fmax(lam - a.K * a.sigma * a.sigma, 0.0));
  const double w = b / (sh + a.eps);
  if (s - w <= 0.0) return 0.0;
  const double dw = sh > 0.0 ? -b / ((sh + a.eps) * (sh + a.eps) * 2.0 * sh) : 0.0;
  return -dw / s + w / (2.0 * s * s * s);
}

// Fused Gram phase of the eigen kernel (image groups): G = M^T M of group g
// into shared memory (row stride GLD, both triangles), on DMMA, with the
// group read straight from the image through a double-buffered cp.async
// tile ring that aliases the G / V^T buffers (neither is live yet). Eight
// warps: warp w owns the Gram kernel's tile rows (w % 4, 7 - w % 4) for the
// row half w / 4 of every 32-row tile; the two halves' partial sums meet in
// shared memory. Running the Gram inside the group loop lets one CTA's DMMA
// phase overlap the other resident CTAs' Jacobi phases (which are bound by
// shared-memory wavefronts and rotation latency, not the fp64 pipe).
__device__ __forceinline__ void eig_fused_gram(const EigArgs& a, const int g, double* sm) {
  using namespace wn;
  const GroupSrc& s = a.src;
  double* T = sm;  // 2 x KMAX x GRS doubles (aliases G and V^T)
  double* G = sm;
  __shared__ long long s_cb[KMAX];
  __shared__ uint32_t s_mx[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w = warp & 3, kh = warp >> 2;
  if (tid < KMAX) s_cb[tid] = tid < s.K ? col_base<true>(s, g, tid) : 0;
  __syncthreads();
  const int ar = lane >> 2, ak = lane & 3;
  double acc[9][2];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q][0] = acc[q][1] = 0.0;
  uint32_t mx = 0;
  const int ntiles = (s.m + GROWS - 1) / GROWS;
  fill_tile<8>(T, s, s_cb, 0, GROWS, GRS);
  for (int tt = 0; tt < ntiles; ++tt) {
    if (tt + 1 < ntiles)
      fill_tile<8>(T + ((tt + 1) & 1) * KMAX * GRS, s, s_cb, (tt + 1) * GROWS, GROWS, GRS);
    else
      cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* Tc = T + (tt & 1) * KMAX * GRS + ar * GRS + ak;
    switch (warp) {  // warp-uniform: compile-time accumulator indices per warp
      case 0: gram_tile_half<0, 0>(acc, Tc, mx); break;
      case 1: gram_tile_half<1, 0>(acc, Tc, mx); break;
      case 2: gram_tile_half<2, 0>(acc, Tc, mx); break;
      case 3: gram_tile_half<3, 0>(acc, Tc, mx); break;
      case 4: gram_tile_half<0, 1>(acc, Tc, mx); break;
      case 5: gram_tile_half<1, 1>(acc, Tc, mx); break;
      case 6: gram_tile_half<2, 1>(acc, Tc, mx); break;
      default: gram_tile_half<3, 1>(acc, Tc, mx); break;
    }
    __syncthreads();
  }
  if (w == 0) {
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) s_mx[kh] = mx;
  }
  // partial sums: the second row half writes, the first adds (both triangles)
#pragma unroll
  for (int pass = 1; pass >= 0; --pass) {
    if (kh == pass) {
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int ti = q < 8 - w ? w : 7 - w;
        const int tj = q < 8 - w ? w + q : q - (8 - w) + 7 - w;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 8 * ti + ar, j = 8 * tj + 2 * ak + e;
          const double v = pass ? acc[q][e] : G[i * GLD + j] + acc[q][e];
          G[i * GLD + j] = v;
          if (tj != ti) G[j * GLD + i] = v;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0 && a.gmax) a.gmax[g] = __hiloint2double((int)max(s_mx[0], s_mx[1]), -1);
}

template <bool FUSED>
__device__ __forceinline__ void eig_group(const EigArgs& a, const int g, double* sm) {
  using namespace wn;
  double* G = sm;               // KMAX x GLD, exactly symmetric throughout
  double* Vt = G + KMAX * GLD;  // KMAX x VLD: Vt[j][i] = V[i][j] (row j = eigenvector j)
  __shared__ double ratio[KMAX];
  __shared__ double s_tiny;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = a.K;
  double* Gg = a.G + (size_t)g * GSZ;
  double* vc = a.vcache ? a.vcache + (size_t)g * GSZ : nullptr;
  const bool warm = vc && (a.warm == 1 || (a.warm == 2 && a.warm_flags[g]));

  if constexpr (FUSED) {
    eig_fused_gram(a, g, sm);
  } else {
    for (int t = tid; t < GSZ / 2; t += EIG_THREADS) {
      const int i = (2 * t) >> 6, j = (2 * t) & 63;
      const double2 v = reinterpret_cast<const double2*>(Gg)[t];
      G[i * GLD + j] = v.x;
      G[i * GLD + j + 1] = v.y;
    }
  }
  for (int t = tid; t < GSZ; t += EIG_THREADS) {
    const int j = t >> 6, i = t & 63;
    Vt[j * VLD + i] = warm ? vc[t] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  if (warp == 0) {  // trace (entries beyond K are zero)
    double tr = fabs(G[lane * GLD + lane]) + fabs(G[(lane + 32) * GLD + lane + 32]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    if (lane == 0) s_tiny = 1e-17 * tr;
  }
  if (warm) {
    // Warm start from this group's eigenvectors of a previous iteration:
    // G <- Vp^T G Vp on DMMA (Y = G Vp to registers, then to G after a
    // barrier), V stays Vp. The sweeps then only remove a small off-diagonal
    // residue.
    const int ar = lane >> 2, ak = lane & 3;
    double d[8][2];
    eig_mm64([&](int i, int k) { return G[i * GLD + k]; },
             [&](int k, int j) { return Vt[j * VLD + k]; }, d);
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        G[mm64_row(warp, t, ar) * GLD + mm64_col(warp, t, ak) + e] = d[t][e];
    __syncthreads();
    eig_mm64([&](int i, int k) { return Vt[i * VLD + k]; },
             [&](int k, int j) { return G[k * GLD + j]; }, d);
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        G[mm64_row(warp, t, ar) * GLD + mm64_col(warp, t, ak) + e] = d[t][e];
    __syncthreads();
    // symmetrise (the product is symmetric up to rounding)
    for (int t = tid; t < GSZ; t += EIG_THREADS) {
      const int i = t >> 6, j = t & 63;
      if (i < j) {
        const double v = 0.5 * (G[i * GLD + j] + G[j * GLD + i]);
        G[i * GLD + j] = v;
        G[j * GLD + i] = v;
      }
    }
  }
  __syncthreads();
  const double tiny = s_tiny, tiny2 = tiny * tiny;

  // ---- parallel cyclic Jacobi in 4x4 block steps (schedule above). Per
  // super-round: phase 1 -- warp 0 lanes 0..15, one quad each, run the
  // quad's three rounds on its own 4x4 diagonal block (accumulating
  // Q_quad) while warps 1..7 apply the PREVIOUS super-round's V <- V Q
  // (double-buffered Q); phase 2 -- thread (w, l) rotates the G block
  // (2w + l/16, l%16): Q_A^T X Q_B. A rotation is skipped once |g_pq| is at
  // rounding level relative to its diagonal pair (or to 1e-17 trace).
  __shared__ double Qs[2][16][16];  // Qs[buf][4*r + c][quad] = Q_quad[r][c]
  __shared__ double Ds[16][16];     // rotated diagonal block, same layout
  __shared__ unsigned s_qrot[2];
  __shared__ unsigned char s_zb[8];  // per warp: zero-shrinkage flags of its 8 rows
  __shared__ unsigned char s_ub[8];  // per warp: rows too close to the shrinkage kink
  __shared__ unsigned s_lines;       // super-rounds holding a pair the finish cannot absorb
  __shared__ unsigned char s_rline[64];  // kRoundLine (lane-indexed reads: shared, not constant)
  __shared__ double s_kd[8];         // per warp: smallest kept diagonal entry
  __shared__ double s_rz[8];         // per warp: largest off-diagonal row sum of an exempt row
  __shared__ double lamv[KMAX];      // final diagonal (first-order finish)
  const int qA = 2 * warp + (lane >> 4), qB = lane & 15;
  int gsr = 0, prev_sr = -1;  // running super-round count; pending V step
  auto v_step = [&](int buf, int srv, int t0, int nthreads) {
    // V <- V Q_srv: V^T rows of quad B at 64 columns; unit u = (column, quad)
    const unsigned m = s_qrot[buf];
    const int B = t0 & 15;
    if (!((m >> B) & 1u)) return;
    int e[4];
    jacobi_quad(srv, B, e);
    double QB[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) QB[i][j] = Qs[buf][4 * i + j][B];
    for (int u = t0; u < 16 * KMAX; u += nthreads) {
      const int i = u >> 4;
      double v[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) v[l] = Vt[e[l] * VLD + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double o = 0.0;
#pragma unroll
        for (int l = 0; l < 4; ++l) o = fma(v[l], QB[l][j], o);
        Vt[e[j] * VLD + i] = o;
      }
    }
  };
  if (tid < 64) s_rline[tid] = kRoundLine[tid];
  int sweep = 0;
  uint64_t zmask = 0;  // indices whose whole Gershgorin disc shrinks to zero
  bool early = false;  // stopped by the first-order finish (residue above kRotTol)
  for (; sweep < MAX_SWEEPS; ++sweep) {
    // Zero-shrinkage exemption: index i is in Z when r(g_ii + sum_k |g_ik|)
    // == 0, i.e. every eigenvalue its Gershgorin disc can hold is mapped to
    // zero by the WNNM shrinkage. Rotations between two Z indices only
    // change the basis inside an invariant subspace whose contribution to
    // Wm = V diag(f(s)/s) V^T is exactly zero (the Z-block's eigenvalues all
    // lie below the threshold, by Gershgorin on that block), so they are
    // skipped; pairs with at least one non-Z index follow the usual test.
    // Z is recomputed from the current G before every sweep, so the sweeps
    // stop only once every non-exempt pair has converged on the final G.
    {
      const int i = tid >> 2, q = tid & 3;
      double r = 0.0;
#pragma unroll 4
      for (int k = 16 * q; k < 16 * q + 16; ++k) r += k == i ? 0.0 : fabs(G[i * GLD + k]);
      r += __shfl_xor_sync(0xffffffffu, r, 1);
      r += __shfl_xor_sync(0xffffffffu, r, 2);
      const double gii = G[i * GLD + i];
      const bool z = shrinks_to_zero(a, gii + r);
      // a kept row is "unsafe" for the first-order finish when its disc
      // (widened by 1e-3 |g_ii|) reaches down to the shrinkage kink
      const bool u = !z && shrinks_to_zero(a, gii - r - 1e-3 * fabs(gii));
      const unsigned bz = __ballot_sync(0xffffffffu, z && q == 0);
      const unsigned bu = __ballot_sync(0xffffffffu, u && q == 0);
      double kd = z ? __longlong_as_double(0x7ff0000000000000ll) : gii, rz = z ? r : 0.0;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        kd = fmin(kd, __shfl_xor_sync(0xffffffffu, kd, o));
        rz = fmax(rz, __shfl_xor_sync(0xffffffffu, rz, o));
      }
      if (tid == 0) s_lines = 0u;
      if (lane == 0) {
        s_kd[warp] = kd;
        s_rz[warp] = rz;
        unsigned char m8 = 0, u8 = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          m8 |= ((bz >> (4 * k)) & 1u) << k;
          u8 |= ((bu >> (4 * k)) & 1u) << k;
        }
        s_zb[warp] = m8;
        s_ub[warp] = u8;
      }
    }
    __syncthreads();
    zmask = 0;
    bool unsafe = false;
    double KD = s_kd[0], RZ = s_rz[0];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      zmask |= (uint64_t)s_zb[k] << (8 * k);
      unsafe |= s_ub[k] != 0;
      KD = fmin(KD, s_kd[k]);
      RZ = fmax(RZ, s_rz[k]);
    }
    // A sweep changes G only if some pair passes the rotation test on the
    // current G (otherwise no round rotates, by induction): test all pairs
    // up front and stop without paying for a no-op sweep. The sweeps also
    // stop once the first-order finish is exact to second order: no kept
    // row near the kink, kept-kept pairs below kFinishTol, and every
    // kept-exempt pair below its own finish bound (see the pair test).
    bool need = false, block_finish = false;
    unsigned lines = 0u;
    const double rot_over_rz2 = (kRotTol / RZ) * (kRotTol / RZ);  // +inf without exempt rows (unused then)
    for (int t = tid; t < GSZ; t += EIG_THREADS) {
      const int i = t >> 6, j = t & 63;
      const unsigned zi = (zmask >> i) & 1ull, zj = (zmask >> j) & 1ull;
      if (i < j && !(zi & zj)) {
        // squared comparisons (no square roots): g_ij^2 against tol^2 |g_ii g_jj|
        const double gij = G[i * GLD + j], g2 = gij * gij;
        const double gi = G[i * GLD + i], gj = G[j * GLD + j];
        const double sc2 = fabs(gi * gj);
        double st2 = kRotTol * kRotTol * sc2, fin2 = kFinishTol * kFinishTol * sc2;
        if (zi | zj) {
          // kept-exempt pair: the exempt eigenvalue is mapped to zero, so only
          // the rotation ANGLE g_ij / gap matters, not the relative accuracy
          // of the small diagonal entry -- the strict test is relative to
          // max(sqrt(g_ii g_jj), gap). The finish may leave an angle theta as
          // long as the first-order term r_i theta (applied below with the
          // diagonal of the exempt block standing in for the block: relative
          // error RZ / gap by a Neumann series of the resolvent) stays exact
          // to kRotTol: theta <= kFinishTol and theta RZ / gap <= kRotTol.
          const double gap = gi - gj, gap2 = gap * gap;
          st2 = kRotTol * kRotTol * fmax(sc2, gap2);
          fin2 = gap2 * fmin(kFinishTol * kFinishTol, gap2 * rot_over_rz2);
        }
        st2 = fmax(st2, tiny2);
#ifdef GLR_EIG_STATS
        if (warm && sweep == 0) {
          const double rel = fabs(gij) / fmax(sqrt(sc2), 1e-300);
          for (int d = 0; d < 6; ++d)
            if (rel > pow(10.0, -(4.0 + d))) atomicAdd(&g_res_hist[1 + d], 1ull);
        }
#endif
        need |= g2 > st2;
        block_finish |= g2 > fmax(st2, fin2);
        // lines the sweep has to visit: pairs above half their finish bound
        if (g2 > fmax(st2, 0.25 * fin2)) lines |= 1u << s_rline[i ^ j];
      }
    }
    lines = __reduce_or_sync(0xffffffffu, lines);
    if (lane == 0 && lines) atomicOr(&s_lines, lines);
    const bool any_need = __syncthreads_or(need);
    const bool any_block = __syncthreads_or(block_finish) || unsafe;
    if (!any_need || !any_block) {
      early = any_need;
      break;
    }
    // Partial sweep: only the lines holding a pair above half its finish bound
    // (rotations stay strict, so a visited quad is cleaned completely and the
    // rest is left to the first-order finish); every line where the finish
    // is ruled out (a kept row near the kink). From ~iteration 15 of C2 a
    // group has 1-3 pairs above the finish tolerance -- a full 21-line sweep
    // for them rotated all ~2000 pairs above the strict test.
    const unsigned run_lines = unsafe ? 0x1FFFFFu : s_lines;
#ifdef GLR_EIG_QUADTOL  // dev A/B: rotate only pairs above GLR_EIG_QUADTOL x the finish tolerance
                        // (measured on C2: 0.5 -> 175.7, 0.1 -> 179.6, strict -> 180.1 iters/s: the
                        // unrotated residues pile up below the threshold and more lines get marked)
    const double rtol2 = unsafe ? kRotTol * kRotTol
                                : (GLR_EIG_QUADTOL * kFinishTol) * (GLR_EIG_QUADTOL * kFinishTol);
#else
    const double rtol2 = kRotTol * kRotTol;
#endif
    for (int sr = 0; sr < 21; ++sr) {
      if (!((run_lines >> sr) & 1u)) continue;
      const int buf = gsr & 1;
      ++gsr;
#ifdef GLR_EIG_STATS
      if (tid == 0 && warm) atomicAdd(&g_res_hist[7], 1ull);
#endif
      if (warp == 0) {
        bool any = false;
        if (lane < 16) {
          int e[4];
          jacobi_quad(sr, lane, e);
          double S[4][4], Q[4][4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              Q[i][j] = i == j ? 1.0 : 0.0;
              if (j >= i) S[i][j] = G[e[i] * GLD + e[j]];
            }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < i; ++j) S[i][j] = S[j][i];
          // rounds a, b, a^b: pairs (0,1)(2,3), (0,2)(1,3), (0,3)(1,2); the
          // two rotations of a round are independent (branch-free, so their
          // latency chains overlap); a skipped rotation is the identity.
          constexpr int PI[6] = {0, 2, 0, 1, 0, 1}, PJ[6] = {1, 3, 2, 3, 3, 2};
#pragma unroll
          for (int rr = 0; rr < 3; ++rr) {
            double c[2], sn[2], t[2], app[2], aqq[2], apq[2];
            bool rotd[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int p = PI[2 * rr + h], q = PJ[2 * rr + h];
              app[h] = S[p][p];
              aqq[h] = S[q][q];
              apq[h] = S[p][q];
              const unsigned zp = (zmask >> e[p]) & 1ull, zq = (zmask >> e[q]) & 1ull;
              // the sweep's pre-check tests, squared (no square root on the rotation's
              // latency chain): kept-exempt pairs relative to max(sc, gap); exempt
              // pairs only under the gap rule (kZGapTol)
              const double a2 = apq[h] * apq[h], dpq = app[h] - aqq[h];
              const double sc2 = fabs(app[h] * aqq[h]);
              const double thr2 = (zp ^ zq) ? kRotTol * kRotTol * fmax(sc2, dpq * dpq)
                                            : rtol2 * sc2;
              const bool rot =
                  a2 > fmax(thr2, tiny2) &&
                  !((zp & zq) && fabs(apq[h]) <= kZGapTol * (KD - fmax(app[h], aqq[h])));
              any |= rot;
              rotd[h] = rot;
              // t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = d / g, as
              // sign(d) g / (|d| + hypot(d, g)): one sqrt, one division, one
              // rsqrt on the latency chain (|t| <= 1)
              const double d = aqq[h] - app[h], g = 2.0 * apq[h];
              const double hh = fma(d, d, g * g);
              // t only has to zero g_pq to ~1e-14 (one Newton step each); c and
              // s = t c are then an exactly consistent rotation (two steps)
              const double tt = (d >= 0.0 ? g : -g) * rcp_nr<1>(fabs(d) + hh * rsqrt_nr<1>(hh));
              t[h] = rot ? tt : 0.0;
              c[h] = rot ? rsqrt_nr<2>(fma(tt, tt, 1.0)) : 1.0;
              sn[h] = rot ? t[h] * c[h] : 0.0;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int p = PI[2 * rr + h], q = PJ[2 * rr + h];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if (k != p && k != q) {
                  jrot(c[h], sn[h], S[k][p], S[k][q]);
                  S[p][k] = S[k][p];
                  S[q][k] = S[k][q];
                }
                jrot(c[h], sn[h], Q[k][p], Q[k][q]);
              }
              S[p][p] = app[h] - t[h] * apq[h];
              S[q][q] = aqq[h] + t[h] * apq[h];
              // a skipped pair keeps its coupling: exempt (zero-shrinkage)
              // pairs can be far from converged, and zeroing their entry
              // would change the matrix being diagonalised
              if (rotd[h]) S[p][q] = S[q][p] = 0.0;
            }
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              Qs[buf][4 * i + j][lane] = Q[i][j];
              Ds[4 * i + j][lane] = S[i][j];
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, any);
        if (lane == 0) s_qrot[buf] = m;
      } else if (prev_sr >= 0) {
        v_step(buf ^ 1, prev_sr, tid - 32, EIG_THREADS - 32);
      }
      __syncthreads();
      const unsigned mask = s_qrot[buf];
      prev_sr = mask ? sr : -1;
      const bool rA = (mask >> qA) & 1u, rB = (mask >> qB) & 1u;
      if (rA || rB) {
        int eA[4], eB[4];
        jacobi_quad(sr, qA, eA);
        jacobi_quad(sr, qB, eB);
        // U = X Q_B (rows of X streamed in), then Y = Q_A^T U row by row
        double U[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double xk[4];
#pragma unroll
          for (int l = 0; l < 4; ++l) xk[l] = G[eA[k] * GLD + eB[l]];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double u = 0.0;
#pragma unroll
            for (int l = 0; l < 4; ++l) u = fma(xk[l], Qs[buf][4 * l + j][qB], u);
            U[k][j] = u;
          }
        }
        const bool diag = qA == qB;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double y[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double qa = Qs[buf][4 * k + i][qA];
#pragma unroll
            for (int j = 0; j < 4; ++j) y[j] = fma(qa, U[k][j], y[j]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) G[eA[i] * GLD + eB[j]] = diag ? Ds[4 * i + j][qA] : y[j];
        }
      }
      __syncthreads();
    }
  }
  if (prev_sr >= 0) {  // the last super-round's V step
    v_step((gsr - 1) & 1, prev_sr, tid, EIG_THREADS);
    __syncthreads();
  }

  if (tid == 0) {
    atomicAdd(&g_eig_work[0], 1ull);
    if (gsr) atomicAdd(&g_eig_work[1], (unsigned long long)gsr);
    if (early) atomicAdd(&g_eig_work[2], 1ull);
  }
#ifdef GLR_EIG_STATS
  if (tid == 0) atomicAdd(&g_eig_hist[warm ? 32 + sweep : sweep], 1u);
  if (tid == 0 && warm) atomicAdd(&g_res_hist[0], 1ull);
#endif
  if (vc && !(warm && sweep == 0)) {  // no sweep from a warm start: the cached V is unchanged
    for (int t = tid; t < GSZ; t += EIG_THREADS) vc[t] = Vt[(t >> 6) * VLD + (t & 63)];
  }
  // ---- shrinkage weights (lowrank.py:58-64) ----
  if (tid < KMAX) {
    const double lam = G[tid * GLD + tid];
    ratio[tid] = tid < K ? shrink_ratio(a, lam) : 0.0;
    lamv[tid] = lam;
  }
  __syncthreads();
#ifdef GLR_EIG_STATS
  if (tid == 0) {
    int kept = 0;
    for (int k = 0; k < KMAX; ++k) kept += ratio[k] != 0.0;
    atomicAdd(&g_rank_hist[kept], 1u);
  }
#endif
  double o[8][2];
  if (!early) {
    // converged to the rotation test: Wm = V diag(ratio) V^T on DMMA
    eig_mm64([&](int i, int k) { return Vt[k * VLD + i] * ratio[k]; },
             [&](int k, int j) { return Vt[k * VLD + j]; }, o);
  } else {
    // Mcorr = diag(f(s)/s) + E o D in place over G: the off-diagonal residue
    // E (all below kFinishTol relative, see the sweep exit; entries at the
    // rotation-test level are dropped as in the converged path) times the
    // divided differences D of the ratio, the derivative where two
    // eigenvalues nearly coincide. Then Wm = (V Mcorr) V^T on DMMA.
    for (int t = tid; t < GSZ; t += EIG_THREADS) {
      const int i = t >> 6, j = t & 63;
      double v = 0.0;
      if (i == j) {
        v = ratio[i];
      } else if (i < K && j < K) {
        const double li = lamv[i], lj = lamv[j], e = G[i * GLD + j];
        if (e * e > kRotTol * kRotTol * fabs(li * lj)) {
          const double d = li - lj;
          const double D = fabs(d) > 1e-4 * fmax(fabs(li), fabs(lj))
                               ? (ratio[i] - ratio[j]) * rcp_nr<2>(d)
                               : shrink_ratio_deriv(a, 0.5 * (li + lj));
          v = e * D;
        }
      }
      G[i * GLD + j] = v;
    }
    __syncthreads();
    eig_mm64([&](int i, int k) { return Vt[k * VLD + i]; },
             [&](int k, int j) { return G[k * GLD + j]; }, o);
    __syncthreads();
    {
      const int ar = lane >> 2, ak = lane & 3;
#pragma unroll
      for (int t = 0; t < 8; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          G[mm64_row(warp, t, ar) * GLD + mm64_col(warp, t, ak) + e] = o[t][e];
    }
    __syncthreads();
    eig_mm64([&](int i, int k) { return G[i * GLD + k]; },
             [&](int k, int j) { return Vt[k * VLD + j]; }, o);
  }
  {
    const int ar = lane >> 2, ak = lane & 3;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      *reinterpret_cast<double2*>(&Gg[mm64_row(warp, t, ar) * KMAX + mm64_col(warp, t, ak)]) =
          make_double2(o[t][0], o[t][1]);
  }
  if (a.wmax) {
    double mx = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) mx = fmax(mx, fmax(fabs(o[t][0]), fabs(o[t][1])));
    for (int o2 = 16; o2 > 0; o2 >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
    __syncthreads();  // ratio[] is free again
    if (lane == 0) ratio[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < EIG_THREADS / 32; ++w) mx = fmax(mx, ratio[w]);
      a.wmax[g] = mx;
    }
  }
}

// Dynamic group scheduling: 3 CTAs per SM take groups from an atomic counter
// (zeroed by the launcher), so the per-group sweep counts balance and the last
// wave's tail shrinks to one group per CTA.
template <bool FUSED>
__global__ void __launch_bounds__(wn::EIG_THREADS, 3) eig_kernel(EigArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_g;
  for (;;) {
    if (threadIdx.x == 0) s_g = atomicAdd(a.counter, 1);
    __syncthreads();
    const int g = s_g;
    __syncthreads();  // every thread has g (and is done with the previous group's smem)
    if (g >= a.n) return;
    eig_group<FUSED>(a, g, sm);
  }
}

// ---------------------------------------------------------------------------
// K3: out = M Wm on DMMA over TR-row tiles of M (cp.async double-buffered,
// column stride TR + 8 or TR + 4: 8 or 4 mod 16 doubles), Wm in shared
// memory (row stride LD = 68 == 4 mod 16). Warp w owns row fragment w % RF
// (8 rows) x NCT = RF column tiles: per k-step one A fragment and NCT B
// fragments feed NCT DMMAs. TR = 32 halves the tile buffers so three CTAs
// fit an SM. The denoised patch entries go to the int64 fixed-point
// numerator with integer atomics (or to `out`).

template <bool IMG, int TR>
__global__ void __launch_bounds__(wn::APPLY_THREADS)
    apply_kernel(GroupSrc s, int n, const double* __restrict__ Wm, double scale,
                 int64_t* __restrict__ acc_out, double* __restrict__ out) {
  using namespace wn;
  constexpr int TRS = TR + (TR == 64 ? 8 : 4);  // tile column stride
  constexpr int RF = TR / 8;                    // row fragments per tile
  constexpr int NCT = RF;                       // column tiles per warp (8 warps)
  extern __shared__ __align__(16) double sm[];
  double* Ws = sm;              // KMAX x LD
  double* T = Ws + KMAX * LD;   // 2 x KMAX x TRS
  __shared__ long long cbase[KMAX];
  const int g = blockIdx.x;
  if (g >= n) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = s.K, m = s.m;
  const int rf = warp % RF, ct0 = (warp / RF) * NCT;
  if (tid < KMAX) cbase[tid] = tid < K ? col_base<IMG>(s, g, tid) : 0;
  __syncthreads();
  fill_tile<APPLY_THREADS / 32>(T, s, cbase, 0, TR, TRS);
  const double* Wg = Wm + (size_t)g * GSZ;
  for (int t = tid; t < GSZ / 2; t += APPLY_THREADS) {
    const int i = (2 * t) >> 6, j = (2 * t) & 63;
    *reinterpret_cast<double2*>(&Ws[i * LD + j]) = reinterpret_cast<const double2*>(Wg)[t];
  }
  const int ar = lane >> 2, ak = lane & 3;
  const int ntiles = (m + TR - 1) / TR;
  for (int tt = 0; tt < ntiles; ++tt) {
    const int r0 = tt * TR;
    if (tt + 1 < ntiles)
      fill_tile<APPLY_THREADS / 32>(T + ((tt + 1) & 1) * KMAX * TRS, s, cbase, r0 + TR, TR, TRS);
    else
      cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* R = T + (tt & 1) * KMAX * TRS;
    double o[NCT][2];
#pragma unroll
    for (int b = 0; b < NCT; ++b) o[b][0] = o[b][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < KMAX; k0 += 4) {  // zero columns beyond K contribute nothing
      const double fa = R[(k0 + ak) * TRS + 8 * rf + ar];
#pragma unroll
      for (int b = 0; b < NCT; ++b)
        dmma(o[b][0], o[b][1], fa, Ws[(k0 + ak) * LD + 8 * (ct0 + b) + ar]);
    }
    const int r = r0 + 8 * rf + ar;
    if (r < m) {
      const int64_t off = (int64_t)(r / s.PC) * s.rs + (r % s.PC);
#pragma unroll
      for (int b = 0; b < NCT; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 8 * (ct0 + b) + 2 * ak + e;
          if (j < K) {
            if constexpr (IMG) {
              const long long val = __double2ll_rn(o[b][e] * scale);
#ifdef GLR_DEV_APPLY_NOATOMIC  // dev experiment: cost of the scatter atomics
              if (val == 0x7edcba9876543210ll) acc_out[cbase[j] + off] = val;
#else
              atomicAdd(reinterpret_cast<unsigned long long*>(acc_out + cbase[j] + off),
                        (unsigned long long)val);
#endif
            } else {
              out[cbase[j] + off] = o[b][e];
            }
          }
        }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K3 on the tensor cores: out = M Wm as an exact-integer split product
// (Ozaki scheme) on tcgen05 kind::i8. Each operand is scaled by a power of
// two (per group: the Gram kernel's max |M|, the eigen kernel's max |Wm|) so
// its entries become integers U with |U| <= 2^46, written as S = 6 balanced
// base-256 digits d_k in [-128, 127] (U = sum_k d_k 256^(5-k)), one int8
// "slice" per digit. The 21 digit products d_k(M) e_l(Wm) with k + l <= 5 are
// int8 MMAs with exact s32 accumulation (<= 6 x 64 x 2^14 < 2^31), one TMEM
// accumulator per level t = k + l. The epilogue joins adjacent levels exactly
// in int32 (a 256 + b < 2^31) and the three pairs in int64, then rounds once
// into the int64 fixed-point numerator. Error: the dropped levels t >= 6 stay
// below 5 2^-40 max|M| max|Wm| in the worst case (measured ~1e-12 on unit
// data), the input rounding 2^-47 of max|M| per entry -- at the numerator's
// 2^-40 resolution and far below the 1e-9 agreement of fp64 WNNM with LAPACK.
//
// Digit extraction is one DFMA per value: fma(v, 2^(46-E), 1.5 2^52 + BIAS)
// leaves U + BIAS (BIAS = 128 sum_k 256^k) in the low 48 mantissa bits, whose
// bytes are the digits + 128; a 4 x 4 byte transpose (PRMT) gathers one digit
// of four values into a word and XOR 0x80 recentres it.
//
// Operand A (the M tile's digits, 128 rows x 6 x 64 bytes) lives in TMEM and
// is written there by the slicers with tcgen05.st, so the tensor core reads
// only the small B operand (Wm's digits) from shared memory: with A in shared
// memory the 2 x 21 x 2 MMAs of N = 32 re-read A 42 times per tile and were
// bound by shared-memory bandwidth. Persistent, warp-specialised: one CTA per
// SM walks groups g = blockIdx.x, + gridDim.x, ...
//   warps 0-7   slicers: per 128-row tile each thread loads its row's 32
//               values (coalesced over rows), forms the digit words, waits for
//               the previous tile's MMAs, and stores 48 TMEM columns; per
//               group, Wm's slices into a 2-buffer shared-memory B ring;
//   warps 16-19 MMA issuers (one lane each): per tile and half of the 64
//               output columns, 21 digit products x 2 K-steps (M = 128,
//               N = 32, K = 32) into one of two TMEM accumulator sets (6
//               levels x 32 columns each); issuer (half, level set) owns its
//               accumulators, so four lanes issue in parallel (one issuing
//               lane was ~10 % slower);
//   warps 8-15  epilogue: per half, the 6 levels of 16 columns, released to
//               the MMA issuer right after tcgen05.ld, then the atomics.

namespace oz {
constexpr int S = 6;                     // digits per operand
constexpr int LV = 6;                    // levels kept: t = k + l <= 5
constexpr int BITS = 46;                 // |U| <= 2^46
constexpr int TR = 128;                  // rows of M per tile (UMMA M)
constexpr int NH = 32;                   // output columns per MMA pass (UMMA N)
constexpr int B_BUF = wn::KMAX * 128;    // 8 KB: two B slices per 128-byte row
constexpr int B_STAGE = (S / 2) * B_BUF; // 24 KB
constexpr int SLICERS = 256, EPI = 256;  // warps 0-7, 8-15; warps 16-19 issue the MMAs
constexpr int ISSUERS = 4;               // (column half) x (level set)
constexpr int THREADS = SLICERS + EPI + 32 * ISSUERS;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t ACC_COLS = LV * NH;   // 192 per accumulator set (sets at 0 and 192)
constexpr uint32_t A_COL = 2 * ACC_COLS; // A: 96 columns, 8 per (K-half, digit)
constexpr size_t SMEM = 2 * B_STAGE + 1024;
// 1.5 * 2^52 + 0x808080808080 (< 2^53, exact)
constexpr double MAGIC = 6755399441055744.0 + 141289400074368.0;
}  // namespace oz

__device__ __forceinline__ double pow2(int e) {  // 2^e for -1022 <= e <= 1023
  return __longlong_as_double((long long)(1023 + e) << 52);
}

// smallest E >= -60 with |v| < 2^E for every |v| <= mx
__device__ __forceinline__ int oz_exp(double mx) {
  return max((int)((((uint32_t)__double2hiint(mx)) >> 20) & 0x7FFu) - 1022, -60);
}

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Digit words of 16 consecutive K-values: w[k * WS + q] packs digit k of
// values 4q .. 4q+3 (byte i = value 4q+i) as signed bytes.
template <int WS>
__device__ __forceinline__ void oz_digits16(const double* v, double scale, uint32_t* w) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double t = fma(v[4 * q + i], scale, oz::MAGIC);
      lo[i] = (uint32_t)__double2loint(t);
      hi[i] = (uint32_t)__double2hiint(t);
    }
    const uint32_t x01 = __byte_perm(lo[0], lo[1], 0x5140), y01 = __byte_perm(lo[0], lo[1], 0x7362);
    const uint32_t x23 = __byte_perm(lo[2], lo[3], 0x5140), y23 = __byte_perm(lo[2], lo[3], 0x7362);
    const uint32_t h01 = __byte_perm(hi[0], hi[1], 0x5140), h23 = __byte_perm(hi[2], hi[3], 0x5140);
    w[5 * WS + q] = __byte_perm(x01, x23, 0x5410) ^ 0x80808080u;  // byte 0: least significant
    w[4 * WS + q] = __byte_perm(x01, x23, 0x7632) ^ 0x80808080u;
    w[3 * WS + q] = __byte_perm(y01, y23, 0x5410) ^ 0x80808080u;
    w[2 * WS + q] = __byte_perm(y01, y23, 0x7632) ^ 0x80808080u;
    w[1 * WS + q] = __byte_perm(h01, h23, 0x5410) ^ 0x80808080u;
    w[0 * WS + q] = __byte_perm(h01, h23, 0x7632) ^ 0x80808080u;  // byte 5: most significant
  }
}

__global__ void __launch_bounds__(oz::THREADS, 1)
    apply_oz_kernel(GroupSrc s, int n, const double* __restrict__ Wm,
                    const double* __restrict__ gmax, const double* __restrict__ wmax,
                    int frac_bits, int64_t* __restrict__ acc_out) {
  using namespace oz;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sB = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  __shared__ __align__(16) long long cb_s[2][wn::KMAX], cb_e[2][wn::KMAX];  // per group (parity)
  // A (TMEM) is handed over per K half: slicer threads jh fill columns
  // 48 jh .. 48 jh + 47, and the issuers run all K-half-0 MMAs of a tile before
  // its K-half-1 MMAs, so half 0 of tile t+1 is written while the K-half-1
  // MMAs of tile t still run (A stays single-buffered: the TMEM columns are
  // taken by the two accumulator sets)
  __shared__ __align__(8) uint64_t full_a[2], empty_a[2], full_b[2], empty_b[2], tfull[2],
      tempty[2];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = s.K, m = s.m;
  const int ntiles = (m + TR - 1) / TR;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full_a[i], SLICERS / 64);  // the slicer warps of K half i
      mbar_init(&empty_a[i], ISSUERS);      // every issuer's MMAs of K half i
      mbar_init(&full_b[i], SLICERS / 32);
      mbar_init(&empty_b[i], ISSUERS);
      mbar_init(&tfull[i], ISSUERS / 2);  // both level sets of the half
      mbar_init(&tempty[i], EPI / 32);
    }
    fence_barrier_init();
  }
  if (warp == 16) tmem_alloc<TMEM_COLS>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < 8) {
    // ---------------- slicers ----------------
    const int st = tid, r_loc = st & (TR - 1), jh = st >> 7;
    const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + A_COL + 48 * jh;
    int it = 0;
    for (int g = blockIdx.x, gi = 0; g < n; g += gridDim.x, ++gi) {
      const int pb = gi & 1;
      if (st < wn::KMAX) cb_s[pb][st] = st < K ? col_base<true>(s, g, st) * 8 : 0;  // bytes
      // Wm -> B slices (shared memory): row nn = output column j', K = j (B[nn][j] = Wm[j][nn]);
      // slice k in buffer k / 2 at bytes (k % 2) 64 + 16 jc, 16-byte chunk XOR (row % 8)
      {
        const int nn = st & 63, jc = st >> 6;
        const double* Wg = Wm + (size_t)g * wn::GSZ;
        double v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = Wg[(16 * jc + i) * wn::KMAX + nn];
        uint32_t w[S * 4];
        oz_digits16<4>(v, pow2(BITS - oz_exp(wmax[g])), w);
        if (gi >= 2) mbar_wait(&empty_b[pb], ((gi >> 1) - 1) & 1);
        uint8_t* b = sB + pb * B_STAGE;
#pragma unroll
        for (int k = 0; k < S; ++k) {
          const int c = ((k & 1) * 4 + jc) ^ (nn & 7);
          *reinterpret_cast<uint4*>(b + (k >> 1) * B_BUF + nn * 128 + c * 16) =
              make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_b[pb]);
      }
      named_bar(1, SLICERS);  // cb_s[pb] written
      const double sc = pow2(BITS - oz_exp(gmax[g]));
      const long long* cb = cb_s[pb] + 32 * jh;
      for (int tt = 0; tt < ntiles; ++tt, ++it) {
        const int r = tt * TR + r_loc;
        const bool rok = r < m;
        const char* src = reinterpret_cast<const char*>(
            s.src + (rok ? (int64_t)(r / s.PC) * s.rs + (r % s.PC) : 0));
        double v[32];
        if (rok && K == wn::KMAX) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __ldg(reinterpret_cast<const double*>(src + cb[i]));
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            v[i] = (rok && 32 * jh + i < K)
                       ? __ldg(reinterpret_cast<const double*>(src + cb[i])) : 0.0;
        }
        // A columns of this thread: 8 per digit k (its 32 K-bytes), digit-major
        uint32_t w[S * 8];
        oz_digits16<8>(v, sc, w);
        oz_digits16<8>(v + 16, sc, w + 4);
        // the previous tile's MMAs of this K half are done
        if (it >= 1) mbar_wait(&empty_a[jh], (it - 1) & 1);
        tc_fence_after();
        tmem_st_32x32b_x32(ta, *reinterpret_cast<const uint32_t(*)[32]>(w));
        tmem_st_32x32b_x16(ta + 32, w + 32);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_a[jh]);
      }
    }
  } else if (warp >= 16) {
    // ---------------- MMA issuers: lane 0 of warps 16-19; warp 16 + 2 ls + hf issues
    // column half hf, levels 0-3 (ls = 0: 10 products) or 4-5 (ls = 1: 11 products) ----------------
    if (lane == 0) {
      const int hf = (warp - 16) & 1, ls = (warp - 16) >> 1;
      constexpr uint32_t idesc = idesc_s8_s32(TR, NH);
      const uint32_t d0 = tmem + (uint32_t)hf * ACC_COLS;
      int it = 0;
      for (int g = blockIdx.x, gi = 0; g < n; g += gridDim.x, ++gi) {
        const int pb = gi & 1;
        mbar_wait(&full_b[pb], (gi >> 1) & 1);
        const uint64_t bd0 = smem_desc_k_sw128(sB + pb * B_STAGE) + (uint64_t)((hf * NH * 128) >> 4);
        for (int tt = 0; tt < ntiles; ++tt, ++it) {
          if (it >= 1) mbar_wait(&tempty[hf], (it - 1) & 1);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            mbar_wait(&full_a[ks], it & 1);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < S; ++k)
#pragma unroll
              for (int l = 0; l + k < LV; ++l)
                if ((k + l >= 4) == (ls == 1)) {  // this issuer's levels (own accumulators)
                  // B: slice l, rows 32 hf.., K bytes 32 ks.. of the slice (desc += bytes >> 4)
                  const uint64_t bd =
                      bd0 + (uint64_t)(((l >> 1) * B_BUF + (l & 1) * 64 + ks * 32) >> 4);
                  umma_i8_ta(d0 + (uint32_t)((k + l) * NH), tmem + A_COL + 48 * ks + 8 * k, bd,
                             idesc, (k | ks) != 0);
                }
            umma_commit(&empty_a[ks]);  // one of the ISSUERS arrivals that free A's K half
          }
          umma_commit(&tfull[hf]);
        }
        umma_commit(&empty_b[pb]);
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int et = tid - SLICERS, q = warp & 3, cc = (warp - 8) >> 2;
    int it = 0;
    for (int g = blockIdx.x, gi = 0; g < n; g += gridDim.x, ++gi) {
      const int pb = gi & 1;
      if (et < wn::KMAX) cb_e[pb][et] = et < K ? col_base<true>(s, g, et) * 8 : 0;  // bytes
      named_bar(2, EPI);
      // value = sum_t acc_t 256^(10-t) 2^(e_m + e_w - 2 BITS) = y 2^(e_m + e_w - 52), with
      // y = c0 2^32 + c1 2^16 + c2, c0 = acc_0 256 + acc_1, c1 = acc_2 256 + acc_3,
      // c2 = acc_4 256 + acc_5 (each exact in int32). Fixed point: round(y 2^-R),
      // R = 52 - e_m - e_w - frac_bits, in integer arithmetic: c0 2^(32-R) + c1 2^(16-R) +
      // ((c2 + 2^(R-1)) >> R) for 2 <= R <= 16 (the normal range: |x| < 2^(41-frac_bits)
      // and |Wm| <= 1 give R ~ 11), a 64-bit path otherwise.
      const int R = max(min(52 - oz_exp(gmax[g]) - oz_exp(wmax[g]) - frac_bits, 62), 0);
      const bool fast = R >= 2 && R <= 16;
      const int half = fast ? 1 << (R - 1) : 0;
      const int m0 = fast ? 1 << (32 - R) : 0, m1 = fast ? 1 << (16 - R) : 0;
      for (int tt = 0; tt < ntiles; ++tt, ++it) {
        const int r = tt * TR + 32 * q + lane;
        const bool rok = r < m;
        char* dst = reinterpret_cast<char*>(
            acc_out + (rok ? (int64_t)(r / s.PC) * s.rs + (r % s.PC) : 0));
        for (int hf = 0; hf < 2; ++hf) {
          mbar_wait(&tfull[hf], it & 1);
          tc_fence_after();
          const uint32_t ta =
              tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(hf * ACC_COLS + 16 * cc);
          int c0[16], c1[16], c2[16];
          {
            uint32_t x[16], y[16], z[16], w[16];
            tmem_ld_32x32b_x16(ta + 0 * NH, x);
            tmem_ld_32x32b_x16(ta + 1 * NH, y);
            tmem_ld_32x32b_x16(ta + 2 * NH, z);
            tmem_ld_32x32b_x16(ta + 3 * NH, w);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              c0[i] = (int)x[i] * 256 + (int)y[i];  // exact: |.| < 2^31
              c1[i] = (int)z[i] * 256 + (int)w[i];
            }
          }
          {
            uint32_t x[16], y[16];
            tmem_ld_32x32b_x16(ta + 4 * NH, x);
            tmem_ld_32x32b_x16(ta + 5 * NH, y);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) c2[i] = (int)x[i] * 256 + (int)y[i];
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[hf]);  // accumulator set hf may be overwritten now
          const int j0 = hf * NH + 16 * cc;
          if (rok && j0 < K) {
            const long long* cb = cb_e[pb] + j0;  // byte offsets of the columns
            if (fast && j0 + 16 <= K) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const long long v = (long long)c0[i] * m0 +
                                    ((long long)c1[i] * m1 + (long long)((c2[i] + half) >> R));
                red_add_u64(reinterpret_cast<unsigned long long*>(dst + cb[i]),
                            (unsigned long long)v);
              }
            } else {
              const int jn = min(16, K - j0);
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                if (i >= jn) break;
                const long long y =
                    (long long)c0[i] * 4294967296ll + (long long)c1[i] * 65536 + c2[i];
                const long long v = R > 0 ? (y + (1ll << (R - 1))) >> R : y;
                red_add_u64(reinterpret_cast<unsigned long long*>(dst + cb[i]),
                            (unsigned long long)v);
              }
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 16) tmem_dealloc<TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// Eigenvector carry-over across a matching refresh: a new group whose anchor
// was also an anchor before (and whose old group lived in this rank's old
// shard) starts its Jacobi sweeps from the old group's eigenvectors.

__global__ void anchor_map_kernel(const int32_t* __restrict__ anchors, int lo, int hi, int W,
                                  int32_t* __restrict__ map, int set) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x)
    map[anchors[2 * i] * W + anchors[2 * i + 1]] = set ? i : -1;
}

// With both position lists given, the cached V^T rows are also re-indexed
// by group column: new column j takes the coordinate of the old column that
// holds the same patch position (t-th occurrence matched to t-th occurrence),
// unmatched new columns take the unmatched old coordinates in order. Any
// such coordinate permutation of an orthogonal V is orthogonal, and a good
// warm start whenever the refreshed group keeps most of its patches.
__global__ void vcache_remap_kernel(const int32_t* __restrict__ new_anchors, int lo, int W,
                                    const int32_t* __restrict__ map,
                                    const double* __restrict__ vc_old, double* __restrict__ vc_new,
                                    uint8_t* __restrict__ flags,
                                    const int32_t* __restrict__ old_pos,
                                    const int32_t* __restrict__ new_pos, int K) {
  __shared__ int perm[wn::KMAX], inv[wn::KMAX], used[wn::KMAX], key_o[wn::KMAX],
      key_n[wn::KMAX];
  const int g = lo + blockIdx.x;
  const int old = map[new_anchors[2 * g] * W + new_anchors[2 * g + 1]];
  const int tid = threadIdx.x;
  if (tid == 0) flags[g] = old >= 0 ? 1 : 0;
  if (old < 0) return;
  if (tid < wn::KMAX) {
    perm[tid] = tid;
    used[tid] = 0;
  }
  if (old_pos && new_pos) {
    if (tid < K) {
      const int32_t* op = old_pos + ((size_t)old * K + tid) * 2;
      const int32_t* np = new_pos + ((size_t)g * K + tid) * 2;
      key_o[tid] = op[0] * W + op[1];
      key_n[tid] = np[0] * W + np[1];
    }
    __syncthreads();
    int match = -1;
    if (tid < K) {
      const int v = key_n[tid];
      int t = 0;  // occurrence rank of v among the new columns before tid
      for (int j = 0; j < tid; ++j) t += key_n[j] == v;
      for (int i = 0; i < K && match < 0; ++i)
        if (key_o[i] == v && t-- == 0) match = i;
      if (match >= 0) used[match] = 1;
    }
    __syncthreads();
    if (tid < K) {
      if (!used[tid]) {  // rank among the unmatched old coordinates
        int r = 0;
        for (int i = 0; i < tid; ++i) r += !used[i];
        inv[r] = tid;
      }
    }
    __syncthreads();
    if (tid < K) {
      if (match < 0) {  // rank among the unmatched new columns
        int r = 0;
        for (int j = 0; j < tid; ++j) {
          const int v = key_n[j];
          int t = 0, m = -1;
          for (int q = 0; q < j; ++q) t += key_n[q] == v;
          for (int i = 0; i < K && m < 0; ++i)
            if (key_o[i] == v && t-- == 0) m = i;
          r += m < 0;
        }
        match = inv[r];
      }
      perm[tid] = match;
    }
  }
  __syncthreads();
  const double* src = vc_old + (size_t)old * wn::GSZ;
  double* dst = vc_new + (size_t)g * wn::GSZ;
  for (int t = tid; t < wn::GSZ; t += blockDim.x) {  // Vt[e][j] = Vt_old[e][perm[j]]
    const int e = t >> 6, j = t & 63;
    dst[t] = src[e * wn::KMAX + perm[j]];
  }
}

// ---------------------------------------------------------------------------
// counters / explicit-group scatter / normalisation

// cnt[pixel] += 1 for every patch covering it (channel-invariant counter)
__global__ void scatter_count_kernel(const int32_t* __restrict__ pos, int n_max,
                                     const int32_t* n_dev, int K, int P, int W,
                                     int32_t* __restrict__ cnt) {
  const int N = n_dev ? min(*n_dev, n_max) : n_max;
  const int64_t total = (int64_t)N * K * P * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i / (P * P);
    const int o = (int)(i - col * P * P);
    const int r = pos[2 * col] + o / P, c = pos[2 * col + 1] + o % P;
    GLR_DCHECK(r >= 0 && c >= 0 && c < W);
    atomicAdd(&cnt[(int64_t)r * W + c], 1);
  }
}

// exact scatter_group: per output element, columns added in group/column order
__global__ void scatter_f64_kernel(const double* __restrict__ groups, const int32_t* __restrict__ pos,
                                   int G, int K, int P, int H, int W, int C,
                                   double* __restrict__ acc, double* __restrict__ cnt) {
  const int64_t total = (int64_t)H * W * C;
  const int m = P * P * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % C);
    const int64_t pix = i / C;
    const int r = (int)(pix / W), c = (int)(pix % W);
    double a = acc[i], n = cnt[i];
    for (int g = 0; g < G; ++g)
      for (int j = 0; j < K; ++j) {
        const int pr = pos[((size_t)g * K + j) * 2], pc = pos[((size_t)g * K + j) * 2 + 1];
        const int dr = r - pr, dc = c - pc;
        if (dr >= 0 && dr < P && dc >= 0 && dc < P) {
          a += groups[((size_t)g * K + j) * m + (dr * P + dc) * C + ch];
          n += 1.0;
        }
      }
    acc[i] = a;
    cnt[i] = n;
  }
}

// fixed-point scatter of explicit fp64 groups (G,K,m) into acc
__global__ void scatter_fixed_kernel(const double* __restrict__ groups,
                                     const int32_t* __restrict__ pos, int G, int K, int P, int W,
                                     int C, double scale, int64_t* __restrict__ acc) {
  const int m = P * P * C;
  const int64_t total = (int64_t)G * K * m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i / m;
    const int e = (int)(i - col * m);
    const int r = pos[2 * col] + e / (P * C);
    const int c = pos[2 * col + 1] + (e / C) % P;
    const long long v = __double2ll_rn(groups[i] * scale);
    atomicAdd(reinterpret_cast<unsigned long long*>(acc + ((int64_t)r * W + c) * C + (e % C)),
              (unsigned long long)v);
  }
}

__global__ void normalize_kernel(int64_t* __restrict__ acc, const int32_t* __restrict__ cnt,
                                 const double* __restrict__ x, int64_t npix, int C, double inv_scale,
                                 double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix * C;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = cnt[i / C];
    if (n > 0) {
      z[i] = ((double)acc[i] * inv_scale) / (double)n;
      acc[i] = 0;  // read-and-clear (the numerator is consumed)
    } else {
      z[i] = x[i];
    }
  }
}

static int blocks_for(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, threads), (int64_t)kNumSMs * 32));
}

constexpr size_t kGramSmem = 2 * wn::KMAX * wn::GRS * sizeof(double);
constexpr size_t kEigSmem = wn::KMAX * (wn::GLD + wn::VLD) * sizeof(double);
#ifndef GLR_APPLY_TR  // apply tile rows: 32 (3 CTAs/SM) measured 2.17 ms vs 2.21 for 64 on C2
#define GLR_APPLY_TR 32
#endif
constexpr int kApplyTR = GLR_APPLY_TR;
constexpr size_t kApplySmem =
    (wn::KMAX * wn::LD + 2 * wn::KMAX * (kApplyTR + (kApplyTR == 64 ? 8 : 4))) * sizeof(double);
// Gram -> eigen/shrink -> apply for n groups; ws holds n x 64 x 64 doubles.
template <bool IMG>
static int run_wnnm(const GroupSrc& s, int n, const EigArgs& ea_in, double scale,
                    int64_t* acc_out, double* out, double* ws, cudaStream_t st) {
  { const int s_ = ensure_smem_attr((const void*)gram_kernel<IMG>, (int)kGramSmem); if (s_) return s_; }
  // Gram inside the eigen kernel for short groups (m <= 512: C1 24.8 vs
  // 25.1 ms per solve, C3 94.7 vs 96.6 ms); the separate DMMA Gram kernel
  // for tall ones (C2, m = 1536: 327.0 vs 332.5 ms -- there the fused Gram
  // phase competes with the Jacobi phases for shared-memory bandwidth)
  const bool kFused = IMG && s.m <= 512;
  {
    const int s_ = ensure_smem_attr(kFused ? (const void*)eig_kernel<true>
                                           : (const void*)eig_kernel<false>, (int)kEigSmem);
    if (s_) return s_;
  }
  {
    const int s_ = ensure_smem_attr((const void*)apply_kernel<IMG, kApplyTR>, (int)kApplySmem);
    if (s_) return s_;
  }
  if (!kFused) {
    gram_kernel<IMG><<<n, wn::GRAM_THREADS, kGramSmem, st>>>(s, n, ws, ws + (size_t)n * wn::GSZ);
    GLR_CUDA(cudaGetLastError());
  }
  EigArgs ea = ea_in;
  ea.src = s;
  ea.gmax = kFused ? ws + (size_t)n * wn::GSZ : nullptr;
  ea.G = ws;
  ea.n = n;
  ea.wmax = ws + (size_t)n * (wn::GSZ + 1);
  ea.counter = reinterpret_cast<int*>(ws + (size_t)n * (wn::GSZ + 2));
  GLR_CUDA(cudaMemsetAsync(ea.counter, 0, sizeof(int), st));
  if (kFused)
    eig_kernel<true><<<std::min(n, 3 * device_sms()), wn::EIG_THREADS, kEigSmem, st>>>(ea);
  else
    eig_kernel<false><<<std::min(n, 3 * device_sms()), wn::EIG_THREADS, kEigSmem, st>>>(ea);
  GLR_CUDA(cudaGetLastError());
#ifndef GLR_APPLY_DMMA  // dev A/B: -DGLR_APPLY_DMMA keeps the fp64 DMMA apply for image groups
  if constexpr (IMG) {
    {
      const int s_ = ensure_smem_attr((const void*)apply_oz_kernel, (int)oz::SMEM);
      if (s_) return s_;
    }
    apply_oz_kernel<<<std::min(n, device_sms()), oz::THREADS, oz::SMEM, st>>>(
        s, n, ws, ws + (size_t)n * wn::GSZ, ws + (size_t)n * (wn::GSZ + 1), ilogb(scale), acc_out);
    return check_launch("wnnm kernels");
  }
#endif
  apply_kernel<IMG, kApplyTR><<<n, wn::APPLY_THREADS, kApplySmem, st>>>(s, n, ws, scale, acc_out,
                                                                        out);
  return check_launch("wnnm kernels");
}


// ---------------------------------------------------------------------------
// Groups wider than 64 columns (lowrank.py:46-65 takes any K): a generic fp64
// path, one CTA per group, G and V in the workspace (2 K^2 doubles per
// group, L2-resident) instead of shared memory:
//   big_gram_kernel    G = M^T M (fp64 FMA), V = I
//   big_jacobi_kernel  cyclic two-sided Jacobi in round-robin order (K/2
//                      disjoint rotations per round, K-1 rounds per sweep),
//                      the same rotation test as the fast kernel; then the
//                      shrinkage and Wm = V diag(f(s)/s) V^T over G
//   big_apply_kernel   out = M Wm, written out or scattered into the int64
//                      fixed-point numerator like every other group
// No warm start (each call is cold). This path exists for conformance with
// the reference's signature; the configurations use K <= 64.
namespace wb {
constexpr int THREADS = 256;
constexpr int MAX_SWEEPS = 40;
}

__device__ __forceinline__ int64_t row_off(const GroupSrc& s, int r) {
  return (int64_t)(r / s.PC) * s.rs + (r % s.PC);
}

template <bool IMG>
__global__ void __launch_bounds__(wb::THREADS) big_gram_kernel(GroupSrc s, int n, double* ws) {
  const int g = blockIdx.x, K = s.K;
  extern __shared__ long long cb[];  // K column bases
  double* G = ws + (size_t)g * 2 * K * K;
  double* V = G + (size_t)K * K;
  for (int j = threadIdx.x; j < K; j += blockDim.x) cb[j] = col_base<IMG>(s, g, j);
  __syncthreads();
  for (int t = threadIdx.x; t < K * K; t += blockDim.x) {
    const int i = t / K, j = t % K;
    V[t] = i == j ? 1.0 : 0.0;
    if (i > j) continue;
    double acc = 0.0;
    for (int r = 0; r < s.m; ++r) {
      const int64_t o = row_off(s, r);
      acc = fma(s.src[cb[i] + o], s.src[cb[j] + o], acc);
    }
    G[(size_t)i * K + j] = acc;
    G[(size_t)j * K + i] = acc;
  }
}

__global__ void __launch_bounds__(wb::THREADS) big_jacobi_kernel(EigArgs a, double* ws) {
  const int g = blockIdx.x, K = a.K, tid = threadIdx.x;
  const int Kp = K + (K & 1);  // even; index K (odd K) is a dummy that never rotates
  const int npair = Kp / 2;
  double* G = ws + (size_t)g * 2 * K * K;
  double* V = G + (size_t)K * K;
  extern __shared__ double sh[];
  double* cs = sh;               // npair
  double* sn = cs + npair;       // npair
  double* tt = sn + npair;       // npair
  int* pp = reinterpret_cast<int*>(tt + npair);
  int* qq = pp + npair;
  __shared__ int s_any;
  __shared__ double s_tiny;
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < K; ++i) tr += fabs(G[(size_t)i * K + i]);
    s_tiny = 1e-17 * tr;
  }
  __syncthreads();
  const double tiny = s_tiny;
  for (int sweep = 0; sweep < wb::MAX_SWEEPS; ++sweep) {
    if (tid == 0) s_any = 0;
    __syncthreads();
    for (int round = 0; round < Kp - 1; ++round) {
      // circle method: (round, Kp-1) and ((round+k) % (Kp-1), (round-k) % (Kp-1))
      for (int k = tid; k < npair; k += blockDim.x) {
        int p, q;
        if (k == 0) {
          p = round;
          q = Kp - 1;
        } else {
          p = (round + k) % (Kp - 1);
          q = (round - k + Kp - 1) % (Kp - 1);
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, sv = 0.0, t = 0.0;
        bool rot = false;
        if (q < K) {
          const double app = G[(size_t)p * K + p], aqq = G[(size_t)q * K + q];
          const double apq = G[(size_t)p * K + q];
          rot = fabs(apq) > fmax(wn::kRotTol * sqrt(fabs(app * aqq)), tiny);
          if (rot) {
            const double tau = (aqq - app) / (2.0 * apq);
            t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            sv = t * c;
          }
        }
        pp[k] = rot ? p : -1;
        qq[k] = q;
        cs[k] = c;
        sn[k] = sv;
        tt[k] = t;
        if (rot) s_any = 1;
      }
      __syncthreads();
      // rows p, q of G (G <- J^T G)
      for (int u = tid; u < npair * K; u += blockDim.x) {
        const int k = u / K, col = u % K, p = pp[k];
        if (p < 0) continue;
        const int q = qq[k];
        const double gp = G[(size_t)p * K + col], gq = G[(size_t)q * K + col];
        G[(size_t)p * K + col] = cs[k] * gp - sn[k] * gq;
        G[(size_t)q * K + col] = sn[k] * gp + cs[k] * gq;
      }
      __syncthreads();
      // columns p, q of G (G <- G J) and of V (V <- V J)
      for (int u = tid; u < npair * K; u += blockDim.x) {
        const int k = u / K, row = u % K, p = pp[k];
        if (p < 0) continue;
        const int q = qq[k];
        const double gp = G[(size_t)row * K + p], gq = G[(size_t)row * K + q];
        G[(size_t)row * K + p] = cs[k] * gp - sn[k] * gq;
        G[(size_t)row * K + q] = sn[k] * gp + cs[k] * gq;
        const double vp = V[(size_t)row * K + p], vq = V[(size_t)row * K + q];
        V[(size_t)row * K + p] = cs[k] * vp - sn[k] * vq;
        V[(size_t)row * K + q] = sn[k] * vp + cs[k] * vq;
      }
      __syncthreads();
      // the rotated 2x2 blocks are diagonal (set exactly)
      for (int k = tid; k < npair; k += blockDim.x) {
        const int p = pp[k];
        if (p < 0) continue;
        const int q = qq[k];
        G[(size_t)p * K + q] = 0.0;
        G[(size_t)q * K + p] = 0.0;
      }
      __syncthreads();
    }
    if (!s_any) break;
  }
  // shrinkage (lowrank.py:58-64), then Wm = V diag(ratio) V^T over G
  double* ratio = sh;  // K doubles (the rotation arrays are done)
  for (int i = tid; i < K; i += blockDim.x) {
    const double lam = G[(size_t)i * K + i];
    const double sv = sqrt(fmax(lam, 0.0));
    double w;
    if (a.uniform_weight >= 0.0) {
      w = a.uniform_weight;
    } else {
      const double sig_hat = sqrt(fmax(sv * sv - K * a.sigma * a.sigma, 0.0));
      w = a.c_weight * sqrt((double)K) * a.sigma * a.sigma / (sig_hat + a.eps);
    }
    const double f = fmax(sv - w, 0.0);
    ratio[i] = sv > 0.0 ? f / sv : 0.0;
  }
  __syncthreads();
  for (int t = tid; t < K * K; t += blockDim.x) {
    const int i = t / K, j = t % K;
    double acc = 0.0;
    for (int k = 0; k < K; ++k)
      acc = fma(V[(size_t)i * K + k] * ratio[k], V[(size_t)j * K + k], acc);
    G[t] = acc;
  }
}

template <bool IMG>
__global__ void __launch_bounds__(wb::THREADS) big_apply_kernel(GroupSrc s, int n, const double* ws,
                                                               double scale, int64_t* acc_out,
                                                               double* out) {
  const int g = blockIdx.x, K = s.K;
  extern __shared__ long long cb[];
  const double* Wm = ws + (size_t)g * 2 * K * K;
  for (int j = threadIdx.x; j < K; j += blockDim.x) cb[j] = col_base<IMG>(s, g, j);
  __syncthreads();
  for (int64_t t = threadIdx.x; t < (int64_t)s.m * K; t += blockDim.x) {
    const int j = (int)(t / s.m), r = (int)(t % s.m);
    const int64_t o = row_off(s, r);
    double v = 0.0;
    for (int k = 0; k < K; ++k) v = fma(s.src[cb[k] + o], Wm[(size_t)k * K + j], v);
    if constexpr (IMG) {
      atomicAdd(reinterpret_cast<unsigned long long*>(acc_out + cb[j] + o),
                (unsigned long long)__double2ll_rn(v * scale));
    } else {
      out[((size_t)g * K + j) * s.m + r] = v;
    }
  }
}

template <bool IMG>
static int run_wnnm_big(const GroupSrc& s, int n, const EigArgs& ea, double scale,
                        int64_t* acc_out, double* out, double* ws, cudaStream_t st) {
  const int K = s.K;
  const int cb_bytes = K * (int)sizeof(long long);
  const int jac_bytes = (K + 1) / 2 * 3 * (int)sizeof(double) + 2 * ((K + 1) / 2) * (int)sizeof(int);
  const int jac_smem = std::max(jac_bytes, K * (int)sizeof(double));
  GLR_REQUIRE(jac_smem <= 200 * 1024, GLR_ERR_UNSUPPORTED, "wnnm: K=%d too large", K);
  if (cb_bytes > 48 * 1024) {
    const int a = ensure_smem_attr((const void*)big_gram_kernel<IMG>, cb_bytes);
    if (a) return a;
    const int b = ensure_smem_attr((const void*)big_apply_kernel<IMG>, cb_bytes);
    if (b) return b;
  }
  if (jac_smem > 48 * 1024) {
    const int a = ensure_smem_attr((const void*)big_jacobi_kernel, jac_smem);
    if (a) return a;
  }
  big_gram_kernel<IMG><<<n, wb::THREADS, cb_bytes, st>>>(s, n, ws);
  GLR_CUDA(cudaGetLastError());
  big_jacobi_kernel<<<n, wb::THREADS, jac_smem, st>>>(ea, ws);
  GLR_CUDA(cudaGetLastError());
  big_apply_kernel<IMG><<<n, wb::THREADS, cb_bytes, st>>>(s, n, ws, scale, acc_out, out);
  return check_launch("wnnm (K > 64) kernels");
}
}  // namespace glr

using namespace glr;

#ifdef GLR_EIG_STATS
extern "C" int glr_debug_eig_hist(unsigned int* out, int reset) {
  cudaMemcpyFromSymbol(out, g_eig_hist, sizeof(unsigned int) * 64);
  cudaMemcpyFromSymbol(out + 64, g_rank_hist, sizeof(unsigned int) * 65);
  cudaMemcpyFromSymbol(out + 130, g_res_hist, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z8[8] = {};
    cudaMemcpyToSymbol(g_res_hist, z8, sizeof(z8));
    unsigned int z[65] = {};
    cudaMemcpyToSymbol(g_eig_hist, z, sizeof(unsigned int) * 64);
    cudaMemcpyToSymbol(g_rank_hist, z, sizeof(unsigned int) * 65);
  }
  return 0;
}
#endif

extern "C" int glr_eig_work(uint64_t* out3_host, int reset) {
  unsigned long long v[3] = {0, 0, 0};
  if (out3_host) {
    GLR_CUDA(cudaMemcpyFromSymbol(v, g_eig_work, sizeof(v)));
    for (int i = 0; i < 3; ++i) out3_host[i] = v[i];
  }
  if (reset) {
    const unsigned long long z[3] = {0, 0, 0};
    GLR_CUDA(cudaMemcpyToSymbol(g_eig_work, z, sizeof(z)));
  }
  return GLR_OK;
}

extern "C" size_t glr_wnnm_workspace(int G, int K) {
  // K > 64 (generic path): G and V, K x K each, per group
  if (K > wn::KMAX) return (size_t)std::max(G, 1) * 2 * K * K * sizeof(double) + 256;
  // G / Wm (64 x 64 per group), then max |M| and max |Wm| per group
  // (+ the eigen kernel's group counter)
  return ((size_t)std::max(G, 1) * (wn::GSZ + 2) + 1) * sizeof(double) + 256;
}

extern "C" int glr_wnnm(const double* groups_d, int G, int m, int K, double sigma, double c_weight,
                        double eps, double uniform_weight, double* out_d, int32_t* nonfinite_d,
                        void* ws_d, size_t ws_bytes, void* stream) {
  GLR_REQUIRE(K >= 1, GLR_ERR_INVALID, "wnnm: K=%d", K);
  GLR_REQUIRE(m >= 1, GLR_ERR_INVALID, "wnnm: m=%d", m);
  GLR_REQUIRE(sigma >= 0, GLR_ERR_INVALID, "noise_sigma must be nonnegative");
  GLR_REQUIRE(c_weight > 0 && eps > 0, GLR_ERR_INVALID, "c_weight and eps must be positive");
  if (G <= 0) return GLR_OK;
  GLR_REQUIRE(ws_bytes >= glr_wnnm_workspace(G, K) - 256, GLR_ERR_WORKSPACE,
              "wnnm: workspace %zu too small", ws_bytes);
  GroupSrc s{};
  s.src = groups_d;
  s.PC = m;
  s.rs = 0;
  s.m = m;
  s.K = K;
  s.vec2 = (m % 2 == 0) && (reinterpret_cast<uintptr_t>(groups_d) % 16 == 0);
  EigArgs ea{};
  ea.K = K;
  ea.sigma = sigma;
  ea.c_weight = c_weight;
  ea.eps = eps;
  ea.uniform_weight = uniform_weight;
  if (K > wn::KMAX)
    return run_wnnm_big<false>(s, G, ea, 1.0, nullptr, out_d, reinterpret_cast<double*>(ws_d),
                               (cudaStream_t)stream);
  return run_wnnm<false>(s, G, ea, 1.0, nullptr, out_d, reinterpret_cast<double*>(ws_d),
                         (cudaStream_t)stream);
}

extern "C" int glr_wnnm_scatter(const double* x_d, int H, int W, int C, int P,
                                const int32_t* positions_d, int n_max, const int32_t* n_dev_d,
                                int K, double sigma, double c_weight, double eps, int frac_bits,
                                int64_t* acc_d, double* vcache_d, int warm,
                                const uint8_t* warm_flags_d, void* ws_d, size_t ws_bytes,
                                void* stream) {
  GLR_REQUIRE(K >= 1, GLR_ERR_INVALID, "wnnm: K=%d", K);
  GLR_REQUIRE(P >= 1 && P <= H && P <= W, GLR_ERR_INVALID, "wnnm_scatter: bad patch size");
  GLR_REQUIRE(frac_bits >= 0 && frac_bits <= 52, GLR_ERR_INVALID, "frac_bits %d", frac_bits);
  GLR_REQUIRE(warm != 2 || warm_flags_d != nullptr, GLR_ERR_INVALID, "warm=2 needs warm flags");
  GLR_REQUIRE(n_dev_d == nullptr, GLR_ERR_UNSUPPORTED, "wnnm_scatter: device-side count unsupported");
  if (n_max <= 0) return GLR_OK;
  GLR_REQUIRE(ws_bytes >= glr_wnnm_workspace(n_max, K) - 256, GLR_ERR_WORKSPACE,
              "wnnm_scatter: workspace %zu too small", ws_bytes);
  GroupSrc s{};
  s.src = x_d;
  s.pos = positions_d;
  s.W = W;
  s.H = H;
  s.C = C;
  s.PC = P * C;
  s.rs = (int64_t)W * C;
  s.m = P * P * C;
  s.K = K;
  s.vec2 = (C % 2 == 0) && (reinterpret_cast<uintptr_t>(x_d) % 16 == 0);
  EigArgs ea{};
  ea.K = K;
  ea.sigma = sigma;
  ea.c_weight = c_weight;
  ea.eps = eps;
  ea.uniform_weight = -1.0;
  if (K > wn::KMAX)  // generic path: cold, no eigenvector cache
    return run_wnnm_big<true>(s, n_max, ea, ldexp(1.0, frac_bits), acc_d, nullptr,
                              reinterpret_cast<double*>(ws_d), (cudaStream_t)stream);
  ea.vcache = vcache_d;
  ea.warm = warm;
  ea.warm_flags = warm_flags_d;
  return run_wnnm<true>(s, n_max, ea, ldexp(1.0, frac_bits), acc_d, nullptr,
                        reinterpret_cast<double*>(ws_d), (cudaStream_t)stream);
}

extern "C" int glr_vcache_remap(const int32_t* old_anchors_d, int old_lo, int old_hi,
                                const int32_t* new_anchors_d, int new_lo, int new_hi, int H,
                                int W, const double* vc_old_d, double* vc_new_d,
                                uint8_t* flags_d, int32_t* map_d, const int32_t* old_pos_d,
                                const int32_t* new_pos_d, int K, void* stream) {
  GLR_REQUIRE((old_pos_d == nullptr) == (new_pos_d == nullptr), GLR_ERR_INVALID,
              "vcache_remap: give both position lists or neither");
  GLR_REQUIRE(old_pos_d == nullptr || (K >= 1 && K <= wn::KMAX), GLR_ERR_INVALID,
              "vcache_remap: K=%d", K);
  cudaStream_t st = (cudaStream_t)stream;
  if (old_hi > old_lo) {
    anchor_map_kernel<<<blocks_for(old_hi - old_lo), 256, 0, st>>>(old_anchors_d, old_lo, old_hi,
                                                                  W, map_d, 1);
    GLR_CUDA(cudaGetLastError());
  }
  if (new_hi > new_lo) {
    vcache_remap_kernel<<<new_hi - new_lo, 256, 0, st>>>(new_anchors_d, new_lo, W, map_d,
                                                        vc_old_d, vc_new_d, flags_d, old_pos_d,
                                                        new_pos_d, K);
    GLR_CUDA(cudaGetLastError());
  }
  if (old_hi > old_lo) {
    anchor_map_kernel<<<blocks_for(old_hi - old_lo), 256, 0, st>>>(old_anchors_d, old_lo, old_hi,
                                                                  W, map_d, 0);
    GLR_CUDA(cudaGetLastError());
  }
  return GLR_OK;
}

extern "C" int glr_scatter_count(const int32_t* positions_d, int n_max, const int32_t* n_dev_d,
                                 int K, int P, int H, int W, int32_t* cnt_d, void* stream) {
  if (n_max <= 0) return GLR_OK;
  scatter_count_kernel<<<blocks_for((int64_t)n_max * K * P * P), 256, 0, (cudaStream_t)stream>>>(
      positions_d, n_max, n_dev_d, K, P, W, cnt_d);
  return check_launch("scatter_count_kernel");
}

extern "C" int glr_scatter_add_f64(const double* groups_d, const int32_t* positions_d, int G, int K,
                                   int P, int H, int W, int C, double* acc_d, double* cnt_d,
                                   void* stream) {
  scatter_f64_kernel<<<blocks_for((int64_t)H * W * C), 256, 0, (cudaStream_t)stream>>>(
      groups_d, positions_d, G, K, P, H, W, C, acc_d, cnt_d);
  return check_launch("scatter_f64_kernel");
}

extern "C" int glr_scatter_fixed(const double* groups_d, const int32_t* positions_d, int G, int K,
                                 int P, int H, int W, int C, int frac_bits, int64_t* acc_d,
                                 void* stream) {
  GLR_REQUIRE(frac_bits >= 0 && frac_bits <= 52, GLR_ERR_INVALID, "frac_bits %d", frac_bits);
  const int64_t total = (int64_t)G * K * P * P * C;
  if (total == 0) return GLR_OK;
  scatter_fixed_kernel<<<blocks_for(total), 256, 0, (cudaStream_t)stream>>>(
      groups_d, positions_d, G, K, P, W, C, ldexp(1.0, frac_bits), acc_d);
  return check_launch("scatter_fixed_kernel");
}

extern "C" int glr_normalize(int64_t* acc_d, const int32_t* cnt_d, const double* x_d, int H,
                             int W, int C, int frac_bits, double* z_d, void* stream) {
  const int64_t npix = (int64_t)H * W;
  normalize_kernel<<<blocks_for(npix * C), 256, 0, (cudaStream_t)stream>>>(
      acc_d, cnt_d, x_d, npix, C, ldexp(1.0, -frac_bits), z_d);
  return check_launch("normalize_kernel");
}
