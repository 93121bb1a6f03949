// Block matching (local KNN by squared pixel distance) and the pixel-L2
// re-rank of global-match groups.
//
//  * glr_block_match  — glr/matching.py:256-283 (`block_match`): for every
//    exemplar, all window positions within `bm_window` (at `bm_stride`),
//    distance d = ((cand - ref)**2).sum(axis=(2,3,4)), the K-1 nearest by
//    (d, row, col) after the exemplar itself, anchor padding.
//  * glr_rerank_pixel — glr/matching.py:243-249 (`rerank_pixel`): slot 0
//    stays, slots 1.. are re-ordered by (pixel distance to the anchor patch,
//    (row, col)).
//
// Distances are bit-identical to numpy's:
//  * block_match: the broadcast difference is a fresh (rows, cols, C, P, P)
//    array whose memory order is (p, q, c), so the 3-axis sum is ONE
//    pairwise summation (numpy loops_utils pairwise_sum, blocks of <= 128
//    with 8 accumulators) over the m = P*P*C squared differences of a patch
//    in (p, q, c) order. The recursion only depends on m: the host turns it
//    into a post-order plan (leaf lengths and adds) that every thread replays
//    on its own candidate.
//  * rerank: `((cand.matrix - ref[:, None]) ** 2).sum(axis=0)` reduces the
//    outer axis of an (m, K) array, i.e. a sequential sum over (p, q, c).
// Each difference is squared as (a - b) * (a - b) with no FMA contraction.
//
// Layout: one CTA per exemplar. The reference patch lives in shared memory;
// the window is walked in bands of candidate rows, each band's image rows
// staged in shared memory with an odd pixel stride (C or C + 1 doubles) so
// a warp's 32 candidates (consecutive columns) hit 32 distinct bank pairs.
// Candidate (distance, ordinal) keys collect in a 2048-entry buffer that is
// bitonic-sorted and cut to the best K-1 whenever it would overflow.

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "internal.cuh"

namespace glr {
namespace bm {
constexpr int THREADS = 512;
constexpr int SORT_CAP = 2048;
constexpr int MAX_PLAN = 512;
constexpr int STACK = 16;
constexpr uint64_t NONE = ~0ull;   // the exemplar's own position / empty slot
}  // namespace bm

struct BmArgs {
  const double* x;
  int H, W, C, P;
  const int32_t* anchors;
  int window, stride, K;
  int32_t* positions;
  int32_t* padded;
  int band;   // candidate rows per band
  int cs;     // shared-memory pixel stride in doubles (odd)
  int ncw;    // staged pixel columns (max over exemplars)
  int n_ops;
  int16_t ops[bm::MAX_PLAN];  // > 0: leaf of that many elements, 0: add top two
};

// Post-order plan of numpy's pairwise_sum recursion for n elements.
static void pairwise_plan(int n, std::vector<int16_t>& ops) {
  if (n <= 128) {
    ops.push_back((int16_t)n);
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  pairwise_plan(n2, ops);
  pairwise_plan(n - n2, ops);
  ops.push_back(0);
}

// Walks the elements of one candidate patch in (p, q, c) order over the
// staged band: offset advances by 1 inside a pixel, by (cs - C) + 1 across
// pixels and by the band row stride across patch rows.
struct PatchWalk {
  int off, c, q;
  int C, P, cs, rowskip;  // rowskip = row stride - P*cs
  __device__ __forceinline__ void next() {
    ++off;
    if (++c == C) {
      c = 0;
      off += cs - C;
      if (++q == P) {
        q = 0;
        off += rowskip;
      }
    }
  }
};

__device__ __forceinline__ double sqdiff(double a, double b) {
  const double d = __dsub_rn(a, b);
  return __dmul_rn(d, d);
}

// numpy pairwise leaf over `len` elements starting at the walk position.
__device__ __forceinline__ double pw_leaf(const double* band, const double* ref, int& i,
                                          PatchWalk& w, int len) {
  if (len < 8) {
    double res = 0.0;
    for (int j = 0; j < len; ++j, ++i) {
      res = __dadd_rn(res, sqdiff(band[w.off], ref[i]));
      w.next();
    }
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    r[j] = sqdiff(band[w.off], ref[i + j]);
    w.next();
  }
  int k = 8;
  const int full = len - (len % 8);
  for (; k < full; k += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      r[j] = __dadd_rn(r[j], sqdiff(band[w.off], ref[i + k + j]));
      w.next();
    }
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; k < len; ++k) {
    res = __dadd_rn(res, sqdiff(band[w.off], ref[i + k]));
    w.next();
  }
  i += len;
  return res;
}

// Bitonic sort of n (a power of two) (key, ordinal) pairs, ascending.
__device__ void bitonic_pairs(uint64_t* key, uint32_t* ord, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
        const int i = 2 * j * (t / j) + (t % j);
        const int l = i + j;
        const bool up = (i & k) == 0;
        const uint64_t ka = key[i], kb = key[l];
        const uint32_t oa = ord[i], ob = ord[l];
        const bool gt = ka > kb || (ka == kb && oa > ob);
        if (gt == up) {
          key[i] = kb;
          key[l] = ka;
          ord[i] = ob;
          ord[l] = oa;
        }
      }
      __syncthreads();
    }
  }
}

__device__ int pow2_ceil(int v) {
  int c = 1;
  while (c < v) c <<= 1;
  return c;
}

__global__ void __launch_bounds__(bm::THREADS, 1) block_match_kernel(BmArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int n = blockIdx.x;
  const int H = a.H, W = a.W, C = a.C, P = a.P, s = a.stride;
  const int m = P * P * C;
  double* ref = smem;
  double* band = ref + ((m + 1) & ~1);
  const int rows_max = (a.band - 1) * s + P;
  uint64_t* key = reinterpret_cast<uint64_t*>(band + (size_t)rows_max * a.ncw * a.cs);
  uint32_t* ord = reinterpret_cast<uint32_t*>(key + bm::SORT_CAP);

  const int r0 = a.anchors[2 * n], c0 = a.anchors[2 * n + 1];
  const int rlo = max(0, r0 - a.window), rhi = min(H - P, r0 + a.window);
  const int clo = max(0, c0 - a.window), chi = min(W - P, c0 + a.window);
  const int nr = (rhi - rlo) / s + 1, nc = (chi - clo) / s + 1;
  const int ncw = (nc - 1) * s + P;  // staged pixel columns
  const int rowstride = ncw * a.cs;

  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const int p = i / (P * C), rem = i - p * P * C;
    ref[i] = a.x[((int64_t)(r0 + p) * W + c0) * C + rem];
  }
  int nbuf = 0;
  const int K1 = a.K - 1;

  for (int br = 0; br < nr; br += a.band) {
    const int nrows = min(a.band, nr - br);
    const int img_r0 = rlo + br * s;
    const int img_rows = (nrows - 1) * s + P;
    // stage image rows [img_r0, img_r0 + img_rows) x cols [clo, clo + ncw)
    const int rowlen = ncw * C;
    for (int t = threadIdx.x; t < img_rows * rowlen; t += blockDim.x) {
      const int rr = t / rowlen, e = t - rr * rowlen;
      const int px = e / C, ch = e - px * C;
      band[rr * rowstride + px * a.cs + ch] =
          a.x[((int64_t)(img_r0 + rr) * W + clo) * C + e];
    }
    const int ncand = nrows * nc;
    if (nbuf + ncand > bm::SORT_CAP) {
      // cut the buffer to its best K-1 before this band's candidates land
      const int n2 = pow2_ceil(nbuf);
      for (int t = nbuf + threadIdx.x; t < n2; t += blockDim.x) key[t] = bm::NONE;
      __syncthreads();
      bitonic_pairs(key, ord, n2);
      nbuf = min(nbuf, K1);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ncand; t += blockDim.x) {
      const int ri = t / nc, ci = t - ri * nc;
      const int rr = img_r0 + ri * s, cc = clo + ci * s;
      uint64_t k = bm::NONE;
      if (rr != r0 || cc != c0) {
        PatchWalk w{ri * s * rowstride + ci * s * a.cs, 0, 0, C, P, a.cs,
                    rowstride - P * a.cs};
        double stk[bm::STACK];
        int sp = 0, i = 0;
        for (int o = 0; o < a.n_ops; ++o) {
          const int op = a.ops[o];
          if (op == 0) {
            const double b = stk[--sp];
            stk[sp - 1] = __dadd_rn(stk[sp - 1], b);
          } else {
            stk[sp++] = pw_leaf(band, ref, i, w, op);
          }
        }
        k = (uint64_t)__double_as_longlong(stk[0]);
      }
      key[nbuf + t] = k;
      ord[nbuf + t] = (uint32_t)((br + ri) * nc + ci);
    }
    nbuf += ncand;
    __syncthreads();
  }
  const int n2 = pow2_ceil(max(nbuf, 2));
  for (int t = nbuf + threadIdx.x; t < n2; t += blockDim.x) key[t] = bm::NONE;
  __syncthreads();
  bitonic_pairs(key, ord, n2);
  // positions: anchor, the K-1 nearest (own position and empty slots carry NONE)
  int32_t* out = a.positions + (int64_t)n * a.K * 2;
  for (int j = threadIdx.x; j < a.K; j += blockDim.x) {
    int pr = r0, pc = c0;
    if (j >= 1 && j - 1 < nbuf && key[j - 1] != bm::NONE) {
      const uint32_t o = ord[j - 1];
      pr = rlo + (int)(o / nc) * s;
      pc = clo + (int)(o % nc) * s;
    }
    out[2 * j] = pr;
    out[2 * j + 1] = pc;
  }
  if (threadIdx.x == 0) {
    int real = 0;
    for (int j = 0; j < min(K1, nbuf); ++j) real += key[j] != bm::NONE;
    a.padded[n] = K1 - real;
  }
}

// rerank_pixel: per exemplar, one thread per group slot.
__global__ void rerank_kernel(const double* __restrict__ x, int H, int W, int C, int P,
                              int32_t* __restrict__ pos, int K) {
  extern __shared__ __align__(16) double rsm[];
  const int n = blockIdx.x;
  const int m = P * P * C;
  double* ref = rsm;
  double* dist = ref + m;
  int32_t* rc = reinterpret_cast<int32_t*>(dist + K);
  int32_t* g = pos + (int64_t)n * K * 2;
  const int r0 = g[0], c0 = g[1];
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const int p = i / (P * C), rem = i - p * P * C;
    ref[i] = x[((int64_t)(r0 + p) * W + c0) * C + rem];
  }
  for (int j = threadIdx.x; j < 2 * K; j += blockDim.x) rc[j] = g[j];
  __syncthreads();
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const int r = rc[2 * j], c = rc[2 * j + 1];
    double d = 0.0;
    int i = 0;
    for (int p = 0; p < P; ++p) {
      const double* row = x + ((int64_t)(r + p) * W + c) * C;
      for (int e = 0; e < P * C; ++e, ++i) d = __dadd_rn(d, sqdiff(row[e], ref[i]));
    }
    dist[j] = d;
  }
  __syncthreads();
  // stable rank of slot j among slots 1..K-1 by (d, (row, col)); sorted() is
  // stable, so equal keys keep slot order
  for (int j = 1 + threadIdx.x; j < K; j += blockDim.x) {
    const double dj = dist[j];
    const int rj = rc[2 * j], cj = rc[2 * j + 1];
    int rank = 0;
    for (int i = 1; i < K; ++i) {
      const double di = dist[i];
      const int ri = rc[2 * i], ci = rc[2 * i + 1];
      const bool less = di < dj || (di == dj && (ri < rj || (ri == rj && (ci < cj ||
                                                  (ci == cj && i < j)))));
      rank += less;
    }
    g[2 * (1 + rank)] = rj;
    g[2 * (1 + rank) + 1] = cj;
  }
}

// xcorr2_valid_batch (matching.py:116-137): out[u][v][n] = sum over (dr, dc,
// ch) of k[n][dr][dc][ch] * x[u+dr][v+dc][ch], accumulated from 0 in that
// order with the product rounded first (the kernel-index loop oracle of the
// reference's tests, bit for bit). One thread per output position, the
// kernel in shared memory (warp-uniform broadcast reads).
__global__ void xcorr_kernel(const double* __restrict__ x, int H, int W, int C,
                             const double* __restrict__ k, int N, int P,
                             double* __restrict__ out) {
  extern __shared__ __align__(16) double ks[];
  const int n = blockIdx.y;
  const int m = P * P * C;
  for (int i = threadIdx.x; i < m; i += blockDim.x) ks[i] = k[(int64_t)n * m + i];
  __syncthreads();
  const int oh = H - P + 1, ow = W - P + 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)oh * ow;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(t / ow), v = (int)(t % ow);
    double acc = 0.0;
    int i = 0;
    for (int dr = 0; dr < P; ++dr) {
      const double* row = x + ((int64_t)(u + dr) * W + v) * C;
      for (int e = 0; e < P * C; ++e, ++i) acc = __dadd_rn(acc, __dmul_rn(ks[i], row[e]));
    }
    out[t * N + n] = acc;
  }
}

}  // namespace glr

using namespace glr;

extern "C" int glr_xcorr_valid(const double* x_d, int H, int W, int C, const double* k_d, int N,
                               int P, double* out_d, void* stream) {
  GLR_REQUIRE(P >= 1 && P <= H && P <= W, GLR_ERR_INVALID, "kernel %dx%d larger than input %dx%d",
              P, P, H, W);
  GLR_REQUIRE(C >= 1 && N >= 0, GLR_ERR_INVALID, "xcorr: bad shape");
  if (N == 0) return GLR_OK;
  const size_t smem = (size_t)P * P * C * 8;
  GLR_REQUIRE(smem <= 227 * 1024, GLR_ERR_UNSUPPORTED, "xcorr: kernel too large");
  { const int s_ = ensure_smem_attr((const void*)xcorr_kernel, (int)smem); if (s_) return s_; }
  const int64_t M = (int64_t)(H - P + 1) * (W - P + 1);
  dim3 grid((unsigned)std::min<int64_t>(cdiv(M, 256), 4 * kNumSMs), (unsigned)N);
  xcorr_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(x_d, H, W, C, k_d, N, P, out_d);
  return check_launch("xcorr_kernel");
}

extern "C" int glr_block_match(const double* x_d, int H, int W, int C, int P,
                               const int32_t* anchors_d, int n, int window, int stride, int K,
                               int32_t* positions_d, int32_t* padded_d, void* stream) {
  GLR_REQUIRE(P >= 2 && P <= H && P <= W, GLR_ERR_INVALID, "patch size %d exceeds image %dx%d",
              P, H, W);
  GLR_REQUIRE(C >= 1, GLR_ERR_INVALID, "block_match: bad channel count %d", C);
  GLR_REQUIRE(K >= 1, GLR_ERR_INVALID, "group_size must be >= 1");
  GLR_REQUIRE(window >= 0, GLR_ERR_INVALID, "bm_window must be >= 0");
  GLR_REQUIRE(stride >= 1, GLR_ERR_INVALID, "bm_stride must be >= 1");
  GLR_REQUIRE(K - 1 <= 1024, GLR_ERR_UNSUPPORTED, "block_match: group_size %d above 1025", K);
  if (n <= 0) return GLR_OK;
  const int m = P * P * C;
  GLR_REQUIRE(m <= 8192, GLR_ERR_UNSUPPORTED, "block_match: patch of %d values above 8192", m);
  BmArgs a{};
  std::vector<int16_t> ops;
  pairwise_plan(m, ops);
  GLR_REQUIRE((int)ops.size() <= bm::MAX_PLAN, GLR_ERR_UNSUPPORTED, "block_match: plan too long");
  a.n_ops = (int)ops.size();
  std::copy(ops.begin(), ops.end(), a.ops);
  a.x = x_d;
  a.H = H, a.W = W, a.C = C, a.P = P;
  a.anchors = anchors_d;
  a.window = window, a.stride = stride, a.K = K;
  a.positions = positions_d;
  a.padded = padded_d;
  a.cs = (C % 2) ? C : C + 1;
  const int nc_max = std::min(2 * window, W - P) / stride + 1;
  a.ncw = std::min((nc_max - 1) * stride + P, W);
  const size_t fixed = (size_t)((m + 1) & ~1) * 8 + (size_t)bm::SORT_CAP * 12;
  const size_t row_bytes = (size_t)a.ncw * a.cs * 8;
  const size_t budget = 200 * 1024;
  // largest band (candidate rows) that fits; at least one row of candidates
  int band = 1;
  const int nr_max = std::min(2 * window, H - P) / stride + 1;
  while (band < nr_max && fixed + (size_t)(band * stride + P) * row_bytes <= budget &&
         (band + 1) * nc_max <= bm::SORT_CAP - std::max(K - 1, 0) - 1 && band * nc_max < 1024)
    ++band;
  a.band = band;
  GLR_REQUIRE(band * nc_max + (K - 1) <= bm::SORT_CAP, GLR_ERR_UNSUPPORTED,
              "block_match: window row of %d candidates too wide", nc_max);
  const size_t smem = fixed + (size_t)((band - 1) * stride + P) * row_bytes;
  GLR_REQUIRE(smem <= 227 * 1024, GLR_ERR_UNSUPPORTED,
              "block_match: window needs %zu bytes of shared memory", smem);
  { const int s_ = ensure_smem_attr((const void*)block_match_kernel, (int)smem); if (s_) return s_; }
  block_match_kernel<<<n, bm::THREADS, smem, (cudaStream_t)stream>>>(a);
  return check_launch("block_match_kernel");
}

extern "C" int glr_rerank_pixel(const double* x_d, int H, int W, int C, int P,
                                int32_t* positions_d, int n, int K, void* stream) {
  GLR_REQUIRE(P >= 1 && P <= H && P <= W, GLR_ERR_INVALID, "rerank: bad patch size");
  GLR_REQUIRE(K >= 1 && K <= 1024, GLR_ERR_UNSUPPORTED, "rerank: group_size %d", K);
  if (n <= 0 || K == 1) return GLR_OK;
  const size_t smem = (size_t)P * P * C * 8 + (size_t)K * 16;
  GLR_REQUIRE(smem <= 227 * 1024, GLR_ERR_UNSUPPORTED, "rerank: patch too large");
  { const int s_ = ensure_smem_attr((const void*)rerank_kernel, (int)smem); if (s_) return s_; }
  const int threads = std::min(1024, std::max(64, (K + 31) / 32 * 32));
  rerank_kernel<<<n, threads, smem, (cudaStream_t)stream>>>(x_d, H, W, C, P, positions_d, K);
  return check_launch("rerank_kernel");
}
