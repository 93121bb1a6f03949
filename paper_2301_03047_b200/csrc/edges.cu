// (1) Edge maps and exemplar detection, fp64, bitwise equal to the reference.
//
// Reference: glr/edges.py:53-162 and glr/solvers.py:154-167. The reference
// evaluates these with scipy.ndimage (C loops) and numpy; the decision stages
// (thresholds, corner ranking) are integer decisions on fp64 values, so the
// kernels here reproduce the exact fp64 operation order of those libraries
// (no FMA contraction: every add/mul is an explicit __dadd_rn/__dmul_rn):
//   * correlate(img, SOBEL, mode="nearest"): acc = 0; acc += w*x over the
//     non-zero taps in row-major order, edge-replicate indexing;
//   * x.mean(axis=2) on a C-contiguous array: numpy pairwise summation
//     (8-way unrolled blocks, recursive halving above 128) then / C;
//   * uniform_filter(size=3, mode="nearest"): per 1-D line a running sum
//     t = (p0+p1)+p2, out = t/3, t += (p[i+2]-p[i-1]); axis 0 then axis 1;
//   * lambda_min = 0.5*((sxx+syy) - sqrt((sxx-syy)^2 + 4*(sxy^2))).
#include <cub/cub.cuh>

#include "common.cuh"
#include "internal.cuh"

namespace glr {

// ---------------------------------------------------------------------------
// fp64 helpers

// Sobel taps (edges.py:18-21): SOBEL_H = [[-1,0,1],[-2,0,2],[-1,0,1]],
// SOBEL_V = SOBEL_H^T. Accumulated in scipy's order over non-zero taps.
template <typename F>
__device__ __forceinline__ double sobel_h(F X, int r0, int r, int r2, int c0, int c, int c2) {
  double acc = 0.0;
  acc = __dadd_rn(acc, -X(r0, c0));
  acc = __dadd_rn(acc, X(r0, c2));
  acc = __dadd_rn(acc, __dmul_rn(-2.0, X(r, c0)));
  acc = __dadd_rn(acc, __dmul_rn(2.0, X(r, c2)));
  acc = __dadd_rn(acc, -X(r2, c0));
  acc = __dadd_rn(acc, X(r2, c2));
  return acc;
}

template <typename F>
__device__ __forceinline__ double sobel_v(F X, int r0, int r, int r2, int c0, int c, int c2) {
  double acc = 0.0;
  acc = __dadd_rn(acc, -X(r0, c0));
  acc = __dadd_rn(acc, __dmul_rn(-2.0, X(r0, c)));
  acc = __dadd_rn(acc, -X(r0, c2));
  acc = __dadd_rn(acc, X(r2, c0));
  acc = __dadd_rn(acc, __dmul_rn(2.0, X(r2, c)));
  acc = __dadd_rn(acc, X(r2, c2));
  return acc;
}

// Order-preserving map double -> uint64 (for max reductions and radix keys).
__device__ __forceinline__ uint64_t ord64(double d) {
  uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord64(uint64_t k) {
  uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

// numpy pairwise summation of n doubles at stride 1 (numpy/_core loops_utils).
__device__ double pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(a, n2), pairwise_sum(a + n2, n - n2));
}

// ---------------------------------------------------------------------------
// A1: per-channel Sobel (edges.py:53-64)

// IDX: int for images below 2^31 elements (cheaper index division), else int64_t
template <typename IDX>
__global__ void sobel_kernel(const double* __restrict__ x, int H, int W, int C,
                             double* __restrict__ gh, double* __restrict__ gv) {
  const IDX total = (IDX)H * W * C;
  for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total;
       i += (IDX)gridDim.x * blockDim.x) {
    const int ch = (int)(i % C);
    const IDX pix = i / C;
    const int r = (int)(pix / W), c = (int)(pix - (IDX)r * W);
    const int r0 = max(r - 1, 0), r2 = min(r + 1, H - 1);
    const int c0 = max(c - 1, 0), c2 = min(c + 1, W - 1);
    auto X = [&](int rr, int cc) { return x[((int64_t)rr * W + cc) * C + ch]; };
    gh[i] = sobel_h(X, r0, r, r2, c0, c, c2);
    gv[i] = sobel_v(X, r0, r, r2, c0, c, c2);
  }
}

// ---------------------------------------------------------------------------
// A2: sign-split binarization (edges.py:67-85) into maps and/or the expanded
// im2col stack consumed by heat_gemm.cu.

__global__ void absmax_kernel(const double* __restrict__ gh, const double* __restrict__ gv,
                              int64_t n, unsigned long long* out) {
  double mh = 0.0, mv = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    mh = fmax(mh, fabs(gh[i]));
    mv = fmax(mv, fabs(gv[i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mh = fmax(mh, __shfl_xor_sync(0xffffffffu, mh, o));
    mv = fmax(mv, __shfl_xor_sync(0xffffffffu, mv, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], (unsigned long long)__double_as_longlong(mh));
    atomicMax(&out[1], (unsigned long long)__double_as_longlong(mv));
  }
}

struct EdgeTh {
  double th;
  int relative;
};

__device__ __forceinline__ void edge_thresholds(const unsigned long long* mx, EdgeTh t, double& th_h,
                                                double& th_v) {
  if (t.relative) {
    th_h = __dmul_rn(t.th, __longlong_as_double((long long)mx[0]));
    th_v = __dmul_rn(t.th, __longlong_as_double((long long)mx[1]));
  } else {
    th_h = t.th;
    th_v = t.th;
  }
}

// map m in {0: h_pos, 1: h_neg, 2: v_pos, 3: v_neg}
__device__ __forceinline__ uint8_t edge_bit(double g, int m, double th_h, double th_v) {
  const double th = (m < 2) ? th_h : th_v;
  const double s = (m & 1) ? -g : g;
  return fmax(s, 0.0) > th ? 1 : 0;
}

__global__ void edge_maps_kernel(const double* __restrict__ gh, const double* __restrict__ gv,
                                 int H, int W, int C, EdgeTh t, const unsigned long long* mx,
                                 uint8_t* __restrict__ maps) {
  double th_h, th_v;
  edge_thresholds(mx, t, th_h, th_v);
  const int64_t plane = (int64_t)H * W * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 4 * plane;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / plane);
    const int64_t j = i - m * plane;
    const double g = (m < 2) ? gh[j] : gv[j];
    maps[i] = edge_bit(g, m, th_h, th_v);
  }
}

// Stack layout (heat_gemm.cu): (H, W, Ce) binary elements, Ce = e*4C, stored
// as packed E2M1 nibbles (1.0 / 0.0), element 2j in the low nibble of byte j.
// One thread per pixel walks its Ce elements in order (p, map, channel) with
// running counters (no per-element index division) and stores the nibbles
// eight at a time as 32-bit words (Cb = Ce/2 bytes per pixel, a multiple of
// 4 whenever e*C is even -- always for the GEMM's e), byte-wise otherwise.
template <bool WORDS>
__global__ void edge_stack_kernel(const double* __restrict__ gh, const double* __restrict__ gv,
                                  int H, int W, int C, int e, EdgeTh t,
                                  const unsigned long long* mx, uint8_t* __restrict__ stack) {
  double th_h, th_v;
  edge_thresholds(mx, t, th_h, th_v);
  const int Cb = e * 2 * C;
  const int64_t npix = (int64_t)H * W;
  for (int64_t pix = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pix < npix;
       pix += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(pix / W);
    uint8_t* out = stack + pix * Cb;
    uint32_t word = 0;
    int nib = 0, nbytes = 0;
    auto emit = [&](uint32_t bit) {
      word |= (bit * kFp4One) << (4 * nib);
      if (++nib == 8) {
        if constexpr (WORDS) {
          *reinterpret_cast<uint32_t*>(out + nbytes) = word;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) out[nbytes + q] = (uint8_t)(word >> (8 * q));
        }
        nbytes += 4;
        word = 0;
        nib = 0;
      }
    };
    for (int p = 0; p < e; ++p) {
      const bool in = r + p < H;
      const int64_t j0 = (pix + (int64_t)p * W) * C;
      for (int m = 0; m < 4; ++m) {
        const double* g = m < 2 ? gh : gv;
        for (int ch = 0; ch < C; ++ch) emit(in ? edge_bit(g[j0 + ch], m, th_h, th_v) : 0u);
      }
    }
    for (int q = 0; 2 * q < nib; ++q) out[nbytes + q] = (uint8_t)(word >> (8 * q));  // tail
  }
}

__global__ void stack_from_maps_kernel(const uint8_t* __restrict__ maps, int H, int W, int C,
                                       int e, uint8_t* __restrict__ stack) {
  const int C4 = 4 * C, Ce = e * C4, Cb = Ce / 2;
  const int64_t plane = (int64_t)H * W * C;
  const int64_t total = (int64_t)H * W * Cb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int cb = (int)(i % Cb);
    const int64_t pix = i / Cb;
    const int r = (int)(pix / W), c = (int)(pix % W);
    uint8_t byte = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ce = 2 * cb + h;
      const int p = ce / C4, k = ce % C4, m = k / C, ch = k % C;
      if (r + p < H && maps[m * plane + ((int64_t)(r + p) * W + c) * C + ch])
        byte |= kFp4One << (4 * h);
    }
    stack[i] = byte;
  }
}

// ---------------------------------------------------------------------------
// A3: Shi-Tomasi response (edges.py:88-97, 110-112)

// per-channel gradient magnitude sqrt(gh^2 + gv^2), (H,W,C)
__global__ void grad_mag_kernel(const double* __restrict__ x, int H, int W, int C,
                                double* __restrict__ t) {
  const int64_t total = (int64_t)H * W * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % C);
    const int64_t pix = i / C;
    const int r = (int)(pix / W), c = (int)(pix % W);
    const int r0 = max(r - 1, 0), r2 = min(r + 1, H - 1);
    const int c0 = max(c - 1, 0), c2 = min(c + 1, W - 1);
    auto X = [&](int rr, int cc) { return x[((int64_t)rr * W + cc) * C + ch]; };
    const double a = sobel_h(X, r0, r, r2, c0, c, c2);
    const double b = sobel_v(X, r0, r, r2, c0, c, c2);
    t[i] = __dsqrt_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
  }
}

__global__ void channel_mean_kernel(const double* __restrict__ t, int64_t npix, int C,
                                    double* __restrict__ mag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x)
    mag[i] = __ddiv_rn(pairwise_sum(t + i * C, C), (double)C);
}

// mag = mean_c sqrt(gh^2 + gv^2) straight from stored Sobel gradients (the
// same values grad_mag_kernel recomputes from x): the block stages its 256
// pixels' per-channel magnitudes in shared memory with coalesced loads (row
// stride C|1 doubles: conflict-free per-thread rows), then each thread takes
// numpy's pairwise mean of its row.
__global__ void grad_mean_kernel(const double* __restrict__ gh, const double* __restrict__ gv,
                                 int64_t npix, int C, double* __restrict__ mag) {
  extern __shared__ double tm[];
  const int ld = C | 1;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x; p0 < npix;
       p0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t left = npix - p0;
    const int np = left < (int64_t)blockDim.x ? (int)left : (int)blockDim.x;
    const int64_t e0 = p0 * C;
    const int ne = np * C;
    for (int e = threadIdx.x; e < ne; e += 4 * blockDim.x) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // four independent loads in flight
        const int eu = e + u * blockDim.x;
        a[u] = eu < ne ? gh[e0 + eu] : 0.0;
        b[u] = eu < ne ? gv[e0 + eu] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int eu = e + u * blockDim.x;
        if (eu < ne) {
          const int q = eu / C;
          tm[q * ld + (eu - q * C)] =
              __dsqrt_rn(__dadd_rn(__dmul_rn(a[u], a[u]), __dmul_rn(b[u], b[u])));
        }
      }
    }
    __syncthreads();
    if ((int)threadIdx.x < np)
      mag[p0 + threadIdx.x] = __ddiv_rn(pairwise_sum(tm + threadIdx.x * ld, C), (double)C);
    __syncthreads();
  }
}

// structure-tensor products of the Sobel gradients of mag
__global__ void st_products_kernel(const double* __restrict__ mag, int H, int W,
                                   double* __restrict__ pxx, double* __restrict__ pyy,
                                   double* __restrict__ pxy) {
  const int64_t total = (int64_t)H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / W), c = (int)(i % W);
    const int r0 = max(r - 1, 0), r2 = min(r + 1, H - 1);
    const int c0 = max(c - 1, 0), c2 = min(c + 1, W - 1);
    auto X = [&](int rr, int cc) { return mag[(int64_t)rr * W + cc]; };
    const double gx = sobel_h(X, r0, r, r2, c0, c, c2);
    const double gy = sobel_v(X, r0, r, r2, c0, c, c2);
    pxx[i] = __dmul_rn(gx, gx);
    pyy[i] = __dmul_rn(gy, gy);
    pxy[i] = __dmul_rn(gx, gy);
  }
}

// 1-D running-sum box filter of width 3 with edge-replicate, along a line of
// n samples at stride `step` (scipy uniform_filter1d order).
__device__ __forceinline__ void box3_line(const double* __restrict__ in, double* __restrict__ out,
                                          int n, int64_t step) {
  auto P = [&](int j) {  // extended line p[j] = a[clamp(j-1, 0, n-1)]
    int k = min(max(j - 1, 0), n - 1);
    return in[k * step];
  };
  double t = __dadd_rn(__dadd_rn(P(0), P(1)), P(2));
  out[0] = __ddiv_rn(t, 3.0);
  // the recurrence is sequential (bitwise scipy order); the loads are not:
  // fetch CH samples ahead so only the two adds sit on the dependency chain
  constexpr int CH = 16;
  for (int i0 = 1; i0 < n; i0 += CH) {
    double nx[CH], pv[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      nx[c] = P(i0 + c + 2);
      pv[c] = P(i0 + c - 1);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (i0 + c < n) {
        t = __dadd_rn(t, __dsub_rn(nx[c], pv[c]));
        out[(int64_t)(i0 + c) * step] = __ddiv_rn(t, 3.0);
      }
    }
  }
}

// axis 0 (down each column) for the three products
__global__ void box3_cols_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                 const double* __restrict__ c, int H, int W,
                                 double* __restrict__ oa, double* __restrict__ ob,
                                 double* __restrict__ oc) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int which = blockIdx.y;
  if (col >= W) return;
  const double* in = which == 0 ? a : (which == 1 ? b : c);
  double* out = which == 0 ? oa : (which == 1 ? ob : oc);
  box3_line(in + col, out + col, H, W);
}

// axis 1 (along each row) for the three products
__global__ void box3_rows_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                 const double* __restrict__ c, int H, int W,
                                 double* __restrict__ oa, double* __restrict__ ob,
                                 double* __restrict__ oc) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int which = blockIdx.y;
  if (row >= H) return;
  const double* in = which == 0 ? a : (which == 1 ? b : c);
  double* out = which == 0 ? oa : (which == 1 ? ob : oc);
  box3_line(in + (int64_t)row * W, out + (int64_t)row * W, W, 1);
}

__global__ void min_eig_kernel(const double* __restrict__ sxx, const double* __restrict__ syy,
                               const double* __restrict__ sxy, int64_t n,
                               double* __restrict__ resp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double a = sxx[i], b = syy[i], c = sxy[i];
    const double tr = __dadd_rn(a, b);
    const double d = __dsub_rn(a, b);
    const double disc = __dsqrt_rn(__dadd_rn(__dmul_rn(d, d), __dmul_rn(4.0, __dmul_rn(c, c))));
    resp[i] = __dmul_rn(0.5, __dsub_rn(tr, disc));
  }
}

// ---------------------------------------------------------------------------
// A3: candidate ordering + greedy NMS (edges.py:113-128)

__global__ void resp_max_kernel(const double* __restrict__ resp, int64_t n,
                                unsigned long long* out) {
  unsigned long long m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)ord64(resp[i]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// key = order-preserving code of the response for candidates (resp >=
// quality * max, only when max > 0), 0 otherwise; values = flat index.
__global__ void cand_keys_kernel(const double* __restrict__ resp, int64_t n, double quality,
                                 const unsigned long long* mx, uint64_t* __restrict__ keys,
                                 int32_t* __restrict__ idx, int* __restrict__ n_cand) {
  const double rmax = unord64(*mx);
  const double thr = __dmul_rn(quality, rmax);
  const bool any = rmax > 0.0;
  int cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = resp[i];
    const bool c = any && v >= thr;
    keys[i] = c ? ord64(v) : 0ull;
    idx[i] = (int32_t)i;
    cnt += c;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_cand, cnt);
}

__global__ void __launch_bounds__(1024) nms_kernel(const uint64_t* __restrict__ keys,
                                                   const int32_t* __restrict__ idx, int64_t total,
                                                   int H, int W, int max_n, int R,
                                                   uint8_t* __restrict__ blocked,
                                                   int32_t* __restrict__ out_rc,
                                                   int32_t* __restrict__ out_n) {
  __shared__ int s_surv[1024];
  __shared__ int s_new[1024];
  __shared__ int warp_tot[32];
  __shared__ int s_nsurv, s_nnew, s_picked;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_picked = 0;
  __syncthreads();
  for (int64_t base = 0; base < total; base += blockDim.x) {
    if (keys[base] == 0) break;  // sorted descending: no candidates left
    const int64_t i = base + tid;
    const bool valid = i < total && keys[i] != 0;
    const int cand = valid ? idx[i] : -1;
    const bool ok = valid && !blocked[cand];
    const int pos = block_excl_scan_1024(ok ? 1 : 0, warp_tot, &s_nsurv);
    if (ok) s_surv[pos] = cand;
    __syncthreads();
    if (warp == 0) {
      int nnew = 0, picked = s_picked;
      const int ns = s_nsurv;
      for (int j = 0; j < ns && picked < max_n; ++j) {
        const int cidx = s_surv[j];
        const int r = cidx / W, c = cidx - (cidx / W) * W;
        bool conflict = false;
        for (int t = lane; t < nnew; t += 32) {
          const int q = s_new[t];
          const int qr = q / W, qc = q - (q / W) * W;
          if (max(abs(r - qr), abs(c - qc)) <= R) conflict = true;
        }
        conflict = __any_sync(0xffffffffu, conflict);
        if (!conflict) {
          if (lane == 0) s_new[nnew] = cidx;
          ++nnew;
          ++picked;
        }
        __syncwarp();
      }
      if (lane == 0) s_nnew = nnew;
    }
    __syncthreads();
    const int nnew = s_nnew, picked0 = s_picked;
    for (int t = tid; t < nnew; t += blockDim.x) {
      const int q = s_new[t];
      out_rc[2 * (picked0 + t)] = q / W;
      out_rc[2 * (picked0 + t) + 1] = q % W;
    }
    const int win = 2 * R + 1;
    const int cells = nnew * win * win;
    for (int t = tid; t < cells; t += blockDim.x) {
      const int k = t / (win * win), o = t % (win * win);
      const int q = s_new[k];
      const int rr = q / W + o / win - R, cc = q % W + o % win - R;
      if (rr >= 0 && rr < H && cc >= 0 && cc < W) blocked[(int64_t)rr * W + cc] = 1;
    }
    __syncthreads();
    if (tid == 0) s_picked = picked0 + nnew;
    __syncthreads();
    if (s_picked >= max_n) break;
  }
  if (tid == 0) *out_n = s_picked;
}

// Same greedy NMS with the blocked set as a shared-memory BITMAP (one bit per
// pixel: 128 KB for 1024 x 1024): one warp walks the ranked candidates 32 at
// a time (prefetched 256 ahead); the first unblocked lane is the next pick
// (exactly the sequential rule), its (2R+1)-row neighbourhood is or-ed into
// the bitmap by 2R+1 lanes, and the remaining lanes are re-tested.
__global__ void __launch_bounds__(1024) nms_bitmap_kernel(const int32_t* __restrict__ idx,
                                                          const int* __restrict__ n_cand, int H,
                                                          int W, int max_n, int R,
                                                          int32_t* __restrict__ out_rc,
                                                          int32_t* __restrict__ out_n) {
  extern __shared__ uint32_t bm[];
  const int nw = (int)(((int64_t)H * W + 31) / 32);
  for (int i = threadIdx.x; i < nw; i += blockDim.x) bm[i] = 0u;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const unsigned full = 0xffffffffu;
  const int total = *n_cand;  // ranked candidates idx[0 .. total)
  constexpr int U = 8;        // batches of 32 fetched per round trip (double-buffered)
  int cur[U], nxt[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = u * 32 + lane;
    cur[u] = i < total ? idx[i] : -1;
  }
  int picked = 0;
  for (int base = 0; base < total && picked < max_n; base += 32 * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + 32 * U + u * 32 + lane;
      nxt[u] = i < total ? idx[i] : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int cand = cur[u];
      if (__ballot_sync(full, cand >= 0) == 0u || picked >= max_n) break;
      const int r = cand >= 0 ? cand / W : 0, c = cand >= 0 ? cand - (cand / W) * W : 0;
      bool live = cand >= 0;
      while (true) {
        const bool free_px = live && !((bm[cand >> 5] >> (cand & 31)) & 1u);
        const unsigned m = __ballot_sync(full, free_px);
        if (m == 0u) break;
        const int first = __ffs(m) - 1;
        const int pr = __shfl_sync(full, r, first), pc = __shfl_sync(full, c, first);
        if (lane == 0) {
          out_rc[2 * picked] = pr;
          out_rc[2 * picked + 1] = pc;
        }
        ++picked;
        if (lane <= 2 * R) {
          const int rr = pr - R + lane;
          if (rr >= 0 && rr < H) {
            const int64_t b0 = (int64_t)rr * W + max(pc - R, 0);
            const int64_t b1 = (int64_t)rr * W + min(pc + R, W - 1);
            const int w0 = (int)(b0 >> 5), w1 = (int)(b1 >> 5);
            const unsigned lo = ~0u << (b0 & 31);
            const unsigned hi = (b1 & 31) == 31 ? ~0u : ((1u << ((b1 & 31) + 1)) - 1u);
            if (w0 == w1) {
              atomicOr(&bm[w0], lo & hi);
            } else {
              atomicOr(&bm[w0], lo);
              atomicOr(&bm[w1], hi);
            }
          }
        }
        __syncwarp();
        if (picked >= max_n) break;
        live = live && lane > first;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
  if (lane == 0) *out_n = picked;
}

constexpr int kNmsBitmapMaxBytes = 200 * 1024;

// Batched exact greedy NMS: 1024 ranked candidates per step. A candidate
// blocked by an earlier batch's pick (shared-memory bitmap) is dead; among
// the live ones the sequential rule "picked iff no earlier PICKED live
// candidate lies within Chebyshev R" is resolved in parallel rounds: a live
// candidate is PICKED once every earlier conflicting live candidate is
// REJECTED, REJECTED as soon as one of them is PICKED (both final, so the
// fixed point is the sequential greedy result, the lexicographically first
// independent set). Picks are emitted in rank order by a block scan, the
// first max_n kept, and their (2R+1)^2 windows or-ed into the bitmap.
namespace nmsb {
constexpr int B = 512;      // candidates per batch (= threads; 1024: 0.67 ms, 256: 0.51 ms on C2)
constexpr int NBR = 8;      // earlier conflicts remembered per candidate
constexpr uint8_t DEAD = 0, UNDEC = 1, PICKED = 2, REJECTED = 3;
constexpr size_t kBatchBytes = (size_t)B * (2 * 4 + NBR * 2 + 1);
}  // namespace nmsb

// GBM: the bitmap of blocked pixels lives in global memory (zeroed by the
// launcher; L2-resident, read with ld.cg and written with atomics, ordered by
// the block barriers) for images whose bitmap exceeds shared memory (C5:
// 2048^2 = 512 KB) -- those used to take the one-warp walk (19.4 ms per C5
// pass with 16 K corners).
template <bool GBM>
__global__ void __launch_bounds__(nmsb::B) nms_batch_kernel(const int32_t* __restrict__ idx,
                                                           const int* __restrict__ n_cand, int H,
                                                           int W, int max_n, int R,
                                                           int32_t* __restrict__ out_rc,
                                                           int32_t* __restrict__ out_n,
                                                           uint32_t* gbm) {
  using namespace nmsb;
  extern __shared__ uint32_t bm_s[];
  const int nw = (int)(((int64_t)H * W + 31) / 32);
  uint32_t* bm = GBM ? gbm : bm_s;
  int32_t* br = reinterpret_cast<int32_t*>(bm_s + (GBM ? 0 : ((nw + 3) & ~3)));
  int32_t* bc = br + B;
  int16_t* nbr = reinterpret_cast<int16_t*>(bc + B);
  uint8_t* st = reinterpret_cast<uint8_t*>(nbr + B * NBR);
  __shared__ int warp_tot[32];
  __shared__ int s_total, s_picked, s_nb, s_pos;
  const int t = threadIdx.x;
  if constexpr (!GBM)
    for (int i = t; i < nw; i += B) bm[i] = 0u;
  if (t == 0) {
    s_picked = 0;
    s_pos = 0;
  }
  __syncthreads();
  const int total = *n_cand;
  while (s_pos < total && s_picked < max_n) {
    // 1. fill the batch with the next B candidates not blocked by earlier
    //    batches' picks, in rank order (stable compaction of 1024-chunks)
    if (t == 0) s_nb = 0;
    __syncthreads();
    while (s_nb < B && s_pos < total) {
      const int pos0 = s_pos, nb0 = s_nb;
      const int i = pos0 + t;
      int cand = 0;
      bool alive = false;
      if (i < total) {
        cand = idx[i];
        GLR_DCHECK(cand >= 0 && (int64_t)cand < (int64_t)H * W);
        const uint32_t word = GBM ? __ldcg(bm + (cand >> 5)) : bm[cand >> 5];
        alive = !((word >> (cand & 31)) & 1u);
      }
      const int e = block_excl_scan_1024(alive ? 1 : 0, warp_tot, &s_total);
      if (alive && nb0 + e < B) {
        const int r = cand / W;
        br[nb0 + e] = r;
        bc[nb0 + e] = cand - r * W;
      }
      if (alive && nb0 + e == B) s_pos = i;  // first candidate left for the next batch
      __syncthreads();
      if (t == 0) {
        if (nb0 + s_total <= B) s_pos = min(total, pos0 + B);
        s_nb = min(B, nb0 + s_total);
      }
      __syncthreads();
    }
    const int nb = s_nb;
    // 2. earlier conflicts inside the batch (Chebyshev <= R)
    const bool live = t < nb;
    const int r = live ? br[t] : 0, c = live ? bc[t] : 0;
    int cnt = 0;
    if (live) {
      for (int j = 0; j < t; ++j) {
        if (abs(br[j] - r) <= R && abs(bc[j] - c) <= R) {
          if (cnt < NBR) nbr[t * NBR + cnt] = (int16_t)j;
          ++cnt;
        }
      }
    }
    st[t] = !live ? DEAD : (cnt == 0 ? PICKED : UNDEC);
    // 3. resolve in rounds (final states only ever set once)
    bool changed;
    do {
      __syncthreads();
      changed = false;
      if (st[t] == UNDEC) {
        bool any_picked = false, all_rejected = true;
        if (cnt <= NBR) {
          for (int q = 0; q < cnt; ++q) {
            const uint8_t s2 = st[nbr[t * NBR + q]];
            any_picked |= s2 == PICKED;
            all_rejected &= s2 == REJECTED;
          }
        } else {  // many earlier conflicts: rescan the batch
          for (int j = 0; j < t; ++j) {
            if (abs(br[j] - r) <= R && abs(bc[j] - c) <= R) {
              const uint8_t s2 = st[j];
              any_picked |= s2 == PICKED;
              all_rejected &= s2 == REJECTED;
            }
          }
        }
        if (any_picked) {
          st[t] = REJECTED;
          changed = true;
        } else if (all_rejected) {
          st[t] = PICKED;
          changed = true;
        }
      }
    } while (__syncthreads_or(changed));
    // 4. emit the picks in rank order, block their windows
    const bool pk = st[t] == PICKED;
    const int slot = s_picked + block_excl_scan_1024(pk ? 1 : 0, warp_tot, &s_total);
    if (pk && slot < max_n) {
      out_rc[2 * slot] = r;
      out_rc[2 * slot + 1] = c;
      for (int rr = max(r - R, 0); rr <= min(r + R, H - 1); ++rr) {
        const int64_t b0 = (int64_t)rr * W + max(c - R, 0);
        const int64_t b1 = (int64_t)rr * W + min(c + R, W - 1);
        for (int64_t w0 = b0 >> 5; w0 <= (b1 >> 5); ++w0) {
          const int64_t lo_b = max(b0, w0 * 32), hi_b = min(b1, w0 * 32 + 31);
          const unsigned lo = ~0u << (lo_b & 31);
          const unsigned hi = (hi_b & 31) == 31 ? ~0u : ((1u << ((hi_b & 31) + 1)) - 1u);
          atomicOr(&bm[w0], lo & hi);
        }
      }
    }
    __syncthreads();
    if (t == 0) s_picked = min(max_n, s_picked + s_total);
    __syncthreads();
  }
  if (t == 0) *out_n = s_picked;
}



// ---------------------------------------------------------------------------
// A4: anchors (edges.py:131-162)

__global__ void __launch_bounds__(1024) anchors_kernel(
    const int32_t* __restrict__ corners, const int32_t* __restrict__ n_corners_d, int max_corners,
    int H, int W, int P, int grid_interval, int max_anchors, int32_t* __restrict__ first,
    int32_t* __restrict__ anchors, uint8_t* __restrict__ tags, int32_t* __restrict__ n_out) {
  __shared__ int warp_tot[32];
  __shared__ int s_total, s_count;
  const int tid = threadIdx.x;
  const int nc = min(*n_corners_d, max_corners);
  const int half = P / 2;
  for (int i = tid; i < nc; i += blockDim.x) {
    const int ar = min(max(corners[2 * i] - half, 0), H - P);
    const int ac = min(max(corners[2 * i + 1] - half, 0), W - P);
    atomicMin(&first[ar * W + ac], i);
  }
  if (tid == 0) s_count = 0;
  __syncthreads();
  // corners, first occurrence of each anchor, in order
  for (int base = 0; base < nc; base += blockDim.x) {
    const int i = base + tid;
    int ar = 0, ac = 0;
    bool keep = false;
    if (i < nc) {
      ar = min(max(corners[2 * i] - half, 0), H - P);
      ac = min(max(corners[2 * i + 1] - half, 0), W - P);
      keep = first[ar * W + ac] == i;
    }
    const int pos = block_excl_scan_1024(keep ? 1 : 0, warp_tot, &s_total);
    const int at = s_count + pos;
    if (keep && at < max_anchors) {
      anchors[2 * at] = ar;
      anchors[2 * at + 1] = ac;
      tags[at] = 0;
    }
    __syncthreads();
    if (tid == 0) s_count += s_total;
    __syncthreads();
  }
  if (grid_interval > 0) {
    const int gr = (H - P) / grid_interval + 1, gc = (W - P) / grid_interval + 1;
    const int ng = gr * gc;
    for (int base = 0; base < ng; base += blockDim.x) {
      const int t = base + tid;
      int r = 0, c = 0;
      bool keep = false;
      if (t < ng) {
        r = (t / gc) * grid_interval;
        c = (t % gc) * grid_interval;
        keep = first[r * W + c] == 0x7f7f7f7f;
      }
      const int pos = block_excl_scan_1024(keep ? 1 : 0, warp_tot, &s_total);
      const int at = s_count + pos;
      if (keep && at < max_anchors) {
        anchors[2 * at] = r;
        anchors[2 * at + 1] = c;
        tags[at] = 1;
      }
      __syncthreads();
      if (tid == 0) s_count += s_total;
      __syncthreads();
    }
  }
  if (tid == 0) *n_out = min(s_count, max_anchors);
}

static int grid_for(int64_t n, int threads = 256) {
  int64_t b = cdiv(n, threads);
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)kNumSMs * 32));
}

}  // namespace glr

using namespace glr;

extern "C" int glr_sobel(const double* x_d, int H, int W, int C, double* gh_d, double* gv_d,
                         void* stream) {
  GLR_REQUIRE(H >= 3 && W >= 3, GLR_ERR_INVALID, "image %dx%d too small for 3x3 Sobel", H, W);
  GLR_REQUIRE(C >= 1, GLR_ERR_INVALID, "channel count %d", C);
  cudaStream_t st = (cudaStream_t)stream;
  int64_t n = (int64_t)H * W * C;
  if (n < (int64_t)INT32_MAX - 65536LL * 256)
    sobel_kernel<int><<<grid_for(n), 256, 0, st>>>(x_d, H, W, C, gh_d, gv_d);
  else
    sobel_kernel<int64_t><<<grid_for(n), 256, 0, st>>>(x_d, H, W, C, gh_d, gv_d);
  return check_launch("sobel_kernel");
}

extern "C" int glr_edge_stack(const double* gh_d, const double* gv_d, int H, int W, int C,
                              double th, int relative, int expand, uint8_t* maps_d,
                              uint8_t* stack_d, double* ws_d, void* stream) {
  GLR_REQUIRE(th >= 0, GLR_ERR_INVALID, "threshold must be nonnegative, got %g", th);
  GLR_REQUIRE(H >= 1 && W >= 1 && C >= 1 && expand >= 1, GLR_ERR_INVALID, "edge_stack: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t n = (int64_t)H * W * C;
  unsigned long long* mx = reinterpret_cast<unsigned long long*>(ws_d);
  GLR_CUDA(cudaMemsetAsync(mx, 0, 2 * sizeof(unsigned long long), st));
  if (relative) {
    absmax_kernel<<<grid_for(n), 256, 0, st>>>(gh_d, gv_d, n, mx);
    GLR_CUDA(cudaGetLastError());
  }
  EdgeTh t{th, relative};
  if (maps_d) {
    edge_maps_kernel<<<grid_for(4 * n), 256, 0, st>>>(gh_d, gv_d, H, W, C, t, mx, maps_d);
    GLR_CUDA(cudaGetLastError());
  }
  if (stack_d) {
    if ((expand * C) % 2 == 0)
      edge_stack_kernel<true><<<grid_for((int64_t)H * W), 256, 0, st>>>(gh_d, gv_d, H, W, C,
                                                                        expand, t, mx, stack_d);
    else
      edge_stack_kernel<false><<<grid_for((int64_t)H * W), 256, 0, st>>>(gh_d, gv_d, H, W, C,
                                                                         expand, t, mx, stack_d);
    GLR_CUDA(cudaGetLastError());
  }
  return GLR_OK;
}

extern "C" int glr_stack_from_maps(const uint8_t* maps_d, int H, int W, int C, int expand,
                                   uint8_t* stack_d, void* stream) {
  GLR_REQUIRE(H >= 1 && W >= 1 && C >= 1 && expand >= 1, GLR_ERR_INVALID,
              "stack_from_maps: bad shape");
  GLR_REQUIRE((4 * C * expand) % 2 == 0, GLR_ERR_INVALID, "stack_from_maps: odd stack width");
  int64_t n = (int64_t)H * W * C * 2 * expand;
  stack_from_maps_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(maps_d, H, W, C, expand,
                                                                       stack_d);
  return check_launch("stack_from_maps_kernel");
}

extern "C" size_t glr_corner_workspace(int H, int W, int C) {
  size_t npix = (size_t)H * W;
  return npix * C * sizeof(double) + 7 * npix * sizeof(double) + 64;
}

extern "C" int glr_corner_response(const double* x_d, int H, int W, int C, double* resp_d,
                                   void* ws_d, void* stream) {
  GLR_REQUIRE(H >= 3 && W >= 3, GLR_ERR_INVALID, "image %dx%d too small for 3x3 Sobel", H, W);
  GLR_REQUIRE(C >= 1, GLR_ERR_INVALID, "channel count %d", C);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npix = (int64_t)H * W;
  double* t = reinterpret_cast<double*>(ws_d);
  double* mag = t + npix * C;
  double* pxx = mag + npix;
  double* pyy = pxx + npix;
  double* pxy = pyy + npix;
  double* qxx = pxy + npix;
  double* qyy = qxx + npix;
  double* qxy = qyy + npix;
  grad_mag_kernel<<<grid_for(npix * C), 256, 0, st>>>(x_d, H, W, C, t);
  channel_mean_kernel<<<grid_for(npix), 256, 0, st>>>(t, npix, C, mag);
  st_products_kernel<<<grid_for(npix), 256, 0, st>>>(mag, H, W, pxx, pyy, pxy);
  box3_cols_kernel<<<dim3((unsigned)cdiv(W, 128), 3), 128, 0, st>>>(pxx, pyy, pxy, H, W, qxx, qyy,
                                                                  qxy);
  box3_rows_kernel<<<dim3((unsigned)cdiv(H, 128), 3), 128, 0, st>>>(qxx, qyy, qxy, H, W, pxx, pyy,
                                                                  pxy);
  min_eig_kernel<<<grid_for(npix), 256, 0, st>>>(pxx, pyy, pxy, npix, resp_d);
  return check_launch("corner_response");
}

// Same response from precomputed Sobel gradients (glr_sobel), skipping the
// second Sobel pass over x.
extern "C" int glr_corner_response_grad(const double* gh_d, const double* gv_d, int H, int W,
                                        int C, double* resp_d, void* ws_d, void* stream) {
  GLR_REQUIRE(H >= 3 && W >= 3, GLR_ERR_INVALID, "image %dx%d too small for 3x3 Sobel", H, W);
  GLR_REQUIRE(C >= 1 && C <= 6000, GLR_ERR_INVALID, "channel count %d", C);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npix = (int64_t)H * W;
  double* mag = reinterpret_cast<double*>(ws_d) + npix * C;  // glr_corner_workspace layout
  double* pxx = mag + npix;
  double* pyy = pxx + npix;
  double* pxy = pyy + npix;
  double* qxx = pxy + npix;
  double* qyy = qxx + npix;
  double* qxy = qyy + npix;
  // 256 pixels per block, fewer for wide channel counts (<= 200 KB staging)
  const int row_bytes = (C | 1) * (int)sizeof(double);
  const int threads = std::max(32, std::min(256, (200 * 1024 / row_bytes) / 32 * 32));
  const int smem = threads * row_bytes;
  if (smem > 48 * 1024) {
    const int s = ensure_smem_attr((const void*)grad_mean_kernel, smem);
    if (s) return s;
  }
  grad_mean_kernel<<<grid_for(npix, threads), threads, smem, st>>>(gh_d, gv_d, npix, C, mag);
  st_products_kernel<<<grid_for(npix), 256, 0, st>>>(mag, H, W, pxx, pyy, pxy);
  box3_cols_kernel<<<dim3((unsigned)cdiv(W, 128), 3), 128, 0, st>>>(pxx, pyy, pxy, H, W, qxx, qyy,
                                                                  qxy);
  box3_rows_kernel<<<dim3((unsigned)cdiv(H, 128), 3), 128, 0, st>>>(qxx, qyy, qxy, H, W, pxx, pyy,
                                                                  pxy);
  min_eig_kernel<<<grid_for(npix), 256, 0, st>>>(pxx, pyy, pxy, npix, resp_d);
  return check_launch("corner_response_grad");
}

static size_t nms_sort_temp(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending((void*)nullptr, bytes, (const uint64_t*)nullptr,
                                            (uint64_t*)nullptr, (const int32_t*)nullptr,
                                            (int32_t*)nullptr, (int)n);
  return bytes;
}

extern "C" size_t glr_nms_workspace(int H, int W) {
  int64_t n = (int64_t)H * W;
  return 256 + n * (2 * sizeof(uint64_t) + 2 * sizeof(int32_t) + 1) + nms_sort_temp(n) + 1024;
}

static inline uint8_t* align256(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
}

extern "C" int glr_corners(const double* resp_d, int H, int W, int max_n, int nms_radius,
                           double quality, int32_t* out_rc_d, int32_t* out_n_d, void* ws_d,
                           size_t ws_bytes, void* stream) {
  GLR_REQUIRE(max_n >= 1, GLR_ERR_INVALID, "max_n must be >= 1");
  GLR_REQUIRE(nms_radius >= 0, GLR_ERR_INVALID, "nms_radius must be >= 0");
  GLR_REQUIRE(ws_bytes >= glr_nms_workspace(H, W), GLR_ERR_WORKSPACE, "corners: workspace");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = (int64_t)H * W;
  uint8_t* p = align256(reinterpret_cast<uint8_t*>(ws_d));
  unsigned long long* mx = reinterpret_cast<unsigned long long*>(p);
  p += 256;
  uint64_t* k_in = reinterpret_cast<uint64_t*>(p);
  p = align256(p + n * sizeof(uint64_t));
  uint64_t* k_out = reinterpret_cast<uint64_t*>(p);
  p = align256(p + n * sizeof(uint64_t));
  int32_t* v_in = reinterpret_cast<int32_t*>(p);
  p = align256(p + n * sizeof(int32_t));
  int32_t* v_out = reinterpret_cast<int32_t*>(p);
  p = align256(p + n * sizeof(int32_t));
  uint8_t* blocked = p;
  p = align256(p + n);
  size_t temp_bytes = nms_sort_temp(n);
  int* n_cand = reinterpret_cast<int*>(mx + 1);
  GLR_CUDA(cudaMemsetAsync(mx, 0, 2 * sizeof(unsigned long long), st));
  resp_max_kernel<<<grid_for(n), 256, 0, st>>>(resp_d, n, mx);
  cand_keys_kernel<<<grid_for(n), 256, 0, st>>>(resp_d, n, quality, mx, k_in, v_in, n_cand);
  GLR_CUDA(cudaGetLastError());
  GLR_CUDA(cub::DeviceRadixSort::SortPairsDescending(p, temp_bytes, k_in, k_out, v_in, v_out,
                                                     (int)n, 0, 64, st));
  const size_t bm_bytes = (size_t)((n + 31) / 32) * sizeof(uint32_t);
  const size_t batch_bytes = ((bm_bytes + 15) & ~size_t(15)) + nmsb::kBatchBytes;
  constexpr int kBatchSmemMax = 226 * 1024;  // 227 KB less the kernel's static shared memory
  if (batch_bytes <= (size_t)kBatchSmemMax && nms_radius <= 64) {
    {
      const int s = ensure_smem_attr((const void*)nms_batch_kernel<false>, kBatchSmemMax);
      if (s) return s;
    }
    nms_batch_kernel<false><<<1, nmsb::B, batch_bytes, st>>>(v_out, n_cand, H, W, max_n,
                                                             nms_radius, out_rc_d, out_n_d, nullptr);
    return check_launch("nms_batch_kernel");
  }
  if (nms_radius <= 64 && n >= 32) {
    // bitmap in global memory (the `blocked` byte map's storage: n >= n / 8 bytes)
    uint32_t* gbm = reinterpret_cast<uint32_t*>(blocked);
    GLR_CUDA(cudaMemsetAsync(gbm, 0, bm_bytes, st));
    nms_batch_kernel<true><<<1, nmsb::B, nmsb::kBatchBytes + 16, st>>>(
        v_out, n_cand, H, W, max_n, nms_radius, out_rc_d, out_n_d, gbm);
    return check_launch("nms_batch_kernel (global bitmap)");
  }
  if (bm_bytes <= (size_t)kNmsBitmapMaxBytes && nms_radius <= 15) {
    {
      const int s = ensure_smem_attr((const void*)nms_bitmap_kernel, kNmsBitmapMaxBytes);
      if (s) return s;
    }
    nms_bitmap_kernel<<<1, 1024, bm_bytes, st>>>(v_out, n_cand, H, W, max_n, nms_radius,
                                                 out_rc_d, out_n_d);
    return check_launch("nms_bitmap_kernel");
  }
  GLR_CUDA(cudaMemsetAsync(blocked, 0, n, st));
  nms_kernel<<<1, 1024, 0, st>>>(k_out, v_out, n, H, W, max_n, nms_radius, blocked, out_rc_d,
                                 out_n_d);
  return check_launch("nms_kernel");
}

extern "C" size_t glr_anchor_workspace(int H, int W) { return (size_t)H * W * sizeof(int32_t); }

extern "C" int glr_select_anchors(const int32_t* corners_rc_d, const int32_t* n_corners_d,
                                  int max_corners, int H, int W, int P, int grid_interval,
                                  int max_anchors, int32_t* anchors_d, uint8_t* tags_d,
                                  int32_t* n_d, void* ws_d, void* stream) {
  GLR_REQUIRE(P <= H && P <= W, GLR_ERR_INVALID, "patch size %d exceeds image %dx%d", P, H, W);
  GLR_REQUIRE(grid_interval >= 0, GLR_ERR_INVALID, "uniform_interval must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* first = reinterpret_cast<int32_t*>(ws_d);
  GLR_CUDA(cudaMemsetAsync(first, 0x7f, (size_t)H * W * sizeof(int32_t), st));
  anchors_kernel<<<1, 1024, 0, st>>>(corners_rc_d, n_corners_d, max_corners, H, W, P,
                                     grid_interval, max_anchors, first, anchors_d, tags_d, n_d);
  return check_launch("anchors_kernel");
}
