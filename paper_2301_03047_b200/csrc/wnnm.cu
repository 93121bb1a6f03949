// (4) Batched WNNM and (5) deterministic aggregation.
//
// Reference: glr/lowrank.py:46-65 (wnnm_prox: thin SVD, sigma_hat =
// sqrt(max(s^2 - K sigma^2, 0)), w = c sqrt(K) sigma^2 / (sigma_hat + eps),
// U diag(max(s - w, 0)) V^T) and :68-87 (glr_regularize: shrink every group,
// scatter_group, divide by the count), glr/patches.py:57-70 (scatter_group).
//
// B200 formulation (one CTA per group, fp64 throughout):
//   G = M^T M (K x K) accumulated over row tiles of the group, which is read
//   straight from the image at its K positions (never materialised);
//   parallel cyclic Jacobi on G (32 disjoint rotations per round) gives
//   G = V diag(lambda) V^T, s = sqrt(lambda);
//   Wm = V diag(f(s)/s) V^T with f the WNNM shrinkage; out = M Wm, since
//   M V = U S makes M V diag(f(s)/s) V^T = U diag(f(s)) V^T.
// The denoised patches are scatter-added into an int64 fixed-point
// numerator with integer atomics: the sum is exact and order-independent,
// hence bitwise deterministic and identical for any exemplar sharding.
#include "common.cuh"

namespace glr {

namespace wn {
constexpr int THREADS = 256;
constexpr int KMAX = 64;
constexpr int LD = KMAX + 1;  // padded leading dimension of G / V / Wm
constexpr int ROWS = 32;      // rows of M per tile
constexpr int MAX_SWEEPS = 24;
}  // namespace wn

struct WnnmArgs {
  // source: either explicit groups (G,K,m) column-major, or image + positions
  const double* groups;
  const double* x;
  int H, W, C, P;
  const int32_t* pos;
  int n_max;
  const int32_t* n_dev;
  int m, K;
  double sigma, c_weight, eps, uniform_weight;
  // outputs: explicit groups or fixed-point scatter
  double* out;
  int64_t* acc;
  double scale;  // 2^frac_bits
  int32_t* nonfinite;
};

template <bool FROM_IMAGE>
__device__ __forceinline__ double load_m(const WnnmArgs& a, int g, int r, int j) {
  if constexpr (FROM_IMAGE) {
    const int32_t* q = a.pos + ((size_t)g * a.K + j) * 2;
    const int PC = a.P * a.C;
    const int rr = q[0] + r / PC;
    const int cc = q[1] + (r / a.C) % a.P;
    return a.x[((int64_t)rr * a.W + cc) * a.C + (r % a.C)];
  } else {
    return a.groups[((size_t)g * a.K + j) * a.m + r];
  }
}

template <bool FROM_IMAGE>
__global__ void __launch_bounds__(wn::THREADS, 2) wnnm_kernel(WnnmArgs a) {
  using namespace wn;
  extern __shared__ __align__(16) double sm[];
  double* G = sm;                 // KMAX x LD
  double* V = G + KMAX * LD;      // KMAX x LD
  double* T = V + KMAX * LD;      // ROWS x KMAX tile of M
  __shared__ double cs_c[KMAX / 2], cs_s[KMAX / 2];
  __shared__ int pair_p[KMAX / 2], pair_q[KMAX / 2];
  __shared__ double ratio[KMAX];
  __shared__ double red[wn::THREADS / 32][2];
  __shared__ int s_stop, s_bad;

  const int g = blockIdx.x;
  const int N = a.n_dev ? min(*a.n_dev, a.n_max) : a.n_max;
  if (g >= N) return;
  const int tid = threadIdx.x;
  const int K = a.K, m = a.m;
  const int Ke = K + (K & 1);  // even size for the round-robin pairing

  // ---- Gram: each thread owns a 4x4 block of G ----
  const int bi = tid / 16, bj = tid % 16;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  bool bad = false;
  for (int r0 = 0; r0 < m; r0 += ROWS) {
    for (int t = tid; t < ROWS * KMAX; t += THREADS) {
      const int rr = t / KMAX, j = t % KMAX;
      double v = 0.0;
      if (r0 + rr < m && j < K) v = load_m<FROM_IMAGE>(a, g, r0 + rr, j);
      bad |= !isfinite(v);
      T[t] = v;
    }
    __syncthreads();
    if (4 * bi < K && 4 * bj < K) {
      const int rmax = min(ROWS, m - r0);
      for (int rr = 0; rr < rmax; ++rr) {
        double x[4], y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          x[k] = T[rr * KMAX + 4 * bi + k];
          y[k] = T[rr * KMAX + 4 * bj + k];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(x[i], y[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
  if (tid == 0) s_bad = 0;
  __syncthreads();
  if (bad) s_bad = 1;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ii = 4 * bi + i, jj = 4 * bj + j;
      if (ii < KMAX && jj < KMAX) G[ii * LD + jj] = (ii < K && jj < K) ? acc[i][j] : 0.0;
    }
  for (int t = tid; t < KMAX * KMAX; t += THREADS) {
    const int i = t / KMAX, j = t % KMAX;
    V[i * LD + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0 && a.nonfinite) atomicExch(a.nonfinite, 1);
    return;
  }

  // ---- parallel cyclic Jacobi (round-robin tournament over Ke indices) ----
  const int npairs = Ke / 2;
  for (int sweep = 0; sweep < MAX_SWEEPS; ++sweep) {
    for (int round = 0; round < Ke - 1; ++round) {
      if (tid < npairs) {
        // tournament: index 0 fixed, others rotate
        auto slot = [&](int s) { return s == 0 ? 0 : 1 + (s - 1 + round) % (Ke - 1); };
        int p = slot(tid), q = slot(Ke - 1 - tid);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, s = 0.0;
        if (q < K) {
          const double app = G[p * LD + p], aqq = G[q * LD + q], apq = G[p * LD + q];
          if (apq != 0.0) {
            const double tau = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(tau) > 1e150) {
              t = 0.5 / tau;
            } else {
              t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            }
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        pair_p[tid] = p;
        pair_q[tid] = q;
        cs_c[tid] = c;
        cs_s[tid] = s;
      }
      __syncthreads();
      // rows: G <- J^T G
      for (int t = tid; t < npairs * K; t += THREADS) {
        const int k = t / K, j = t % K;
        const double s = cs_s[k];
        if (s == 0.0) continue;
        const double c = cs_c[k];
        const int p = pair_p[k], q = pair_q[k];
        const double gp = G[p * LD + j], gq = G[q * LD + j];
        G[p * LD + j] = c * gp - s * gq;
        G[q * LD + j] = s * gp + c * gq;
      }
      __syncthreads();
      // columns: G <- G J, V <- V J
      for (int t = tid; t < 2 * npairs * K; t += THREADS) {
        const int which = t / (npairs * K);
        const int u = t % (npairs * K);
        const int k = u / K, i = u % K;
        const double s = cs_s[k];
        if (s == 0.0) continue;
        const double c = cs_c[k];
        const int p = pair_p[k], q = pair_q[k];
        double* Mx = which ? V : G;
        const double xp = Mx[i * LD + p], xq = Mx[i * LD + q];
        Mx[i * LD + p] = c * xp - s * xq;
        Mx[i * LD + q] = s * xp + c * xq;
      }
      __syncthreads();
    }
    // convergence: off-diagonal mass vs total
    double off = 0.0, tot = 0.0;
    for (int t = tid; t < K * K; t += THREADS) {
      const int i = t / K, j = t % K;
      const double v = G[i * LD + j];
      tot += v * v;
      if (i != j) off += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if ((tid & 31) == 0) {
      red[tid >> 5][0] = off;
      red[tid >> 5][1] = tot;
    }
    __syncthreads();
    if (tid == 0) {
      double o = 0.0, s = 0.0;
      for (int w = 0; w < THREADS / 32; ++w) {
        o += red[w][0];
        s += red[w][1];
      }
      s_stop = (o <= 1e-30 * s) || s == 0.0;
    }
    __syncthreads();
    if (s_stop) break;
  }

  // ---- shrinkage weights (lowrank.py:58-64) ----
  if (tid < K) {
    const double lam = G[tid * LD + tid];
    const double s = sqrt(fmax(lam, 0.0));
    double w;
    if (a.uniform_weight >= 0.0) {
      w = a.uniform_weight;
    } else {
      const double sig_hat = sqrt(fmax(s * s - K * a.sigma * a.sigma, 0.0));
      w = a.c_weight * sqrt((double)K) * a.sigma * a.sigma / (sig_hat + a.eps);
    }
    const double f = fmax(s - w, 0.0);
    ratio[tid] = s > 0.0 ? f / s : 0.0;
  }
  __syncthreads();
  // Wm = V diag(ratio) V^T into G
  for (int t = tid; t < K * K; t += THREADS) {
    const int i = t / K, j = t % K;
    double v = 0.0;
    for (int k = 0; k < K; ++k) v = fma(V[i * LD + k] * ratio[k], V[j * LD + k], v);
    G[i * LD + j] = v;
  }
  __syncthreads();

  // ---- out = M Wm, row tiles; thread -> (row, 8 consecutive columns) ----
  const int cb = tid % 8, rr = tid / 8;  // 8 column blocks x 32 rows
  for (int r0 = 0; r0 < m; r0 += ROWS) {
    for (int t = tid; t < ROWS * KMAX; t += THREADS) {
      const int r2 = t / KMAX, j = t % KMAX;
      T[t] = (r0 + r2 < m && j < K) ? load_m<FROM_IMAGE>(a, g, r0 + r2, j) : 0.0;
    }
    __syncthreads();
    const int r = r0 + rr;
    if (r < m) {
      double o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = 0.0;
      for (int i = 0; i < K; ++i) {
        const double mv = T[rr * KMAX + i];
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = fma(mv, G[i * LD + cb * 8 + k], o[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = cb * 8 + k;
        if (j >= K) break;
        if constexpr (FROM_IMAGE) {
          const int32_t* q = a.pos + ((size_t)g * K + j) * 2;
          const int PC = a.P * a.C;
          const int prow = q[0] + r / PC;
          const int pcol = q[1] + (r / a.C) % a.P;
          const int64_t idx = ((int64_t)prow * a.W + pcol) * a.C + (r % a.C);
          const long long v = __double2ll_rn(o[k] * a.scale);
          atomicAdd(reinterpret_cast<unsigned long long*>(a.acc + idx), (unsigned long long)v);
        } else {
          a.out[((size_t)g * K + j) * m + r] = o[k];
        }
      }
    }
    __syncthreads();
  }
}

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

__global__ void normalize_kernel(const int64_t* __restrict__ acc, const int32_t* __restrict__ cnt,
                                 const double* __restrict__ x, int64_t npix, int C, double inv_scale,
                                 double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix * C;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = cnt[i / C];
    z[i] = n > 0 ? ((double)acc[i] * inv_scale) / (double)n : x[i];
  }
}

static int blocks_for(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, threads), (int64_t)kNumSMs * 32));
}

static size_t wnnm_smem() {
  return (size_t)(2 * wn::KMAX * wn::LD + wn::ROWS * wn::KMAX) * sizeof(double);
}

template <bool FROM_IMAGE>
static int launch_wnnm(const WnnmArgs& a, int grid, cudaStream_t st) {
  const size_t smem = wnnm_smem();
  GLR_CUDA(cudaFuncSetAttribute(wnnm_kernel<FROM_IMAGE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  wnnm_kernel<FROM_IMAGE><<<grid, wn::THREADS, smem, st>>>(a);
  return check_launch("wnnm_kernel");
}

}  // namespace glr

using namespace glr;

extern "C" size_t glr_wnnm_workspace(int G, int K) { return 0; }

extern "C" int glr_wnnm(const double* groups_d, int G, int m, int K, double sigma, double c_weight,
                        double eps, double uniform_weight, double* out_d, int32_t* nonfinite_d,
                        void* ws_d, size_t ws_bytes, void* stream) {
  GLR_REQUIRE(K >= 1 && K <= wn::KMAX, GLR_ERR_UNSUPPORTED, "wnnm: K=%d outside [1, %d]", K,
              wn::KMAX);
  GLR_REQUIRE(m >= 1, GLR_ERR_INVALID, "wnnm: m=%d", m);
  GLR_REQUIRE(sigma >= 0, GLR_ERR_INVALID, "noise_sigma must be nonnegative");
  GLR_REQUIRE(c_weight > 0 && eps > 0, GLR_ERR_INVALID, "c_weight and eps must be positive");
  if (G <= 0) return GLR_OK;
  WnnmArgs a{};
  a.groups = groups_d;
  a.n_max = G;
  a.m = m;
  a.K = K;
  a.sigma = sigma;
  a.c_weight = c_weight;
  a.eps = eps;
  a.uniform_weight = uniform_weight;
  a.out = out_d;
  a.nonfinite = nonfinite_d;
  return launch_wnnm<false>(a, G, (cudaStream_t)stream);
}

extern "C" int glr_wnnm_scatter(const double* x_d, int H, int W, int C, int P,
                                const int32_t* positions_d, int n_max, const int32_t* n_dev_d,
                                int K, double sigma, double c_weight, double eps, int frac_bits,
                                int64_t* acc_d, void* ws_d, size_t ws_bytes, void* stream) {
  GLR_REQUIRE(K >= 1 && K <= wn::KMAX, GLR_ERR_UNSUPPORTED, "wnnm: K=%d outside [1, %d]", K,
              wn::KMAX);
  GLR_REQUIRE(P >= 1 && P <= H && P <= W, GLR_ERR_INVALID, "wnnm_scatter: bad patch size");
  GLR_REQUIRE(frac_bits >= 0 && frac_bits <= 52, GLR_ERR_INVALID, "frac_bits %d", frac_bits);
  if (n_max <= 0) return GLR_OK;
  WnnmArgs a{};
  a.x = x_d;
  a.H = H;
  a.W = W;
  a.C = C;
  a.P = P;
  a.pos = positions_d;
  a.n_max = n_max;
  a.n_dev = n_dev_d;
  a.m = P * P * C;
  a.K = K;
  a.sigma = sigma;
  a.c_weight = c_weight;
  a.eps = eps;
  a.uniform_weight = -1.0;
  a.acc = acc_d;
  a.scale = ldexp(1.0, frac_bits);
  return launch_wnnm<true>(a, n_max, (cudaStream_t)stream);
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

extern "C" int glr_normalize(const int64_t* acc_d, const int32_t* cnt_d, const double* x_d, int H,
                             int W, int C, int frac_bits, double* z_d, void* stream) {
  const int64_t npix = (int64_t)H * W;
  normalize_kernel<<<blocks_for(npix * C), 256, 0, (cudaStream_t)stream>>>(
      acc_d, cnt_d, x_d, npix, C, ldexp(1.0, -frac_bits), z_d);
  return check_launch("normalize_kernel");
}
