// (6) Sensing operators and the fused GAP projection.
//
// Reference: glr/operators.py (CACTI :35-59, masked Fourier :65-89, MSFA
// :160-185) and glr/solvers.py:284-308 (gap_solve projection
// x = clip(z + A^T(safe_div(y - A z, gram)), -p/2, 3p/2), residual
// ||y - A x||, _safe_div :220-226).
//
// The mask-sum family (CACTI and MSFA share A x = sum_t M_t x_t) is one
// pixel-local kernel that fuses: count-normalisation of the aggregated
// numerator (lowrank.py:84-87), the projection, the clip, and a
// deterministic per-block partial of the squared residual of the NEW
// iterate. Channel sums use numpy's pairwise order (operators.py:39 sums
// over axis 2) so A x matches the reference to the last bit for T <= 128.
//
// The Fourier family uses a hand-written fp64 complex FFT (fft.cu).
#include "common.cuh"
#include "fft.cuh"

namespace glr {

namespace gap {
constexpr int THREADS = 256;
constexpr int TMAX = 128;
}  // namespace gap

// numpy pairwise sum over a small register/local array
__device__ __forceinline__ double pw_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__global__ void masksum_forward_kernel(const double* __restrict__ x, const double* __restrict__ mk,
                                       int64_t npix, int T, double* __restrict__ y) {
  double prod[gap::TMAX];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int t = 0; t < T; ++t) prod[t] = __dmul_rn(mk[i * T + t], x[i * T + t]);
    y[i] = pw_sum(prod, T);
  }
}

__global__ void masksum_adjoint_kernel(const double* __restrict__ y, const double* __restrict__ mk,
                                       int64_t npix, int T, double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix * T;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __dmul_rn(mk[i], y[i / T]);
}

// deterministic block partial sums -> out[blockIdx.x]
__device__ __forceinline__ void block_sum_store(double v, double* out) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = __dadd_rn(s, red[w]);
    out[blockIdx.x] = s;
  }
}

__global__ void final_sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v = __dadd_rn(v, part[i]);
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = __dadd_rn(s, red[w]);
    *out = s;
  }
}

struct GapArgs {
  int64_t* acc;  // consumed: read, then reset to zero (read-and-clear)
  const int32_t* cnt;
  double inv_scale;
  const double* x_in;
  const double* mk;
  const double* y;
  const double* gram;
  int64_t npix;
  int T;
  double lo, hi, rho;
  double* x_out;
  double* part;
};

// TT > 0: channel count fixed at compile time (arrays in registers, 16-byte
// loads); TT = 0: any T <= TMAX (arrays in local memory).
template <int TT>
__global__ void __launch_bounds__(gap::THREADS, 2) gap_masksum_kernel(GapArgs a) {
  constexpr int TA = TT > 0 ? TT : gap::TMAX;
  const int T = TT > 0 ? TT : a.T;
  double z[TA], mk[TA], prod[TA];
  double acc_sq = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = a.cnt ? a.cnt[i] : 0;
    if constexpr (TT > 0 && TT % 2 == 0) {
      const double2* mk2 = reinterpret_cast<const double2*>(a.mk + i * TT);
#pragma unroll
      for (int t = 0; t < TT / 2; ++t) {
        const double2 m = mk2[t];
        mk[2 * t] = m.x;
        mk[2 * t + 1] = m.y;
      }
      if (n > 0) {
        longlong2* ac2 = reinterpret_cast<longlong2*>(a.acc + i * TT);
#pragma unroll
        for (int t = 0; t < TT / 2; ++t) {
          const longlong2 v = ac2[t];
          z[2 * t] = ((double)v.x * a.inv_scale) / (double)n;
          z[2 * t + 1] = ((double)v.y * a.inv_scale) / (double)n;
        }
        // read-and-clear: the numerator is zero again for the next
        // iteration's scatter (uncovered pixels were never written)
#pragma unroll
        for (int t = 0; t < TT / 2; ++t) __stcs(ac2 + t, make_longlong2(0, 0));
      } else {
        const double2* x2 = reinterpret_cast<const double2*>(a.x_in + i * TT);
#pragma unroll
        for (int t = 0; t < TT / 2; ++t) {
          const double2 v = x2[t];
          z[2 * t] = v.x;
          z[2 * t + 1] = v.y;
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int64_t k = i * T + t;
        mk[t] = a.mk[k];
        if (n > 0) {
          z[t] = ((double)a.acc[k] * a.inv_scale) / (double)n;
          a.acc[k] = 0;
        } else {
          z[t] = a.x_in[k];
        }
      }
    }
    double gram;
    if (a.gram) {
      gram = a.gram[i];
    } else {
#pragma unroll
      for (int t = 0; t < T; ++t) prod[t] = __dmul_rn(mk[t], mk[t]);
      gram = pw_sum(prod, T);
    }
#pragma unroll
    for (int t = 0; t < T; ++t) prod[t] = __dmul_rn(mk[t], z[t]);
    const double az = pw_sum(prod, T);
    const double yi = a.y[i];
    // GAP: safe_div(y - Az, gram) (solvers.py:220-226, rho = 0);
    // ADMM: (y - Am) / (rho + gram) (solvers.py:329)
    const double den = a.rho != 0.0 ? __dadd_rn(a.rho, gram) : gram;
    const double r = den != 0.0 ? __ddiv_rn(__dsub_rn(yi, az), den) : 0.0;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      double v = __dadd_rn(z[t], __dmul_rn(mk[t], r));
      z[t] = fmin(fmax(v, a.lo), a.hi);
      prod[t] = __dmul_rn(mk[t], z[t]);
    }
    if constexpr (TT > 0 && TT % 2 == 0) {
      double2* o2 = reinterpret_cast<double2*>(a.x_out + i * TT);
#pragma unroll
      for (int t = 0; t < TT / 2; ++t) o2[t] = make_double2(z[2 * t], z[2 * t + 1]);
    } else {
#pragma unroll
      for (int t = 0; t < T; ++t) a.x_out[i * T + t] = z[t];
    }
    const double d = __dsub_rn(yi, pw_sum(prod, T));
    acc_sq = fma(d, d, acc_sq);
  }
  block_sum_store(acc_sq, a.part);
}

__global__ void sq_err_kernel(const double* __restrict__ x, const double* __restrict__ ref,
                              int64_t n, double peak, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = peak > 0.0 ? fmin(fmax(x[i], 0.0), peak) : x[i];
    const double d = ref[i] - v;
    s = fma(d, d, s);
  }
  block_sum_store(s, part);
}

constexpr int kGapBlocks = 8 * kNumSMs;

// out = clip((a x + b y) + c z) elementwise (z optional), evaluated in that
// order so ADMM's m = z - u, v = x + u, u' = (u + x) - z match numpy bitwise
// (solvers.py:327, 332, 334).
__global__ void lincomb_kernel(const double* __restrict__ x, double a, const double* __restrict__ y,
                               double b, const double* __restrict__ z, double c, int64_t n,
                               int clip, double lo, double hi, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = __dmul_rn(a, x[i]);
    if (y) v = __dadd_rn(v, __dmul_rn(b, y[i]));
    if (z) v = __dadd_rn(v, __dmul_rn(c, z[i]));
    if (clip) v = fmin(fmax(v, lo), hi);
    out[i] = v;
  }
}

}  // namespace glr

using namespace glr;

extern "C" int glr_masksum_forward(const double* x_d, const double* masks_d, int H, int W, int T,
                                   double* y_d, void* stream) {
  GLR_REQUIRE(T >= 1 && T <= gap::TMAX, GLR_ERR_UNSUPPORTED, "masksum: T=%d", T);
  const int64_t npix = (int64_t)H * W;
  masksum_forward_kernel<<<kGapBlocks, gap::THREADS, 0, (cudaStream_t)stream>>>(x_d, masks_d,
                                                                               npix, T, y_d);
  return check_launch("masksum_forward_kernel");
}

extern "C" int glr_masksum_adjoint(const double* y_d, const double* masks_d, int H, int W, int T,
                                   double* x_d, void* stream) {
  const int64_t npix = (int64_t)H * W;
  masksum_adjoint_kernel<<<kGapBlocks * 4, gap::THREADS, 0, (cudaStream_t)stream>>>(
      y_d, masks_d, npix, T, x_d);
  return check_launch("masksum_adjoint_kernel");
}

extern "C" size_t glr_gap_workspace(int H, int W) { return (kGapBlocks + 8) * sizeof(double); }

extern "C" int glr_gap_masksum(int64_t* acc_d, const int32_t* cnt_d, int frac_bits,
                               const double* x_in_d, const double* masks_d, const double* y_d,
                               const double* gram_d, int H, int W, int T, double lo, double hi,
                               double rho, double* x_out_d, double* resid_d, void* ws_d,
                               void* stream) {
  GLR_REQUIRE(T >= 1 && T <= gap::TMAX, GLR_ERR_UNSUPPORTED, "gap_masksum: T=%d", T);
  GLR_REQUIRE(rho >= 0, GLR_ERR_INVALID, "rho must be nonnegative");
  cudaStream_t st = (cudaStream_t)stream;
  GapArgs a;
  a.rho = rho;
  a.acc = acc_d;
  a.cnt = acc_d ? cnt_d : nullptr;
  a.inv_scale = ldexp(1.0, -frac_bits);
  a.x_in = x_in_d;
  a.mk = masks_d;
  a.y = y_d;
  a.gram = gram_d;
  a.npix = (int64_t)H * W;
  a.T = T;
  a.lo = lo;
  a.hi = hi;
  a.x_out = x_out_d;
  a.part = reinterpret_cast<double*>(ws_d);
  switch (T) {
    case 8: gap_masksum_kernel<8><<<kGapBlocks, gap::THREADS, 0, st>>>(a); break;
    case 16: gap_masksum_kernel<16><<<kGapBlocks, gap::THREADS, 0, st>>>(a); break;
    case 24: gap_masksum_kernel<24><<<kGapBlocks, gap::THREADS, 0, st>>>(a); break;
    case 32: gap_masksum_kernel<32><<<kGapBlocks, gap::THREADS, 0, st>>>(a); break;
    default: gap_masksum_kernel<0><<<kGapBlocks, gap::THREADS, 0, st>>>(a); break;
  }
  GLR_CUDA(cudaGetLastError());
  final_sum_kernel<<<1, 256, 0, st>>>(a.part, kGapBlocks, resid_d);
  return check_launch("final_sum_kernel");
}

// ---------------------------------------------------------------------------
// init="interp" (solvers.py:237-254): scipy gaussian_filter(sigma=1.5) of the
// adjoint and of the masks, per channel, mode "reflect", radius 6, evaluated
// in scipy's symmetric correlate1d order: out = x[i] w[0] + sum over
// j = -R..-1 of (x[i+j] + x[i-j]) w[j]; axis 0 then axis 1. Bit-identical to
// scipy (the weights come from the host, computed with numpy like scipy).

__device__ __forceinline__ int reflect_idx(int i, int n) {
  i %= 2 * n;
  if (i < 0) i += 2 * n;
  return i < n ? i : 2 * n - 1 - i;
}

struct GaussW {
  double w[16];  // w[R + j], j in [-R, R]
  int R;
};

// one separable pass over both images (x and masks) along `axis` (0: rows, 1: cols)
__global__ void gauss_pass_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                  int H, int W, int C, int axis, GaussW gw,
                                  double* __restrict__ oa, double* __restrict__ ob) {
  const int64_t total = (int64_t)H * W * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % C);
    const int64_t pix = i / C;
    const int r = (int)(pix / W), c = (int)(pix % W);
    const int n = axis == 0 ? H : W, pos = axis == 0 ? r : c;
    auto at = [&](const double* src, int k) {
      const int q = reflect_idx(k, n);
      return axis == 0 ? src[((int64_t)q * W + c) * C + ch] : src[((int64_t)r * W + q) * C + ch];
    };
    double va = __dmul_rn(at(a, pos), gw.w[gw.R]);
    double vb = __dmul_rn(at(b, pos), gw.w[gw.R]);
    for (int j = -gw.R; j < 0; ++j) {
      va = __dadd_rn(va, __dmul_rn(__dadd_rn(at(a, pos + j), at(a, pos - j)), gw.w[gw.R + j]));
      vb = __dadd_rn(vb, __dmul_rn(__dadd_rn(at(b, pos + j), at(b, pos - j)), gw.w[gw.R + j]));
    }
    oa[i] = va;
    ob[i] = vb;
  }
}

__global__ void interp_div_kernel(const double* __restrict__ num, const double* __restrict__ den,
                                  int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = den[i] > 1e-12 ? __ddiv_rn(num[i], den[i]) : 0.0;
}

// CACTI interp: xt / max(gram, 1e-12) (solvers.py:252-253)
__global__ void gram_div_kernel(const double* __restrict__ xt, const double* __restrict__ gram,
                                int64_t npix, int C, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix * C;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ddiv_rn(xt[i], fmax(gram[i / C], 1e-12));
}

extern "C" int glr_interp_msfa(const double* xt_d, const double* masks_d, int H, int W, int C,
                               const double* weights, int radius, double* out_d, void* ws_d,
                               void* stream) {
  GLR_REQUIRE(radius >= 0 && radius <= 7, GLR_ERR_UNSUPPORTED, "interp: radius %d", radius);
  cudaStream_t st = (cudaStream_t)stream;
  GaussW gw;
  gw.R = radius;
  for (int i = 0; i <= 2 * radius; ++i) gw.w[i] = weights[i];
  const int64_t n = (int64_t)H * W * C;
  double* t = reinterpret_cast<double*>(ws_d);  // 4 x n doubles
  gauss_pass_kernel<<<kGapBlocks * 4, gap::THREADS, 0, st>>>(xt_d, masks_d, H, W, C, 0, gw, t,
                                                             t + n);
  gauss_pass_kernel<<<kGapBlocks * 4, gap::THREADS, 0, st>>>(t, t + n, H, W, C, 1, gw, t + 2 * n,
                                                             t + 3 * n);
  interp_div_kernel<<<kGapBlocks * 4, gap::THREADS, 0, st>>>(t + 2 * n, t + 3 * n, n, out_d);
  return check_launch("interp_msfa");
}

extern "C" int glr_interp_cacti(const double* xt_d, const double* gram_d, int H, int W, int C,
                                double* out_d, void* stream) {
  gram_div_kernel<<<kGapBlocks * 4, gap::THREADS, 0, (cudaStream_t)stream>>>(
      xt_d, gram_d, (int64_t)H * W, C, out_d);
  return check_launch("interp_cacti");
}

extern "C" int glr_lincomb(const double* x_d, double a, const double* y_d, double b,
                           const double* z_d, double c, int64_t n, int clip, double lo, double hi,
                           double* out_d, void* stream) {
  lincomb_kernel<<<kGapBlocks * 4, gap::THREADS, 0, (cudaStream_t)stream>>>(x_d, a, y_d, b, z_d,
                                                                            c, n, clip, lo, hi,
                                                                            out_d);
  return check_launch("lincomb_kernel");
}

// ---------------------------------------------------------------------------
// f3: on-device SSIM (metrics.py:40-78): per channel, an 11x11 Gaussian window
// (sigma 1.5, normalised) over every valid position, SSIM map averaged over the
// positions and the channels. The separable form g/sum(g) (x) g/sum(g) of the
// reference's outer-product window; a = clip(x, 0, peak) as in _record
// (solvers.py:262-264), b = ref. Deterministic block sums. Reporting metric:
// compared with the reference to 1e-10, not bitwise.

struct SsimW {
  double g[16];
  int S;
};

// pass 1 (along rows): five windowed sums per (row, valid col, channel)
__global__ void ssim_rows_kernel(const double* __restrict__ x, const double* __restrict__ ref,
                                 int H, int W, int C, double peak, int clip, SsimW w,
                                 double* __restrict__ t) {
  const int Wv = W - w.S + 1;
  const int64_t n = (int64_t)H * Wv * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % C);
    const int64_t rc = i / C;
    const int r = (int)(rc / Wv), c = (int)(rc % Wv);
    double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
    for (int k = 0; k < w.S; ++k) {
      const int64_t j = ((int64_t)r * W + c + k) * C + ch;
      double a = x[j];
      if (clip) a = fmin(fmax(a, 0.0), peak);
      const double b = ref[j], g = w.g[k];
      sa = fma(g, a, sa);
      sb = fma(g, b, sb);
      saa = fma(g, a * a, saa);
      sbb = fma(g, b * b, sbb);
      sab = fma(g, a * b, sab);
    }
    t[i] = sa;
    t[i + n] = sb;
    t[i + 2 * n] = saa;
    t[i + 3 * n] = sbb;
    t[i + 4 * n] = sab;
  }
}

// pass 2 (along columns) + SSIM map + block partial sums
__global__ void ssim_cols_kernel(const double* __restrict__ t, int H, int W, int C, double peak,
                                 SsimW w, double* __restrict__ part) {
  const int Wv = W - w.S + 1, Hv = H - w.S + 1;
  const int64_t n = (int64_t)H * Wv * C, nv = (int64_t)Hv * Wv * C;
  const double c1 = (0.01 * peak) * (0.01 * peak), c2 = (0.03 * peak) * (0.03 * peak);
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % C);
    const int64_t rc = i / C;
    const int r = (int)(rc / Wv), c = (int)(rc % Wv);
    double m[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k < w.S; ++k) {
      const int64_t j = ((int64_t)(r + k) * Wv + c) * C + ch;
      const double g = w.g[k];
#pragma unroll
      for (int q = 0; q < 5; ++q) m[q] = fma(g, t[j + q * n], m[q]);
    }
    const double ma = m[0], mb = m[1];
    const double va = m[2] - ma * ma, vb = m[3] - mb * mb, cov = m[4] - ma * mb;
    const double num = (2 * ma * mb + c1) * (2 * cov + c2);
    const double den = (ma * ma + mb * mb + c1) * (va + vb + c2);
    acc += num / den;
  }
  block_sum_store(acc, part);
}

extern "C" size_t glr_ssim_workspace(int H, int W, int C) {
  return (5 * (size_t)H * W * C + kGapBlocks + 8) * sizeof(double);
}

extern "C" int glr_ssim(const double* x_d, const double* ref_d, int H, int W, int C, double peak,
                        int clip, const double* window, int win_size, double* out_d, void* ws_d,
                        void* stream) {
  GLR_REQUIRE(win_size >= 1 && win_size <= 16, GLR_ERR_UNSUPPORTED, "ssim: window %d", win_size);
  GLR_REQUIRE(H >= win_size && W >= win_size, GLR_ERR_INVALID,
              "image %dx%d smaller than %dx%d window", H, W, win_size, win_size);
  cudaStream_t st = (cudaStream_t)stream;
  SsimW w;
  w.S = win_size;
  for (int i = 0; i < win_size; ++i) w.g[i] = window[i];
  double* t = reinterpret_cast<double*>(ws_d);
  double* part = t + 5 * (size_t)H * W * C;
  ssim_rows_kernel<<<kGapBlocks * 2, 256, 0, st>>>(x_d, ref_d, H, W, C, peak, clip, w, t);
  GLR_CUDA(cudaGetLastError());
  ssim_cols_kernel<<<kGapBlocks, 256, 0, st>>>(t, H, W, C, peak, w, part);
  GLR_CUDA(cudaGetLastError());
  final_sum_kernel<<<1, 256, 0, st>>>(part, kGapBlocks, out_d);
  return check_launch("ssim");
}

extern "C" int glr_sq_err(const double* x_d, const double* ref_d, int n, double peak,
                          double* out_d, void* ws_d, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* part = reinterpret_cast<double*>(ws_d);
  sq_err_kernel<<<kGapBlocks, 256, 0, st>>>(x_d, ref_d, n, peak, part);
  GLR_CUDA(cudaGetLastError());
  final_sum_kernel<<<1, 256, 0, st>>>(part, kGapBlocks, out_d);
  return check_launch("sq_err");
}
