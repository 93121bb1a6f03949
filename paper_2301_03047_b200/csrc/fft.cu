// (6) Masked unitary 2-D Fourier operator (MRI) on a hand-written fp64 FFT.
//
// Reference: glr/operators.py:65-89 — y = M * fft2(x, norm="ortho"),
// A^T y = Re(ifft2(M * y, norm="ortho")), gram = M — plus the complex
// (re, im) variant of SURVEY.md §8c for the MRI config (x_shape (H, W, 2),
// adjoint keeps both parts). The GAP update (solvers.py:298-301) is fused
// around the transforms: normalise -> F z -> safe_div(y - M F z, M) -> M r ->
// F^-1 -> z + A^T r -> optional clip -> residual ||y - M F x||.
//
// Transforms: radix-2 decimation-in-time in shared memory, one CTA per line
// (rows, then columns with strided loads), twiddles from sincospi on exact
// dyadic fractions; lengths that are not powers of two use a direct DFT.
#include "common.cuh"
#include "internal.cuh"
#include "fft.cuh"

namespace glr {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ unsigned bitrev(unsigned v, int bits) {
  return __brev(v) >> (32 - bits);
}

// one CTA per line; line i starts at data + i*line_stride, elements at elem_stride
__global__ void fft_pow2_kernel(double2* __restrict__ data, int n, int log2n, int64_t line_stride,
                                int64_t elem_stride, int sign, double scale) {
  extern __shared__ double2 buf[];
  double2* line = data + (int64_t)blockIdx.x * line_stride;
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    buf[bitrev((unsigned)j, log2n)] = line[(int64_t)j * elem_stride];
  __syncthreads();
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1;
    for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
      const int grp = b / half, k = b - grp * half;
      const int i = grp * len + k, j = i + half;
      double s, c;
      sincospi((double)sign * (2.0 * k) / (double)len, &s, &c);
      const double2 t = cmul(make_double2(c, s), buf[j]);
      const double2 u = buf[i];
      buf[i] = make_double2(u.x + t.x, u.y + t.y);
      buf[j] = make_double2(u.x - t.x, u.y - t.y);
    }
    __syncthreads();
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double2 v = buf[j];
    line[(int64_t)j * elem_stride] = make_double2(v.x * scale, v.y * scale);
  }
}

// direct DFT for other lengths
__global__ void dft_kernel(double2* __restrict__ data, int n, int64_t line_stride,
                           int64_t elem_stride, int sign, double scale) {
  extern __shared__ double2 buf[];
  double2* line = data + (int64_t)blockIdx.x * line_stride;
  for (int j = threadIdx.x; j < n; j += blockDim.x) buf[j] = line[(int64_t)j * elem_stride];
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int j = 0; j < n; ++j) {
      const long long jk = ((long long)j * k) % n;
      double s, c;
      sincospi((double)sign * 2.0 * (double)jk / (double)n, &s, &c);
      const double2 v = buf[j];
      re += v.x * c - v.y * s;
      im += v.x * s + v.y * c;
    }
    buf[n + k] = make_double2(re * scale, im * scale);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) line[(int64_t)j * elem_stride] = buf[n + j];
}

static int fft_lines(double2* data, int n, int lines, int64_t line_stride, int64_t elem_stride,
                     int sign, double scale, cudaStream_t st) {
  int log2n = 0;
  while ((1 << log2n) < n) ++log2n;
  const bool pow2 = (1 << log2n) == n;
  const int threads = std::min(512, std::max(32, pow2 ? n / 2 : n));
  const size_t smem = (size_t)(pow2 ? n : 2 * n) * sizeof(double2);
  GLR_REQUIRE(smem <= 200 * 1024, GLR_ERR_UNSUPPORTED, "fft: length %d too large", n);
  if (pow2) {
    { const int s_ = ensure_smem_attr((const void*)fft_pow2_kernel, (int)smem); if (s_) return s_; }
    fft_pow2_kernel<<<lines, threads, smem, st>>>(data, n, log2n, line_stride, elem_stride, sign,
                                                  scale);
  } else {
    { const int s_ = ensure_smem_attr((const void*)dft_kernel, (int)smem); if (s_) return s_; }
    dft_kernel<<<lines, threads, smem, st>>>(data, n, line_stride, elem_stride, sign, scale);
  }
  return check_launch("fft_lines");
}

int fft2_ortho(double2* data, int H, int W, int sign, cudaStream_t st) {
  int s = fft_lines(data, W, H, W, 1, sign, 1.0, st);  // rows
  if (s) return s;
  return fft_lines(data, H, W, 1, W, sign, 1.0 / sqrt((double)H * (double)W), st);  // columns
}

// ---------------------------------------------------------------------------
// elementwise stages

// z = normalised aggregate (or x), written to z_out; packed complex to buf
__global__ void pack_kernel(int64_t* __restrict__ acc, const int32_t* __restrict__ cnt,
                            double inv_scale, const double* __restrict__ x_in, int64_t npix, int C,
                            double* __restrict__ z_out, double2* __restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (acc && cnt) ? cnt[i] : 0;
    double v[2] = {0.0, 0.0};
    for (int c = 0; c < C; ++c) {
      const int64_t k = i * C + c;
      if (n > 0) {
        v[c] = ((double)acc[k] * inv_scale) / (double)n;
        acc[k] = 0;  // read-and-clear (the numerator is consumed)
      } else {
        v[c] = x_in[k];
      }
      if (z_out) z_out[k] = v[c];
    }
    buf[i] = make_double2(v[0], C == 2 ? v[1] : 0.0);
  }
}

__global__ void mask_mul_kernel(double2* __restrict__ buf, const double* __restrict__ mask,
                                int64_t npix) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double m = mask[i];
    buf[i] = make_double2(buf[i].x * m, buf[i].y * m);
  }
}

__global__ void mask_copy_kernel(const double2* __restrict__ src, const double* __restrict__ mask,
                                 int64_t npix, double2* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double m = mask[i];
    dst[i] = make_double2(src[i].x * m, src[i].y * m);
  }
}

// buf <- M * (y - M * buf) / (rho + M) (ADMM, solvers.py:329; rho = 0 is
// GAP's safe_div, zero where the divisor is zero)
__global__ void spectral_residual_kernel(double2* __restrict__ buf, const double2* __restrict__ y,
                                         const double* __restrict__ mask, int64_t npix,
                                         double rho) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double m = mask[i];
    const double den = rho != 0.0 ? rho + m : m;
    double2 r = make_double2(0.0, 0.0);
    if (den != 0.0) {
      const double2 f = buf[i];
      r = make_double2((y[i].x - m * f.x) / den, (y[i].y - m * f.y) / den);
    }
    buf[i] = make_double2(m * r.x, m * r.y);
  }
}

// x = z + A^T r (real part, or re/im), optional clip; repack x into buf
__global__ void fourier_update_kernel(double2* __restrict__ buf, double* __restrict__ x, int64_t npix,
                                      int C, int clip, double lo, double hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = buf[i];
    double v0 = x[i * C] + a.x;
    if (clip) v0 = fmin(fmax(v0, lo), hi);
    x[i * C] = v0;
    double v1 = 0.0;
    if (C == 2) {
      v1 = x[i * C + 1] + a.y;
      if (clip) v1 = fmin(fmax(v1, lo), hi);
      x[i * C + 1] = v1;
    }
    buf[i] = make_double2(v0, v1);
  }
}

__global__ void adjoint_out_kernel(const double2* __restrict__ buf, int64_t npix, int C,
                                   double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i * C] = buf[i].x;
    if (C == 2) x[i * C + 1] = buf[i].y;
  }
}

// partial sums of |y - M * buf|^2
__global__ void fourier_resid_kernel(const double2* __restrict__ buf, const double2* __restrict__ y,
                                     const double* __restrict__ mask, int64_t npix,
                                     double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double m = mask[i];
    const double dr = y[i].x - m * buf[i].x, di = y[i].y - m * buf[i].y;
    s = fma(dr, dr, fma(di, di, s));
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void fsum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

constexpr int kFBlocks = 2 * kNumSMs;

static int eblocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)kFBlocks * 4));
}

}  // namespace glr

using namespace glr;

extern "C" size_t glr_fft_workspace(int H, int W) {
  return (size_t)H * W * sizeof(double2) + (kFBlocks + 8) * sizeof(double) + 256;
}

extern "C" int glr_fourier_forward(const double* x_d, const double* mask_d, int H, int W, int C,
                                   double* y_d, void* ws_d, void* stream) {
  GLR_REQUIRE(C == 1 || C == 2, GLR_ERR_INVALID, "fourier: C=%d (1 real, 2 complex)", C);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npix = (int64_t)H * W;
  double2* buf = reinterpret_cast<double2*>(y_d);
  pack_kernel<<<eblocks(npix), 256, 0, st>>>(nullptr, nullptr, 1.0, x_d, npix, C, nullptr, buf);
  GLR_CUDA(cudaGetLastError());
  int s = fft2_ortho(buf, H, W, -1, st);
  if (s) return s;
  mask_mul_kernel<<<eblocks(npix), 256, 0, st>>>(buf, mask_d, npix);
  return check_launch("fourier_forward");
}

extern "C" int glr_fourier_adjoint(const double* y_d, const double* mask_d, int H, int W, int C,
                                   double* x_d, void* ws_d, void* stream) {
  GLR_REQUIRE(C == 1 || C == 2, GLR_ERR_INVALID, "fourier: C=%d (1 real, 2 complex)", C);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npix = (int64_t)H * W;
  double2* buf = reinterpret_cast<double2*>(ws_d);
  mask_copy_kernel<<<eblocks(npix), 256, 0, st>>>(reinterpret_cast<const double2*>(y_d), mask_d,
                                                  npix, buf);
  GLR_CUDA(cudaGetLastError());
  int s = fft2_ortho(buf, H, W, +1, st);
  if (s) return s;
  adjoint_out_kernel<<<eblocks(npix), 256, 0, st>>>(buf, npix, C, x_d);
  return check_launch("fourier_adjoint");
}

extern "C" int glr_gap_fourier(int64_t* acc_d, const int32_t* cnt_d, int frac_bits,
                               const double* x_in_d, const double* mask_d, const double* y_d, int H,
                               int W, int C, int clip, double lo, double hi, double rho,
                               double* x_out_d, double* resid_d, void* ws_d, void* stream) {
  GLR_REQUIRE(C == 1 || C == 2, GLR_ERR_INVALID, "fourier: C=%d (1 real, 2 complex)", C);
  GLR_REQUIRE(rho >= 0, GLR_ERR_INVALID, "rho must be nonnegative");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npix = (int64_t)H * W;
  double2* buf = reinterpret_cast<double2*>(ws_d);
  double* part = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(buf + npix) + 255) & ~uintptr_t(255));
  const double2* y = reinterpret_cast<const double2*>(y_d);
  pack_kernel<<<eblocks(npix), 256, 0, st>>>(acc_d, acc_d ? cnt_d : nullptr, ldexp(1.0, -frac_bits),
                                             x_in_d, npix, C, x_out_d, buf);
  GLR_CUDA(cudaGetLastError());
  int s = fft2_ortho(buf, H, W, -1, st);
  if (s) return s;
  spectral_residual_kernel<<<eblocks(npix), 256, 0, st>>>(buf, y, mask_d, npix, rho);
  GLR_CUDA(cudaGetLastError());
  s = fft2_ortho(buf, H, W, +1, st);
  if (s) return s;
  fourier_update_kernel<<<eblocks(npix), 256, 0, st>>>(buf, x_out_d, npix, C, clip, lo, hi);
  GLR_CUDA(cudaGetLastError());
  s = fft2_ortho(buf, H, W, -1, st);
  if (s) return s;
  fourier_resid_kernel<<<kFBlocks, 256, 0, st>>>(buf, y, mask_d, npix, part);
  GLR_CUDA(cudaGetLastError());
  fsum_kernel<<<1, 32, 0, st>>>(part, kFBlocks, resid_d);
  return check_launch("gap_fourier");
}
