// Anisotropic TV proximal step (the "tv" baseline regularizer,
// glr/solvers.py:101-139): dual projected gradient, per channel,
//   z  = x - w * div(ph, pv)
//   ph = clip(ph - (tau / w) * grad_h(z), -1, 1),  pv likewise,  tau = 1/8,
// `iters` times, then out = x - w * div(ph, pv).
// Channels are independent, so all of them run at once in the (H, W, C)
// layout. One launch per dual step reads the old (ph, pv) and writes the new
// pair (ping-pong); every product and difference is rounded as numpy rounds
// it (no FMA contraction), so the result is bit-identical to the reference.

#include <algorithm>

#include "common.cuh"

namespace glr {

// div(ph, pv) at (i, j) (solvers.py:111-117): the horizontal part first, then
// the vertical part added to it.
__device__ __forceinline__ double tv_div(const double* __restrict__ ph,
                                         const double* __restrict__ pv, int i, int j, int W,
                                         int C, int64_t e) {
  const int64_t rs = (int64_t)W * C;
  const double dh = j == 0 ? ph[e] : __dsub_rn(ph[e], ph[e - C]);
  const double dv = i == 0 ? pv[e] : __dsub_rn(pv[e], pv[e - rs]);
  return __dadd_rn(dh, dv);
}

__global__ void tv_step_kernel(const double* __restrict__ x, const double* __restrict__ ph,
                               const double* __restrict__ pv, int H, int W, int C, double w,
                               double step, double* __restrict__ ph_out,
                               double* __restrict__ pv_out) {
  const int64_t n = (int64_t)H * W * C;
  const int64_t rs = (int64_t)W * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / rs), j = (int)((e % rs) / C);
    const double z = __dsub_rn(x[e], __dmul_rn(w, tv_div(ph, pv, i, j, W, C, e)));
    double gh = 0.0, gv = 0.0;  // _grad (solvers.py:103-108): forward differences
    if (j + 1 < W)
      gh = __dsub_rn(__dsub_rn(x[e + C], __dmul_rn(w, tv_div(ph, pv, i, j + 1, W, C, e + C))), z);
    if (i + 1 < H)
      gv = __dsub_rn(__dsub_rn(x[e + rs], __dmul_rn(w, tv_div(ph, pv, i + 1, j, W, C, e + rs))),
                     z);
    ph_out[e] = fmin(fmax(__dsub_rn(ph[e], __dmul_rn(step, gh)), -1.0), 1.0);
    pv_out[e] = fmin(fmax(__dsub_rn(pv[e], __dmul_rn(step, gv)), -1.0), 1.0);
  }
}

__global__ void tv_out_kernel(const double* __restrict__ x, const double* __restrict__ ph,
                              const double* __restrict__ pv, int H, int W, int C, double w,
                              double* __restrict__ out) {
  const int64_t n = (int64_t)H * W * C;
  const int64_t rs = (int64_t)W * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / rs), j = (int)((e % rs) / C);
    out[e] = __dsub_rn(x[e], __dmul_rn(w, tv_div(ph, pv, i, j, W, C, e)));
  }
}

}  // namespace glr

using namespace glr;

extern "C" size_t glr_tv_workspace(int H, int W, int C) {
  return (size_t)4 * H * W * C * sizeof(double);
}

extern "C" int glr_tv_denoise(const double* x_d, int H, int W, int C, double weight, int iters,
                              double* out_d, void* ws_d, size_t ws_bytes, void* stream) {
  GLR_REQUIRE(H >= 1 && W >= 1 && C >= 1, GLR_ERR_INVALID, "tv: empty image");
  GLR_REQUIRE(iters >= 0, GLR_ERR_INVALID, "tv: iters must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = (int64_t)H * W * C;
  if (!(weight > 0.0)) {  // solvers.py:125-126: x.copy()
    if (out_d != x_d)
      GLR_CUDA(cudaMemcpyAsync(out_d, x_d, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return GLR_OK;
  }
  GLR_REQUIRE(ws_d && ws_bytes >= glr_tv_workspace(H, W, C), GLR_ERR_WORKSPACE,
              "tv: workspace too small");
  GLR_REQUIRE(out_d != x_d, GLR_ERR_INVALID, "tv: out must not alias x");
  double* buf = reinterpret_cast<double*>(ws_d);
  double* ph[2] = {buf, buf + 2 * n};
  double* pv[2] = {buf + n, buf + 3 * n};
  GLR_CUDA(cudaMemsetAsync(buf, 0, 2 * n * sizeof(double), st));
  const double step = 0.125 / weight;  // (tau / weight), solvers.py:136-137
  const int blocks = (int)std::min<int64_t>(cdiv(n, 256), kNumSMs * 16);
  int cur = 0;
  for (int it = 0; it < iters; ++it) {
    tv_step_kernel<<<blocks, 256, 0, st>>>(x_d, ph[cur], pv[cur], H, W, C, weight, step,
                                           ph[cur ^ 1], pv[cur ^ 1]);
    cur ^= 1;
  }
  tv_out_kernel<<<blocks, 256, 0, st>>>(x_d, ph[cur], pv[cur], H, W, C, weight, out_d);
  return check_launch("tv_kernels");
}
