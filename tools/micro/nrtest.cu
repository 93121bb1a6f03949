#include <cstdio>
#include <cmath>
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  for (int i = 0; i < 2; ++i) y = fma(y, fma(-x, y, 1.0), y);
  return y;
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  for (int i = 0; i < 2; ++i) y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
  return y;
}
__global__ void k(double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = exp2(-40.0 + 80.0 * (i / (double)n)) * (1.0 + 0.37 * sin((double)i));
  out[4 * i] = x; out[4*i+1] = rcp_nr(x); out[4*i+2] = rsqrt_nr(x); out[4*i+3] = 0;
}
int main() {
  int n = 1 << 20; double* d; cudaMalloc(&d, 32 * n);
  k<<<n / 256, 256>>>(d, n);
  double* h = new double[4 * n]; cudaMemcpy(h, d, 32 * n, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < n; ++i) {
    long double x = h[4*i];
    e1 = fmax(e1, (double)fabsl(h[4*i+1] * x - 1.0L));
    e2 = fmax(e2, (double)fabsl(h[4*i+2] * h[4*i+2] * x - 1.0L));
  }
  printf("max rel err rcp %.3e rsqrt^2 %.3e (ulp %.3e)\n", e1, e2, 1.1e-16);
  return 0;
}
