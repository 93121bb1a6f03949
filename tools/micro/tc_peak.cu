// Microbenchmark: dense tcgen05.mma throughput per kind on this GPU (one CTA
// per SM, operands resident in shared memory, one issuing thread, M = 128,
// N = 256, one TMEM accumulator). Gives the measured peaks the heat map
// (kind::mxf4) and the split-integer WNNM apply (kind::i8) are reported
// against; kind::f16 (bf16) is printed beside them to calibrate against the
// driver's cuBLAS bf16 figure in MEASURED_PEAKS.json.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2301_03047_b200/csrc \
//        tools/micro/tc_peak.cu -o build/tc_peak && build/tc_peak
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace glr;

enum Kind { F16 = 0, I8 = 1, MXF4 = 2 };

template <int KIND>
__global__ void __launch_bounds__(128, 1) tc_peak_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;                 // 128 rows x 128 B
  uint8_t* B = sm + 128 * 128;     // 256 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // pseudo-random operand bytes (not all zeros: realistic datapath activity)
  for (int i = tid; i < 384 * 128 / 4; i += 128) {
    uint32_t v = (uint32_t)i * 2654435761u ^ 0x5bd1e995u;
    if (KIND == MXF4) v &= 0x22222222u;  // E2M1 0.0 / 1.0 nibbles
    if (KIND == F16) v &= 0x3f803f80u;   // bf16 0.0 / 1.0
    reinterpret_cast<uint32_t*>(sm)[i] = v;
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (KIND == MXF4) {  // scale factors = UE8M0 127 (2^0) in columns 448.. / 480..
    uint32_t ones[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) ones[i] = 0x7f7f7f7fu;
    const uint32_t lanes = (uint32_t)(warp * 32) << 16;
    tmem_st_32x32b_x32(tmem + lanes + 448, ones);
    tmem_st_32x32b_x32(tmem + lanes + 480, ones);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint64_t ad = smem_desc_k_sw128(A), bd = smem_desc_k_sw128(B);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i != 0;
      if (KIND == MXF4) {
        umma_mxf4(tmem, ad, bd, idesc_mxf4(128, 256), acc, tmem + 448, tmem + 480);
      } else if (KIND == I8) {
        umma_i8(tmem, ad, bd, idesc_s8_s32(128, 256), acc);
      } else {
        const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) |
                            ((128u >> 4) << 24);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(id), "r"(acc));
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) *cycles = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int KIND>
static void run(const char* name, double flop_per_mma, int sms) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const int smem = 384 * 128 + 2048;
  cudaFuncSetAttribute(tc_peak_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  tc_peak_kernel<KIND><<<sms, 128, smem>>>(1000, cyc);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    tc_peak_kernel<KIND><<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const cudaError_t err = cudaGetLastError();
  const double tf = flop_per_mma * iters * sms / (best * 1e-3) / 1e12;
  printf("{\"kind\": \"%s\", \"tflops\": %.1f, \"ms\": %.3f, \"clk_per_mma\": %.1f, \"sms\": %d, "
         "\"err\": \"%s\"}\n", name, tf, best, (double)c / iters, sms, cudaGetErrorString(err));
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<F16>("bf16 (kind::f16, M128 N256 K16)", 2.0 * 128 * 256 * 16, sms);
  run<I8>("s8 (kind::i8, M128 N256 K32)", 2.0 * 128 * 256 * 32, sms);
  run<MXF4>("e2m1 (kind::mxf4 block32, M128 N256 K64)", 2.0 * 128 * 256 * 64, sms);
  return 0;
}
