// (2) Global similarity heat map as an implicit GEMM on tcgen05 tensor cores.
//
// Reference: glr/matching.py:140-167 (similarity_heatmap, im2col branch
// :145-156): heat[u,v,n] = sum over the P x P x 4C window of the product of
// the binary edge stack at position (u,v) and at exemplar anchor n. The
// reference runs this as an OpenBLAS sgemm on an explicit im2col copy; here
// the im2col is never materialised:
//
//   * The edge stack holds the binary maps as (H, W, Ce) elements with
//     Ce = e*4C ("e-row expanded": channel p*4C+k of pixel (r,c) holds
//     map_k(r+p, c)), each element an E2M1 (fp4) 1.0 or 0.0 packed two per
//     byte, so a pixel is Cb = Ce/2 bytes. For a fixed output row u and slab
//     s, the K-run of position v is the contiguous byte range
//     stack[u+s*e][v .. v+P-1][*] of length L = P*Cb, and consecutive v are
//     Cb bytes apart. A 3-D TMA map with dims {L, ow, H} and strides
//     {Cb, W*Cb} therefore addresses the overlapping im2col rows directly;
//     one TMA box = 128 positions x 128 bytes (256 K-elements).
//   * The exemplar operand B (Npad x Kp bytes, K-major, zero-padded) is
//     gathered once per refresh from the same stack (exemplar_pack_kernel).
//   * tcgen05.mma kind::mxf4 (block-scaled fp4, f32 accumulate) with every
//     UE8M0 scale factor = 2^0: products of 0/1 are exact and the f32 sums
//     are exact integers (max 4*C*P^2 < 2^24). fp4 halves the operand bytes
//     per multiply-add of the u8 formulation (this kernel is bound by the
//     L2 -> shared-memory operand stream) and runs at twice the i8 rate.
//     Accumulators live in TMEM (2 x 128 lanes x 224 columns), the constant
//     scale factors in the remaining 64 columns.
//   * Output: exemplar-major u16 heat[n][u*ow+v] (flat index = the
//     reference's row-major slice index, matching.py:177-178), rows padded
//     to a multiple of 8 entries (glr_heat_stride) for 16-byte loads.
//
// Persistent, warp-specialised kernel (256 threads, one CTA per SM), launched
// as clusters of CL CTAs that work on adjacent position tiles of the same
// exemplar tile: each CTA loads its own A box and 1/CL of the B box,
// multicast into every CTA's shared memory, so the L2 -> SM operand stream
// (the bound) carries 16 + 28/CL KB per stage instead of 16 + 28 KB.
//   warp 0 (one lane)  TMA producer, 5-stage smem ring (full/empty mbarriers;
//                      a stage is refilled once ALL CTAs' MMAs released it);
//   warp 1 (one lane)  tcgen05.mma issuer into one of two TMEM accumulators;
//   warp 2             owns the 512-column TMEM allocation;
//   warps 4-7          also write the constant scale factors at start-up;
//   warps 4-7          epilogue: tcgen05.ld -> u16 stores, then release the
//                      accumulator, so tile i's epilogue overlaps tile i+1's
//                      MMAs (accumulator handoff via tmem_full/tmem_empty).
#include <cstdio>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace glr {

namespace heat {
constexpr int BM = 128;      // positions per tile (UMMA M)
constexpr int BN = 224;      // exemplars per tile (UMMA N)
constexpr int BK = 128;      // bytes of K per stage (one 128B swizzle row = 256 fp4)
constexpr int UK = 32;       // bytes of K per tcgen05.mma kind::mxf4 (64 fp4)
constexpr int STAGES = 5;
constexpr int CL = 2;        // CTAs per cluster sharing one exemplar tile (multicast)
constexpr int ACC = 2;       // TMEM accumulators (2 x 224 columns)
constexpr int THREADS = 256;
constexpr int A_BYTES = BM * BK;
constexpr int B_BYTES = BN * BK;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t SFA_COL = 448;  // 32 columns of scale factors for A
constexpr uint32_t SFB_COL = 480;  // 32 columns of scale factors for B
}  // namespace heat

struct HeatGeom {
  int H, W, C4, P, e, Ce, Cb, S, L, kchunks, Kp, oh, ow;
};

static HeatGeom heat_geom(int H, int W, int C, int P, int e) {
  HeatGeom g;
  g.H = H;
  g.W = W;
  g.C4 = 4 * C;
  g.P = P;
  g.e = e;
  g.Ce = e * 4 * C;
  g.Cb = g.Ce / 2;
  g.S = (int)cdiv(P, e);
  g.L = P * g.Cb;
  g.kchunks = (int)cdiv(g.L, heat::BK);
  g.Kp = g.S * g.kchunks * heat::BK;
  g.oh = H - P + 1;
  g.ow = W - P + 1;
  return g;
}

struct HeatParams {
  int oh, ow, Mpad, n_max, m_tiles_per_row, S, kchunks, e;
  const int32_t* n_dev;
  uint16_t* heat;
};

__global__ void __launch_bounds__(heat::THREADS, 1)
    heat_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, HeatParams p) {
  using namespace heat;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + ACC);

  const int N = p.n_dev ? min(*p.n_dev, p.n_max) : p.n_max;
  const int n_tiles = (N + BN - 1) / BN;
  // tile pairs (two m tiles, one n tile), n fastest: clusters share A tiles in L2
  const int total = p.oh * (p.m_tiles_per_row / CL) * n_tiles;
  const int num_k = p.S * p.kchunks;
  const int rank = (int)cluster_ctarank();
  const int cl = blockIdx.x / CL, n_cl = gridDim.x / CL;
  constexpr uint16_t kAll = (1u << CL) - 1;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // every CTA's MMA commit
    }
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peers' barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp >= 4) {
    // every scale-factor byte = UE8M0 127 = 2^0, whatever the layout the MMA reads
    uint32_t ones[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) ones[j] = 0x7F7F7F7Fu;
    const uint32_t lanes = (uint32_t)((warp - 4) * 32) << 16;
    tmem_st_32x32b_x32(tmem + lanes + SFA_COL, ones);
    tmem_st_32x32b_x32(tmem + lanes + SFB_COL, ones);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      int it = 0;
      for (int t = cl; t < total; t += n_cl) {
        const int n0 = (t % n_tiles) * BN;
        const int m_tile = CL * (t / n_tiles) + rank;
        const int u = m_tile / p.m_tiles_per_row;
        const int v0 = (m_tile % p.m_tiles_per_row) * BM;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          if (it >= STAGES) mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          const int slab = kb / p.kchunks;
          const int kc = kb - slab * p.kchunks;
          tma_load_3d(sA + s * A_BYTES, &tmA, &full[s], kc * BK, v0, u + slab * p.e);
          tma_load_2d_mc(sB + s * B_BYTES + rank * (B_BYTES / CL), &tmB, &full[s], kb * BK,
                         n0 + rank * (BN / CL), kAll);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      constexpr uint32_t idesc = idesc_mxf4(BM, BN);
      int it = 0, lt = 0;
      for (int t = cl; t < total; t += n_cl, ++lt) {
        const int acc = lt & 1, use = lt >> 1;
        if (use > 0) mbar_wait(&tempty[acc], (use - 1) & 1);  // epilogue drained it
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = smem_desc_k_sw128(sA + s * A_BYTES);
          const uint64_t bd = smem_desc_k_sw128(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)  // +32 bytes inside the 128B swizzle atom
            umma_mxf4(d, ad + (uint64_t)((k * UK) >> 4), bd + (uint64_t)((k * UK) >> 4), idesc,
                      (kb | k) != 0, tmem + SFA_COL, tmem + SFB_COL);
          umma_commit_mc(&empty[s], kAll);  // frees stage s in every CTA
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> registers -> u16 exemplar-major rows ----
    const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31 (warp id % 4)
    int lt = 0;
    for (int t = cl; t < total; t += n_cl, ++lt) {
      const int acc = lt & 1, use = lt >> 1;
      const int n0 = (t % n_tiles) * BN;
      const int m_tile = CL * (t / n_tiles) + rank;
      const int u = m_tile / p.m_tiles_per_row;
      const int v = (m_tile % p.m_tiles_per_row) * BM + ew * 32 + lane;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const bool v_ok = v < p.ow;
      uint16_t* out = p.heat + (size_t)u * p.ow + v;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * BN + c * 32), r);
        tmem_ld_wait();
        const int nb = n0 + c * 32;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = nb + j;
          if (v_ok && n < N) out[(size_t)n * p.Mpad] = (uint16_t)__float2uint_rn(__uint_as_float(r[j]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still multicast into it
  if (warp == 2) tmem_dealloc<TMEM_COLS>(tmem);
}

// B operand (bytes): bmat[n][s*kchunks*BK + k'] = stack[r_n + s*e][c_n + k'/Cb][k' % Cb]
// for k' < L, zero for the K padding, for the padded exemplars and past row H.
__global__ void exemplar_pack_kernel(const uint8_t* __restrict__ stack, HeatGeom g,
                                     const int32_t* __restrict__ anchors, int n_max,
                                     const int32_t* n_dev, int n_pad, uint8_t* __restrict__ bmat) {
  const int N = n_dev ? min(*n_dev, n_max) : n_max;
  const int row_bytes = g.Kp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n_pad * row_bytes;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / row_bytes);
    const int k = (int)(i - (int64_t)n * row_bytes);
    const int slab = k / (g.kchunks * heat::BK);
    const int kk = k - slab * g.kchunks * heat::BK;
    uint8_t val = 0;
    if (n < N && kk < g.L) {
      const int cb = kk % g.Cb;
      // the byte's two expanded channels 2cb, 2cb+1 (same row: 4C is even) hold
      // map row (anchor row + slab*e + 2cb / 4C); rows at or past P belong to
      // no patch and stay zero
      if (slab * g.e + (2 * cb) / g.C4 < g.P) {
        const int r = anchors[2 * n] + slab * g.e;
        const int c = anchors[2 * n + 1] + kk / g.Cb;
        val = stack[((size_t)r * g.W + c) * g.Cb + cb];
      }
    }
    bmat[i] = val;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

}  // namespace glr

using namespace glr;

extern "C" int glr_heat_expand_factor(int C, int P) {
  // Smallest padded K (then the smallest expansion) among e in [1, max(P,8)]
  // whose pixel stride e*4C/2 bytes is a multiple of 16 (TMA stride rule);
  // e = 8 always qualifies. Expanded rows at or past P are zero in B.
  int best_e = -1;
  int64_t best_k = 0;
  for (int e = 1; e <= (P > 8 ? P : 8); ++e) {
    if ((4 * C * e) % 32 != 0) continue;
    HeatGeom g = heat_geom(P, P, C, P, e);
    if (best_e < 0 || g.Kp < best_k) {
      best_e = e;
      best_k = g.Kp;
    }
  }
  return best_e;
}

extern "C" int64_t glr_heat_stride(int H, int W, int P) {
  return cdiv((int64_t)(H - P + 1) * (W - P + 1), 8) * 8;
}

extern "C" size_t glr_heat_workspace(int C, int P, int n_max) {
  int e = glr_heat_expand_factor(C, P);
  if (e < 1) return 0;
  HeatGeom g = heat_geom(P, P, C, P, e);
  size_t n_pad = (size_t)cdiv(n_max, heat::BN) * heat::BN;
  return n_pad * (size_t)g.Kp + 256;
}

extern "C" int glr_heat_map(const uint8_t* stack_d, int H, int W, int C, int P, int expand,
                            const int32_t* anchors_d, int n_max, const int32_t* n_dev_d,
                            uint16_t* heat_d, void* ws_d, size_t ws_bytes, void* stream) {
  GLR_REQUIRE(P >= 1 && P <= H && P <= W && C >= 1, GLR_ERR_INVALID,
              "heat_map: bad shape H=%d W=%d C=%d P=%d", H, W, C, P);
  GLR_REQUIRE(expand >= 1 && expand <= (P > 8 ? P : 8) && (4 * C * expand) % 32 == 0,
              GLR_ERR_INVALID,
              "heat_map: expand factor %d invalid for C=%d", expand, C);
  if (n_max <= 0) return GLR_OK;
  HeatGeom g = heat_geom(H, W, C, P, expand);
  GLR_REQUIRE(4 * C * P * P <= 65535, GLR_ERR_UNSUPPORTED,
              "heat_map: max score %d does not fit u16", 4 * C * P * P);
  const int n_pad = (int)cdiv(n_max, heat::BN) * heat::BN;
  GLR_REQUIRE(ws_bytes >= (size_t)n_pad * g.Kp, GLR_ERR_WORKSPACE,
              "heat_map: workspace %zu < %zu", ws_bytes, (size_t)n_pad * g.Kp);
  auto encode = get_encode_fn();
  GLR_REQUIRE(encode != nullptr, GLR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* bmat = reinterpret_cast<uint8_t*>(ws_d);

  {
    int64_t total = (int64_t)n_pad * g.Kp;
    int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
    exemplar_pack_kernel<<<blocks, 256, 0, st>>>(stack_d, g, anchors_d, n_max, n_dev_d, n_pad,
                                                 bmat);
    GLR_CUDA(cudaGetLastError());
  }

  CUtensorMap tmA, tmB;
  {
    cuuint64_t dims[3] = {(cuuint64_t)g.L, (cuuint64_t)g.ow, (cuuint64_t)H};
    cuuint64_t strides[2] = {(cuuint64_t)g.Cb, (cuuint64_t)W * g.Cb};
    cuuint32_t box[3] = {heat::BK, heat::BM, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)stack_d, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GLR_REQUIRE(r == CUDA_SUCCESS, GLR_ERR_CUDA, "cuTensorMapEncodeTiled(A) failed: %d", (int)r);
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)g.Kp, (cuuint64_t)n_pad};
    cuuint64_t strides[1] = {(cuuint64_t)g.Kp};
    cuuint32_t box[2] = {heat::BK, heat::BN / heat::CL};  // each CTA loads its slice
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)bmat, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GLR_REQUIRE(r == CUDA_SUCCESS, GLR_ERR_CUDA, "cuTensorMapEncodeTiled(B) failed: %d", (int)r);
  }

  HeatParams hp;
  hp.oh = g.oh;
  hp.ow = g.ow;
  hp.Mpad = (int)glr_heat_stride(H, W, P);
  hp.n_max = n_max;
  hp.m_tiles_per_row = (int)cdiv(g.ow, heat::CL * heat::BM) * heat::CL;  // tiles go in clusters
  hp.S = g.S;
  hp.kchunks = g.kchunks;
  hp.e = g.e;
  hp.n_dev = n_dev_d;
  hp.heat = heat_d;
  static bool attr_set = false;
  if (!attr_set) {
    GLR_CUDA(cudaFuncSetAttribute(heat_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  heat::SMEM_BYTES));
    attr_set = true;
  }
  const int64_t pairs = (int64_t)g.oh * (hp.m_tiles_per_row / heat::CL) * (n_pad / heat::BN);
  GLR_REQUIRE(pairs < (1ll << 31), GLR_ERR_UNSUPPORTED, "heat_map: too many tiles");
  int sms = kNumSMs;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(heat::THREADS);
  cfg.dynamicSmemBytes = heat::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = heat::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent: one CTA per SM, in clusters of two -- as many clusters as can
  // be co-resident (the GPCs need not split into pairs evenly)
  static int max_clusters = 0;
  if (max_clusters == 0) {
    cfg.gridDim = dim3(heat::CL * (sms / heat::CL));
    if (cudaOccupancyMaxActiveClusters(&max_clusters, heat_gemm_kernel, &cfg) != cudaSuccess ||
        max_clusters < 1)
      max_clusters = sms / heat::CL;
    cudaGetLastError();
  }
  cfg.gridDim = dim3(heat::CL * (unsigned)std::min<int64_t>(pairs, max_clusters));
  GLR_CUDA(cudaLaunchKernelEx(&cfg, heat_gemm_kernel, tmA, tmB, hp));
  return GLR_OK;
}
