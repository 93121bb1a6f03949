// Internal cross-file entry points (not part of the C ABI).
#pragma once
#include <cstddef>
#include <cstdint>

namespace glr {

// Per-device native state (common.cu). Kernel attributes and occupancy
// queries are per device in CUDA, so every cache below is keyed by the
// CURRENT device (cudaGetDevice) and guarded by a mutex: a process may drive
// several GPUs, from several threads, through the same library.
//   ensure_smem_attr: cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once
//                     per (kernel, device, size);
//   device_sms:       multiprocessor count of the current device;
//   cached_per_device: a per-(key, device) integer computed once by `init`.
int ensure_smem_attr(const void* kernel, int bytes);
int device_sms();
int cached_per_device(const void* key, int (*init)(void* ctx), void* ctx);

// top-K over the heat GEMM's candidate lists (topk.cu)
int topk_cand_launch(const uint64_t* cand_d, const uint32_t* cnt_d, const uint16_t* thr_d,
                     int cap, int n_max, int oh, int ow, int max_score,
                     const int32_t* anchors_d, int K, int sep, int32_t* positions_d,
                     int32_t* padded_d, uint8_t* fallback_d, void* stream);

}  // namespace glr
