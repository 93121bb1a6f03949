// Internal cross-file entry points (not part of the C ABI).
#pragma once
#include <cstddef>
#include <cstdint>

namespace glr {

// top-K over the heat GEMM's candidate lists (topk.cu)
int topk_cand_launch(const uint64_t* cand_d, const uint32_t* cnt_d, const uint16_t* thr_d,
                     int cap, int n_max, int oh, int ow, int max_score,
                     const int32_t* anchors_d, int K, int sep, int32_t* positions_d,
                     int32_t* padded_d, uint8_t* fallback_d, void* stream);

}  // namespace glr
