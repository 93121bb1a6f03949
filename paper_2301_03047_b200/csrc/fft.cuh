// fp64 complex 2-D DFT used by the masked-Fourier operator (fft.cu).
#pragma once
#include <cuda_runtime.h>

namespace glr {

// In-place unitary ("ortho") 2-D DFT of an H x W complex128 array (row-major,
// interleaved re/im). sign = -1 forward (numpy fft2), +1 inverse (ifft2).
int fft2_ortho(double2* data, int H, int W, int sign, cudaStream_t st);

}  // namespace glr
