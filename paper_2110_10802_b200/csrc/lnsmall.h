// lnsmall.h — LayerNorm(+swish) over short channels-last rows (lnsmall.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dfx {
// true when cols is 1, 2, 4, 8, 16 or 32 vectors (bf16: 8 channels, f32: 4)
bool ln_small_ok(int dtype, int64_t cols);
int ln_small_fwd(int dtype, int64_t rows, int64_t cols, const void* x, const float* gamma, const float* beta,
                 float eps, int act, void* y, cudaStream_t st);
int ln_small_bwd(int dtype, int64_t rows, int64_t cols, const void* dy, const void* x, const float* gamma,
                 const float* beta, float eps, int act, void* dx, float* dgamma, float* dbeta, void* workspace,
                 size_t ws_bytes, cudaStream_t st);
}  // namespace dfx
