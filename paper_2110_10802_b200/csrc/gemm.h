// gemm.h — internal entry points of the two contraction paths.
#pragma once
#include <cuda_runtime.h>

#include "dfx.h"

namespace dfx {
int gemm_simt(const dfx_gemm_args& p, cudaStream_t st);
// Returns DFX_OK after launching, or DFX_ERR_UNSUPPORTED (no error recorded)
// when the shape/layout does not tile for tcgen05.
bool gemm_tc_supported(const dfx_gemm_args& p);
int gemm_tc(const dfx_gemm_args& p, cudaStream_t st);
size_t gemm_tc_workspace(const dfx_gemm_args& p);
void gemm_tc_set_trace(void* buf);
}  // namespace dfx
