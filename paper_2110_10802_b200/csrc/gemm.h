// gemm.h — internal entry points of the two contraction paths.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "dfx.h"

namespace dfx {
int gemm_simt(const dfx_gemm_args& p, cudaStream_t st);
size_t gemm_simt_workspace(const dfx_gemm_args& p);
// Returns DFX_OK after launching, or DFX_ERR_UNSUPPORTED (no error recorded)
// when the shape/layout does not tile for tcgen05.
bool gemm_tc_supported(const dfx_gemm_args& p);
int gemm_tc(const dfx_gemm_args& p, cudaStream_t st);
size_t gemm_tc_workspace(const dfx_gemm_args& p);
void gemm_tc_set_trace(void* buf);
int gemm_excite(int64_t m, int64_t k, int64_t n, const void* z, int64_t hw, const float* mean, const float* rstd,
                const float* gamma, const float* beta, const float* gate, const void* w, void* d, void* y_out,
                cudaStream_t st);
// 4-D TMA tensor map (gemm_tc.cu): dims (inner..outer) = {d0, d1, nb2, nb1}, strides in elements
int make_map(CUtensorMap* map, const void* base, int esz, uint64_t d0, uint64_t d1, int64_t s1, int64_t nb2,
             int64_t sb2, int64_t nb1, int64_t sb1, uint32_t box0, uint32_t box1, bool swizzle128);
int make_map_sw(CUtensorMap* map, const void* base, int esz, uint64_t d0, uint64_t d1, int64_t s1, int64_t nb2,
                int64_t sb2, int64_t nb1, int64_t sb1, uint32_t box0, uint32_t box1, CUtensorMapSwizzle swz);
}  // namespace dfx
