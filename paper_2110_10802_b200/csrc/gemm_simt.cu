// gemm_simt.cu — CUDA-core FP32 contraction path.
//
// Used for f32 operands (the C1 parity config: tensor-core TF32 would miss
// the 1e-4 bar, SURVEY.md §7 "hard parts") and for shapes the tcgen05 path
// does not tile.  Semantics: Gemm/MatMul/Einsum (frontend.py:335-481) and the
// Einsum VJPs (autodiff.py:1363-1459): D = epi(alpha * A·Bᵀ) with arbitrary
// element strides, two batch levels and the fused epilogues of dfx.h.
#include "common.cuh"
#include "gemm.h"

namespace dfx {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) simt_gemm_kernel(dfx_gemm_args p) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t z = blockIdx.z;
  const int64_t b1 = z / p.batch2, b2 = z % p.batch2;
  const TI* A = (const TI*)p.a + b1 * p.a_stride_b1 + b2 * p.a_stride_b2;
  const TI* B = (const TI*)p.b + b1 * p.b_stride_b1 + b2 * p.b_stride_b2;
  const bool a_kc = p.a_stride_k == 1, b_kc = p.b_stride_k == 1;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < p.k; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * 256;
      int mm, kk;
      if (a_kc) { kk = idx % BK; mm = idx / BK; } else { mm = idx % BM; kk = idx / BM; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < p.m && gk < p.k) ? to_f<TI>(A[gm * p.a_stride_m + gk * p.a_stride_k]) : 0.f;
      int nn;
      if (b_kc) { kk = idx % BK; nn = idx / BK; } else { nn = idx % BN; kk = idx / BN; }
      const int64_t gn = n0 + nn, gk2 = k0 + kk;
      Bs[kk][nn] = (gn < p.n && gk2 < p.k) ? to_f<TI>(B[gn * p.b_stride_n + gk2 * p.b_stride_k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  TO* D = (TO*)p.d + b1 * p.d_stride_b1 + b2 * p.d_stride_b2;
  const TO* AUX = p.aux ? (const TO*)p.aux + b1 * p.aux_stride_b1 + b2 * p.aux_stride_b2 : nullptr;
  TO* AO = p.aux_out ? (TO*)p.aux_out + b1 * p.aux_out_stride_b1 + b2 * p.aux_out_stride_b2 : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= p.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn >= p.n) continue;
      float v = p.alpha * acc[i][j];
      switch (p.epilogue) {
        case DFX_EPI_BIAS: v += p.bias[gn]; break;
        case DFX_EPI_BIAS_GELU:
          v += p.bias ? p.bias[gn] : 0.f;
          if (AO) AO[gm * p.aux_out_stride_m + gn] = from_f<TO>(v);
          v = gelu_f(v);
          break;
        case DFX_EPI_GELU_BWD: v *= gelu_grad_f(to_f<TO>(AUX[gm * p.aux_stride_m + gn])); break;
        case DFX_EPI_ADD: v += p.beta * to_f<TO>(AUX[gm * p.aux_stride_m + gn]); break;
        default: break;
      }
      D[gm * p.d_stride_m + gn] = from_f<TO>(v);
    }
  }
}

}  // namespace

int gemm_simt(const dfx_gemm_args& p, cudaStream_t st) {
  const int64_t nb = p.batch1 * p.batch2;
  DFX_REQUIRE(nb <= 65535, DFX_ERR_SHAPE, "dfx_gemm: too many batches for the SIMT path");
  dim3 grid((unsigned)((p.n + BN - 1) / BN), (unsigned)((p.m + BM - 1) / BM), (unsigned)nb);
  DFX_REQUIRE(grid.y <= 65535, DFX_ERR_SHAPE, "dfx_gemm: m too large for the SIMT path");
  if (p.in_dtype == DFX_F32 && p.out_dtype == DFX_F32)
    launch_k(simt_gemm_kernel<float, float>, grid, 256, 0, st, p);
  else if (p.in_dtype == DFX_BF16 && p.out_dtype == DFX_BF16)
    launch_k(simt_gemm_kernel<__nv_bfloat16, __nv_bfloat16>, grid, 256, 0, st, p);
  else if (p.in_dtype == DFX_BF16 && p.out_dtype == DFX_F32)
    launch_k(simt_gemm_kernel<__nv_bfloat16, float>, grid, 256, 0, st, p);
  else if (p.in_dtype == DFX_F32 && p.out_dtype == DFX_BF16)
    launch_k(simt_gemm_kernel<float, __nv_bfloat16>, grid, 256, 0, st, p);
  else
    return fail(DFX_ERR_DTYPE, "dfx_gemm: in/out dtype must be f32 or bf16");
  DFX_LAUNCH_CHECK("dfx_gemm (simt)");
  return DFX_OK;
}

}  // namespace dfx
