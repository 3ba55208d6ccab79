// gemm_simt.cu — CUDA-core FP32 contraction path.
//
// Used for f32 operands (the C1 parity config: tensor-core TF32 would miss
// the 1e-4 bar, SURVEY.md §7 "hard parts") and for shapes the tcgen05 path
// does not tile.  Semantics: Gemm/MatMul/Einsum (frontend.py:335-481) and the
// Einsum VJPs (autodiff.py:1363-1459): D = epi(alpha * A·Bᵀ) with arbitrary
// element strides, two batch levels and the fused epilogues of dfx.h.
#include <algorithm>

#include "common.cuh"
#include "gemm.h"

namespace dfx {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

// epilogue of one output element (shared by the direct path and the split-K reduce)
template <typename TO>
__device__ __forceinline__ void simt_epilogue(const dfx_gemm_args& p, int64_t b1, int64_t b2, int64_t gm, int64_t gn,
                                              float acc) {
  TO* D = (TO*)p.d + b1 * p.d_stride_b1 + b2 * p.d_stride_b2;
  const TO* AUX = p.aux ? (const TO*)p.aux + b1 * p.aux_stride_b1 + b2 * p.aux_stride_b2 : nullptr;
  TO* AO = p.aux_out ? (TO*)p.aux_out + b1 * p.aux_out_stride_b1 + b2 * p.aux_out_stride_b2 : nullptr;
  float v = p.alpha * acc;
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

// 64 x 64 tile, 16-deep K steps, 4 x 4 outputs per thread; the next K step's
// operands are fetched into registers while the current one is multiplied
// out of shared memory (double buffering).  gridDim.z = splits x batches:
// with splits > 1 each z-slice covers a K range and writes f32 partials
// [split][batch][m][n] that simt_splitk_reduce sums and finishes.
template <typename TI, typename TO>
__global__ void __launch_bounds__(256) simt_gemm_kernel(dfx_gemm_args p, int splits, int64_t kps,
                                                        float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t nb = p.batch1 * p.batch2;
  const int64_t z = blockIdx.z % nb;
  const int split = (int)(blockIdx.z / nb);
  const int64_t b1 = z / p.batch2, b2 = z % p.batch2;
  const TI* A = (const TI*)p.a + b1 * p.a_stride_b1 + b2 * p.a_stride_b2;
  const TI* B = (const TI*)p.b + b1 * p.b_stride_b1 + b2 * p.b_stride_b2;
  const bool a_kc = p.a_stride_k == 1, b_kc = p.b_stride_k == 1;
  const int64_t kbeg = (int64_t)split * kps, kend = min(p.k, kbeg + kps);
  float2 acc2[4][2];  // packed fp32 pairs along n: FFMA2 issues two FMAs
#pragma unroll
  for (int i = 0; i < 4; ++i) acc2[i][0] = acc2[i][1] = make_float2(0.f, 0.f);
  float ra[4], rb[4];
  int am[4], ak[4], bn_[4], bk[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = tid + i * 256;
    if (a_kc) { ak[i] = idx % BK; am[i] = idx / BK; } else { am[i] = idx % BM; ak[i] = idx / BM; }
    if (b_kc) { bk[i] = idx % BK; bn_[i] = idx / BK; } else { bn_[i] = idx % BN; bk[i] = idx / BN; }
  }
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t gm = m0 + am[i], gk = k0 + ak[i];
      ra[i] = (gm < p.m && gk < kend) ? to_f<TI>(A[gm * p.a_stride_m + gk * p.a_stride_k]) : 0.f;
      const int64_t gn = n0 + bn_[i], gk2 = k0 + bk[i];
      rb[i] = (gn < p.n && gk2 < kend) ? to_f<TI>(B[gn * p.b_stride_n + gk2 * p.b_stride_k]) : 0.f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      As[buf][ak[i]][am[i]] = ra[i];
      Bs[buf][bk[i]][bn_[i]] = rb[i];
    }
  };
  int buf = 0;
  if (kbeg < kend) {
    fetch(kbeg);
    stash(0);
  }
  __syncthreads();
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) fetch(k0 + BK);  // in flight while the current step computes
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float2 b01 = make_float2(b.x, b.y), b23 = make_float2(b.z, b.w);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 ai = make_float2(av[i], av[i]);
        acc2[i][0] = __ffma2_rn(ai, b01, acc2[i][0]);
        acc2[i][1] = __ffma2_rn(ai, b23, acc2[i][1]);
      }
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= p.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn >= p.n) continue;
      const float v = (j & 1) ? acc2[i][j >> 1].y : acc2[i][j >> 1].x;
      if (splits > 1)
        part[(((int64_t)split * nb + z) * p.m + gm) * p.n + gn] = v;
      else
        simt_epilogue<TO>(p, b1, b2, gm, gn, v);
    }
  }
}

// fixed-order sum of the split-K partials, then the epilogue
template <typename TO>
__global__ void __launch_bounds__(256) simt_splitk_reduce(dfx_gemm_args p, int splits, const float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  const int64_t nb = p.batch1 * p.batch2;
  const int64_t total = nb * p.m * p.n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += part[(int64_t)s * total + i];
    const int64_t gn = i % p.n, gm = (i / p.n) % p.m, z = i / (p.n * p.m);
    simt_epilogue<TO>(p, z / p.batch2, z % p.batch2, gm, gn, acc);
  }
}

// split-K plan: few output tiles + long K (the C1 fp32 layer: 256 x 768 x 3072)
int simt_splits(const dfx_gemm_args& p) {
  const int64_t nb = p.batch1 * p.batch2;
  const int64_t tiles = nb * ((p.m + BM - 1) / BM) * ((p.n + BN - 1) / BN);
  const int sms = num_sms();
  if (nb != 1 || tiles >= sms || p.k < 512) return 1;
  int64_t s = std::min<int64_t>(16, std::min<int64_t>((2 * sms) / std::max<int64_t>(tiles, 1), p.k / 256));
  return (int)std::max<int64_t>(1, s);
}

}  // namespace

size_t gemm_simt_workspace(const dfx_gemm_args& p) {
  const int s = simt_splits(p);
  return s > 1 ? (size_t)s * p.batch1 * p.batch2 * p.m * p.n * sizeof(float) + 256 : 0;
}

int gemm_simt(const dfx_gemm_args& p, cudaStream_t st) {
  const int64_t nb = p.batch1 * p.batch2;
  int splits = simt_splits(p);
  float* part = nullptr;
  if (splits > 1) {
    if (!p.workspace || p.workspace_bytes < gemm_simt_workspace(p) || !aligned16(p.workspace)) splits = 1;
    else part = (float*)p.workspace;
  }
  const int64_t kps = (p.k + splits - 1) / splits;
  DFX_REQUIRE(nb * splits <= 65535, DFX_ERR_SHAPE, "dfx_gemm: too many batches for the SIMT path");
  dim3 grid((unsigned)((p.n + BN - 1) / BN), (unsigned)((p.m + BM - 1) / BM), (unsigned)(nb * splits));
  DFX_REQUIRE(grid.y <= 65535, DFX_ERR_SHAPE, "dfx_gemm: m too large for the SIMT path");
#define SIMT_LAUNCH(TI, TO)                                                                              \
  {                                                                                                      \
    launch_k(simt_gemm_kernel<TI, TO>, grid, 256, 0, st, p, splits, kps, part);                          \
    if (splits > 1) {                                                                                    \
      DFX_LAUNCH_CHECK("dfx_gemm (simt split-K)");                                                       \
      const int64_t total = nb * p.m * p.n;                                                              \
      const int g2 = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);                \
      launch_k(simt_splitk_reduce<TO>, g2, 256, 0, st, p, splits, (const float*)part);                   \
    }                                                                                                    \
  }
  if (p.in_dtype == DFX_F32 && p.out_dtype == DFX_F32) SIMT_LAUNCH(float, float)
  else if (p.in_dtype == DFX_BF16 && p.out_dtype == DFX_BF16) SIMT_LAUNCH(__nv_bfloat16, __nv_bfloat16)
  else if (p.in_dtype == DFX_BF16 && p.out_dtype == DFX_F32) SIMT_LAUNCH(__nv_bfloat16, float)
  else if (p.in_dtype == DFX_F32 && p.out_dtype == DFX_BF16) SIMT_LAUNCH(float, __nv_bfloat16)
  else return fail(DFX_ERR_DTYPE, "dfx_gemm: in/out dtype must be f32 or bf16");
#undef SIMT_LAUNCH
  DFX_LAUNCH_CHECK("dfx_gemm (simt)");
  return DFX_OK;
}

}  // namespace dfx
