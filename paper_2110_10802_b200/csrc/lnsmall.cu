// lnsmall.cu — LayerNorm (+ swish) over SHORT rows (C <= 32 vectors, the
// channels-last normalisation sweep of config C4: C = 32 / 64 channels),
// sm_100a.  The BDRLN row kernels give a whole warp to one row, which leaves
// 24 of 32 lanes idle at C = 64 bf16; here a row is a group of G = C/V lanes
// (G in {1, 2, 4, 8, 16, 32}), a warp holds 32/G rows, and each thread keeps
// four rows' vectors in flight.  Mean / variance / the VJP means reduce with
// xor-shuffles inside the group.
//
// Reference: LayerNormalization over the last axis (frontend.py:519-529,
// biased variance) followed by swish = Mul(u, Sigmoid(u)) (frontend.py:229,
// 293); VJP _bwd_layernorm (autodiff.py:1490-1545) with the swish derivative.
// dgamma / dbeta: per-thread column accumulators -> per-CTA partials ->
// fixed-order f64 column sums (bitwise reproducible).
#include <algorithm>

#include "common.cuh"
#include "lnsmall.h"

namespace dfx {
namespace {

constexpr int kU = 4;   // rows in flight per thread (forward)
constexpr int kUb = 2;  // backward: x and dy rows in flight; bf16 rows of <= 64 channels fit 80 registers -> 3 CTAs per SM

template <int G> __device__ __forceinline__ float gsum(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T> __device__ __forceinline__ float sig_small(float u) {
  if constexpr (sizeof(T) == 2) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(0.5f * u));
    return fmaf(0.5f, y, 0.5f);
  } else {
    return sigmoid_f(u);
  }
}

template <typename T, int V, int G, int ACT>
__global__ void __launch_bounds__(256) ln_small_fwd_kernel(int64_t rows, const T* __restrict__ x,
                                                           const float* __restrict__ gamma,
                                                           const float* __restrict__ beta, float eps,
                                                           T* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  constexpr int C = G * V, RPW = 32 / G;
  const int lane = threadIdx.x & 31, gl = lane % G, rs = lane / G;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  float g[V], b[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    g[i] = gamma[gl * V + i];
    b[i] = beta[gl * V + i];
  }
  for (int64_t r0 = wid * RPW * kU; r0 < rows; r0 += nw * RPW * kU) {
    Vec<T, V> xv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t r = r0 + u * RPW + rs;
      if (r < rows) xv[u].load(x + r * C + gl * V);
      else {
#pragma unroll
        for (int i = 0; i < V; ++i) xv[u].v[i] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) s += xv[u].v[i];
      const float mean = gsum<G>(s) * (1.f / C);
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float d = xv[u].v[i] - mean;
        q = fmaf(d, d, q);
      }
      const float rstd = rsqrtf(gsum<G>(q) * (1.f / C) + eps);
      Vec<T, V> yv;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float uu = fmaf((xv[u].v[i] - mean) * rstd, g[i], b[i]);
        yv.v[i] = ACT ? uu * sig_small<T>(uu) : uu;
      }
      const int64_t r = r0 + u * RPW + rs;
      if (r < rows) yv.store(y + r * C + gl * V);
    }
  }
}

template <typename T, int V, int G, int ACT>
__global__ void __launch_bounds__(256, (sizeof(T) == 2 && G <= 8) ? 3 : 2) ln_small_bwd_kernel(int64_t rows, const T* __restrict__ dy,
                                                           const T* __restrict__ x, const float* __restrict__ gamma,
                                                           const float* __restrict__ beta, float eps,
                                                           T* __restrict__ dx, float* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  constexpr int C = G * V, RPW = 32 / G;
  __shared__ float red[8 * 32 * V];  // [warp * RPW + rs][C] for one of (dgamma, dbeta)
  const int lane = threadIdx.x & 31, gl = lane % G, rs = lane / G, warp = threadIdx.x / 32;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + warp;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  float g[V], b[V], ag[V], ab[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    g[i] = gamma[gl * V + i];
    b[i] = beta[gl * V + i];
    ag[i] = 0.f;
    ab[i] = 0.f;
  }
  for (int64_t r0 = wid * RPW * kUb; r0 < rows; r0 += nw * RPW * kUb) {
    Vec<T, V> xv[kUb], dv[kUb];
#pragma unroll
    for (int u = 0; u < kUb; ++u) {
      const int64_t r = r0 + u * RPW + rs;
      if (r < rows) {
        xv[u].load(x + r * C + gl * V);
        dv[u].load(dy + r * C + gl * V);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) {
          xv[u].v[i] = 0.f;
          dv[u].v[i] = 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUb; ++u) {
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) s += xv[u].v[i];
      const float mean = gsum<G>(s) * (1.f / C);
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float d = xv[u].v[i] - mean;
        q = fmaf(d, d, q);
      }
      const float rstd = rsqrtf(gsum<G>(q) * (1.f / C) + eps);
      float xh[V], dxh[V], s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        xh[i] = (xv[u].v[i] - mean) * rstd;
        float du = dv[u].v[i];
        if (ACT) {
          const float uu = fmaf(xh[i], g[i], b[i]);
          const float sg = sig_small<T>(uu);
          du *= sg * fmaf(uu, 1.f - sg, 1.f);
        }
        ag[i] = fmaf(du, xh[i], ag[i]);  // padded rows contribute du = 0
        ab[i] += du;
        dxh[i] = du * g[i];
        s1 += dxh[i];
        s2 = fmaf(dxh[i], xh[i], s2);
      }
      const float m1 = gsum<G>(s1) * (1.f / C), m2 = gsum<G>(s2) * (1.f / C);
      Vec<T, V> o;
#pragma unroll
      for (int i = 0; i < V; ++i) o.v[i] = rstd * (dxh[i] - m1 - xh[i] * m2);
      const int64_t r = r0 + u * RPW + rs;
      if (r < rows) o.store(dx + r * C + gl * V);
    }
  }
  // CTA partials: fixed order over the block's (warp, row-slot) lanes
  const int nslot = (blockDim.x / 32) * RPW;
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int i = 0; i < V; ++i) red[(warp * RPW + rs) * C + gl * V + i] = q == 0 ? ag[i] : ab[i];
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      float acc = 0.f;
      for (int j = 0; j < nslot; ++j) acc += red[j * C + c];
      part[((size_t)blockIdx.x * 2 + q) * C + c] = acc;
    }
    __syncthreads();
  }
}

// dgamma / dbeta = fixed-order f64 sums of the CTA partials [nb][2][C]
// (1024 threads per 32 columns, sum_part_rows)
__global__ void __launch_bounds__(1024) ln_small_finalize_kernel(int nb, int C, const float* __restrict__ part,
                                                                 float* __restrict__ dgamma,
                                                                 float* __restrict__ dbeta) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sred[32][33];
  const int idx = blockIdx.x * 32 + (threadIdx.x & 31);  // over 2C
  const double v = sum_part_rows(nb, part, (size_t)2 * C, idx, idx < 2 * C, sred);
  if (threadIdx.x < 32 && idx < 2 * C) {
    if (idx < C) dgamma[idx] = (float)v;
    else dbeta[idx - C] = (float)v;
  }
}

constexpr int kMaxBlocks = 8 * 148;

template <typename T, int V, int G>
int fwd_launch(int64_t rows, const void* x, const float* gamma, const float* beta, float eps, int act, void* y,
               cudaStream_t st) {
  constexpr int RPW = 32 / G;
  const int64_t per_block = 8LL * RPW * kU;
  const int grid = (int)std::min<int64_t>((rows + per_block - 1) / per_block, (int64_t)num_sms() * 8);
  if (act)
    launch_k(ln_small_fwd_kernel<T, V, G, 1>, grid, 256, 0, st, rows, (const T*)x, gamma, beta, eps, (T*)y);
  else
    launch_k(ln_small_fwd_kernel<T, V, G, 0>, grid, 256, 0, st, rows, (const T*)x, gamma, beta, eps, (T*)y);
  DFX_LAUNCH_CHECK("dfx_layernorm_act_fwd (short rows)");
  return DFX_OK;
}

template <typename T, int V, int G>
int bwd_launch(int64_t rows, const void* dy, const void* x, const float* gamma, const float* beta, float eps,
               int act, void* dx, float* dgamma, float* dbeta, float* part, size_t part_floats, cudaStream_t st) {
  constexpr int RPW = 32 / G, C = G * V;
  const int64_t per_block = 8LL * RPW * kUb;
  int grid = (int)std::min<int64_t>((rows + per_block - 1) / per_block, (int64_t)std::min(kMaxBlocks, num_sms() * 8));
  grid = (int)std::min<int64_t>(grid, (int64_t)(part_floats / (2 * C)));
  if (grid < 1) return fail(DFX_ERR_WORKSPACE, "dfx_layernorm_act_bwd: workspace too small");
  if (act)
    launch_k(ln_small_bwd_kernel<T, V, G, 1>, grid, 256, 0, st, rows, (const T*)dy, (const T*)x, gamma, beta, eps,
             (T*)dx, part);
  else
    launch_k(ln_small_bwd_kernel<T, V, G, 0>, grid, 256, 0, st, rows, (const T*)dy, (const T*)x, gamma, beta, eps,
             (T*)dx, part);
  DFX_LAUNCH_CHECK("dfx_layernorm_act_bwd (short rows)");
  launch_k(ln_small_finalize_kernel, (unsigned)((2 * C + 31) / 32), 1024, 0, st, grid, C, (const float*)part, dgamma,
           dbeta);
  DFX_LAUNCH_CHECK("dfx_layernorm_act_bwd (short rows) finalize");
  return DFX_OK;
}

#define LN_SMALL_DISPATCH(FN, T, V, ...)                          \
  switch (cols / (V)) {                                           \
    case 1: return FN<T, V, 1>(__VA_ARGS__);                      \
    case 2: return FN<T, V, 2>(__VA_ARGS__);                      \
    case 4: return FN<T, V, 4>(__VA_ARGS__);                      \
    case 8: return FN<T, V, 8>(__VA_ARGS__);                      \
    case 16: return FN<T, V, 16>(__VA_ARGS__);                    \
    case 32: return FN<T, V, 32>(__VA_ARGS__);                    \
    default: return DFX_ERR_UNSUPPORTED;                          \
  }

}  // namespace

bool ln_small_ok(int dtype, int64_t cols) {
  const int V = dtype == DFX_BF16 ? 8 : 4;
  if (cols % V) return false;
  const int64_t g = cols / V;
  return g == 1 || g == 2 || g == 4 || g == 8 || g == 16 || g == 32;
}

int ln_small_fwd(int dtype, int64_t rows, int64_t cols, const void* x, const float* gamma, const float* beta,
                 float eps, int act, void* y, cudaStream_t st) {
  if (rows <= 0) return DFX_OK;
  if (dtype == DFX_BF16) { LN_SMALL_DISPATCH(fwd_launch, __nv_bfloat16, 8, rows, x, gamma, beta, eps, act, y, st) }
  LN_SMALL_DISPATCH(fwd_launch, float, 4, rows, x, gamma, beta, eps, act, y, st)
}

int ln_small_bwd(int dtype, int64_t rows, int64_t cols, const void* dy, const void* x, const float* gamma,
                 const float* beta, float eps, int act, void* dx, float* dgamma, float* dbeta, void* workspace,
                 size_t ws_bytes, cudaStream_t st) {
  if (rows <= 0) return DFX_OK;
  float* part = (float*)workspace;
  const size_t pf = ws_bytes / sizeof(float);
  if (dtype == DFX_BF16) {
    LN_SMALL_DISPATCH(bwd_launch, __nv_bfloat16, 8, rows, dy, x, gamma, beta, eps, act, dx, dgamma, dbeta, part, pf, st)
  }
  LN_SMALL_DISPATCH(bwd_launch, float, 4, rows, dy, x, gamma, beta, eps, act, dx, dgamma, dbeta, part, pf, st)
}

}  // namespace dfx
