// norm.cu — BatchNorm (training) over the channel axis fused with an
// activation, channels-last [rows, C] (rows = N * spatial...), sm_100a.
// Config C4 of the north star ("LayerNorm vs BatchNorm on 4D/5D tensors,
// fused with elementwise"); the LayerNorm half lives in rowops.cu
// (dfx_layernorm_act_*).
//
// Reference: BatchNormalization training mode (frontend.py:544-591): batch
// statistics over every axis but 1, biased variance, running statistics
// run*m + batch*(1-m); VJP autodiff.py:1557-1617.  swish = Mul(u, Sigmoid(u))
// (frontend.py:229, 293).
//
//   stats    x -> per-block Welford (n, mean, M2) per channel, merged in fixed
//            order -> [3][C] (SyncBN all-gathers these; dfx_bn_finalize merges)
//   apply    y = act((x - mean) * rstd * gamma + beta)
//   bwd_reduce  (dy, x) -> [2][C] = (sum du, sum du*xhat), du = dy * act'(u)
//   bwd_dx   dx = gamma*rstd*(du - sum du/M - xhat*sum(du*xhat)/M)
#include "common.cuh"

namespace dfx {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 4 * 148;

struct Wf {
  float n, mean, m2;
};
__device__ __forceinline__ Wf wmerge(Wf a, Wf b) {
  const float n = a.n + b.n;
  if (n == 0.f) return a;
  const float d = b.mean - a.mean;
  const float f = b.n / n;
  return {n, a.mean + d * f, a.m2 + b.m2 + d * d * a.n * f};
}

template <typename T> struct NV { static constexpr int value = 8; };
template <> struct NV<float> { static constexpr int value = 4; };

// block b handles rows [b*rpb, min((b+1)*rpb, rows)); thread (cv, py)
template <typename T, int V>
__global__ void __launch_bounds__(kThreads) bn_stats_kernel(int64_t rows, int C, int64_t rpb, const T* __restrict__ x,
                                                           float* __restrict__ part /*[blocks][3][C]*/) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int CV = C / V, PY = blockDim.x / CV;
  const int cv = threadIdx.x % CV, py = threadIdx.x / CV;
  const int c0 = cv * V;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, rows);
  float cnt = 0.f, mean[V], m2[V];
#pragma unroll
  for (int i = 0; i < V; ++i) { mean[i] = 0.f; m2[i] = 0.f; }
  for (int64_t r = r0 + py; r < r1; r += PY) {
    Vec<T, V> v;
    v.load(x + r * C + c0);
    cnt += 1.f;
    const float inv = 1.f / cnt;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float d = v.v[i] - mean[i];
      mean[i] += d * inv;
      m2[i] += d * (v.v[i] - mean[i]);
    }
  }
  float* s_n = sm;
  float* s_mean = sm + PY;
  float* s_m2 = s_mean + PY * C;
  if (cv == 0) s_n[py] = cnt;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    s_mean[py * C + c0 + i] = mean[i];
    s_m2[py * C + c0 + i] = m2[i];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    Wf acc = {0.f, 0.f, 0.f};
    for (int j = 0; j < PY; ++j) acc = wmerge(acc, Wf{s_n[j], s_mean[j * C + c], s_m2[j * C + c]});
    part[((size_t)blockIdx.x * 3 + 0) * C + c] = acc.n;
    part[((size_t)blockIdx.x * 3 + 1) * C + c] = acc.mean;
    part[((size_t)blockIdx.x * 3 + 2) * C + c] = acc.m2;
  }
}

// one block per channel: merge block partials in a fixed tree order
__global__ void __launch_bounds__(kThreads) bn_merge_kernel(int nparts, int C, const float* __restrict__ part,
                                                           float* __restrict__ out /*[3][C]*/) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sn[kThreads], smn[kThreads], sm2[kThreads];
  const int c = blockIdx.x;
  Wf acc = {0.f, 0.f, 0.f};
  for (int b = threadIdx.x; b < nparts; b += blockDim.x)
    acc = wmerge(acc, Wf{part[((size_t)b * 3) * C + c], part[((size_t)b * 3 + 1) * C + c],
                         part[((size_t)b * 3 + 2) * C + c]});
  sn[threadIdx.x] = acc.n; smn[threadIdx.x] = acc.mean; sm2[threadIdx.x] = acc.m2;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      Wf m = wmerge(Wf{sn[threadIdx.x], smn[threadIdx.x], sm2[threadIdx.x]},
                    Wf{sn[threadIdx.x + s], smn[threadIdx.x + s], sm2[threadIdx.x + s]});
      sn[threadIdx.x] = m.n; smn[threadIdx.x] = m.mean; sm2[threadIdx.x] = m.m2;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[c] = sn[0]; out[C + c] = smn[0]; out[2 * C + c] = sm2[0]; }
}

template <typename T, int V, int ACT>
__global__ void __launch_bounds__(kThreads) bn_apply_kernel(int64_t nvec, int C, const T* __restrict__ x,
                                                           const float* __restrict__ mean, const float* __restrict__ rstd,
                                                           const float* __restrict__ gamma, const float* __restrict__ beta,
                                                           T* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  const int CV = C / V;
  for (int64_t vi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; vi < nvec; vi += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(vi % CV) * V;
    Vec<T, V> xv, yv;
    xv.load(x + vi * V);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = c0 + i;
      const float u = (xv.v[i] - mean[c]) * rstd[c] * gamma[c] + beta[c];
      yv.v[i] = ACT ? u * sigmoid_f(u) : u;
    }
    yv.store(y + vi * V);
  }
}

template <typename T, int V, int ACT>
__global__ void __launch_bounds__(kThreads) bn_bwd_reduce_kernel(int64_t rows, int C, int64_t rpb,
                                                                 const T* __restrict__ dy, const T* __restrict__ x,
                                                                 const float* __restrict__ mean,
                                                                 const float* __restrict__ rstd,
                                                                 const float* __restrict__ gamma,
                                                                 const float* __restrict__ beta,
                                                                 float* __restrict__ part /*[blocks][2][C]*/) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int CV = C / V, PY = blockDim.x / CV;
  const int cv = threadIdx.x % CV, py = threadIdx.x / CV;
  const int c0 = cv * V;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, rows);
  float mu[V], rs[V], gm[V], bt[V], s1[V], s2[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    mu[i] = mean[c0 + i]; rs[i] = rstd[c0 + i]; gm[i] = gamma[c0 + i]; bt[i] = beta[c0 + i];
    s1[i] = 0.f; s2[i] = 0.f;
  }
  for (int64_t r = r0 + py; r < r1; r += PY) {
    Vec<T, V> dv, xv;
    dv.load(dy + r * C + c0);
    xv.load(x + r * C + c0);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float xh = (xv.v[i] - mu[i]) * rs[i];
      float du = dv.v[i];
      if (ACT) {
        const float u = xh * gm[i] + bt[i];
        const float sg = sigmoid_f(u);
        du *= sg + u * sg * (1.f - sg);
      }
      s1[i] += du;
      s2[i] += du * xh;
    }
  }
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int i = 0; i < V; ++i) sm[py * C + c0 + i] = q == 0 ? s1[i] : s2[i];
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      float acc = 0.f;
      for (int j = 0; j < PY; ++j) acc += sm[j * C + c];
      part[((size_t)blockIdx.x * 2 + q) * C + c] = acc;
    }
    __syncthreads();
  }
}

__global__ void bn_sum_parts_kernel(int nparts, int C, const float* __restrict__ part, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 2 * C) return;
  float acc = 0.f;
  for (int b = 0; b < nparts; ++b) acc += part[(size_t)b * 2 * C + idx];
  out[idx] = acc;
}

template <typename T, int V, int ACT>
__global__ void __launch_bounds__(kThreads) bn_bwd_dx_kernel(int64_t nvec, int C, const T* __restrict__ dy,
                                                            const T* __restrict__ x, const float* __restrict__ mean,
                                                            const float* __restrict__ rstd,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ beta,
                                                            const float* __restrict__ sums, float inv_count,
                                                            T* __restrict__ dx) {
  pdl_trigger();
  pdl_wait();
  const int CV = C / V;
  for (int64_t vi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; vi < nvec; vi += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(vi % CV) * V;
    Vec<T, V> dv, xv, o;
    dv.load(dy + vi * V);
    xv.load(x + vi * V);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = c0 + i;
      const float xh = (xv.v[i] - mean[c]) * rstd[c];
      float du = dv.v[i];
      if (ACT) {
        const float u = xh * gamma[c] + beta[c];
        const float sg = sigmoid_f(u);
        du *= sg + u * sg * (1.f - sg);
      }
      o.v[i] = gamma[c] * rstd[c] * (du - sums[c] * inv_count - xh * sums[C + c] * inv_count);
    }
    o.store(dx + vi * V);
  }
}

// vector width: 128-bit when C allows it, scalar lanes otherwise
int vec_width(int dtype, int64_t C) {
  const int V = dtype == DFX_BF16 ? 8 : 4;
  return C % V == 0 ? V : 1;
}

int check_bn(int dtype, int64_t rows, int64_t C, const char* op) {
  DFX_REQUIRE(dtype == DFX_BF16 || dtype == DFX_F32, DFX_ERR_DTYPE, std::string(op) + ": dtype must be f32 or bf16");
  DFX_REQUIRE(rows > 0 && C > 0, DFX_ERR_SHAPE, std::string(op) + ": empty tensor");
  DFX_REQUIRE(C / vec_width(dtype, C) <= kThreads, DFX_ERR_SHAPE, std::string(op) + ": too many channels");
  return DFX_OK;
}

// DISPATCH(MACRO, ACT): expands MACRO(T, V, ACT) for the (dtype, width) at hand
#define BN_DISPATCH(M, ACTV)                                                    \
  do {                                                                          \
    const int vw__ = vec_width(dtype, C);                                       \
    if (dtype == DFX_BF16) {                                                    \
      if (vw__ == 8) { if (ACTV) M(__nv_bfloat16, 8, 1) else M(__nv_bfloat16, 8, 0) } \
      else { if (ACTV) M(__nv_bfloat16, 1, 1) else M(__nv_bfloat16, 1, 0) }    \
    } else {                                                                    \
      if (vw__ == 4) { if (ACTV) M(float, 4, 1) else M(float, 4, 0) }           \
      else { if (ACTV) M(float, 1, 1) else M(float, 1, 0) }                     \
    }                                                                           \
  } while (0)

void blocks_for(int64_t rows, int64_t* rpb, int* nb) {
  int64_t b = std::min<int64_t>(kMaxBlocks, (rows + 63) / 64);
  if (b < 1) b = 1;
  *rpb = (rows + b - 1) / b;
  *nb = (int)((rows + *rpb - 1) / *rpb);
}

}  // namespace
}  // namespace dfx

using namespace dfx;

extern "C" {

size_t dfx_batchnorm_workspace(int64_t rows, int64_t C) {
  (void)rows;
  return (size_t)kMaxBlocks * 3 * C * sizeof(float) + 256;
}

int dfx_batchnorm_stats(int dtype, int64_t rows, int64_t C, const void* x, float* local, void* workspace,
                        size_t ws_bytes, void* stream) {
  if (int rc = check_bn(dtype, rows, C, "dfx_batchnorm_stats")) return rc;
  DFX_REQUIRE(x && local && workspace, DFX_ERR_SHAPE, "dfx_batchnorm_stats: null pointer");
  DFX_REQUIRE(ws_bytes >= dfx_batchnorm_workspace(rows, C), DFX_ERR_WORKSPACE, "dfx_batchnorm_stats: workspace too small");
  cudaStream_t st = as_stream(stream);
  int64_t rpb;
  int nb;
  blocks_for(rows, &rpb, &nb);
  const int V = vec_width(dtype, C);
  const int CV = (int)C / V, PY = kThreads / CV;
  const size_t sm = (size_t)(PY + 2 * PY * C) * sizeof(float);
#define S(TT, VV, ACT)                                                                                    \
  {                                                                                                       \
    auto k = bn_stats_kernel<TT, VV>;                                                                     \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);   \
    launch_k(k, nb, CV * PY, sm, st, rows, (int)C, rpb, (const TT*)x, (float*)workspace);                       \
  }
  BN_DISPATCH(S, 0);
#undef S
  DFX_LAUNCH_CHECK("dfx_batchnorm_stats");
  launch_k(bn_merge_kernel, (unsigned)C, kThreads, 0, st, nb, (int)C, (const float*)workspace, local);
  DFX_LAUNCH_CHECK("dfx_batchnorm_stats merge");
  return DFX_OK;
}

int dfx_batchnorm_act_apply(int dtype, int64_t rows, int64_t C, const void* x, const float* mean, const float* rstd,
                            const float* gamma, const float* beta, int act, void* y, void* stream) {
  if (int rc = check_bn(dtype, rows, C, "dfx_batchnorm_act_apply")) return rc;
  DFX_REQUIRE(x && mean && rstd && gamma && beta && y, DFX_ERR_SHAPE, "dfx_batchnorm_act_apply: null pointer");
  DFX_REQUIRE(act == 0 || act == 1, DFX_ERR_UNSUPPORTED, "dfx_batchnorm_act_apply: act must be 0 or 1");
  cudaStream_t st = as_stream(stream);
  const int V = vec_width(dtype, C);
  const int64_t nvec = rows * C / V;
  const int grid = (int)std::min<int64_t>((nvec + 255) / 256, (int64_t)num_sms() * 16);
#define A(TT, VV, ACT) { launch_k(bn_apply_kernel<TT, VV, ACT>, grid, 256, 0, st, nvec, (int)C, (const TT*)x, mean, rstd, gamma, beta, (TT*)y); }
  BN_DISPATCH(A, act);
#undef A
  DFX_LAUNCH_CHECK("dfx_batchnorm_act_apply");
  return DFX_OK;
}

int dfx_batchnorm_act_bwd_reduce(int dtype, int64_t rows, int64_t C, const void* dy, const void* x,
                                 const float* mean, const float* rstd, const float* gamma, const float* beta,
                                 int act, float* bnsum, void* workspace, size_t ws_bytes, void* stream) {
  if (int rc = check_bn(dtype, rows, C, "dfx_batchnorm_act_bwd_reduce")) return rc;
  DFX_REQUIRE(dy && x && mean && rstd && gamma && beta && bnsum && workspace, DFX_ERR_SHAPE,
              "dfx_batchnorm_act_bwd_reduce: null pointer");
  DFX_REQUIRE(ws_bytes >= dfx_batchnorm_workspace(rows, C), DFX_ERR_WORKSPACE,
              "dfx_batchnorm_act_bwd_reduce: workspace too small");
  cudaStream_t st = as_stream(stream);
  int64_t rpb;
  int nb;
  blocks_for(rows, &rpb, &nb);
  const int V = vec_width(dtype, C);
  const int CV = (int)C / V, PY = kThreads / CV;
  const size_t sm = (size_t)PY * C * sizeof(float);
#define R(TT, VV, ACT)                                                                                      \
  {                                                                                                         \
    auto k = bn_bwd_reduce_kernel<TT, VV, ACT>;                                                             \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
    launch_k(k, nb, CV * PY, sm, st, rows, (int)C, rpb, (const TT*)dy, (const TT*)x, mean, rstd, gamma, beta,     \
                               (float*)workspace);                                                          \
  }
  BN_DISPATCH(R, act);
#undef R
  DFX_LAUNCH_CHECK("dfx_batchnorm_act_bwd_reduce");
  launch_k(bn_sum_parts_kernel, (unsigned)((2 * C + 255) / 256), 256, 0, st, nb, (int)C, (const float*)workspace, bnsum);
  DFX_LAUNCH_CHECK("dfx_batchnorm_act_bwd_reduce sum");
  return DFX_OK;
}

int dfx_batchnorm_act_bwd_dx(int dtype, int64_t rows, int64_t C, const void* dy, const void* x, const float* mean,
                             const float* rstd, const float* gamma, const float* beta, int act, const float* bnsum,
                             double count, void* dx, void* stream) {
  if (int rc = check_bn(dtype, rows, C, "dfx_batchnorm_act_bwd_dx")) return rc;
  DFX_REQUIRE(dy && x && mean && rstd && gamma && beta && bnsum && dx, DFX_ERR_SHAPE,
              "dfx_batchnorm_act_bwd_dx: null pointer");
  DFX_REQUIRE(count > 0, DFX_ERR_SHAPE, "dfx_batchnorm_act_bwd_dx: count must be positive");
  cudaStream_t st = as_stream(stream);
  const int V = vec_width(dtype, C);
  const int64_t nvec = rows * C / V;
  const int grid = (int)std::min<int64_t>((nvec + 255) / 256, (int64_t)num_sms() * 16);
  const float ic = (float)(1.0 / count);
#define D(TT, VV, ACT) \
  { launch_k(bn_bwd_dx_kernel<TT, VV, ACT>, grid, 256, 0, st, nvec, (int)C, (const TT*)dy, (const TT*)x, mean, rstd, gamma, beta, bnsum, ic, (TT*)dx); }
  BN_DISPATCH(D, act);
#undef D
  DFX_LAUNCH_CHECK("dfx_batchnorm_act_bwd_dx");
  return DFX_OK;
}

}  // extern "C"
