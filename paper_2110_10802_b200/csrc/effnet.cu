// effnet.cu — the EfficientNet-B0 training step's glue kernels (config C5),
// NHWC, sm_100a: stem im2col, global average pool, softmax cross-entropy,
// residual add.  The hot work of the step runs elsewhere (dwconv.cu /
// mbconv.cu for depthwise+BN+swish+SE, gemm_tc.cu for every 1x1 conv, the
// stem and the classifier, norm.cu for the GEMM-side BatchNorms).
//
// Reference semantics: Conv (frontend.py:598-678), GlobalAveragePool
// (frontend.py:681-706), Gemm (369-405), Softmax (488-501) — the loss is the
// mean over the batch of -log softmax(logits)[label]; Add (frontend.py:291).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace dfx {
namespace {

// stem: cols[m][k] for a 3x3 conv with Cin input channels, k = (ky*3+kx)*Cin + c,
// zero for padding taps and for k in [9*Cin, Kp) (Kp = GEMM K, a multiple of 8).
// One thread per output pixel: the 9*Cin taps are gathered into registers and
// the Kp-wide row leaves as 16-byte stores (one index decomposition per pixel).
template <typename T, int KP>
__global__ void __launch_bounds__(256) im2col3x3_kernel(int N, int H, int W, int Cin, int Ho, int Wo, int stride,
                                                        int pt, int pl, const T* __restrict__ x,
                                                        T* __restrict__ cols) {
  pdl_wait();
  pdl_trigger();
  constexpr int EPV = 16 / sizeof(T);
  const int64_t total = (int64_t)N * Ho * Wo;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < total; m += (int64_t)gridDim.x * blockDim.x) {
    const int ox = (int)(m % Wo);
    const int64_t t2 = m / Wo;
    const int oy = (int)(t2 % Ho);
    const int n = (int)(t2 / Ho);
    float v[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) v[k] = 0.f;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int iy = oy * stride + t / 3 - pt, ix = ox * stride + t % 3 - pl;
      if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
        const T* px = x + (((size_t)n * H + iy) * W + ix) * Cin;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[t * 3 + c] = to_f(px[c]);  // Cin == 3 (host-checked)
      }
    }
    T* out = cols + m * KP;
#pragma unroll
    for (int q = 0; q < KP / EPV; ++q) {
      Vec<T, EPV> o;
#pragma unroll
      for (int i = 0; i < EPV; ++i) o.v[i] = v[q * EPV + i];
      o.store(out + q * EPV);
    }
  }
}

// pooled[n][c] = mean over HW of x[n][p][c]; one block per (n, 256-channel slab)
template <typename T>
__global__ void __launch_bounds__(256) avgpool_fwd_kernel(int HW, int C, const T* __restrict__ x,
                                                          T* __restrict__ pooled) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.y;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int lane_p = threadIdx.x >> 5;  // 8 pixel lanes
  __shared__ float red[8][33];
  float acc = 0.f;
  if (c < C)
    for (int p = lane_p; p < HW; p += 8) acc += to_f(x[((size_t)n * HW + p) * C + c]);
  red[lane_p][threadIdx.x & 31] = acc;
  __syncthreads();
  if (lane_p == 0 && c < C) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += red[j][threadIdx.x & 31];
    pooled[(size_t)n * C + c] = from_f<T>(s / (float)HW);
  }
}

// dx[n][p][c] = dpooled[n][c] / HW (the GlobalAveragePool VJP)
template <typename T>
__global__ void __launch_bounds__(256) avgpool_bwd_kernel(int N, int HW, int C, const T* __restrict__ dpooled,
                                                          T* __restrict__ dx) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = (int64_t)N * HW * C;
  const float inv = 1.f / (float)HW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int n = (int)(i / ((int64_t)HW * C));
    dx[i] = from_f<T>(to_f(dpooled[(size_t)n * C + c]) * inv);
  }
}

// one block per sample: loss_rows[n] = -log softmax(z)[label], dz = (softmax - onehot) / N
template <typename TG>
__global__ void __launch_bounds__(256) xent_kernel(int N, int classes, const float* __restrict__ logits,
                                                   const int32_t* __restrict__ labels, float* __restrict__ loss_rows,
                                                   TG* __restrict__ dlogits) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x;
  const float* z = logits + (size_t)n * classes;
  __shared__ float sred[32];
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) mx = fmaxf(mx, z[j]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? sred[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) sred[0] = v;
  }
  __syncthreads();
  mx = sred[0];
  __syncthreads();
  float se = 0.f;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) se += __expf(z[j] - mx);
  se = warp_sum(se);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = se;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? sred[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) sred[0] = v;
  }
  __syncthreads();
  const float lse = mx + logf(sred[0]);
  const int lab = labels[n];
  const float inv_n = 1.f / (float)N;
  // a label outside [0, classes) (e.g. an ignore index) is not a class of
  // this head: its row gets zero gradient and a NaN loss, so the mean loss
  // reports the bad batch instead of reading z out of bounds
  const bool ok = lab >= 0 && lab < classes;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) {
    const float p = __expf(z[j] - lse);
    dlogits[(size_t)n * classes + j] = from_f<TG>(ok ? (p - (j == lab ? 1.f : 0.f)) * inv_n : 0.f);
  }
  if (threadIdx.x == 0) loss_rows[n] = ok ? lse - z[lab] : __int_as_float(0x7fc00000);
}

// loss = mean(loss_rows), fixed order
__global__ void mean_kernel(int N, const float* __restrict__ rows, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < N; ++i) s += rows[i];
    out[0] = s / (float)N;
  }
}

template <typename T, int V>
__global__ void __launch_bounds__(256) add_kernel(int64_t nvec, const T* __restrict__ a, const T* __restrict__ b,
                                                  T* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    Vec<T, V> va, vb;
    va.load(a + i * V);
    vb.load(b + i * V);
#pragma unroll
    for (int j = 0; j < V; ++j) va.v[j] += vb.v[j];
    va.store(out + i * V);
  }
}

int grid_for(int64_t work) { return (int)std::min<int64_t>((work + 255) / 256, (int64_t)num_sms() * 8); }

}  // namespace
}  // namespace dfx

using namespace dfx;

extern "C" {

int dfx_im2col3x3(int dtype, int64_t N, int64_t H, int64_t W, int64_t Cin, int stride, const int* pads, int64_t Kp,
                  const void* x, void* cols, void* stream) {
  DFX_REQUIRE(N > 0 && H > 0 && W > 0 && Cin > 0 && x && cols && pads, DFX_ERR_SHAPE, "dfx_im2col3x3: bad arguments");
  DFX_REQUIRE(stride == 1 || stride == 2, DFX_ERR_UNSUPPORTED, "dfx_im2col3x3: stride must be 1 or 2");
  DFX_REQUIRE(Kp >= 9 * Cin, DFX_ERR_SHAPE, "dfx_im2col3x3: Kp must be >= 9*Cin");
  const int64_t Ho = (H + pads[0] + pads[2] - 3) / stride + 1, Wo = (W + pads[1] + pads[3] - 3) / stride + 1;
  DFX_REQUIRE(Ho > 0 && Wo > 0, DFX_ERR_SHAPE, "dfx_im2col3x3: empty output");
  cudaStream_t st = as_stream(stream);
  DFX_REQUIRE(Kp == 32 && Cin == 3, DFX_ERR_UNSUPPORTED, "dfx_im2col3x3: the stem layout (Cin = 3, Kp = 32)");
  const int grid = grid_for(N * Ho * Wo);
  if (dtype == DFX_BF16)
    launch_k(im2col3x3_kernel<__nv_bfloat16, 32>, grid, 256, 0, st, (int)N, (int)H, (int)W, (int)Cin, (int)Ho,
             (int)Wo, stride, pads[0], pads[1], (const __nv_bfloat16*)x, (__nv_bfloat16*)cols);
  else if (dtype == DFX_F32)
    launch_k(im2col3x3_kernel<float, 32>, grid, 256, 0, st, (int)N, (int)H, (int)W, (int)Cin, (int)Ho, (int)Wo,
             stride, pads[0], pads[1], (const float*)x, (float*)cols);
  else
    return fail(DFX_ERR_DTYPE, "dfx_im2col3x3: dtype must be f32 or bf16");
  DFX_LAUNCH_CHECK("dfx_im2col3x3");
  return DFX_OK;
}

int dfx_avgpool_fwd(int dtype, int64_t N, int64_t HW, int64_t C, const void* x, void* pooled, void* stream) {
  DFX_REQUIRE(N > 0 && HW > 0 && C > 0 && x && pooled, DFX_ERR_SHAPE, "dfx_avgpool_fwd: bad arguments");
  cudaStream_t st = as_stream(stream);
  const dim3 grid((unsigned)((C + 31) / 32), (unsigned)N);
  if (dtype == DFX_BF16)
    launch_k(avgpool_fwd_kernel<__nv_bfloat16>, grid, 256, 0, st, (int)HW, (int)C, (const __nv_bfloat16*)x,
             (__nv_bfloat16*)pooled);
  else if (dtype == DFX_F32)
    launch_k(avgpool_fwd_kernel<float>, grid, 256, 0, st, (int)HW, (int)C, (const float*)x, (float*)pooled);
  else
    return fail(DFX_ERR_DTYPE, "dfx_avgpool_fwd: dtype must be f32 or bf16");
  DFX_LAUNCH_CHECK("dfx_avgpool_fwd");
  return DFX_OK;
}

int dfx_avgpool_bwd(int dtype, int64_t N, int64_t HW, int64_t C, const void* dpooled, void* dx, void* stream) {
  DFX_REQUIRE(N > 0 && HW > 0 && C > 0 && dpooled && dx, DFX_ERR_SHAPE, "dfx_avgpool_bwd: bad arguments");
  cudaStream_t st = as_stream(stream);
  const int grid = grid_for(N * HW * C);
  if (dtype == DFX_BF16)
    launch_k(avgpool_bwd_kernel<__nv_bfloat16>, grid, 256, 0, st, (int)N, (int)HW, (int)C,
             (const __nv_bfloat16*)dpooled, (__nv_bfloat16*)dx);
  else if (dtype == DFX_F32)
    launch_k(avgpool_bwd_kernel<float>, grid, 256, 0, st, (int)N, (int)HW, (int)C, (const float*)dpooled, (float*)dx);
  else
    return fail(DFX_ERR_DTYPE, "dfx_avgpool_bwd: dtype must be f32 or bf16");
  DFX_LAUNCH_CHECK("dfx_avgpool_bwd");
  return DFX_OK;
}

int dfx_softmax_xent(int64_t N, int64_t classes, const float* logits, const int32_t* labels, float* loss,
                     float* loss_rows, int grad_dtype, void* dlogits, void* stream) {
  DFX_REQUIRE(N > 0 && classes > 0 && logits && labels && loss && loss_rows && dlogits, DFX_ERR_SHAPE,
              "dfx_softmax_xent: bad arguments");
  cudaStream_t st = as_stream(stream);
  if (grad_dtype == DFX_BF16)
    launch_k(xent_kernel<__nv_bfloat16>, (unsigned)N, 256, 0, st, (int)N, (int)classes, logits, labels, loss_rows,
             (__nv_bfloat16*)dlogits);
  else if (grad_dtype == DFX_F32)
    launch_k(xent_kernel<float>, (unsigned)N, 256, 0, st, (int)N, (int)classes, logits, labels, loss_rows,
             (float*)dlogits);
  else
    return fail(DFX_ERR_DTYPE, "dfx_softmax_xent: grad dtype must be f32 or bf16");
  DFX_LAUNCH_CHECK("dfx_softmax_xent");
  launch_k(mean_kernel, 1, 32, 0, st, (int)N, (const float*)loss_rows, loss);
  DFX_LAUNCH_CHECK("dfx_softmax_xent mean");
  return DFX_OK;
}

int dfx_add(int dtype, int64_t n, const void* a, const void* b, void* out, void* stream) {
  DFX_REQUIRE(n >= 0 && a && b && out, DFX_ERR_SHAPE, "dfx_add: bad arguments");
  cudaStream_t st = as_stream(stream);
  if (dtype == DFX_BF16) {
    DFX_REQUIRE(n % 8 == 0 && aligned16(a) && aligned16(b) && aligned16(out), DFX_ERR_SHAPE,
                "dfx_add: bf16 needs n % 8 == 0 and 16-byte aligned buffers");
    launch_k(add_kernel<__nv_bfloat16, 8>, grid_for(n / 8), 256, 0, st, n / 8, (const __nv_bfloat16*)a,
             (const __nv_bfloat16*)b, (__nv_bfloat16*)out);
  } else if (dtype == DFX_F32) {
    DFX_REQUIRE(n % 4 == 0 && aligned16(a) && aligned16(b) && aligned16(out), DFX_ERR_SHAPE,
                "dfx_add: f32 needs n % 4 == 0 and 16-byte aligned buffers");
    launch_k(add_kernel<float, 4>, grid_for(n / 4), 256, 0, st, n / 4, (const float*)a, (const float*)b,
             (float*)out);
  } else {
    return fail(DFX_ERR_DTYPE, "dfx_add: dtype must be f32 or bf16");
  }
  DFX_LAUNCH_CHECK("dfx_add");
  return DFX_OK;
}

}  // extern "C"
