// mbconv.cu — EfficientNet-B0 MBConv hot path, NHWC, sm_100a.
//
// Forward  (depthwise 3x3 -> BatchNorm(train) -> swish -> squeeze-excite):
//   K1 dwconv_fwd      x -> z (stored), per-tile Welford (mean, M2) per channel
//   K2 bn_reduce       tiles -> (n, mean, M2) per channel   [SyncBN: allgather]
//   K3 bn_finalize     ranks -> mean, rstd, running stats   (frontend.py:558-591)
//   K4 bn_swish_pool   z -> per-(n, tile) channel sums of a = swish(BN(z))
//   K5 se_fwd          pooled -> r = Wr p + br, e = We swish(r) + be, s = sigmoid(e)
//   K6 excite          z -> y = swish(BN(z)) * s[n, c]
// a = swish(BN(z)) is never stored: K4 and K6 recompute it from z (the
// paper's recompute-instead-of-stash) — 5 full-tensor
// passes instead of the 6 of a stash-everything schedule.
//
// Backward:
//   B1 bwd_reduce      (dy, z) -> per (n, c): A1=sum dy*a, A2=sum dy*sw', A3=sum sw',
//                      A4=sum dy*sw'*xhat, A5=sum sw'*xhat   (sw' = d swish/du)
//   B2 se_bwd          SE-MLP VJP per sample -> dpool[n,c], and per-sample
//                      BN-VJP sums  sum du = s*A2 + dpool/HW*A3,
//                                   sum du*xhat = s*A4 + dpool/HW*A5
//   B3 se_bwd_reduce   fixed-order sums over samples -> dWe, dbe, dWr, dbr,
//                      dgamma, dbeta, and the BN sums (SyncBN: allreduce them)
//   B4 dwconv_bwd      dz = gamma*rstd*(du - mean(du) - xhat*mean(du*xhat))
//                      (autodiff.py:1557-1617) computed into shared memory for
//                      an output tile + halo, then dx (transposed depthwise
//                      conv, the VJP of the lowered loop nest lowering.py:930-1004)
//                      and per-block dw partials; B5 finalizes dw.
// Only two full-tensor backward passes read (dy, z) + (dy, z, x) and one
// writes dx.  All reductions are fixed-order (Welford/Chan merges, no float
// atomics): results are bitwise reproducible.
#include <algorithm>

#include "common.cuh"
#include "dwconv.h"

namespace dfx {
namespace {

constexpr int kThreads = 256;

template <typename T> struct MbVec { static constexpr int value = 8; };
template <> struct MbVec<float> { static constexpr int value = 4; };

struct Geo {
  int N, H, W, C;        // input
  int Ho, Wo;            // output
  int stride, pt, pl;    // stride, top/left pad
  int ks;                // taps per side (3 or 5)
  int tile_rows;         // output rows per tile
  int tiles_per_img;
};

__device__ __forceinline__ float sigmoidf_(float u) { return 1.f / (1.f + __expf(-u)); }
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// sigmoid for the bf16 path: one MUFU op (tanh.approx, rel. error ~2^-11,
// far below bf16 rounding); the f32 path keeps the exact form for 1e-4 parity.
template <typename T> __device__ __forceinline__ float sigm(float u) {
  if constexpr (sizeof(T) == 2) return fmaf(0.5f, tanh_approx(0.5f * u), 0.5f);
  else return sigmoidf_(u);
}

__host__ __device__ __forceinline__ int floordiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

struct Welford {
  float n, mean, m2;
};
__device__ __forceinline__ Welford merge(Welford a, Welford b) {
  const float n = a.n + b.n;
  if (n == 0.f) return a;
  const float d = b.mean - a.mean;
  const float f = b.n / n;
  return {n, a.mean + d * f, a.m2 + b.m2 + d * d * a.n * f};
}

// ---------------------------------------------------------------- K1
// tile = (image n, output rows [r0, r0+tile_rows)), all columns, all channels.
// thread (cv, py): channel vector cv, pixel lane py.
template <typename T, int V>
__global__ void __launch_bounds__(kThreads) dwconv_fwd_kernel(Geo g, const T* __restrict__ x,
                                                              const float* __restrict__ w,
                                                              T* __restrict__ z,
                                                              float* __restrict__ part /*[tiles][2][C]*/) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int CV = g.C / V;
  const int PY = blockDim.x / CV;
  const int cv = threadIdx.x % CV, py = threadIdx.x / CV;
  const int tile = blockIdx.x;
  const int n = tile / g.tiles_per_img;
  const int r0 = (tile % g.tiles_per_img) * g.tile_rows;
  const int r1 = min(r0 + g.tile_rows, g.Ho);
  const int npix = (r1 - r0) * g.Wo;
  const int c0 = cv * V;
  float wr[9][V];
  if (py < PY) {
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      Vec<float, V> wv;
      wv.load(w + t * g.C + c0);
#pragma unroll
      for (int i = 0; i < V; ++i) wr[t][i] = wv.v[i];
    }
  }
  float cnt = 0.f, mean[V], m2[V];
#pragma unroll
  for (int i = 0; i < V; ++i) { mean[i] = 0.f; m2[i] = 0.f; }
  if (py < PY) {
    for (int p = py; p < npix; p += PY) {
      const int oy = r0 + p / g.Wo, ox = p % g.Wo;
      float acc[V];
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = 0.f;
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        const int iy = oy * g.stride + ky - g.pt;
        if (iy < 0 || iy >= g.H) continue;
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const int ix = ox * g.stride + kx - g.pl;
          if (ix < 0 || ix >= g.W) continue;
          Vec<T, V> xv;
          xv.load(x + (((size_t)n * g.H + iy) * g.W + ix) * g.C + c0);
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = fmaf(xv.v[i], wr[ky * 3 + kx][i], acc[i]);
        }
      }
      Vec<T, V> zv;
#pragma unroll
      for (int i = 0; i < V; ++i) zv.v[i] = acc[i];
      zv.store(z + (((size_t)n * g.Ho + oy) * g.Wo + ox) * g.C + c0);
      cnt += 1.f;
      const float inv = 1.f / cnt;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float d = acc[i] - mean[i];
        mean[i] += d * inv;
        m2[i] += d * (acc[i] - mean[i]);
      }
    }
  }
  // fixed-order merge over pixel lanes: sm layout [PY][3][C]
  float* s_n = sm;                 // [PY]
  float* s_mean = sm + PY;         // [PY][C]
  float* s_m2 = s_mean + PY * g.C; // [PY][C]
  if (py < PY) {
    if (cv == 0) s_n[py] = cnt;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      s_mean[py * g.C + c0 + i] = mean[i];
      s_m2[py * g.C + c0 + i] = m2[i];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
    Welford acc = {0.f, 0.f, 0.f};
    for (int j = 0; j < PY; ++j) acc = merge(acc, Welford{s_n[j], s_mean[j * g.C + c], s_m2[j * g.C + c]});
    part[((size_t)tile * 2 + 0) * g.C + c] = acc.mean;
    part[((size_t)tile * 2 + 1) * g.C + c] = acc.m2;
  }
}

// ---------------------------------------------------------------- K2
// one block per channel: merge tiles (count per tile from geometry) -> out[3][C]
__global__ void __launch_bounds__(kThreads) bn_reduce_kernel(Geo g, int ntiles, const float* __restrict__ part,
                                                             float* __restrict__ out /*[3][C]: n, mean, M2*/) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sn[kThreads], smn[kThreads], sm2[kThreads];
  const int c = blockIdx.x;
  Welford acc = {0.f, 0.f, 0.f};
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    const int r0 = (t % g.tiles_per_img) * g.tile_rows;
    const float cnt = (float)((min(r0 + g.tile_rows, g.Ho) - r0) * g.Wo);
    acc = merge(acc, Welford{cnt, part[((size_t)t * 2) * g.C + c], part[((size_t)t * 2 + 1) * g.C + c]});
  }
  sn[threadIdx.x] = acc.n; smn[threadIdx.x] = acc.mean; sm2[threadIdx.x] = acc.m2;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      Welford m = merge(Welford{sn[threadIdx.x], smn[threadIdx.x], sm2[threadIdx.x]},
                        Welford{sn[threadIdx.x + s], smn[threadIdx.x + s], sm2[threadIdx.x + s]});
      sn[threadIdx.x] = m.n; smn[threadIdx.x] = m.mean; sm2[threadIdx.x] = m.m2;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[c] = sn[0];
    out[g.C + c] = smn[0];
    out[2 * g.C + c] = sm2[0];
  }
}

// ---------------------------------------------------------------- K3
__global__ void bn_finalize_kernel(int C, int nsets, const float* __restrict__ sets /*[nsets][3][C]*/, float eps,
                                   float momentum, float* __restrict__ mean, float* __restrict__ var,
                                   float* __restrict__ rstd, float* run_mean, float* run_var) {
  pdl_trigger();
  pdl_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  Welford acc = {0.f, 0.f, 0.f};
  for (int r = 0; r < nsets; ++r)
    acc = merge(acc, Welford{sets[(size_t)r * 3 * C + c], sets[(size_t)r * 3 * C + C + c],
                             sets[(size_t)r * 3 * C + 2 * C + c]});
  const float v = acc.m2 / acc.n;  // biased variance (frontend.py:565)
  if (mean) mean[c] = acc.mean;
  if (var) var[c] = v;
  rstd[c] = rsqrtf(v + eps);
  if (run_mean) run_mean[c] = run_mean[c] * momentum + acc.mean * (1.f - momentum);
  if (run_var) run_var[c] = run_var[c] * momentum + v * (1.f - momentum);
}

struct BnParams {
  const float* mean;
  const float* rstd;
  const float* gamma;
  const float* beta;
};

// ---------------------------------------------------------------- K4
template <typename T, int V>
__global__ void __launch_bounds__(kThreads) bn_swish_pool_kernel(Geo g, const T* __restrict__ z, BnParams bn,
                                                                 float* __restrict__ part /*[tiles][C]*/) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  // channel chunks across gridDim.y (wide C at small H x W: enough CTAs/lanes)
  const int CVt = g.C / V, CVc = (CVt + gridDim.y - 1) / gridDim.y, PY = blockDim.x / CVc;
  const int lcv = threadIdx.x % CVc, py = threadIdx.x / CVc;
  const int cv = blockIdx.y * CVc + lcv;
  const bool on = cv < CVt;
  const int cbeg = blockIdx.y * CVc * V, cend = min(cbeg + CVc * V, g.C);
  const int tile = blockIdx.x;
  const int n = tile / g.tiles_per_img;
  const int r0 = (tile % g.tiles_per_img) * g.tile_rows;
  const int r1 = min(r0 + g.tile_rows, g.Ho);
  const int c0 = (on ? cv : 0) * V;
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;
  if (py < PY && on) {
    float sc[V], sh[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      sc[i] = bn.rstd[c0 + i] * bn.gamma[c0 + i];
      sh[i] = bn.beta[c0 + i] - bn.mean[c0 + i] * sc[i];
    }
    const T* base = z + ((size_t)n * g.Ho + r0) * g.Wo * g.C + c0;
    const int npix = (r1 - r0) * g.Wo;
    int p = py;
    for (; p + 3 * PY < npix; p += 4 * PY) {  // 4 loads in flight per thread
      Vec<T, V> zv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) zv[q].load(base + (size_t)(p + q * PY) * g.C);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float u = fmaf(zv[q].v[i], sc[i], sh[i]);
          acc[i] = fmaf(u, sigm<T>(u), acc[i]);
        }
    }
    for (; p < npix; p += PY) {
      Vec<T, V> zv;
      zv.load(base + (size_t)p * g.C);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float u = fmaf(zv.v[i], sc[i], sh[i]);
        acc[i] = fmaf(u, sigm<T>(u), acc[i]);
      }
    }
    for (int i = 0; i < V; ++i) sm[py * g.C + c0 + i] = acc[i];
  }
  __syncthreads();
  for (int c = cbeg + threadIdx.x; c < cend; c += blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < PY; ++j) s += sm[j * g.C + c];
    part[(size_t)tile * g.C + c] = s;
  }
}

// ---------------------------------------------------------------- K5
// one block per sample.  Wr [SE][C], We [C][SE] (Gemm transB=1 layout).
__global__ void __launch_bounds__(1024) se_fwd_kernel(Geo g, int SE, const float* __restrict__ part,
                                                          const float* __restrict__ wr, const float* __restrict__ br,
                                                          const float* __restrict__ we, const float* __restrict__ be,
                                                          float* __restrict__ pooled, float* __restrict__ r_out,
                                                          float* __restrict__ s_out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  float* p = sm;       // [C]
  float* r2 = sm + g.C; // [SE]
  const int n = blockIdx.x;
  const float inv_hw = 1.f / (float)(g.Ho * g.Wo);
  for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
    float s = 0.f;
#pragma unroll 4
    for (int t = 0; t < g.tiles_per_img; ++t) s += part[((size_t)n * g.tiles_per_img + t) * g.C + c];
    p[c] = s * inv_hw;
    pooled[(size_t)n * g.C + c] = s * inv_hw;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = warp; j < SE; j += nw) {
    float acc = 0.f;
#pragma unroll 8
    for (int c = lane; c < g.C; c += 32) acc += wr[(size_t)j * g.C + c] * p[c];
    acc = warp_sum(acc) + br[j];
    if (lane == 0) {
      r_out[(size_t)n * SE + j] = acc;
      r2[j] = acc * sigmoidf_(acc);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
    float e = be[c];
#pragma unroll 8
    for (int j = 0; j < SE; ++j) e += we[(size_t)c * SE + j] * r2[j];
    s_out[(size_t)n * g.C + c] = sigmoidf_(e);
  }
}

// ---------------------------------------------------------------- K6
// tile = (image n, rows), thread (channel vector cv, pixel lane py): the
// per-channel BN/SE constants are loaded once per thread, not per element.
template <typename T, int V>
__global__ void __launch_bounds__(kThreads) excite_kernel(Geo g, const T* __restrict__ z, BnParams bn,
                                                          const float* __restrict__ s, T* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  // channel chunks across gridDim.y (wide C at small H x W: enough CTAs/lanes)
  const int CVt = g.C / V, CVc = (CVt + gridDim.y - 1) / gridDim.y, PY = blockDim.x / CVc;
  const int lcv = threadIdx.x % CVc, py = threadIdx.x / CVc;
  const int cv = blockIdx.y * CVc + lcv;
  const bool on = cv < CVt;
  const int cbeg = blockIdx.y * CVc * V, cend = min(cbeg + CVc * V, g.C);
  if (py >= PY || !on) return;
  const int tile = blockIdx.x;
  const int n = tile / g.tiles_per_img;
  const int r0 = (tile % g.tiles_per_img) * g.tile_rows;
  const int r1 = min(r0 + g.tile_rows, g.Ho);
  const int c0 = (on ? cv : 0) * V;
  float sc[V], sh[V], se[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    sc[i] = bn.rstd[c0 + i] * bn.gamma[c0 + i];
    sh[i] = bn.beta[c0 + i] - bn.mean[c0 + i] * sc[i];
    se[i] = s[(size_t)n * g.C + c0 + i];
  }
  const size_t base = ((size_t)n * g.Ho + r0) * g.Wo * g.C + c0;
  const int npix = (r1 - r0) * g.Wo;
  int p = py;
  for (; p + PY < npix; p += 2 * PY) {  // two pixels in flight per thread
    Vec<T, V> z0, z1;
    z0.load(z + base + (size_t)p * g.C);
    z1.load(z + base + (size_t)(p + PY) * g.C);
    Vec<T, V> y0, y1;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float u0 = fmaf(z0.v[i], sc[i], sh[i]), u1 = fmaf(z1.v[i], sc[i], sh[i]);
      y0.v[i] = u0 * sigm<T>(u0) * se[i];
      y1.v[i] = u1 * sigm<T>(u1) * se[i];
    }
    y0.store(y + base + (size_t)p * g.C);
    y1.store(y + base + (size_t)(p + PY) * g.C);
  }
  if (p < npix) {
    Vec<T, V> z0, y0;
    z0.load(z + base + (size_t)p * g.C);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float u0 = fmaf(z0.v[i], sc[i], sh[i]);
      y0.v[i] = u0 * sigm<T>(u0) * se[i];
    }
    y0.store(y + base + (size_t)p * g.C);
  }
}

// ---------------------------------------------------------------- B1
template <typename T, int V>
__global__ void __launch_bounds__(kThreads) bwd_reduce_kernel(Geo g, const T* __restrict__ dy, const T* __restrict__ z,
                                                              BnParams bn, float* __restrict__ part /*[tiles][5][C]*/) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  // channel chunks across gridDim.y (wide C at small H x W: enough CTAs/lanes)
  const int CVt = g.C / V, CVc = (CVt + gridDim.y - 1) / gridDim.y, PY = blockDim.x / CVc;
  const int lcv = threadIdx.x % CVc, py = threadIdx.x / CVc;
  const int cv = blockIdx.y * CVc + lcv;
  const bool on = cv < CVt;
  const int cbeg = blockIdx.y * CVc * V, cend = min(cbeg + CVc * V, g.C);
  const int tile = blockIdx.x;
  const int n = tile / g.tiles_per_img;
  const int r0 = (tile % g.tiles_per_img) * g.tile_rows;
  const int r1 = min(r0 + g.tile_rows, g.Ho);
  const int c0 = (on ? cv : 0) * V;
  float a[5][V];
#pragma unroll
  for (int k = 0; k < 5; ++k)
#pragma unroll
    for (int i = 0; i < V; ++i) a[k][i] = 0.f;
  if (py < PY && on) {
    float mu[V], rs[V], gm[V], bt[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      mu[i] = bn.mean[c0 + i]; rs[i] = bn.rstd[c0 + i]; gm[i] = bn.gamma[c0 + i]; bt[i] = bn.beta[c0 + i];
    }
    float P[V], Q[V], R[V], M[V];  // u = z*P + Q, xhat = z*R + M
#pragma unroll
    for (int i = 0; i < V; ++i) {
      P[i] = gm[i] * rs[i];
      Q[i] = bt[i] - mu[i] * P[i];
      R[i] = rs[i];
      M[i] = -mu[i] * rs[i];
    }
    const size_t base = ((size_t)n * g.Ho + r0) * g.Wo * g.C + c0;
    const int npix = (r1 - r0) * g.Wo;
    auto body = [&](const Vec<T, V>& dv, const Vec<T, V>& zv) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float zz = zv.v[i];
        const float xh = fmaf(zz, R[i], M[i]);
        const float u = fmaf(zz, P[i], Q[i]);
        const float sg = sigm<T>(u);
        const float swp = sg * fmaf(u, 1.f - sg, 1.f);
        const float d = dv.v[i];
        const float dswp = d * swp;
        a[0][i] = fmaf(d * u, sg, a[0][i]);
        a[1][i] += dswp;
        a[2][i] += swp;
        a[3][i] = fmaf(dswp, xh, a[3][i]);
        a[4][i] = fmaf(swp, xh, a[4][i]);
      }
    };
    // four pixels per iteration: 8 independent 128-bit loads in flight per thread
    int p = py;
    for (; p + 3 * PY < npix; p += 4 * PY) {
      Vec<T, V> dv[4], zv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        dv[q].load(dy + base + (size_t)(p + q * PY) * g.C);
        zv[q].load(z + base + (size_t)(p + q * PY) * g.C);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) body(dv[q], zv[q]);
    }
    for (; p < npix; p += PY) {
      Vec<T, V> dv, zv;
      dv.load(dy + base + (size_t)p * g.C);
      zv.load(z + base + (size_t)p * g.C);
      body(dv, zv);
    }
  }
  for (int k = 0; k < 5; ++k) {
    if (py < PY && on) {
#pragma unroll
      for (int i = 0; i < V; ++i) sm[py * g.C + c0 + i] = a[k][i];
    }
    __syncthreads();
    for (int c = cbeg + threadIdx.x; c < cend; c += blockDim.x) {
      float s = 0.f;
      for (int j = 0; j < PY; ++j) s += sm[j * g.C + c];
      part[((size_t)tile * 5 + k) * g.C + c] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- B2
// one block per sample: SE VJP + per-sample BN-VJP sums.
__global__ void __launch_bounds__(1024) se_bwd_kernel(Geo g, int SE, const float* __restrict__ part,
                                                          const float* __restrict__ s, const float* __restrict__ r,
                                                          const float* __restrict__ wr, const float* __restrict__ we,
                                                          float* __restrict__ de_out /*[N][C]*/,
                                                          float* __restrict__ dr_out /*[N][SE]*/,
                                                          float* __restrict__ dpool /*[N][C]*/,
                                                          float* __restrict__ nsum /*[N][2][C]*/) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  float* A = sm;               // [5][C]
  float* de = A + 5 * g.C;     // [C]
  float* dr = de + g.C;        // [SE]
  const int n = blockIdx.x;
  for (int idx = threadIdx.x; idx < 5 * g.C; idx += blockDim.x) {
    const int k = idx / g.C, c = idx % g.C;
    float acc = 0.f;
#pragma unroll 4
    for (int t = 0; t < g.tiles_per_img; ++t) acc += part[(((size_t)n * g.tiles_per_img + t) * 5 + k) * g.C + c];
    A[idx] = acc;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
    const float sv = s[(size_t)n * g.C + c];
    const float d = A[c] * sv * (1.f - sv);  // d loss / d e  (ds = A1, sigmoid')
    de[c] = d;
    de_out[(size_t)n * g.C + c] = d;
  }
  __syncthreads();
  // dr[j] = Σ_c We[c][j] de[c]: thread (j, part) walks c = part, part + P, ...
  // so consecutive threads read consecutive We entries (We is [C][SE]); the P
  // partial sums of each j are then added in part order (deterministic)
  const int P = (int)blockDim.x / SE;  // SE <= blockDim.x (host check)
  float* red = dr + SE;                 // [P][SE] <= 1024 floats after dr
  __syncthreads();
  if ((int)threadIdx.x < P * SE) {
    const int j = (int)threadIdx.x % SE, part = (int)threadIdx.x / SE;
    float acc = 0.f;
#pragma unroll 4
    for (int c = part; c < g.C; c += P) acc = fmaf(we[(size_t)c * SE + j], de[c], acc);
    red[part * SE + j] = acc;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < SE; j += blockDim.x) {
    float acc = 0.f;
    for (int q = 0; q < P; ++q) acc += red[q * SE + j];
    const float rv = r[(size_t)n * SE + j];
    const float sg = sigmoidf_(rv);
    const float v = acc * (sg + rv * sg * (1.f - sg));
    dr[j] = v;
    dr_out[(size_t)n * SE + j] = v;
  }
  __syncthreads();
  const float inv_hw = 1.f / (float)(g.Ho * g.Wo);
  for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
    float dp = 0.f;
#pragma unroll 8
    for (int j = 0; j < SE; ++j) dp += wr[(size_t)j * g.C + c] * dr[j];
    dp *= inv_hw;  // d loss / d a contribution per pixel
    dpool[(size_t)n * g.C + c] = dp;
    const float sv = s[(size_t)n * g.C + c];
    nsum[((size_t)n * 2 + 0) * g.C + c] = sv * A[1 * g.C + c] + dp * A[2 * g.C + c];
    nsum[((size_t)n * 2 + 1) * g.C + c] = sv * A[3 * g.C + c] + dp * A[4 * g.C + c];
  }
}

// ---------------------------------------------------------------- B3
// Sample reductions of the SE-MLP and BN parameter gradients.  A block owns 32
// consecutive outputs (lanes; channel-fastest flat index, so loads of one
// sample row are coalesced and the per-(n, j) factor is a broadcast) and its 8
// warps take samples n = w, w + 8, ...; the 8 partials of each output are then
// added in warp order (deterministic).  Outputs: dWe [C][SE] (written through
// the transposed index), dWr [SE][C], dbe [C], dbr [SE], bnsum [2][C].
__global__ void __launch_bounds__(256) se_bwd_reduce_kernel(int N, int C, int SE, const float* __restrict__ de,
                                                            const float* __restrict__ dr, const float* __restrict__ r,
                                                            const float* __restrict__ pooled,
                                                            const float* __restrict__ nsum, float* __restrict__ dwe /*[C][SE]*/,
                                                            float* __restrict__ dbe, float* __restrict__ dwr /*[SE][C]*/,
                                                            float* __restrict__ dbr, float* __restrict__ bnsum /*[2][C]*/) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t total = (int64_t)C * SE * 2 + C + SE + 2 * C;
  const int64_t n_w = (int64_t)C * SE;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < total; base += (int64_t)gridDim.x * 32) {
    int64_t k = base + lane;
    float acc = 0.f;
    if (k < total) {
      if (k < n_w) {  // dWe[c][j] = Σ_n de[n][c] swish(r[n][j]),  k = j * C + c
        const int j = (int)(k / C), c = (int)(k % C);
        for (int n = w; n < N; n += 8) {
          const float rv = __ldg(r + (size_t)n * SE + j);
          acc = fmaf(__ldg(de + (size_t)n * C + c), rv * sigmoidf_(rv), acc);
        }
      } else if ((k -= n_w) < n_w) {  // dWr[j][c] = Σ_n dr[n][j] pooled[n][c],  k = j * C + c
        const int j = (int)(k / C), c = (int)(k % C);
        for (int n = w; n < N; n += 8) acc = fmaf(__ldg(dr + (size_t)n * SE + j), __ldg(pooled + (size_t)n * C + c), acc);
      } else if ((k -= n_w) < C) {
        for (int n = w; n < N; n += 8) acc += __ldg(de + (size_t)n * C + k);
      } else if ((k -= C) < SE) {
        for (int n = w; n < N; n += 8) acc += __ldg(dr + (size_t)n * SE + k);
      } else {
        k -= SE;
        const int q = (int)(k / C), c = (int)(k % C);
        for (int n = w; n < N; n += 8) acc += __ldg(nsum + ((size_t)n * 2 + q) * C + c);
      }
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0 && base + lane < total) {
      float t = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) t += red[q][lane];
      int64_t kk = base + lane;
      if (kk < n_w) {
        dwe[(size_t)(kk % C) * SE + kk / C] = t;
      } else if ((kk -= n_w) < n_w) {
        dwr[kk] = t;
      } else if ((kk -= n_w) < C) {
        dbe[kk] = t;
      } else if ((kk -= C) < SE) {
        dbr[kk] = t;
      } else {
        bnsum[kk - SE] = t;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- B4
// Block = output tile TO x TO of one image (+1 halo), all channels.  Persistent
// over tiles; dw partials accumulate in registers.
constexpr int TO = 8;
constexpr int TH = TO + 2;

template <typename T, int V>
__global__ void __launch_bounds__(kThreads) dwconv_bwd_kernel(Geo g, const T* __restrict__ dy, const T* __restrict__ z,
                                                              const T* __restrict__ x, const float* __restrict__ w,
                                                              BnParams bn, const float* __restrict__ s,
                                                              const float* __restrict__ dpool,
                                                              const float* __restrict__ bnsum /*[2][C]*/,
                                                              float inv_count, T* __restrict__ dx,
                                                              float* __restrict__ dw_part /*[grid][9][C]*/) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float dzs[];  // [TH*TH][C]
  const int CV = g.C / V;
  const int PY = blockDim.x / CV;
  const int cv = threadIdx.x % CV, py = threadIdx.x / CV;
  const int c0 = cv * V;
  const int ty_n = (g.Ho + TO - 1) / TO, tx_n = (g.Wo + TO - 1) / TO;
  const int ntiles = g.N * ty_n * tx_n;
  float wr[9][V], dwa[9][V];
  float mu[V], rs[V], gm[V], bt[V], mdu[V], mdux[V];
  if (py < PY) {
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      Vec<float, V> wv;
      wv.load(w + t * g.C + c0);
#pragma unroll
      for (int i = 0; i < V; ++i) { wr[t][i] = wv.v[i]; dwa[t][i] = 0.f; }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = c0 + i;
      mu[i] = bn.mean[c]; rs[i] = bn.rstd[c]; gm[i] = bn.gamma[c]; bt[i] = bn.beta[c];
      const float ic = inv_count > 0.f ? inv_count : 1.f / bnsum[2 * g.C + c];  // SyncBN: allreduced count
      mdu[i] = bnsum[c] * ic;
      mdux[i] = bnsum[g.C + c] * ic;
    }
  }
  // dz region needed by the input pixels a tile owns, relative to its first
  // output row/col: [lo, lo + TH)  (always <= TO + 2 wide for pads <= 2)
  const int lo_y = floordiv(g.pt - 2, g.stride), lo_x = floordiv(g.pl - 2, g.stride);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int n = tile / (ty_n * tx_n);
    const int oy0 = ((tile / tx_n) % ty_n) * TO, ox0 = (tile % tx_n) * TO;
    // dz over output rows/cols [o0+lo, o0+lo+TH) into shared memory (0 outside)
    if (py < PY) {
      float sv[V], dp[V];
#pragma unroll
      for (int i = 0; i < V; ++i) { sv[i] = s[(size_t)n * g.C + c0 + i]; dp[i] = dpool[(size_t)n * g.C + c0 + i]; }
      for (int q = py; q < TH * TH; q += PY) {
        const int oy = oy0 + lo_y + q / TH, ox = ox0 + lo_x + q % TH;
        float* dst = dzs + q * g.C + c0;
        if (oy < 0 || oy >= g.Ho || ox < 0 || ox >= g.Wo) {
#pragma unroll
          for (int i = 0; i < V; ++i) dst[i] = 0.f;
          continue;
        }
        const size_t off = (((size_t)n * g.Ho + oy) * g.Wo + ox) * g.C + c0;
        Vec<T, V> dv, zv;
        dv.load(dy + off);
        zv.load(z + off);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float xh = (zv.v[i] - mu[i]) * rs[i];
          const float u = fmaf(xh, gm[i], bt[i]);
          const float sg = sigmoidf_(u);
          const float du = (dv.v[i] * sv[i] + dp[i]) * (sg + u * sg * (1.f - sg));
          dst[i] = gm[i] * rs[i] * (du - mdu[i] - xh * mdux[i]);
        }
      }
    }
    __syncthreads();
    if (py < PY) {
      // dw partials over the tile's own outputs
      for (int q = py; q < TO * TO; q += PY) {
        const int oy = oy0 + q / TO, ox = ox0 + q % TO;
        if (oy >= g.Ho || ox >= g.Wo) continue;
        const float* dz = dzs + ((oy - oy0 - lo_y) * TH + (ox - ox0 - lo_x)) * g.C + c0;
        float d[V];
#pragma unroll
        for (int i = 0; i < V; ++i) d[i] = dz[i];
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
          const int iy = oy * g.stride + ky - g.pt;
          if (iy < 0 || iy >= g.H) continue;
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
            const int ix = ox * g.stride + kx - g.pl;
            if (ix < 0 || ix >= g.W) continue;
            Vec<T, V> xv;
            xv.load(x + (((size_t)n * g.H + iy) * g.W + ix) * g.C + c0);
#pragma unroll
            for (int i = 0; i < V; ++i) dwa[ky * 3 + kx][i] = fmaf(d[i], xv.v[i], dwa[ky * 3 + kx][i]);
          }
        }
      }
      // dx over the input pixels owned by this tile: [o0*stride, (o0+TO)*stride);
      // the last tile of a row/column also owns the input tail past Ho*stride
      const int iy0 = oy0 * g.stride, ix0 = ox0 * g.stride;
      const int side_y = (oy0 + TO >= g.Ho) ? g.H - iy0 : TO * g.stride;
      const int side_x = (ox0 + TO >= g.Wo) ? g.W - ix0 : TO * g.stride;
      for (int q = py; q < side_y * side_x; q += PY) {
        const int iy = iy0 + q / side_x, ix = ix0 + q % side_x;
        if (iy >= g.H || ix >= g.W) continue;
        float acc[V];
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = 0.f;
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
          const int ty = iy + g.pt - ky;
          if (((ty % g.stride) + g.stride) % g.stride != 0) continue;
          const int oy = floordiv(ty, g.stride);
          if (oy < 0 || oy >= g.Ho) continue;
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
            const int tx = ix + g.pl - kx;
            if (((tx % g.stride) + g.stride) % g.stride != 0) continue;
            const int ox = floordiv(tx, g.stride);
            if (ox < 0 || ox >= g.Wo) continue;
            const float* dz = dzs + ((oy - oy0 - lo_y) * TH + (ox - ox0 - lo_x)) * g.C + c0;
#pragma unroll
            for (int i = 0; i < V; ++i) acc[i] = fmaf(dz[i], wr[ky * 3 + kx][i], acc[i]);
          }
        }
        Vec<T, V> o;
#pragma unroll
        for (int i = 0; i < V; ++i) o.v[i] = acc[i];
        o.store(dx + (((size_t)n * g.H + iy) * g.W + ix) * g.C + c0);
      }
    }
    __syncthreads();
  }
  // dw partials: fixed-order merge over pixel lanes via shared memory
  for (int t = 0; t < 9; ++t) {
    if (py < PY) {
#pragma unroll
      for (int i = 0; i < V; ++i) dzs[py * g.C + c0 + i] = dwa[t][i];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
      float acc = 0.f;
      for (int j = 0; j < PY; ++j) acc += dzs[j * g.C + c];
      dw_part[((size_t)blockIdx.x * 9 + t) * g.C + c] = acc;
    }
    __syncthreads();
  }
}

// B5: dw[t][c] = sum_b part[b][t][c]
__global__ void dw_finalize_kernel(int nparts, int C, const float* __restrict__ part, float* __restrict__ dw) {
  pdl_trigger();
  pdl_wait();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 9 * C) return;
  float acc = 0.f;
  for (int b = 0; b < nparts; ++b) acc += part[(size_t)b * 9 * C + idx];
  dw[idx] = acc;
}

// ---------------------------------------------------------------- host
int make_geo(int64_t N, int64_t H, int64_t W, int64_t C, int stride, int ks, const int* pads, int vec, Geo* g,
             const char* op) {
  DFX_REQUIRE(N > 0 && H > 0 && W > 0 && C > 0, DFX_ERR_SHAPE, std::string(op) + ": empty tensor");
  DFX_REQUIRE(stride == 1 || stride == 2, DFX_ERR_UNSUPPORTED, std::string(op) + ": stride must be 1 or 2");
  DFX_REQUIRE(ks == 3 || ks == 5, DFX_ERR_UNSUPPORTED, std::string(op) + ": kernel size must be 3 or 5");
  DFX_REQUIRE(C % vec == 0, DFX_ERR_SHAPE, std::string(op) + ": channels must be a multiple of " + std::to_string(vec));
  DFX_REQUIRE(C / vec <= kThreads, DFX_ERR_SHAPE, std::string(op) + ": too many channels");
  for (int i = 0; i < 4; ++i)
    DFX_REQUIRE(pads[i] >= 0 && pads[i] <= ks - 1, DFX_ERR_UNSUPPORTED,
                std::string(op) + ": pads must be in [0, ksize-1]");
  g->N = (int)N; g->H = (int)H; g->W = (int)W; g->C = (int)C;
  g->stride = stride; g->pt = pads[0]; g->pl = pads[1]; g->ks = ks;
  g->Ho = (int)((H + pads[0] + pads[2] - ks) / stride + 1);
  g->Wo = (int)((W + pads[1] + pads[3] - ks) / stride + 1);
  DFX_REQUIRE(g->Ho > 0 && g->Wo > 0, DFX_ERR_SHAPE, std::string(op) + ": output would be empty");
  // rows per pixel tile of the stream kernels (pool / excite / bwd_reduce,
  // grid = images x tiles x channel chunks): fewest (whole waves x rows per
  // tile) at the 2-CTA/SM residency of bwd_reduce (128 registers), so the
  // last wave is not a sliver (C3: 13-row tiles, 864 CTAs = 2.9 waves, instead
  // of 18-row tiles, 672 CTAs = 2.3 waves)
  {
    const int cvt = (int)C / vec;
    const int nch = cvt > 64 ? (cvt + 63) / 64 : 1;
    const long slots = 2L * num_sms();
    const int rmax = std::max(1, std::min(g->Ho, 4096 / g->Wo));
    long best = -1;
    int bestR = std::min(g->Ho, std::max(1, 2048 / g->Wo));
    for (int R = rmax; R >= 1; --R) {
      const long ctas = (long)N * ((g->Ho + R - 1) / R) * nch;
      const long cost = (ctas + slots - 1) / slots * (long)(R * g->Wo + 64);  // + per-tile fixed cost
      if (best < 0 || cost < best) {
        best = cost;
        bestR = R;
      }
    }
    g->tile_rows = bestR;
  }
  g->tiles_per_img = (g->Ho + g->tile_rows - 1) / g->tile_rows;
  return DFX_OK;
}

template <typename T> constexpr int vec_of() { return MbVec<T>::value; }

// channel chunking of the stream kernels: <= 64 vectors per CTA row
struct Lanes {
  int nch, cvc, py;
};
inline Lanes lanes_for(int C, int V) {
  const int cvt = C / V;
  const int nch = cvt > 64 ? (cvt + 63) / 64 : 1;
  const int cvc = (cvt + nch - 1) / nch;
  return Lanes{nch, cvc, kThreads / cvc};
}

// TMA ring path (dwconv.cu) geometry of this block: 3x3 taps
inline DwShape dw_shape(const Geo& g) { return DwShape{g.N, g.H, g.W, g.Ho, g.Wo, g.C, g.ks, g.stride, g.pt, g.pl}; }
inline bool ring_ok(const Geo& g) { return dw_ring_ok(dw_shape(g), 2) && dw_ring_ok(dw_shape(g), 4); }
// ring-path scratch (floats): partials [tiles][9][C] (>= [tiles][3][C]) then dz
inline size_t ring_part_floats(const Geo& g) {
  const DwShape d = dw_shape(g);
  size_t t = 0;
  for (int esz : {2, 4}) t = std::max(t, std::max(dw_stat_tiles(d, esz) * 3, dw_dzw_tiles(d, esz) * 9));
  return (t * g.C + 63) / 64 * 64;
}

}  // namespace
}  // namespace dfx

using namespace dfx;

namespace {

template <typename T>
int mb_forward(const Geo& g, const void* x, const float* w, void* z, float* bn_part, float* bn_local,
               cudaStream_t st) {
  constexpr int V = vec_of<T>();
  if (ring_ok(g)) return dw_conv_stats(sizeof(T) == 2 ? DFX_BF16 : DFX_F32, dw_shape(g), x, w, z, bn_part, bn_local, st);
  DFX_REQUIRE(g.ks == 3, DFX_ERR_UNSUPPORTED, "dfx_mbconv_fwd_stats: 5x5 needs the TMA ring path (C % 8 == 0)");
  const int CV = g.C / V, PY = kThreads / CV, threads = CV * PY;
  const int ntiles = g.N * g.tiles_per_img;
  const size_t sm1 = (size_t)(PY + 2 * PY * g.C) * sizeof(float);
  auto k1 = dwconv_fwd_kernel<T, V>;
  if (sm1 > 48 * 1024) cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
  launch_k(k1, ntiles, threads, sm1, st, g, (const T*)x, w, (T*)z, bn_part);
  DFX_LAUNCH_CHECK("dfx_mbconv_fwd dwconv");
  launch_k(bn_reduce_kernel, g.C, kThreads, 0, st, g, ntiles, bn_part, bn_local);
  DFX_LAUNCH_CHECK("dfx_mbconv_fwd bn_reduce");
  return DFX_OK;
}

}  // namespace

extern "C" {

/* Workspace sizes (floats) are computed by dfx_mbconv_workspace. */
size_t dfx_mbconv_workspace(int64_t N, int64_t H, int64_t W, int64_t C, int stride, int ksize, const int* pads,
                            int SE) {
  Geo g;
  if (make_geo(N, H, W, C, stride, ksize, pads, C % 8 == 0 ? 8 : 4, &g, "dfx_mbconv_workspace")) return 0;
  const size_t ntiles = (size_t)g.N * g.tiles_per_img;
  const size_t nsm = (size_t)4 * num_sms();
  // bn_part 2C*tiles | pool_part C*tiles | bwd_part 5C*tiles | de N*C | dr N*SE | nsum 2NC | dw_part 9C*grid
  size_t fl = ntiles * 2 * C + ntiles * C + ntiles * 5 * C + (size_t)N * C + (size_t)N * SE + 2 * (size_t)N * C +
              9 * (size_t)C * nsm;
  if (ring_ok(g)) {
    // ring path: partials at the head (the generic scratch is not live across
    // the dwconv calls), dz ([N, Ho, Wo, C], f32-sized) after everything
    fl = (std::max(fl, ring_part_floats(g)) + 63) / 64 * 64 + (size_t)g.N * g.Ho * g.Wo * C;
  }
  return sizeof(float) * fl + 256;
}

int dfx_mbconv_fwd_stats(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int stride, int ksize,
    const int* pads,
                         const void* x, const float* w_dw, void* z, float* bn_local, void* workspace,
                         size_t ws_bytes, void* stream) {
  const int V = dtype == DFX_BF16 ? 8 : 4;
  Geo g;
  if (int rc = make_geo(N, H, W, C, stride, ksize, pads, V, &g, "dfx_mbconv_fwd_stats")) return rc;
  DFX_REQUIRE(x && w_dw && z && bn_local && workspace, DFX_ERR_SHAPE, "dfx_mbconv_fwd_stats: null pointer");
  DFX_REQUIRE(ws_bytes >= dfx_mbconv_workspace(N, H, W, C, stride, ksize, pads, 1), DFX_ERR_WORKSPACE,
              "dfx_mbconv_fwd_stats: workspace too small");
  float* bn_part = (float*)workspace;
  if (dtype == DFX_BF16)
    return mb_forward<__nv_bfloat16>(g, x, w_dw, z, bn_part, bn_local, as_stream(stream));
  if (dtype == DFX_F32)
    return mb_forward<float>(g, x, w_dw, z, bn_part, bn_local, as_stream(stream));
  return fail(DFX_ERR_DTYPE, "dfx_mbconv_fwd_stats: dtype must be f32 or bf16");
}

int dfx_bn_finalize(int64_t C, int nsets, const float* sets, float eps, float momentum, float* mean, float* var,
                    float* rstd, float* run_mean, float* run_var, void* stream) {
  DFX_REQUIRE(C > 0 && nsets > 0 && sets && rstd, DFX_ERR_SHAPE, "dfx_bn_finalize: bad arguments");
  launch_k(bn_finalize_kernel, (unsigned)((C + 127) / 128), 128, 0, as_stream(stream), (int)C, nsets, sets, eps, momentum,
                                                                                 mean, var, rstd, run_mean, run_var);
  DFX_LAUNCH_CHECK("dfx_bn_finalize");
  return DFX_OK;
}

int dfx_mbconv_fwd_se(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int stride, int ksize,
    const int* pads, int64_t SE,
                      const void* z, const float* mean, const float* rstd, const float* gamma, const float* beta,
                      const float* w_r, const float* b_r, const float* w_e, const float* b_e, float* pooled,
                      float* r, float* s, void* y, void* workspace, size_t ws_bytes, void* stream) {
  const int V = dtype == DFX_BF16 ? 8 : 4;
  Geo g;
  if (int rc = make_geo(N, H, W, C, stride, ksize, pads, V, &g, "dfx_mbconv_fwd_se")) return rc;
  DFX_REQUIRE(SE > 0 && z && mean && rstd && gamma && beta && w_r && b_r && w_e && b_e && pooled && r && s,
              DFX_ERR_SHAPE, "dfx_mbconv_fwd_se: null pointer");
  DFX_REQUIRE(ws_bytes >= dfx_mbconv_workspace(N, H, W, C, stride, ksize, pads, (int)SE), DFX_ERR_WORKSPACE,
              "dfx_mbconv_fwd_se: workspace too small");
  cudaStream_t st = as_stream(stream);
  const int ntiles = g.N * g.tiles_per_img;
  float* pool_part = (float*)workspace + (size_t)ntiles * 2 * C;
  BnParams bn{mean, rstd, gamma, beta};
  const Lanes ln = lanes_for(g.C, V);
  const int PY = ln.py, threads = ln.cvc * ln.py;
  const dim3 grid2((unsigned)ntiles, (unsigned)ln.nch);
  const size_t sm4 = (size_t)PY * g.C * sizeof(float);
  if (dtype == DFX_BF16) {
    auto k4 = bn_swish_pool_kernel<__nv_bfloat16, 8>;
    if (sm4 > 48 * 1024) cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
    launch_k(k4, grid2, threads, sm4, st, g, (const __nv_bfloat16*)z, bn, pool_part);
  } else if (dtype == DFX_F32) {
    auto k4 = bn_swish_pool_kernel<float, 4>;
    if (sm4 > 48 * 1024) cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
    launch_k(k4, grid2, threads, sm4, st, g, (const float*)z, bn, pool_part);
  } else {
    return fail(DFX_ERR_DTYPE, "dfx_mbconv_fwd_se: dtype must be f32 or bf16");
  }
  DFX_LAUNCH_CHECK("dfx_mbconv_fwd_se pool");
  launch_k(se_fwd_kernel, g.N, 1024, (size_t)(g.C + SE) * sizeof(float), st, g, (int)SE, pool_part, w_r, b_r, w_e, b_e,
                                                                           pooled, r, s);
  DFX_LAUNCH_CHECK("dfx_mbconv_fwd_se se");
  if (!y) return DFX_OK;  // excite folded into the consumer (dfx_gemm_excite)
  if (dtype == DFX_BF16)
    launch_k(excite_kernel<__nv_bfloat16, 8>, grid2, threads, 0, st, g, (const __nv_bfloat16*)z, bn, s,
             (__nv_bfloat16*)y);
  else
    launch_k(excite_kernel<float, 4>, grid2, threads, 0, st, g, (const float*)z, bn, s, (float*)y);
  DFX_LAUNCH_CHECK("dfx_mbconv_fwd_se excite");
  return DFX_OK;
}

int dfx_mbconv_bwd_reduce(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int stride, int ksize,
    const int* pads,
                          int64_t SE, const void* dy, const void* z, const float* mean, const float* rstd,
                          const float* gamma, const float* beta, const float* s, const float* r,
                          const float* pooled, const float* w_r, const float* w_e, float* dw_e, float* db_e,
                          float* dw_r, float* db_r, float* dpool, float* bnsum, void* workspace, size_t ws_bytes,
                          void* stream) {
  const int V = dtype == DFX_BF16 ? 8 : 4;
  Geo g;
  if (int rc = make_geo(N, H, W, C, stride, ksize, pads, V, &g, "dfx_mbconv_bwd_reduce")) return rc;
  DFX_REQUIRE(dy && z && mean && rstd && gamma && beta && s && r && pooled && w_r && w_e && dw_e && db_e && dw_r &&
                  db_r && dpool && bnsum,
              DFX_ERR_SHAPE, "dfx_mbconv_bwd_reduce: null pointer");
  DFX_REQUIRE(ws_bytes >= dfx_mbconv_workspace(N, H, W, C, stride, ksize, pads, (int)SE), DFX_ERR_WORKSPACE,
              "dfx_mbconv_bwd_reduce: workspace too small");
  cudaStream_t st = as_stream(stream);
  const int ntiles = g.N * g.tiles_per_img;
  float* bwd_part = (float*)workspace + (size_t)ntiles * 3 * C;
  float* de = bwd_part + (size_t)ntiles * 5 * C;
  float* dr = de + (size_t)N * C;
  float* nsum = dr + (size_t)N * SE;
  BnParams bn{mean, rstd, gamma, beta};
  const Lanes ln = lanes_for(g.C, V);
  const int PY = ln.py, threads = ln.cvc * ln.py;
  const dim3 grid2((unsigned)ntiles, (unsigned)ln.nch);
  const size_t sm = (size_t)PY * g.C * sizeof(float);
  if (dtype == DFX_BF16) {
    auto k = bwd_reduce_kernel<__nv_bfloat16, 8>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(k, grid2, threads, sm, st, g, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)z, bn, bwd_part);
  } else if (dtype == DFX_F32) {
    auto k = bwd_reduce_kernel<float, 4>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(k, grid2, threads, sm, st, g, (const float*)dy, (const float*)z, bn, bwd_part);
  } else {
    return fail(DFX_ERR_DTYPE, "dfx_mbconv_bwd_reduce: dtype must be f32 or bf16");
  }
  DFX_LAUNCH_CHECK("dfx_mbconv_bwd_reduce reduce");
  DFX_REQUIRE(SE <= 1024, DFX_ERR_UNSUPPORTED, "dfx_mbconv_bwd_reduce: squeeze width must be <= 1024");
  const size_t sm_se = (size_t)(6 * g.C + SE + 1024) * sizeof(float);
  if (sm_se > 48 * 1024) cudaFuncSetAttribute(se_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_se);
  launch_k(se_bwd_kernel, g.N, 1024, sm_se, st, g, (int)SE, bwd_part, s, r, w_r, w_e,
                                                                                de, dr, dpool, nsum);
  DFX_LAUNCH_CHECK("dfx_mbconv_bwd_reduce se_bwd");
  const int64_t total = (int64_t)C * SE * 2 + C + SE + 2 * C;
  const int grid5 = (int)std::min<int64_t>((total + 31) / 32, (int64_t)num_sms() * 16);
  launch_k(se_bwd_reduce_kernel, grid5, 256, 0, st, g.N, g.C, (int)SE, de, dr, r, pooled, nsum, dw_e, db_e,
           dw_r, db_r, bnsum);
  DFX_LAUNCH_CHECK("dfx_mbconv_bwd_reduce se_reduce");
  return DFX_OK;
}

int dfx_mbconv_bwd_dx(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int stride, int ksize,
    const int* pads,
                      const void* dy, const void* z, const void* x, const float* w_dw, const float* mean,
                      const float* rstd, const float* gamma, const float* beta, const float* s, const float* dpool,
                      const float* bnsum, double count, void* dx, float* dw_dw, void* workspace, size_t ws_bytes,
                      void* stream) {
  const int V = dtype == DFX_BF16 ? 8 : 4;
  Geo g;
  if (int rc = make_geo(N, H, W, C, stride, ksize, pads, V, &g, "dfx_mbconv_bwd_dx")) return rc;
  DFX_REQUIRE(dy && z && x && w_dw && mean && rstd && gamma && beta && s && dpool && bnsum && dx && dw_dw,
              DFX_ERR_SHAPE, "dfx_mbconv_bwd_dx: null pointer");
  DFX_REQUIRE(count >= 0, DFX_ERR_SHAPE, "dfx_mbconv_bwd_dx: count must be >= 0");
  DFX_REQUIRE(ws_bytes >= dfx_mbconv_workspace(N, H, W, C, stride, ksize, pads, 1), DFX_ERR_WORKSPACE,
              "dfx_mbconv_bwd_dx: workspace too small");
  cudaStream_t st = as_stream(stream);
  if (ring_ok(g)) {
    // dz (stored) + dw from the x window, then dx = transposed conv of dz
    const DwShape d = dw_shape(g);
    const size_t nt = (size_t)g.N * g.tiles_per_img, nsm = (size_t)4 * num_sms();
    const size_t fl1 = nt * 8 * C + (size_t)N * C + (size_t)N + 2 * (size_t)N * C + 9 * (size_t)C * nsm;
    float* part = (float*)workspace;
    void* dzb = (float*)workspace + (std::max(fl1, ring_part_floats(g)) + 63) / 64 * 64;  // TMA: 16-B aligned
    const DzConsts k{mean, rstd, gamma, beta, s, dpool, bnsum, count > 0 ? (float)(1.0 / count) : -1.f};
    if (int rc = dw_dz_dw(dtype, d, x, dy, z, k, dzb, part, dw_dw, st)) return rc;
    return dw_dx(dtype, d, dzb, w_dw, dx, st);
  }
  DFX_REQUIRE(g.ks == 3, DFX_ERR_UNSUPPORTED, "dfx_mbconv_bwd_dx: 5x5 needs the TMA ring path (C % 8 == 0)");
  const int ntiles_conv = g.N * ((g.Ho + TO - 1) / TO) * ((g.Wo + TO - 1) / TO);
  const int grid = std::min(ntiles_conv, 4 * num_sms());
  const size_t ntiles = (size_t)g.N * g.tiles_per_img;
  (void)ntiles;
  float* dw_part = (float*)workspace;  // [grid][9][C]; the forward/reduce scratch is dead by now
  BnParams bn{mean, rstd, gamma, beta};
  const int CV = g.C / V, PY = kThreads / CV, threads = CV * PY;
  const size_t sm = std::max((size_t)TH * TH * g.C, (size_t)PY * g.C) * sizeof(float);
  const float inv_count = count > 0 ? (float)(1.0 / count) : -1.f;
  if (dtype == DFX_BF16) {
    auto k = dwconv_bwd_kernel<__nv_bfloat16, 8>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(k, grid, threads, sm, st, g, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)z, (const __nv_bfloat16*)x, w_dw,
                                 bn, s, dpool, bnsum, inv_count, (__nv_bfloat16*)dx, dw_part);
  } else if (dtype == DFX_F32) {
    auto k = dwconv_bwd_kernel<float, 4>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(k, grid, threads, sm, st, g, (const float*)dy, (const float*)z, (const float*)x, w_dw, bn, s, dpool, bnsum,
                                 inv_count, (float*)dx, dw_part);
  } else {
    return fail(DFX_ERR_DTYPE, "dfx_mbconv_bwd_dx: dtype must be f32 or bf16");
  }
  DFX_LAUNCH_CHECK("dfx_mbconv_bwd_dx conv");
  launch_k(dw_finalize_kernel, (9 * (int)C + 255) / 256, 256, 0, st, grid, (int)C, dw_part, dw_dw);
  DFX_LAUNCH_CHECK("dfx_mbconv_bwd_dx dw");
  return DFX_OK;
}

}  // extern "C"
