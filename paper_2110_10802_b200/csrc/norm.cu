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

// block b handles rows [b*rpb, min((b+1)*rpb, rows)); thread (cv, py) owns
// channel vector cv and every PY-th row; rows are loaded four at a time (four
// 128-bit loads in flight per thread).  Statistics are shifted sums (shift =
// the thread's first row: no per-element division, no cancellation), turned
// into a Welford (n, mean, M2) set per thread and merged in a fixed order.
template <typename T, int V>
__global__ void __launch_bounds__(kThreads) bn_stats_kernel(int64_t rows, int C, int64_t rpb, const T* __restrict__ x,
                                                           float* __restrict__ part /*[blocks][3][C]*/) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  // channel chunks across gridDim.y (wide C, few rows: enough CTAs and lanes)
  const int CVt = C / V, CVc = (CVt + gridDim.y - 1) / gridDim.y, PY = blockDim.x / CVc;
  const int lcv = threadIdx.x % CVc, py = threadIdx.x / CVc;
  const int cv = blockIdx.y * CVc + lcv;
  const bool on = cv < CVt;
  const int c0 = (on ? cv : 0) * V;
  const int cbeg = blockIdx.y * CVc * V, cend = min(cbeg + CVc * V, C);
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, rows);
  float sh[V], s1[V], s2[V];
  int cnt = 0;
  int64_t r = on ? r0 + py : r1;
  {
    Vec<T, V> v;
    if (r < r1) v.load(x + r * C + c0);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      sh[i] = r < r1 ? v.v[i] : 0.f;
      s1[i] = 0.f;
      s2[i] = 0.f;
    }
  }
  for (; r + 3 * PY < r1; r += 4 * PY) {
    Vec<T, V> v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q].load(x + (r + q * PY) * C + c0);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float d = v[q].v[i] - sh[i];
        s1[i] += d;
        s2[i] = fmaf(d, d, s2[i]);
      }
    cnt += 4;
  }
  for (; r < r1; r += PY) {
    Vec<T, V> v;
    v.load(x + r * C + c0);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float d = v.v[i] - sh[i];
      s1[i] += d;
      s2[i] = fmaf(d, d, s2[i]);
    }
    ++cnt;
  }
  float* s_n = sm;
  float* s_mean = sm + PY;
  float* s_m2 = s_mean + PY * C;
  if (lcv == 0) s_n[py] = (float)cnt;
  if (on) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float m = cnt ? s1[i] / (float)cnt : 0.f;
      s_mean[py * C + c0 + i] = sh[i] + m;
      s_m2[py * C + c0 + i] = cnt ? fmaxf(s2[i] - s1[i] * m, 0.f) : 0.f;
    }
  }
  __syncthreads();
  for (int c = cbeg + threadIdx.x; c < cend; c += blockDim.x) {
    Wf acc = {0.f, 0.f, 0.f};
    for (int j = 0; j < PY; ++j) acc = wmerge(acc, Wf{s_n[j], s_mean[j * C + c], s_m2[j * C + c]});
    part[((size_t)blockIdx.x * 3 + 0) * C + c] = acc.n;
    part[((size_t)blockIdx.x * 3 + 1) * C + c] = acc.mean;
    part[((size_t)blockIdx.x * 3 + 2) * C + c] = acc.m2;
  }
}

// single-replica finalize fused into the merge (dfx_batchnorm_stats_finalize):
// the statistics of the one set, exactly as dfx_bn_finalize computes them
struct BnFin {
  float eps, momentum;
  float *mean, *var, *rstd, *run_mean, *run_var;  // rstd == null: merge only
};

// one block per channel: merge block partials in a fixed tree order
__global__ void __launch_bounds__(kThreads) bn_merge_kernel(int nparts, int C, const float* __restrict__ part,
                                                           float* __restrict__ out /*[3][C]*/, BnFin fin) {
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
  if (threadIdx.x == 0) {
    out[c] = sn[0]; out[C + c] = smn[0]; out[2 * C + c] = sm2[0];
    if (fin.rstd) {
      const float v = sm2[0] / sn[0];  // biased variance (frontend.py:565)
      if (fin.mean) fin.mean[c] = smn[0];
      if (fin.var) fin.var[c] = v;
      fin.rstd[c] = rsqrtf(v + fin.eps);
      if (fin.run_mean) fin.run_mean[c] = fin.run_mean[c] * fin.momentum + smn[0] * (1.f - fin.momentum);
      if (fin.run_var) fin.run_var[c] = fin.run_var[c] * fin.momentum + v * (1.f - fin.momentum);
    }
  }
}

// swish'(u) = s + u s (1 - s); bf16 storage uses the one-MUFU sigmoid
template <typename T> __device__ __forceinline__ float sig_t(float u) {
  if constexpr (sizeof(T) == 2) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(0.5f * u));
    return fmaf(0.5f, y, 0.5f);
  } else {
    return sigmoid_f(u);
  }
}

// rows-chunk grid, thread (cv, py): the per-channel constants live in
// registers (u = x*P + Q), four rows in flight per thread
template <typename T, int V, int ACT>
__global__ void __launch_bounds__(kThreads) bn_apply_kernel(int64_t rows, int C, int64_t rpb, const T* __restrict__ x,
                                                           const float* __restrict__ mean, const float* __restrict__ rstd,
                                                           const float* __restrict__ gamma, const float* __restrict__ beta,
                                                           T* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  // channel chunks across gridDim.y (wide C, few rows: enough CTAs and lanes)
  const int CVt = C / V, CVc = (CVt + gridDim.y - 1) / gridDim.y, PY = blockDim.x / CVc;
  const int lcv = threadIdx.x % CVc, py = threadIdx.x / CVc;
  const int cv = blockIdx.y * CVc + lcv;
  const bool on = cv < CVt;
  const int c0 = (on ? cv : 0) * V;
  const int cbeg = blockIdx.y * CVc * V, cend = min(cbeg + CVc * V, C);
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, rows);
  float P[V], Q[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    P[i] = rstd[c0 + i] * gamma[c0 + i];
    Q[i] = beta[c0 + i] - mean[c0 + i] * P[i];
  }
  auto f = [&](const Vec<T, V>& xv, T* out) {
    Vec<T, V> yv;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float u = fmaf(xv.v[i], P[i], Q[i]);
      yv.v[i] = ACT ? u * sig_t<T>(u) : u;
    }
    yv.store(out);
  };
  int64_t r = on ? r0 + py : r1;
  for (; r + 3 * PY < r1; r += 4 * PY) {
    Vec<T, V> v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q].load(x + (r + q * PY) * C + c0);
#pragma unroll
    for (int q = 0; q < 4; ++q) f(v[q], y + (r + q * PY) * C + c0);
  }
  for (; r < r1; r += PY) {
    Vec<T, V> v;
    v.load(x + r * C + c0);
    f(v, y + r * C + c0);
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
  // channel chunks across gridDim.y (wide C, few rows: enough CTAs and lanes)
  const int CVt = C / V, CVc = (CVt + gridDim.y - 1) / gridDim.y, PY = blockDim.x / CVc;
  const int lcv = threadIdx.x % CVc, py = threadIdx.x / CVc;
  const int cv = blockIdx.y * CVc + lcv;
  const bool on = cv < CVt;
  const int c0 = (on ? cv : 0) * V;
  const int cbeg = blockIdx.y * CVc * V, cend = min(cbeg + CVc * V, C);
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, rows);
  float P[V], Q[V], R[V], M[V], s1[V], s2[V];  // u = x*P + Q, xhat = x*R + M
#pragma unroll
  for (int i = 0; i < V; ++i) {
    R[i] = rstd[c0 + i];
    M[i] = -mean[c0 + i] * R[i];
    P[i] = gamma[c0 + i] * R[i];
    Q[i] = beta[c0 + i] - mean[c0 + i] * P[i];
    s1[i] = 0.f;
    s2[i] = 0.f;
  }
  auto f = [&](const Vec<T, V>& dv, const Vec<T, V>& xv) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float xh = fmaf(xv.v[i], R[i], M[i]);
      float du = dv.v[i];
      if (ACT) {
        const float u = fmaf(xv.v[i], P[i], Q[i]);
        const float sg = sig_t<T>(u);
        du *= sg * fmaf(u, 1.f - sg, 1.f);
      }
      s1[i] += du;
      s2[i] = fmaf(du, xh, s2[i]);
    }
  };
  int64_t r = on ? r0 + py : r1;
  for (; r + 3 * PY < r1; r += 4 * PY) {
    Vec<T, V> dv[4], xv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      dv[q].load(dy + (r + q * PY) * C + c0);
      xv[q].load(x + (r + q * PY) * C + c0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) f(dv[q], xv[q]);
  }
  for (; r < r1; r += PY) {
    Vec<T, V> dv, xv;
    dv.load(dy + r * C + c0);
    xv.load(x + r * C + c0);
    f(dv, xv);
  }
  for (int q = 0; q < 2; ++q) {
    if (on) {
#pragma unroll
      for (int i = 0; i < V; ++i) sm[py * C + c0 + i] = q == 0 ? s1[i] : s2[i];
    }
    __syncthreads();
    for (int c = cbeg + threadIdx.x; c < cend; c += blockDim.x) {
      double acc = 0.0;  // the cross-lane / cross-block merges run in f64
      for (int j = 0; j < PY; ++j) acc += sm[j * C + c];
      part[((size_t)blockIdx.x * 2 + q) * C + c] = (float)acc;
    }
    __syncthreads();
  }
}

// out[i] = sum_b part[b][i] (i over 2C): block = 32 outputs x 8 part lanes,
// fixed-order f64 combine
__global__ void __launch_bounds__(1024) bn_sum_parts_kernel(int nparts, int C, const float* __restrict__ part,
                                                            float* __restrict__ out, float* __restrict__ dbeta,
                                                            float* __restrict__ dgamma) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[32][33];
  const int idx = blockIdx.x * 32 + (threadIdx.x & 31);
  const double v = sum_part_rows(nparts, part, (size_t)2 * C, idx, idx < 2 * C, red);
  if (threadIdx.x < 32 && idx < 2 * C) {
    out[idx] = (float)v;
    float* g = idx < C ? dbeta : dgamma;  // the local parameter gradients (bnsum before any SyncBN allreduce)
    if (g) g[idx < C ? idx : idx - C] = (float)v;
  }
}

// dx = A*du + Cx*x + B with A = gamma*rstd and the BN-VJP means folded into
// per-channel constants (autodiff.py:1557-1617)
template <typename T, int V, int ACT>
__global__ void __launch_bounds__(kThreads) bn_bwd_dx_kernel(int64_t rows, int C, int64_t rpb, const T* __restrict__ dy,
                                                            const T* __restrict__ x, const float* __restrict__ mean,
                                                            const float* __restrict__ rstd,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ beta,
                                                            const float* __restrict__ sums, float inv_count,
                                                            T* __restrict__ dx) {
  pdl_trigger();
  pdl_wait();
  // channel chunks across gridDim.y (wide C, few rows: enough CTAs and lanes)
  const int CVt = C / V, CVc = (CVt + gridDim.y - 1) / gridDim.y, PY = blockDim.x / CVc;
  const int lcv = threadIdx.x % CVc, py = threadIdx.x / CVc;
  const int cv = blockIdx.y * CVc + lcv;
  const bool on = cv < CVt;
  const int c0 = (on ? cv : 0) * V;
  const int cbeg = blockIdx.y * CVc * V, cend = min(cbeg + CVc * V, C);
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(r0 + rpb, rows);
  float A[V], Cx[V], B[V], P[V], Q[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = c0 + i;
    const float rs = rstd[c], mu = mean[c];
    A[i] = gamma[c] * rs;
    // inv_count <= 0: SyncBN — the allreduced per-channel count is sums[2][c]
    const float ic = inv_count > 0.f ? inv_count : 1.f / sums[2 * C + c];
    const float mdu = sums[c] * ic, mdux = sums[C + c] * ic;
    Cx[i] = -A[i] * mdux * rs;
    B[i] = -A[i] * mdu + A[i] * mdux * rs * mu;
    P[i] = A[i];
    Q[i] = beta[c] - mu * A[i];
  }
  auto f = [&](const Vec<T, V>& dv, const Vec<T, V>& xv, T* out) {
    Vec<T, V> o;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      float du = dv.v[i];
      if (ACT) {
        const float u = fmaf(xv.v[i], P[i], Q[i]);
        const float sg = sig_t<T>(u);
        du *= sg * fmaf(u, 1.f - sg, 1.f);
      }
      o.v[i] = fmaf(A[i], du, fmaf(Cx[i], xv.v[i], B[i]));
    }
    o.store(out);
  };
  int64_t r = on ? r0 + py : r1;
  for (; r + 3 * PY < r1; r += 4 * PY) {
    Vec<T, V> dv[4], xv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      dv[q].load(dy + (r + q * PY) * C + c0);
      xv[q].load(x + (r + q * PY) * C + c0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) f(dv[q], xv[q], dx + (r + q * PY) * C + c0);
  }
  for (; r < r1; r += PY) {
    Vec<T, V> dv, xv;
    dv.load(dy + r * C + c0);
    xv.load(x + r * C + c0);
    f(dv, xv, dx + r * C + c0);
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
  DFX_REQUIRE(C / vec_width(dtype, C) <= 64 * kThreads, DFX_ERR_SHAPE, std::string(op) + ": too many channels");
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

// elementwise passes: >= 8 rows per thread lane, at most 8 blocks per SM
// (rounded to whole waves of the kernel's resident CTAs when there is enough work)
void stream_blocks(int64_t rows, int PY, int64_t* rpb, int* nb, int resident = 8, int nch = 1) {
  int64_t b = std::min<int64_t>((int64_t)num_sms() * 8, (rows + 8 * PY - 1) / (8 * PY));
  const int64_t wave = std::max<int64_t>(1, (int64_t)resident * num_sms() / std::max(nch, 1));
  if (b > wave) b = (b + wave - 1) / wave * wave;  // whole waves
  if (b < 1) b = 1;
  *rpb = (rows + b - 1) / b;
  *nb = (int)((rows + *rpb - 1) / *rpb);
}

// reductions: partial sets per block (<= kMaxBlocks), >= 4 rows per thread lane
// channel chunking: <= 64 vectors per CTA row so a wide C still gets >= 4 row lanes
struct Lanes {
  int nch, cvc, py;
};
Lanes lanes_for(int64_t C, int V) {
  const int cvt = (int)C / V;
  const int nch = cvt > 64 ? (cvt + 63) / 64 : 1;
  const int cvc = (cvt + nch - 1) / nch;
  return Lanes{nch, cvc, kThreads / cvc};
}

// `resident`: CTAs of the launched kernel that fit one SM at once (its
// register / shared-memory occupancy); the row blocks x channel chunks then
// fill exactly one wave (a 4-per-SM grid of an 80-register kernel that only
// fits 3 per SM ran a 1/3-full second wave)
void blocks_for(int64_t rows, int64_t* rpb, int* nb, int resident = 4, int nch = 1) {
  const int64_t wave = std::max<int64_t>(1, (int64_t)resident * num_sms() / std::max(nch, 1));
  int64_t b = std::min<int64_t>(std::min<int64_t>(kMaxBlocks, wave), (rows + 63) / 64);
  if (b < 1) b = 1;
  *rpb = (rows + b - 1) / b;
  *nb = (int)((rows + *rpb - 1) / *rpb);
}

template <typename K> int resident_ctas(K kern, int threads, size_t smem) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  return occ;
}

int bn_stats_impl(int dtype, int64_t rows, int64_t C, const void* x, float* local, void* workspace, size_t ws_bytes,
                  const BnFin& fin, void* stream) {
  if (int rc = check_bn(dtype, rows, C, "dfx_batchnorm_stats")) return rc;
  DFX_REQUIRE(x && local && workspace, DFX_ERR_SHAPE, "dfx_batchnorm_stats: null pointer");
  DFX_REQUIRE(ws_bytes >= dfx_batchnorm_workspace(rows, C), DFX_ERR_WORKSPACE, "dfx_batchnorm_stats: workspace too small");
  cudaStream_t st = as_stream(stream);
  int64_t rpb = 0;
  int nb = 0;
  const int V = vec_width(dtype, C);
  const Lanes ln = lanes_for(C, V);
  const int PY = ln.py;
  const size_t sm = (size_t)(PY + 2 * PY * C) * sizeof(float);
#define S(TT, VV, ACT)                                                                                    \
  {                                                                                                       \
    auto k = bn_stats_kernel<TT, VV>;                                                                     \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);   \
    blocks_for(rows, &rpb, &nb, resident_ctas(k, ln.cvc * PY, sm), ln.nch);                               \
    launch_k(k, dim3(nb, ln.nch), ln.cvc * PY, sm, st, rows, (int)C, rpb, (const TT*)x, (float*)workspace);     \
  }
  BN_DISPATCH(S, 0);
#undef S
  DFX_LAUNCH_CHECK("dfx_batchnorm_stats");
  launch_k(bn_merge_kernel, (unsigned)C, kThreads, 0, st, nb, (int)C, (const float*)workspace, local, fin);
  DFX_LAUNCH_CHECK("dfx_batchnorm_stats merge");
  return DFX_OK;
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
  return bn_stats_impl(dtype, rows, C, x, local, workspace, ws_bytes, BnFin{0.f, 0.f, nullptr, nullptr, nullptr,
                                                                           nullptr, nullptr}, stream);
}

int dfx_batchnorm_stats_finalize(int dtype, int64_t rows, int64_t C, const void* x, float* local, float eps,
                                 float momentum, float* mean, float* var, float* rstd, float* run_mean,
                                 float* run_var, void* workspace, size_t ws_bytes, void* stream) {
  DFX_REQUIRE(rstd, DFX_ERR_SHAPE, "dfx_batchnorm_stats_finalize: rstd is required");
  return bn_stats_impl(dtype, rows, C, x, local, workspace, ws_bytes,
                       BnFin{eps, momentum, mean, var, rstd, run_mean, run_var}, stream);
}

int dfx_batchnorm_act_apply(int dtype, int64_t rows, int64_t C, const void* x, const float* mean, const float* rstd,
                            const float* gamma, const float* beta, int act, void* y, void* stream) {
  if (int rc = check_bn(dtype, rows, C, "dfx_batchnorm_act_apply")) return rc;
  DFX_REQUIRE(x && mean && rstd && gamma && beta && y, DFX_ERR_SHAPE, "dfx_batchnorm_act_apply: null pointer");
  DFX_REQUIRE(act == 0 || act == 1, DFX_ERR_UNSUPPORTED, "dfx_batchnorm_act_apply: act must be 0 or 1");
  cudaStream_t st = as_stream(stream);
  const int V = vec_width(dtype, C);
  const Lanes ln = lanes_for(C, V);
  int64_t rpb = 0;
  int nb = 0;
#define A(TT, VV, ACT) { stream_blocks(rows, ln.py * ln.nch, &rpb, &nb, resident_ctas(bn_apply_kernel<TT, VV, ACT>, ln.cvc * ln.py, 0), ln.nch); launch_k(bn_apply_kernel<TT, VV, ACT>, dim3(nb, ln.nch), ln.cvc * ln.py, 0, st, rows, (int)C, rpb, (const TT*)x, mean, rstd, gamma, beta, (TT*)y); }
  BN_DISPATCH(A, act);
#undef A
  DFX_LAUNCH_CHECK("dfx_batchnorm_act_apply");
  return DFX_OK;
}

int dfx_batchnorm_act_bwd_reduce(int dtype, int64_t rows, int64_t C, const void* dy, const void* x,
                                 const float* mean, const float* rstd, const float* gamma, const float* beta,
                                 int act, float* bnsum, void* workspace, size_t ws_bytes, void* stream) {
  return dfx_batchnorm_act_bwd_reduce_grads(dtype, rows, C, dy, x, mean, rstd, gamma, beta, act, bnsum, nullptr,
                                            nullptr, workspace, ws_bytes, stream);
}

int dfx_batchnorm_act_bwd_reduce_grads(int dtype, int64_t rows, int64_t C, const void* dy, const void* x,
                                       const float* mean, const float* rstd, const float* gamma, const float* beta,
                                       int act, float* bnsum, float* dbeta, float* dgamma, void* workspace,
                                       size_t ws_bytes, void* stream) {
  if (int rc = check_bn(dtype, rows, C, "dfx_batchnorm_act_bwd_reduce")) return rc;
  DFX_REQUIRE(dy && x && mean && rstd && gamma && beta && bnsum && workspace, DFX_ERR_SHAPE,
              "dfx_batchnorm_act_bwd_reduce: null pointer");
  DFX_REQUIRE(ws_bytes >= dfx_batchnorm_workspace(rows, C), DFX_ERR_WORKSPACE,
              "dfx_batchnorm_act_bwd_reduce: workspace too small");
  cudaStream_t st = as_stream(stream);
  int64_t rpb = 0;
  int nb = 0;
  const int V = vec_width(dtype, C);
  const Lanes ln = lanes_for(C, V);
  const int PY = ln.py;
  const size_t sm = (size_t)PY * C * sizeof(float);
#define R(TT, VV, ACT)                                                                                      \
  {                                                                                                         \
    auto k = bn_bwd_reduce_kernel<TT, VV, ACT>;                                                             \
    if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
    blocks_for(rows, &rpb, &nb, resident_ctas(k, ln.cvc * PY, sm), ln.nch);                                 \
    launch_k(k, dim3(nb, ln.nch), ln.cvc * PY, sm, st, rows, (int)C, rpb, (const TT*)dy, (const TT*)x, mean, rstd, gamma, beta, \
                               (float*)workspace);                                                          \
  }
  BN_DISPATCH(R, act);
#undef R
  DFX_LAUNCH_CHECK("dfx_batchnorm_act_bwd_reduce");
  launch_k(bn_sum_parts_kernel, (unsigned)((2 * C + 31) / 32), 1024, 0, st, nb, (int)C, (const float*)workspace, bnsum,
           dbeta, dgamma);
  DFX_LAUNCH_CHECK("dfx_batchnorm_act_bwd_reduce sum");
  return DFX_OK;
}

int dfx_batchnorm_act_bwd_dx(int dtype, int64_t rows, int64_t C, const void* dy, const void* x, const float* mean,
                             const float* rstd, const float* gamma, const float* beta, int act, const float* bnsum,
                             double count, void* dx, void* stream) {
  if (int rc = check_bn(dtype, rows, C, "dfx_batchnorm_act_bwd_dx")) return rc;
  DFX_REQUIRE(dy && x && mean && rstd && gamma && beta && bnsum && dx, DFX_ERR_SHAPE,
              "dfx_batchnorm_act_bwd_dx: null pointer");
  DFX_REQUIRE(count >= 0, DFX_ERR_SHAPE, "dfx_batchnorm_act_bwd_dx: count must be >= 0");
  cudaStream_t st = as_stream(stream);
  const int V = vec_width(dtype, C);
  const Lanes ln = lanes_for(C, V);
  int64_t rpb = 0;
  int nb = 0;
  const float ic = count > 0 ? (float)(1.0 / count) : -1.f;  // -1: per-channel count from bnsum[2]
#define D(TT, VV, ACT) \
  { stream_blocks(rows, ln.py * ln.nch, &rpb, &nb, resident_ctas(bn_bwd_dx_kernel<TT, VV, ACT>, ln.cvc * ln.py, 0), ln.nch); launch_k(bn_bwd_dx_kernel<TT, VV, ACT>, dim3(nb, ln.nch), ln.cvc * ln.py, 0, st, rows, (int)C, rpb, (const TT*)dy, (const TT*)x, mean, rstd, gamma, beta, bnsum, ic, (TT*)dx); }
  BN_DISPATCH(D, act);
#undef D
  DFX_LAUNCH_CHECK("dfx_batchnorm_act_bwd_dx");
  return DFX_OK;
}

}  // extern "C"
