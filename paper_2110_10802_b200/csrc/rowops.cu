// rowops.cu — HBM-bound row kernels of the BERT encoder hot path (sm_100a).
//
//  * bias + dropout + residual + LayerNorm, forward and backward
//      reference: Add/Mul/Add (frontend.py:291-293) + LayerNormalization
//      (frontend.py:519-529), VJP autodiff.py:1490-1545.
//  * scaled + masked softmax + dropout, forward and backward
//      reference: Div (frontend.py:294) + Add (175-188) + Softmax (493-501) +
//      Mul (293), VJP autodiff.py:1465-1484.
//  * bias + tanh-GELU forward/backward (frontend.py:223-295 chain).
//  * deterministic column sums (bias gradients, autodiff.py:1452-1458).
//
// Layout: one warp per row, every lane owns NCH chunks of V contiguous
// elements (128-bit accesses: V=8 for bf16, V=4 for f32), so the row lives in
// registers between the reduction and the write-back: each tensor is read once
// and written once.  Row statistics use warp shuffles only.  Column
// reductions keep per-lane partials for the lane's fixed columns across a
// grid-stride loop over rows, reduce the 8 warps of a block in fixed order
// through shared memory and finish with a fixed-order pass over blocks — no
// float atomics, so results are bitwise reproducible.
#include "common.cuh"
#include "lnsmall.h"
#include "tc_ptx.cuh"

namespace dfx {
namespace {

constexpr int kWarps = 8;            // rows per 256-thread block
constexpr int kMaxColBlocks = 296;   // 2 x 148 SMs: partial-sum slots

template <typename T> struct VecWidth { static constexpr int value = 8; };
template <> struct VecWidth<float> { static constexpr int value = 4; };

// ---------------------------------------------------------------------------
// bias + dropout + residual + LayerNorm

template <typename T, int V, int NCH, int ACT = 0>
__global__ void __launch_bounds__(256, 4) bdrln_fwd_kernel(
    int64_t rows, int cols, const T* __restrict__ h, const float* __restrict__ bias,
    const uint8_t* __restrict__ keep, const uint8_t* __restrict__ kbits, float ks, const T* __restrict__ res,
    const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
    T* __restrict__ y, T* __restrict__ s_out, float* __restrict__ mean_out,
    float* __restrict__ rstd_out) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = cols / V;
  const float inv_n = 1.f / (float)cols;
  // gamma/beta/bias are re-read per row (L1-resident): holding them in
  // registers would cap occupancy below one wave of row-warps
  for (int64_t row = (int64_t)blockIdx.x * kWarps + warp; row < rows; row += (int64_t)gridDim.x * kWarps) {
    const size_t base = (size_t)row * cols;
    float x[NCH][V];
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int vi = lane + c * 32;
      if (vi < nvec) {
        const int col = vi * V;
        Vec<T, V> hv;
        hv.load(h + base + col);
        float pb[V];
        if (bias) {
          Vec<float, V> bv;
          bv.load(bias + col);
#pragma unroll
          for (int i = 0; i < V; ++i) pb[i] = bv.v[i];
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) pb[i] = 0.f;
        }
        float m[V], r[V];
        if (keep) load_keep<V>(keep + base + col, ks, m);
        else if (kbits) load_keep_bits<V>(kbits, base + col, ks, m);
        else {
#pragma unroll
          for (int i = 0; i < V; ++i) m[i] = 1.f;
        }
        if (res) { Vec<T, V> rv; rv.load(res + base + col);
#pragma unroll
          for (int i = 0; i < V; ++i) r[i] = rv.v[i];
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) r[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < V; ++i) {
          x[c][i] = (hv.v[i] + pb[i]) * m[i] + r[i];
          sum += x[c][i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) x[c][i] = 0.f;
      }
    }
    const float mu = warp_sum(sum) * inv_n;
    float sq = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (lane + c * 32 < nvec) {
#pragma unroll
        for (int i = 0; i < V; ++i) { const float d = x[c][i] - mu; sq += d * d; }
      }
    }
    const float rstd = rsqrtf(warp_sum(sq) * inv_n + eps);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int vi = lane + c * 32;
      if (vi < nvec) {
        const int col = vi * V;
        if (s_out) {
          Vec<T, V> sv;
#pragma unroll
          for (int i = 0; i < V; ++i) sv.v[i] = x[c][i];
          sv.store(s_out + base + col);
        }
        Vec<float, V> gv, btv;
        gv.load(gamma + col);
        btv.load(beta + col);
        Vec<T, V> yv;
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float u = (x[c][i] - mu) * rstd * gv.v[i] + btv.v[i];
          yv.v[i] = ACT ? u * sigmoid_f(u) : u;
        }
        yv.store(y + base + col);
      }
    }
    if (lane == 0) {
      if (mean_out) mean_out[row] = mu;
      if (rstd_out) rstd_out[row] = rstd;
    }
  }
}

// Fixed-order reduction of per-lane column partials of the 8 warps of a block
// into part[blockIdx.x * cols + col].  acc is [NCH][V] per lane.
template <int V, int NCH>
__device__ __forceinline__ void block_colsum_store(float (&acc)[NCH][V], int cols, float* red,
                                                   float* __restrict__ part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = cols / V;
  // staging position of column c: c + (c >> 5).  Lanes write V-strided
  // columns; the one-float skew per 32-column group spreads them over all 32
  // banks (unskewed: 32 / V distinct banks), the column readers stay linear.
  const int pst = cols + ((cols + 31) >> 5);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int col = vi * V + i;
        red[warp * pst + col + (col >> 5)] = acc[c][i];
      }
    }
  }
  __syncthreads();
  for (int col = threadIdx.x; col < cols; col += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[w * pst + col + (col >> 5)];
    part[(size_t)blockIdx.x * cols + col] = s;
  }
  __syncthreads();
}

template <typename T, int V, int NCH, int ACT = 0>
__global__ void __launch_bounds__(256, 2) bdrln_bwd_kernel(
    int64_t rows, int cols, const T* __restrict__ dy, const T* __restrict__ s,
    const float* __restrict__ gamma, const float* __restrict__ beta,
    const uint8_t* __restrict__ keep, const uint8_t* __restrict__ kbits, float ks, float eps,
    T* __restrict__ ds_out, T* __restrict__ dh_out, float* __restrict__ part_g,
    float* __restrict__ part_b, float* __restrict__ part_h) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float red[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = cols / V;
  const float inv_n = 1.f / (float)cols;
  float acc_g[NCH][V], acc_b[NCH][V], acc_h[NCH][V];
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int i = 0; i < V; ++i) { acc_g[c][i] = 0.f; acc_b[c][i] = 0.f; acc_h[c][i] = 0.f; }
  for (int64_t row = (int64_t)blockIdx.x * kWarps + warp; row < rows;
       row += (int64_t)gridDim.x * kWarps) {
    const size_t base = (size_t)row * cols;
    float x[NCH][V], g[NCH][V];
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int vi = lane + c * 32;
      if (vi < nvec) {
        Vec<T, V> sv, dv;
        sv.load(s + base + vi * V);
        dv.load(dy + base + vi * V);
#pragma unroll
        for (int i = 0; i < V; ++i) { x[c][i] = sv.v[i]; g[c][i] = dv.v[i]; sum += sv.v[i]; }
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) { x[c][i] = 0.f; g[c][i] = 0.f; }
      }
    }
    const float mu = warp_sum(sum) * inv_n;
    float sq = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c)
      if (lane + c * 32 < nvec) {
#pragma unroll
        for (int i = 0; i < V; ++i) { const float d = x[c][i] - mu; sq += d * d; }
      }
    const float rstd = rsqrtf(warp_sum(sq) * inv_n + eps);
    // gamma (and beta) are re-read per row from L1: keeping them in
    // registers would cost 2 blocks/SM of occupancy
    float gam[NCH][V];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int vi = lane + c * 32;
#pragma unroll
      for (int i = 0; i < V; ++i) gam[c][i] = 0.f;
      if (vi < nvec) {
        Vec<float, V> gv;
        gv.load(gamma + vi * V);
#pragma unroll
        for (int i = 0; i < V; ++i) gam[c][i] = gv.v[i];
        if constexpr (ACT) {
          Vec<float, V> bv;
          bv.load(beta + vi * V);
#pragma unroll
          for (int i = 0; i < V; ++i) {  // dy w.r.t. the LN output through swish
            const float u = (x[c][i] - mu) * rstd * gam[c][i] + bv.v[i];
            const float sg = sigmoid_f(u);
            g[c][i] *= sg + u * sg * (1.f - sg);
          }
        }
      }
    }
    float m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
      for (int i = 0; i < V; ++i) {
        x[c][i] = (x[c][i] - mu) * rstd;  // xhat (0 on padding lanes: gamma=0, dy=0)
        const float dyg = g[c][i] * gam[c][i];
        m1 += dyg;
        m2 += dyg * x[c][i];
      }
    m1 = warp_sum(m1) * inv_n;
    m2 = warp_sum(m2) * inv_n;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int vi = lane + c * 32;
      if (vi < nvec) {
        const int col = vi * V;
        float m[V];
        if (keep) load_keep<V>(keep + base + col, ks, m);
        else if (kbits) load_keep_bits<V>(kbits, base + col, ks, m);
        else {
#pragma unroll
          for (int i = 0; i < V; ++i) m[i] = 1.f;
        }
        Vec<T, V> dsv, dhv;
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float dsi = rstd * (g[c][i] * gam[c][i] - m1 - x[c][i] * m2);
          dsv.v[i] = dsi;
          dhv.v[i] = dsi * m[i];
          acc_g[c][i] += g[c][i] * x[c][i];
          acc_b[c][i] += g[c][i];
          acc_h[c][i] += dsi * m[i];
        }
        if (ds_out) dsv.store(ds_out + base + col);
        if (dh_out) dhv.store(dh_out + base + col);
      }
    }
  }
  block_colsum_store<V, NCH>(acc_g, cols, red, part_g);
  block_colsum_store<V, NCH>(acc_b, cols, red, part_b);
  block_colsum_store<V, NCH>(acc_h, cols, red, part_h);
}


unsigned long long* g_row_trace = nullptr;  // debug timeline of the one-wave BDRLN backward

// One-wave variant (bf16, rows <= 16 * kMaxColBlocks — the BERT C2 shape):
// every warp owns exactly ONE row, so all rows are in flight at once (the
// grid-stride kernel above is latency-bound there), and nothing is carried
// across rows.  The row stays in registers as raw bf16 (24 registers for s
// and dy at 768 columns) and is unpacked on each use, which keeps the kernel
// at 64 registers = 2 CTAs x 16 warps per SM without spills.  All arithmetic
// is packed fp32 (FADD2 / FMUL2 / FFMA2 on column pairs): one wave of this
// kernel is instruction-issue bound, not HBM bound.  The CTA's 16 rows are
// reduced per column in a fixed order through two shared-memory planes
// (dbias and dgamma staged by the output pass, then dbeta).
__device__ __forceinline__ float2 bf2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}
__device__ __forceinline__ uint32_t pk_bf2(float2 v) {
  __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
  return *reinterpret_cast<uint32_t*>(&h);
}

// bf16 forward, no activation (the BERT case): every global load of the row
// (h, residual, keep flags) is issued before any use, and gamma / beta / bias
// are staged once per CTA in shared memory in the meantime, so a warp pays
// one DRAM round trip per row instead of one per chunk plus a parameter
// round trip after the reductions (the generic kernel's branches per chunk
// keep the compiler from hoisting its loads).  Arithmetic as bdrln_fwd_kernel.
constexpr int kFwdWarps = 7;  // 224-thread CTAs: 4 per SM at <= 72 registers, 28 row-warps per SM (one wave at C2)

template <int NCH> struct BdrlnRow {
  uint4 hv[NCH], rv[NCH];
  uint32_t kw[NCH];  // keep flags of the lane's 8 columns per chunk, as bits
};

template <int NCH>
__device__ __forceinline__ BdrlnRow<NCH> bdrln_load_row(int64_t r, int64_t rows, int cols, int lane,
                                                        const __nv_bfloat16* __restrict__ h,
                                                        const __nv_bfloat16* __restrict__ res,
                                                        const uint8_t* __restrict__ keep,
                                                        const uint8_t* __restrict__ kbits) {
  BdrlnRow<NCH> d;
  const size_t base = (size_t)r * cols;
  const int nvec = cols / 8;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    const bool on = r < rows && vi < nvec;
    d.hv[c] = on ? __ldg(reinterpret_cast<const uint4*>(h + base + vi * 8)) : make_uint4(0, 0, 0, 0);
    d.rv[c] = on && res ? __ldg(reinterpret_cast<const uint4*>(res + base + vi * 8)) : make_uint4(0, 0, 0, 0);
    if (on && keep) {
      const uint2 k2 = __ldg(reinterpret_cast<const uint2*>(keep + base + vi * 8));
      d.kw[c] = ((k2.x * 0x01020408u) >> 24) | (((k2.y * 0x01020408u) >> 24) << 4);
    } else if (on && kbits) {
      d.kw[c] = __ldg(kbits + ((base + vi * 8) >> 3));
    } else {
      d.kw[c] = 0xFFu;
    }
  }
  return d;
}

template <int NCH>
__device__ __forceinline__ void bdrln_row(const BdrlnRow<NCH>& d, int64_t row, int cols, int lane, bool masked,
                                          float ks, float eps, const float* gam, const float* bet, const float* bia,
                                          __nv_bfloat16* __restrict__ y, __nv_bfloat16* __restrict__ s_out,
                                          float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  constexpr int V = 8;
  const int nvec = cols / V;
  const float inv_n = 1.f / (float)cols;
  const size_t base = (size_t)row * cols;
  float x[NCH][V];
  float sum = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      const float4 b0 = reinterpret_cast<const float4*>(bia + vi * V)[0];
      const float4 b1 = reinterpret_cast<const float4*>(bia + vi * V)[1];
      const float pb[V] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      float hf[V], rf[V];
      unpack4<__nv_bfloat16>(d.hv[c], hf);
      unpack4<__nv_bfloat16>(d.rv[c], rf);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float m = masked ? (((d.kw[c] >> i) & 1u) ? ks : 0.f) : 1.f;
        x[c][i] = (hf[i] + pb[i]) * m + rf[i];
        sum += x[c][i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) x[c][i] = 0.f;
    }
  }
  const float mu = warp_sum(sum) * inv_n;
  float sq = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (lane + c * 32 < nvec) {
#pragma unroll
      for (int i = 0; i < V; ++i) { const float dd = x[c][i] - mu; sq += dd * dd; }
    }
  }
  const float rstd = rsqrtf(warp_sum(sq) * inv_n + eps);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      const int col = vi * V;
      if (s_out) *reinterpret_cast<uint4*>(s_out + base + col) = pack4<__nv_bfloat16>(x[c]);
      const float4 g0 = reinterpret_cast<const float4*>(gam + col)[0];
      const float4 g1 = reinterpret_cast<const float4*>(gam + col)[1];
      const float4 e0 = reinterpret_cast<const float4*>(bet + col)[0];
      const float4 e1 = reinterpret_cast<const float4*>(bet + col)[1];
      const float gv[V] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float bv[V] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
      float yv[V];
#pragma unroll
      for (int i = 0; i < V; ++i) yv[i] = (x[c][i] - mu) * rstd * gv[i] + bv[i];
      *reinterpret_cast<uint4*>(y + base + col) = pack4<__nv_bfloat16>(yv);
    }
  }
  if (lane == 0) {
    if (mean_out) mean_out[row] = mu;
    if (rstd_out) rstd_out[row] = rstd;
  }
}

template <int NCH>
__global__ void __launch_bounds__(kFwdWarps * 32, 4) bdrln_fwd_bf16_kernel(
    int64_t rows, int cols, const __nv_bfloat16* __restrict__ h, const float* __restrict__ bias,
    const uint8_t* __restrict__ keep, const uint8_t* __restrict__ kbits, float ks,
    const __nv_bfloat16* __restrict__ res, const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
    __nv_bfloat16* __restrict__ y, __nv_bfloat16* __restrict__ s_out, float* __restrict__ mean_out,
    float* __restrict__ rstd_out) {
  extern __shared__ float prm[];  // gamma [cols] | beta [cols] | bias [cols]
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (int64_t)blockIdx.x * kFwdWarps + warp;
  const int64_t stride = (int64_t)gridDim.x * kFwdWarps;
  // the first row's loads go out before the parameter staging
  const BdrlnRow<NCH> first = bdrln_load_row<NCH>(row0, rows, cols, lane, h, res, keep, kbits);
  float* gam = prm;
  float* bet = prm + cols;
  float* bia = prm + 2 * cols;
  for (int i = threadIdx.x; i < cols / 4; i += blockDim.x) {
    reinterpret_cast<float4*>(gam)[i] = __ldg(reinterpret_cast<const float4*>(gamma) + i);
    reinterpret_cast<float4*>(bet)[i] = __ldg(reinterpret_cast<const float4*>(beta) + i);
    reinterpret_cast<float4*>(bia)[i] = bias ? __ldg(reinterpret_cast<const float4*>(bias) + i)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  const bool masked = keep || kbits;
  if (row0 < rows) bdrln_row<NCH>(first, row0, cols, lane, masked, ks, eps, gam, bet, bia, y, s_out, mean_out, rstd_out);
  for (int64_t row = row0 + stride; row < rows; row += stride) {
    const BdrlnRow<NCH> d = bdrln_load_row<NCH>(row, rows, cols, lane, h, res, keep, kbits);
    bdrln_row<NCH>(d, row, cols, lane, masked, ks, eps, gam, bet, bia, y, s_out, mean_out, rstd_out);
  }
}

template <int NCH>
__global__ void __launch_bounds__(512, 2) bdrln_bwd_wave_kernel(
    int64_t rows, int cols, const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ s,
    const float* __restrict__ gamma, const uint8_t* __restrict__ keep, const uint8_t* __restrict__ kbits, float ks,
    float eps, __nv_bfloat16* __restrict__ ds_out, __nv_bfloat16* __restrict__ dh_out,
    float* __restrict__ part /*[3][grid][cols]*/, int rpc /* rows per CTA, <= 16 */,
    unsigned long long* trace /* debug timeline (tools/bdrln_trace.py), normally null */) {
  pdl_trigger();
  pdl_wait();
#define RTRACE(k)                                                                                  \
  do {                                                                                             \
    if (trace && threadIdx.x == 0) {                                                               \
      unsigned long long t_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
      trace[blockIdx.x * 8 + (k)] = t_;                                                            \
    }                                                                                              \
  } while (0)
  constexpr int V = 8;
  extern __shared__ float red[];  // [2][16][pst] staging planes, then gamma [cols]
  // plane position of column c: c + 2 * (c >> 5) (every 32-column group shifted
  // two floats further).  The writers (lane l holds columns 8l..8l+7 of a
  // 256-column chunk) then hit 16 distinct bank pairs per float2 store instead
  // of 4 (8-way conflicts), and the column-sum readers (consecutive threads,
  // consecutive columns) stay conflict-free.
  const int pst = cols + 2 * ((cols + 31) >> 5);
  auto ppos = [](int c) { return c + 2 * (c >> 5); };
  float* red2 = red + 16 * pst;
  float* gam = red2 + 16 * pst;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = cols / V;
  const float inv_n = 1.f / (float)cols;
  const int64_t row = (int64_t)blockIdx.x * rpc + warp;
  const bool valid = warp < rpc && row < rows;
  const size_t base = (size_t)(valid ? row : 0) * cols;
  uint4 sr[NCH], dr[NCH];
  uint32_t kb[NCH];  // the lane's 8 keep flags of each chunk as bits
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    const bool on = valid && vi < nvec;
    sr[c] = on ? *reinterpret_cast<const uint4*>(s + base + vi * V) : make_uint4(0, 0, 0, 0);
    dr[c] = on ? *reinterpret_cast<const uint4*>(dy + base + vi * V) : make_uint4(0, 0, 0, 0);
    if (on && keep) {  // 8 bytes of 0/1 -> 8 bits (byte k -> bit k, no carries)
      const uint2 k2 = *reinterpret_cast<const uint2*>(keep + base + vi * V);
      kb[c] = ((k2.x * 0x01020408u) >> 24) | (((k2.y * 0x01020408u) >> 24) << 4);
    } else if (on && kbits) {
      kb[c] = __ldg(kbits + ((base + vi * V) >> 3));
    } else {
      kb[c] = 0xFFu;
    }
  }
  // gamma -> smem once per CTA: the per-chunk reads below are then LDS, not
  // one dependent L2 round trip per chunk (1.5 us of the kernel, measured)
  for (int i = threadIdx.x * 4; i < cols; i += blockDim.x * 4)
    *reinterpret_cast<float4*>(gam + i) = __ldg(reinterpret_cast<const float4*>(gamma + i));
  __syncthreads();
  RTRACE(0);
  // mean, then variance (two passes over the registers)
  float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const uint32_t w[4] = {sr[c].x, sr[c].y, sr[c].z, sr[c].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) a2 = __fadd2_rn(a2, bf2(w[i]));
  }
  const float mu = warp_sum(a2.x + a2.y) * inv_n;
  RTRACE(1);
  const float2 nmu2 = make_float2(-mu, -mu);
  a2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (lane + c * 32 < nvec) {
      const uint32_t w[4] = {sr[c].x, sr[c].y, sr[c].z, sr[c].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 d = __fadd2_rn(bf2(w[i]), nmu2);
        a2 = __ffma2_rn(d, d, a2);
      }
    }
  }
  const float rstd = rsqrtf(warp_sum(a2.x + a2.y) * inv_n + eps);
  RTRACE(2);
  const float2 rstd2 = make_float2(rstd, rstd);
  // m1 = mean(dy*g), m2 = mean(dy*g*xhat)
  float2 m1a = make_float2(0.f, 0.f), m2a = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      const float4 g0 = reinterpret_cast<const float4*>(gam + vi * V)[0];
      const float4 g1 = reinterpret_cast<const float4*>(gam + vi * V)[1];
      const float2 gg[4] = {make_float2(g0.x, g0.y), make_float2(g0.z, g0.w), make_float2(g1.x, g1.y),
                            make_float2(g1.z, g1.w)};
      const uint32_t ws[4] = {sr[c].x, sr[c].y, sr[c].z, sr[c].w};
      const uint32_t wd[4] = {dr[c].x, dr[c].y, dr[c].z, dr[c].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 dyg = __fmul2_rn(bf2(wd[i]), gg[i]);
        const float2 xh = __fmul2_rn(__fadd2_rn(bf2(ws[i]), nmu2), rstd2);
        m1a = __fadd2_rn(m1a, dyg);
        m2a = __ffma2_rn(dyg, xh, m2a);
      }
    }
  }
  const float m1 = warp_sum(m1a.x + m1a.y) * inv_n, m2 = warp_sum(m2a.x + m2a.y) * inv_n;
  RTRACE(3);
  const float2 nm1v = make_float2(-m1, -m1), nm2v = make_float2(-m2, -m2);
  // ds = rstd * (dy*g - (xhat*m2 + m1)) and dh = ds * keep * ks -> HBM;
  // dh (the dbias contribution) and dy*xhat (dgamma) -> the two planes
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      const int col = vi * V;
      const float4 g0 = reinterpret_cast<const float4*>(gam + col)[0];
      const float4 g1 = reinterpret_cast<const float4*>(gam + col)[1];
      const float2 gg[4] = {make_float2(g0.x, g0.y), make_float2(g0.z, g0.w), make_float2(g1.x, g1.y),
                            make_float2(g1.z, g1.w)};
      const uint32_t ws[4] = {sr[c].x, sr[c].y, sr[c].z, sr[c].w};
      const uint32_t wd[4] = {dr[c].x, dr[c].y, dr[c].z, dr[c].w};
      uint32_t pds[4], pdh[4];
      float2* r1 = reinterpret_cast<float2*>(red + warp * pst + ppos(col));
      float2* r2 = reinterpret_cast<float2*>(red2 + warp * pst + ppos(col));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 y = bf2(wd[i]);
        const float2 dyg = __fmul2_rn(y, gg[i]);
        const float2 xh = __fmul2_rn(__fadd2_rn(bf2(ws[i]), nmu2), rstd2);
        const float2 ds = __fmul2_rn(__ffma2_rn(xh, nm2v, __fadd2_rn(dyg, nm1v)), rstd2);
        const float2 kf = make_float2((kb[c] >> (2 * i)) & 1u ? ks : 0.f, (kb[c] >> (2 * i + 1)) & 1u ? ks : 0.f);
        const float2 dh = __fmul2_rn(ds, kf);
        pds[i] = pk_bf2(ds);
        pdh[i] = pk_bf2(dh);
        // invalid rows (the grid's tail) stage zeros
        r1[i] = valid ? dh : make_float2(0.f, 0.f);
        r2[i] = valid ? __fmul2_rn(y, xh) : make_float2(0.f, 0.f);
      }
      if (valid) {
        if (ds_out) *reinterpret_cast<uint4*>(ds_out + base + col) = make_uint4(pds[0], pds[1], pds[2], pds[3]);
        if (dh_out) *reinterpret_cast<uint4*>(dh_out + base + col) = make_uint4(pdh[0], pdh[1], pdh[2], pdh[3]);
      }
    }
  }
  const int64_t nparts = gridDim.x;
  RTRACE(4);
  // column partials of the CTA's 16 rows, rows summed in fixed order:
  // dbias (plane 1) and dgamma (plane 2), then dbeta (dy, plane 1 again)
  __syncthreads();
  RTRACE(5);
  for (int col = threadIdx.x; col < cols; col += blockDim.x) {
    float th = 0.f, tg = 0.f;
#pragma unroll
    for (int w = 0; w < 16; ++w) {
      th += red[w * pst + ppos(col)];
      tg += red2[w * pst + ppos(col)];
    }
    part[((size_t)2 * nparts + blockIdx.x) * cols + col] = th;
    part[((size_t)0 * nparts + blockIdx.x) * cols + col] = tg;
  }
  RTRACE(6);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      const uint32_t wd[4] = {dr[c].x, dr[c].y, dr[c].z, dr[c].w};
      float2* r1 = reinterpret_cast<float2*>(red + warp * pst + ppos(vi * V));  // 8-byte aligned (skewed planes)
#pragma unroll
      for (int i = 0; i < 4; ++i) r1[i] = bf2(wd[i]);
    }
  }
  __syncthreads();
  for (int col = threadIdx.x; col < cols; col += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 16; ++w) t += red[w * pst + ppos(col)];
    part[((size_t)1 * nparts + blockIdx.x) * cols + col] = t;
  }
  RTRACE(7);
#undef RTRACE
}

// out_q[col] (+)= sum_b part[q][b][col] for q = blockIdx.y.  Warp w sums
// partial rows b = w, w+8, ... for 32 consecutive columns (coalesced), then
// the 8 warp sums are added in fixed order: deterministic.
constexpr int kFinWarps = 16;
__global__ void __launch_bounds__(kFinWarps * 32) finalize_colsum_kernel(int nparts, int cols,
                                                              const float* __restrict__ part,
                                                              float* out0, float* out1, float* out2,
                                                              int accumulate) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[kFinWarps][33];
  const int q = blockIdx.y;
  float* out = q == 0 ? out0 : (q == 1 ? out1 : out2);
  if (out == nullptr) return;
  const float* pq = part + (size_t)q * nparts * cols;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (col < cols) {
#pragma unroll 8
    for (int b = warp; b < nparts; b += kFinWarps) s += pq[(size_t)b * cols + col];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && col < cols) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kFinWarps; ++w) t += red[w][lane];
    out[col] = accumulate ? out[col] + t : t;
  }
}

// ---------------------------------------------------------------------------
// scaled + masked softmax + dropout

template <typename T, int V, int NCH>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(
    int64_t rows, int cols, int64_t rows_per_batch, const T* __restrict__ x, float inv_div,
    const float* __restrict__ am, const uint8_t* __restrict__ keep, float ks,
    T* __restrict__ p_out, T* __restrict__ pd_out) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarps + warp;
  if (row >= rows) return;
  const int nvec = cols / V;
  const size_t base = (size_t)row * cols;
  const float* amr = am ? am + (size_t)(row / rows_per_batch) * cols : nullptr;
  constexpr float kLog2e = 1.4426950408889634f;
  float z[NCH][V];
  float mx = -INFINITY;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      Vec<T, V> xv;
      xv.load(x + base + vi * V);
      float a[V];
      if (amr) { Vec<float, V> av; av.load(amr + vi * V);
#pragma unroll
        for (int i = 0; i < V; ++i) a[i] = av.v[i];
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) a[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < V; ++i) {
        z[c][i] = (xv.v[i] * inv_div + a[i]) * kLog2e;
        mx = fmaxf(mx, z[c][i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) z[c][i] = -INFINITY;
    }
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int i = 0; i < V; ++i) {
      z[c][i] = exp2f(z[c][i] - mx);
      sum += z[c][i];
    }
  const float inv = 1.f / warp_sum(sum);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      const int col = vi * V;
      Vec<T, V> pv;
#pragma unroll
      for (int i = 0; i < V; ++i) pv.v[i] = z[c][i] * inv;
      if (p_out) pv.store(p_out + base + col);
      if (pd_out) {
        float m[V];
        if (keep) load_keep<V>(keep + base + col, ks, m);
        else {
#pragma unroll
          for (int i = 0; i < V; ++i) m[i] = 1.f;
        }
        Vec<T, V> dv;
#pragma unroll
        for (int i = 0; i < V; ++i) dv.v[i] = pv.v[i] * m[i];
        dv.store(pd_out + base + col);
      }
    }
  }
}

template <typename T, int V, int NCH>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(
    int64_t rows, int cols, const T* __restrict__ dpd, const T* __restrict__ p,
    const uint8_t* __restrict__ keep, float ks, float inv_div, T* __restrict__ dx) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarps + warp;
  if (row >= rows) return;
  const int nvec = cols / V;
  const size_t base = (size_t)row * cols;
  float gv[NCH][V], pv[NCH][V];
  float dot = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      const int col = vi * V;
      Vec<T, V> a, b;
      a.load(dpd + base + col);
      b.load(p + base + col);
      float m[V];
      if (keep) load_keep<V>(keep + base + col, ks, m);
      else {
#pragma unroll
        for (int i = 0; i < V; ++i) m[i] = 1.f;
      }
#pragma unroll
      for (int i = 0; i < V; ++i) {
        gv[c][i] = a.v[i] * m[i];
        pv[c][i] = b.v[i];
        dot += gv[c][i] * pv[c][i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) { gv[c][i] = 0.f; pv[c][i] = 0.f; }
    }
  }
  dot = warp_sum(dot);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int vi = lane + c * 32;
    if (vi < nvec) {
      Vec<T, V> o;
#pragma unroll
      for (int i = 0; i < V; ++i) o.v[i] = (gv[c][i] - dot) * pv[c][i] * inv_div;
      o.store(dx + base + vi * V);
    }
  }
}

// ---------------------------------------------------------------------------
// bias + GELU (elementwise; one V-vector per thread, grid-stride)

template <typename T, int V>
__global__ void __launch_bounds__(256) bias_gelu_fwd_kernel(int64_t nvec, int cols,
                                                            const T* __restrict__ f,
                                                            const float* __restrict__ bias,
                                                            T* __restrict__ pre, T* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  for (int64_t vi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; vi < nvec;
       vi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = vi * V;
    const int col = (int)(e % cols);
    Vec<T, V> fv;
    fv.load(f + e);
    Vec<T, V> pv, yv;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float x = fv.v[i] + (bias ? bias[col + i] : 0.f);
      pv.v[i] = x;
      yv.v[i] = gelu_f(x);
    }
    if (pre) pv.store(pre + e);
    yv.store(y + e);
  }
}

template <typename T, int V>
__global__ void __launch_bounds__(256) gelu_bwd_kernel(int64_t nvec, const T* __restrict__ dy,
                                                       const T* __restrict__ pre,
                                                       T* __restrict__ dpre) {
  pdl_trigger();
  pdl_wait();
  for (int64_t vi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; vi < nvec;
       vi += (int64_t)gridDim.x * blockDim.x) {
    Vec<T, V> a, b, o;
    a.load(dy + vi * V);
    b.load(pre + vi * V);
#pragma unroll
    for (int i = 0; i < V; ++i) o.v[i] = a.v[i] * gelu_grad_f(b.v[i]);
    o.store(dpre + vi * V);
  }
}

// ---------------------------------------------------------------------------
// column sums: grid (col strips of 32*V, row groups); part[y][cols]

template <typename T, int V>
__global__ void __launch_bounds__(256) colsum_kernel(int64_t rows, int cols, int64_t ld,
                                                     const T* __restrict__ x,
                                                     float* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[kWarps][32 * V];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col0 = blockIdx.x * 32 * V + lane * V;
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;
  if (col0 < cols) {
    // four rows' loads in flight per warp (a lone load per iteration left the
    // kernel latency-bound at 2.4 TB/s); the sum order stays fixed
    const int64_t step = (int64_t)gridDim.y * kWarps;
    int64_t r = (int64_t)blockIdx.y * kWarps + warp;
    for (; r + 3 * step < rows; r += 4 * step) {
      Vec<T, V> v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u].load(x + (r + u * step) * ld + col0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += v[u].v[i];
    }
    for (; r < rows; r += step) {
      Vec<T, V> v;
      v.load(x + r * ld + col0);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += v.v[i];
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) red[warp][lane * V + i] = acc[i];
  __syncthreads();
  for (int j = threadIdx.x; j < 32 * V; j += blockDim.x) {
    const int col = blockIdx.x * 32 * V + j;
    if (col < cols) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += red[w][j];
      part[(size_t)blockIdx.y * cols + col] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// optimizer / casts

__global__ void sgd_kernel(int64_t n, float* __restrict__ w, const float* __restrict__ g, float lr,
                           __nv_bfloat16* __restrict__ wb) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = w[i] - lr * g[i];
    w[i] = v;
    if (wb) wb[i] = __float2bfloat16_rn(v);
  }
}

// 16-byte form (n4 float4 groups, 16-byte aligned w / g, 8-byte aligned wb):
// two groups per thread per iteration, so each thread keeps 64 bytes of loads
// in flight (the scalar form streamed at ~5.5 TB/s)
__global__ void sgd4_kernel(int64_t n4, float4* __restrict__ w, const float4* __restrict__ g, float lr,
                            uint2* __restrict__ wb) {
  pdl_trigger();
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float2 nl = make_float2(-lr, -lr);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 2 * stride) {
    const bool two = i + stride < n4;
    const float4 w0 = w[i], g0 = g[i];
    float4 w1 = make_float4(0.f, 0.f, 0.f, 0.f), g1 = w1;
    if (two) { w1 = w[i + stride]; g1 = g[i + stride]; }
    float4 v[2] = {w0, w1};
    const float4 gg[2] = {g0, g1};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float2 a = __ffma2_rn(make_float2(gg[u].x, gg[u].y), nl, make_float2(v[u].x, v[u].y));
      const float2 b = __ffma2_rn(make_float2(gg[u].z, gg[u].w), nl, make_float2(v[u].z, v[u].w));
      v[u] = make_float4(a.x, a.y, b.x, b.y);
    }
    w[i] = v[0];
    if (wb) {
      __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0].x, v[0].y), h1 = __floats2bfloat162_rn(v[0].z, v[0].w);
      wb[i] = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
    }
    if (two) {
      w[i + stride] = v[1];
      if (wb) {
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[1].x, v[1].y), h1 = __floats2bfloat162_rn(v[1].z, v[1].w);
        wb[i + stride] = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
      }
    }
  }
}

__global__ void scale_kernel(int64_t n, float* __restrict__ x, float s) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= s;
}

// two equal-length casts in one launch (the BN parameter gradients dbeta and
// dgamma of every normalisation layer: one tiny launch instead of two)
template <typename S, typename D>
__global__ void cast2_kernel(int64_t n, const S* __restrict__ s0, const S* __restrict__ s1, D* __restrict__ d0,
                             D* __restrict__ d1) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n)
      d0[i] = from_f<D>(to_f<S>(s0[i]));
    else
      d1[i - n] = from_f<D>(to_f<S>(s1[i - n]));
  }
}

template <typename S, typename D>
__global__ void cast_kernel(int64_t n, const S* __restrict__ s, D* __restrict__ d) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = from_f<D>(to_f<S>(s[i]));
}

// ---------------------------------------------------------------------------
// host dispatch helpers

inline int grid_for(int64_t n, int per_block, int cap) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// Row kernels are instantiated for NCH in this list (chunks of 32*V columns).
#define DFX_NCH_LIST(X) X(1) X(2) X(3) X(4) X(6) X(8) X(12) X(16)

inline int pick_nch(int nvec) {
  const int need = (nvec + 31) / 32;
  static const int opts[] = {1, 2, 3, 4, 6, 8, 12, 16};
  for (int o : opts)
    if (o >= need) return o;
  return -1;
}

template <typename T, int V> int check_row_shape(int64_t cols, const char* op) {
  if (cols <= 0 || cols % V != 0)
    return fail(DFX_ERR_SHAPE, std::string(op) + ": cols must be a positive multiple of " + std::to_string(V));
  if (pick_nch((int)(cols / V)) < 0)
    return fail(DFX_ERR_SHAPE, std::string(op) + ": cols too large (max " + std::to_string(16 * 32 * V) + ")");
  return DFX_OK;
}

size_t colsum_ws_bytes(int64_t rows, int64_t cols) {
  (void)rows;
  return (size_t)kMaxColBlocks * (size_t)cols * sizeof(float);
}

template <typename T, int V>
int bdrln_fwd_t(int64_t rows, int64_t cols, const void* h, const float* bias, const uint8_t* keep,
                const uint8_t* kbits, float ks, const void* res, const float* gamma, const float* beta, float eps, void* y,
                void* s_out, float* mean, float* rstd, cudaStream_t st, int act = 0) {
  if (int rc = check_row_shape<T, V>(cols, "dfx_bdrln_fwd")) return rc;
  const int nch = pick_nch((int)(cols / V));
  const int grid = grid_for(rows, kWarps, 4 * num_sms());
  if (rows == 0) return DFX_OK;
  if constexpr (sizeof(T) == 2) {
    // bf16, no activation, <= 768 columns with 16-byte aligned parameters: loads-first kernel
    const bool al = ((reinterpret_cast<uintptr_t>(gamma) | reinterpret_cast<uintptr_t>(beta) |
                      reinterpret_cast<uintptr_t>(bias)) & 15) == 0;
    if (!act && nch <= 3 && cols % 4 == 0 && al && (!keep || (reinterpret_cast<uintptr_t>(keep) & 7) == 0)) {
      const size_t sm = (size_t)3 * cols * sizeof(float);
#define LF(N)                                                                                      \
  if (nch == N)                                                                                    \
    launch_k(bdrln_fwd_bf16_kernel<N>, grid_for(rows, kFwdWarps, 4 * num_sms()), kFwdWarps * 32, sm, st, rows, (int)cols, (const __nv_bfloat16*)h, bias, keep, \
             kbits, ks, (const __nv_bfloat16*)res, gamma, beta, eps, (__nv_bfloat16*)y, (__nv_bfloat16*)s_out, mean, rstd);
      LF(1) LF(2) LF(3)
#undef LF
      DFX_LAUNCH_CHECK("dfx_bdrln_fwd");
      return DFX_OK;
    }
  }
#define L(N)                                                                                        \
  if (nch == N) {                                                                                   \
    if (act)                                                                                        \
      launch_k(bdrln_fwd_kernel<T, V, N, 1>, grid, 256, 0, st, rows, (int)cols, (const T*)h, bias, keep, kbits, ks, \
                                                         (const T*)res, gamma, beta, eps, (T*)y,    \
                                                         (T*)s_out, mean, rstd);                   \
    else                                                                                            \
      launch_k(bdrln_fwd_kernel<T, V, N, 0>, grid, 256, 0, st, rows, (int)cols, (const T*)h, bias, keep, kbits, ks, \
                                                         (const T*)res, gamma, beta, eps, (T*)y,    \
                                                         (T*)s_out, mean, rstd);                   \
  }
  DFX_NCH_LIST(L)
#undef L
  DFX_LAUNCH_CHECK("dfx_bdrln_fwd");
  return DFX_OK;
}

template <typename T, int V, int ACT>
int bdrln_bwd_launch(int nch, int grid, size_t smem, int64_t rows, int64_t cols, const void* dy, const void* s,
                     const float* gamma, const float* beta, const uint8_t* keep, const uint8_t* kbits, float ks,
                     float eps, void* ds, void* dh, float* pg, float* pb, float* ph, cudaStream_t st) {
#define L(N)                                                                                       \
  if (nch == N) {                                                                                  \
    auto kfn = bdrln_bwd_kernel<T, V, N, ACT>;                                                     \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    launch_k(kfn, grid, 256, smem, st, rows, (int)cols, (const T*)dy, (const T*)s, gamma, beta, keep, kbits, ks, eps, \
                                 (T*)ds, (T*)dh, pg, pb, ph);                                      \
  }
  DFX_NCH_LIST(L)
#undef L
  DFX_LAUNCH_CHECK("dfx_bdrln_bwd");
  return DFX_OK;
}

// partial-set count of the backward (the finalize must use the same one)
// rows per CTA of the one-wave backward: two CTAs on every SM with an even
// share of the rows (<= 16, one per warp), so no SM runs a second CTA while
// others idle (256 CTAs of 16 rows left 40 SMs with one CTA at C2)
inline int bdrln_wave_rpc(int64_t rows) {
  const int64_t slots = std::min<int64_t>(2 * (int64_t)num_sms(), kMaxColBlocks);  // <= the workspace's partial sets
  return (int)std::min<int64_t>(16, std::max<int64_t>(1, (rows + slots - 1) / slots));
}

template <typename T, int V> int bdrln_bwd_grid(int64_t rows, int64_t cols, int act) {
  const int nch = pick_nch((int)(cols / V));
  const bool wave = sizeof(T) == 2 && act == 0 && rows <= 16 * (int64_t)kMaxColBlocks && nch <= 3;
  if (!wave) return grid_for(rows, kWarps, kMaxColBlocks);
  const int rpc = bdrln_wave_rpc(rows);
  return (int)((rows + rpc - 1) / rpc);
}

template <typename T, int V>
int bdrln_bwd_t(int64_t rows, int64_t cols, const void* dy, const void* s, const float* gamma,
                const uint8_t* keep, const uint8_t* kbits, float ks, float eps, void* ds, void* dh, float* dgamma,
                float* dbeta, float* dbias, void* ws, size_t ws_bytes, cudaStream_t st, int act = 0,
                const float* beta = nullptr) {
  if (int rc = check_row_shape<T, V>(cols, "dfx_bdrln_bwd")) return rc;
  if (rows == 0) return DFX_OK;
  const int nch = pick_nch((int)(cols / V));
  const bool wave = sizeof(T) == 2 && act == 0 && rows <= 16 * (int64_t)kMaxColBlocks && nch <= 3;
  const int grid = bdrln_bwd_grid<T, V>(rows, cols, act);
  const size_t need = 3 * (size_t)grid * cols * sizeof(float);
  DFX_REQUIRE(ws_bytes >= need, DFX_ERR_WORKSPACE, "dfx_bdrln_bwd: workspace too small");
  float* pg = (float*)ws;
  float* pb = pg + (size_t)grid * cols;
  float* ph = pb + (size_t)grid * cols;
  int rc;
  if (wave) {
    const size_t wsm = ((size_t)2 * 16 * (cols + 2 * ((cols + 31) / 32)) + cols) * sizeof(float);  // planes + gamma
#define LW(N)                                                                                      \
  if (nch == N) {                                                                                  \
    auto kfn = bdrln_bwd_wave_kernel<N>;                                                           \
    if (wsm > 48 * 1024) cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm); \
    launch_k(kfn, grid, 512, wsm, st, rows, (int)cols, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)s, gamma, keep, kbits, \
                                ks, eps, (__nv_bfloat16*)ds, (__nv_bfloat16*)dh, pg, bdrln_wave_rpc(rows), g_row_trace); \
  }
    LW(1) LW(2) LW(3)
#undef LW
    DFX_LAUNCH_CHECK("dfx_bdrln_bwd");
    if (dgamma || dbeta || dbias) {
      launch_k(finalize_colsum_kernel, dim3((unsigned)((cols + 31) / 32), 3), kFinWarps * 32, 0, st, grid, (int)cols, pg,
                                                                                      dgamma, dbeta, dbias, 0);
      DFX_LAUNCH_CHECK("dfx_bdrln_bwd finalize");
    }
    return DFX_OK;
  }
  const size_t smem = (size_t)kWarps * (cols + (cols + 31) / 32) * sizeof(float);  // skewed staging (block_colsum_store)
  rc = act ? bdrln_bwd_launch<T, V, 1>(nch, grid, smem, rows, cols, dy, s, gamma, beta, keep, kbits, ks, eps, ds, dh,
                                        pg, pb, ph, st)
               : bdrln_bwd_launch<T, V, 0>(nch, grid, smem, rows, cols, dy, s, gamma, beta, keep, kbits, ks, eps, ds, dh,
                                        pg, pb, ph, st);
  if (rc) return rc;
  if (dgamma || dbeta || dbias) {
    launch_k(finalize_colsum_kernel, dim3((unsigned)((cols + 31) / 32), 3), kFinWarps * 32, 0, st, grid, (int)cols, pg, dgamma,
                                                                               dbeta, dbias, 0);
    DFX_LAUNCH_CHECK("dfx_bdrln_bwd finalize");
  }
  return DFX_OK;
}

template <typename T, int V>
int softmax_fwd_t(int64_t batch, int64_t heads, int64_t q, int64_t cols, const void* x, float inv_div,
                  const float* am, const uint8_t* keep, float ks, void* p, void* pd, cudaStream_t st) {
  if (int rc = check_row_shape<T, V>(cols, "dfx_softmax_fwd")) return rc;
  const int64_t rows = batch * heads * q;
  if (rows == 0) return DFX_OK;
  const int nch = pick_nch((int)(cols / V));
  const int64_t grid = (rows + kWarps - 1) / kWarps;
#define L(N)                                                                                    \
  if (nch == N)                                                                                 \
    launch_k(softmax_fwd_kernel<T, V, N>, (unsigned)grid, 256, 0, st, rows, (int)cols, heads * q,     \
                                                                (const T*)x, inv_div, am, keep, \
                                                                ks, (T*)p, (T*)pd);
  DFX_NCH_LIST(L)
#undef L
  DFX_LAUNCH_CHECK("dfx_softmax_fwd");
  return DFX_OK;
}

template <typename T, int V>
int softmax_bwd_t(int64_t rows, int64_t cols, const void* dpd, const void* p, const uint8_t* keep,
                  float ks, float inv_div, void* dx, cudaStream_t st) {
  if (int rc = check_row_shape<T, V>(cols, "dfx_softmax_bwd")) return rc;
  if (rows == 0) return DFX_OK;
  const int nch = pick_nch((int)(cols / V));
  const int64_t grid = (rows + kWarps - 1) / kWarps;
#define L(N)                                                                                     \
  if (nch == N)                                                                                  \
    launch_k(softmax_bwd_kernel<T, V, N>, (unsigned)grid, 256, 0, st, rows, (int)cols, (const T*)dpd,  \
                                                                (const T*)p, keep, ks, inv_div,  \
                                                                (T*)dx);
  DFX_NCH_LIST(L)
#undef L
  DFX_LAUNCH_CHECK("dfx_softmax_bwd");
  return DFX_OK;
}

// Width dispatch: 128-bit vectors when cols is a multiple of the vector width,
// scalar lanes otherwise (the reference accepts any extent).
#define DFX_VDISPATCH(FN)                                                              \
  template <typename T, typename... A> int FN##_any(int64_t cols, A... a) {             \
    if (cols % VecWidth<T>::value == 0) return FN<T, VecWidth<T>::value>(a...);        \
    return FN<T, 1>(a...);                                                              \
  }
DFX_VDISPATCH(bdrln_fwd_t)
DFX_VDISPATCH(bdrln_bwd_t)
DFX_VDISPATCH(softmax_fwd_t)
DFX_VDISPATCH(softmax_bwd_t)

template <typename T>
int colsum_t(int64_t rows, int64_t cols, const void* x, int64_t ld, float* out, int accumulate,
             void* ws, size_t ws_bytes, cudaStream_t st) {
  constexpr int V = VecWidth<T>::value;
  DFX_REQUIRE(cols > 0 && cols % V == 0 && ld % V == 0, DFX_ERR_SHAPE,
              "dfx_colsum: cols and ld must be multiples of the vector width");
  DFX_REQUIRE(aligned16(x), DFX_ERR_ALIGN, "dfx_colsum: x must be 16-byte aligned");
  const int gx = (int)((cols + 32 * V - 1) / (32 * V));
  int gy = (int)std::max<int64_t>(1, std::min<int64_t>((rows + kWarps - 1) / kWarps, kMaxColBlocks / gx));
  DFX_REQUIRE(ws_bytes >= (size_t)gy * cols * sizeof(float), DFX_ERR_WORKSPACE,
              "dfx_colsum: workspace too small");
  launch_k(colsum_kernel<T, V>, dim3(gx, gy), 256, 0, st, rows, (int)cols, ld, (const T*)x, (float*)ws);
  DFX_LAUNCH_CHECK("dfx_colsum");
  launch_k(finalize_colsum_kernel, dim3((unsigned)((cols + 31) / 32), 1), kFinWarps * 32, 0, st, gy, (int)cols, (const float*)ws, out,
                                                                              nullptr, nullptr, accumulate);
  DFX_LAUNCH_CHECK("dfx_colsum finalize");
  return DFX_OK;
}

}  // namespace
}  // namespace dfx

using namespace dfx;

extern "C" {

static int bdrln_fwd_entry(int dtype, int64_t rows, int64_t cols, const void* h, const float* bias,
                           const uint8_t* keep, const uint8_t* kbits, float keep_scale, const void* residual,
                           const float* gamma, const float* beta, float eps, void* y, void* s_stash, float* mean,
                           float* rstd, void* stream) {
  DFX_REQUIRE(h && gamma && beta && y, DFX_ERR_SHAPE, "dfx_bdrln_fwd: null required pointer");
  if (dtype == DFX_BF16)
    return bdrln_fwd_t_any<__nv_bfloat16>(cols, rows, cols, h, bias, keep, kbits, keep_scale, residual, gamma, beta,
                                      eps, y, s_stash, mean, rstd, as_stream(stream));
  if (dtype == DFX_F32)
    return bdrln_fwd_t_any<float>(cols, rows, cols, h, bias, keep, kbits, keep_scale, residual, gamma, beta, eps, y,
                              s_stash, mean, rstd, as_stream(stream));
  return fail(DFX_ERR_DTYPE, "dfx_bdrln_fwd: dtype must be f32 or bf16");
}

int dfx_bdrln_fwd(int dtype, int64_t rows, int64_t cols, const void* h, const float* bias,
                  const uint8_t* keep, float keep_scale, const void* residual, const float* gamma,
                  const float* beta, float eps, void* y, void* s_stash, float* mean, float* rstd,
                  void* stream) {
  return bdrln_fwd_entry(dtype, rows, cols, h, bias, keep, nullptr, keep_scale, residual, gamma, beta, eps, y,
                         s_stash, mean, rstd, stream);
}

int dfx_bdrln_fwd_kb(int dtype, int64_t rows, int64_t cols, const void* h, const float* bias,
                     const uint32_t* keep_bits, float keep_scale, const void* residual, const float* gamma,
                     const float* beta, float eps, void* y, void* s_stash, float* mean, float* rstd,
                     void* stream) {
  DFX_REQUIRE(keep_bits && (rows * cols) % 32 == 0, DFX_ERR_SHAPE,
              "dfx_bdrln_fwd_kb: keep_bits required and rows*cols must be a multiple of 32");
  return bdrln_fwd_entry(dtype, rows, cols, h, bias, nullptr, reinterpret_cast<const uint8_t*>(keep_bits), keep_scale,
                         residual, gamma, beta, eps, y, s_stash, mean, rstd, stream);
}

size_t dfx_bdrln_bwd_workspace(int64_t rows, int64_t cols) {
  return 3 * colsum_ws_bytes(rows, cols);
}

int dfx_bdrln_bwd_finalize(int dtype, int64_t rows, int64_t cols, const void* workspace, size_t ws_bytes,
                           float* dgamma, float* dbeta, float* dbias, void* stream) {
  DFX_REQUIRE(workspace && rows > 0 && cols > 0, DFX_ERR_SHAPE, "dfx_bdrln_bwd_finalize: bad arguments");
  int grid;
  if (dtype == DFX_BF16) grid = bdrln_bwd_grid<__nv_bfloat16, 8>(rows, cols, 0);
  else if (dtype == DFX_F32) grid = bdrln_bwd_grid<float, 4>(rows, cols, 0);
  else return fail(DFX_ERR_DTYPE, "dfx_bdrln_bwd_finalize: dtype must be f32 or bf16");
  DFX_REQUIRE(ws_bytes >= 3 * (size_t)grid * cols * sizeof(float), DFX_ERR_WORKSPACE,
              "dfx_bdrln_bwd_finalize: workspace too small");
  if (!(dgamma || dbeta || dbias)) return DFX_OK;
  launch_k(finalize_colsum_kernel, dim3((unsigned)((cols + 31) / 32), 3), kFinWarps * 32, 0, as_stream(stream), grid,
           (int)cols, (const float*)workspace, dgamma, dbeta, dbias, 0);
  DFX_LAUNCH_CHECK("dfx_bdrln_bwd_finalize");
  return DFX_OK;
}

static int bdrln_bwd_entry(int dtype, int64_t rows, int64_t cols, const void* dy, const void* s_stash,
                           const float* gamma, const uint8_t* keep, const uint8_t* kbits, float keep_scale, float eps,
                           void* ds, void* dh, float* dgamma, float* dbeta, float* dbias, void* workspace,
                           size_t ws_bytes, void* stream) {
  DFX_REQUIRE(dy && s_stash && gamma, DFX_ERR_SHAPE, "dfx_bdrln_bwd: null required pointer");
  if (dtype == DFX_BF16)
    return bdrln_bwd_t_any<__nv_bfloat16>(cols, rows, cols, dy, s_stash, gamma, keep, kbits, keep_scale, eps, ds, dh,
                                      dgamma, dbeta, dbias, workspace, ws_bytes, as_stream(stream));
  if (dtype == DFX_F32)
    return bdrln_bwd_t_any<float>(cols, rows, cols, dy, s_stash, gamma, keep, kbits, keep_scale, eps, ds, dh, dgamma,
                              dbeta, dbias, workspace, ws_bytes, as_stream(stream));
  return fail(DFX_ERR_DTYPE, "dfx_bdrln_bwd: dtype must be f32 or bf16");
}

int dfx_bdrln_bwd(int dtype, int64_t rows, int64_t cols, const void* dy, const void* s_stash,
                  const float* gamma, const uint8_t* keep, float keep_scale, float eps, void* ds,
                  void* dh, float* dgamma, float* dbeta, float* dbias, void* workspace,
                  size_t ws_bytes, void* stream) {
  return bdrln_bwd_entry(dtype, rows, cols, dy, s_stash, gamma, keep, nullptr, keep_scale, eps, ds, dh, dgamma, dbeta,
                         dbias, workspace, ws_bytes, stream);
}

int dfx_bdrln_bwd_kb(int dtype, int64_t rows, int64_t cols, const void* dy, const void* s_stash,
                     const float* gamma, const uint32_t* keep_bits, float keep_scale, float eps, void* ds,
                     void* dh, float* dgamma, float* dbeta, float* dbias, void* workspace,
                     size_t ws_bytes, void* stream) {
  DFX_REQUIRE(keep_bits && (rows * cols) % 32 == 0, DFX_ERR_SHAPE,
              "dfx_bdrln_bwd_kb: keep_bits required and rows*cols must be a multiple of 32");
  return bdrln_bwd_entry(dtype, rows, cols, dy, s_stash, gamma, nullptr, reinterpret_cast<const uint8_t*>(keep_bits),
                         keep_scale, eps, ds, dh, dgamma, dbeta, dbias, workspace, ws_bytes, stream);
}

int dfx_softmax_fwd(int dtype, int64_t batch, int64_t heads, int64_t q, int64_t cols,
                    const void* scores, float inv_divisor, const float* add_mask,
                    const uint8_t* keep, float keep_scale, void* p, void* pd, void* stream) {
  DFX_REQUIRE(scores && (p || pd), DFX_ERR_SHAPE, "dfx_softmax_fwd: null required pointer");
  if (dtype == DFX_BF16)
    return softmax_fwd_t_any<__nv_bfloat16>(cols, batch, heads, q, cols, scores, inv_divisor, add_mask, keep,
                                        keep_scale, p, pd, as_stream(stream));
  if (dtype == DFX_F32)
    return softmax_fwd_t_any<float>(cols, batch, heads, q, cols, scores, inv_divisor, add_mask, keep,
                                keep_scale, p, pd, as_stream(stream));
  return fail(DFX_ERR_DTYPE, "dfx_softmax_fwd: dtype must be f32 or bf16");
}

int dfx_softmax_bwd(int dtype, int64_t rows, int64_t cols, const void* dpd, const void* p,
                    const uint8_t* keep, float keep_scale, float inv_divisor, void* dscores,
                    void* stream) {
  DFX_REQUIRE(dpd && p && dscores, DFX_ERR_SHAPE, "dfx_softmax_bwd: null required pointer");
  if (dtype == DFX_BF16)
    return softmax_bwd_t_any<__nv_bfloat16>(cols, rows, cols, dpd, p, keep, keep_scale, inv_divisor, dscores,
                                        as_stream(stream));
  if (dtype == DFX_F32)
    return softmax_bwd_t_any<float>(cols, rows, cols, dpd, p, keep, keep_scale, inv_divisor, dscores,
                                as_stream(stream));
  return fail(DFX_ERR_DTYPE, "dfx_softmax_bwd: dtype must be f32 or bf16");
}

int dfx_bias_gelu_fwd(int dtype, int64_t rows, int64_t cols, const void* f, const float* bias,
                      void* pre, void* y, void* stream) {
  DFX_REQUIRE(f && y, DFX_ERR_SHAPE, "dfx_bias_gelu_fwd: null required pointer");
  const int V = dtype == DFX_BF16 ? 8 : 4;
  DFX_REQUIRE(cols > 0 && cols % V == 0, DFX_ERR_SHAPE, "dfx_bias_gelu_fwd: cols must be a multiple of the vector width");
  const int64_t nvec = rows * cols / V;
  if (nvec == 0) return DFX_OK;
  const int grid = grid_for(nvec, 256, 148 * 16);
  cudaStream_t st = as_stream(stream);
  if (dtype == DFX_BF16)
    launch_k(bias_gelu_fwd_kernel<__nv_bfloat16, 8>, grid, 256, 0, st, nvec, (int)cols, (const __nv_bfloat16*)f, bias, (__nv_bfloat16*)pre, (__nv_bfloat16*)y);
  else if (dtype == DFX_F32)
    launch_k(bias_gelu_fwd_kernel<float, 4>, grid, 256, 0, st, nvec, (int)cols, (const float*)f, bias, (float*)pre, (float*)y);
  else
    return fail(DFX_ERR_DTYPE, "dfx_bias_gelu_fwd: dtype must be f32 or bf16");
  DFX_LAUNCH_CHECK("dfx_bias_gelu_fwd");
  return DFX_OK;
}

int dfx_bias_gelu_bwd(int dtype, int64_t rows, int64_t cols, const void* dy, const void* pre,
                      void* dpre, float* dbias, void* workspace, size_t ws_bytes, void* stream) {
  DFX_REQUIRE(dy && pre && dpre, DFX_ERR_SHAPE, "dfx_bias_gelu_bwd: null required pointer");
  const int V = dtype == DFX_BF16 ? 8 : 4;
  DFX_REQUIRE(cols > 0 && cols % V == 0, DFX_ERR_SHAPE, "dfx_bias_gelu_bwd: cols must be a multiple of the vector width");
  const int64_t nvec = rows * cols / V;
  if (nvec == 0) return DFX_OK;
  const int grid = grid_for(nvec, 256, 148 * 16);
  cudaStream_t st = as_stream(stream);
  if (dtype == DFX_BF16)
    launch_k(gelu_bwd_kernel<__nv_bfloat16, 8>, grid, 256, 0, st, nvec, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)pre, (__nv_bfloat16*)dpre);
  else if (dtype == DFX_F32)
    launch_k(gelu_bwd_kernel<float, 4>, grid, 256, 0, st, nvec, (const float*)dy, (const float*)pre, (float*)dpre);
  else
    return fail(DFX_ERR_DTYPE, "dfx_bias_gelu_bwd: dtype must be f32 or bf16");
  DFX_LAUNCH_CHECK("dfx_bias_gelu_bwd");
  if (dbias) return dfx_colsum(dtype, rows, cols, dpre, cols, dbias, 0, workspace, ws_bytes, stream);
  return DFX_OK;
}

size_t dfx_colsum_workspace(int64_t rows, int64_t cols) { return colsum_ws_bytes(rows, cols); }

int dfx_colsum(int dtype, int64_t rows, int64_t cols, const void* x, int64_t ld, float* out,
               int accumulate, void* workspace, size_t ws_bytes, void* stream) {
  DFX_REQUIRE(x && out, DFX_ERR_SHAPE, "dfx_colsum: null pointer");
  if (dtype == DFX_BF16)
    return colsum_t<__nv_bfloat16>(rows, cols, x, ld, out, accumulate, workspace, ws_bytes, as_stream(stream));
  if (dtype == DFX_F32)
    return colsum_t<float>(rows, cols, x, ld, out, accumulate, workspace, ws_bytes, as_stream(stream));
  return fail(DFX_ERR_DTYPE, "dfx_colsum: dtype must be f32 or bf16");
}

int dfx_layernorm_act_fwd(int dtype, int64_t rows, int64_t cols, const void* x, const float* gamma,
                          const float* beta, float eps, int act, void* y, void* stream) {
  DFX_REQUIRE(x && gamma && beta && y, DFX_ERR_SHAPE, "dfx_layernorm_act_fwd: null pointer");
  DFX_REQUIRE(act == 0 || act == 1, DFX_ERR_UNSUPPORTED, "dfx_layernorm_act_fwd: act must be 0 (none) or 1 (swish)");
  if ((dtype == DFX_BF16 || dtype == DFX_F32) && ln_small_ok(dtype, cols))  // C4's short rows
    return ln_small_fwd(dtype, rows, cols, x, gamma, beta, eps, act, y, as_stream(stream));
  if (dtype == DFX_BF16)
    return bdrln_fwd_t_any<__nv_bfloat16>(cols, rows, cols, x, nullptr, nullptr, nullptr, 1.f, nullptr, gamma, beta, eps, y, nullptr,
                                      nullptr, nullptr, as_stream(stream), act);
  if (dtype == DFX_F32)
    return bdrln_fwd_t_any<float>(cols, rows, cols, x, nullptr, nullptr, nullptr, 1.f, nullptr, gamma, beta, eps, y, nullptr, nullptr,
                              nullptr, as_stream(stream), act);
  return fail(DFX_ERR_DTYPE, "dfx_layernorm_act_fwd: dtype must be f32 or bf16");
}

int dfx_layernorm_act_bwd(int dtype, int64_t rows, int64_t cols, const void* dy, const void* x,
                          const float* gamma, const float* beta, float eps, int act, void* dx, float* dgamma,
                          float* dbeta, void* workspace, size_t ws_bytes, void* stream) {
  DFX_REQUIRE(dy && x && gamma && beta && dx, DFX_ERR_SHAPE, "dfx_layernorm_act_bwd: null pointer");
  DFX_REQUIRE(act == 0 || act == 1, DFX_ERR_UNSUPPORTED, "dfx_layernorm_act_bwd: act must be 0 (none) or 1 (swish)");
  if ((dtype == DFX_BF16 || dtype == DFX_F32) && ln_small_ok(dtype, cols)) {
    DFX_REQUIRE(dgamma && dbeta && workspace, DFX_ERR_SHAPE, "dfx_layernorm_act_bwd: dgamma/dbeta/workspace required");
    return ln_small_bwd(dtype, rows, cols, dy, x, gamma, beta, eps, act, dx, dgamma, dbeta, workspace, ws_bytes,
                        as_stream(stream));
  }
  if (dtype == DFX_BF16)
    return bdrln_bwd_t_any<__nv_bfloat16>(cols, rows, cols, dy, x, gamma, nullptr, nullptr, 1.f, eps, dx, nullptr, dgamma, dbeta, nullptr,
                                      workspace, ws_bytes, as_stream(stream), act, beta);
  if (dtype == DFX_F32)
    return bdrln_bwd_t_any<float>(cols, rows, cols, dy, x, gamma, nullptr, nullptr, 1.f, eps, dx, nullptr, dgamma, dbeta, nullptr,
                              workspace, ws_bytes, as_stream(stream), act, beta);
  return fail(DFX_ERR_DTYPE, "dfx_layernorm_act_bwd: dtype must be f32 or bf16");
}

int dfx_sgd_update(int64_t n, float* master, const float* grad, float lr, void* weights_bf16,
                   void* stream) {
  DFX_REQUIRE(master && grad, DFX_ERR_SHAPE, "dfx_sgd_update: null pointer");
  if (n == 0) return DFX_OK;
  if (n % 4 == 0 && aligned16(master) && aligned16(grad) && (reinterpret_cast<uintptr_t>(weights_bf16) & 7) == 0) {
    const int64_t n4 = n / 4;
    launch_k(sgd4_kernel, grid_for((n4 + 1) / 2, 256, 148 * 8), 256, 0, as_stream(stream), n4,
             reinterpret_cast<float4*>(master), reinterpret_cast<const float4*>(grad), lr,
             reinterpret_cast<uint2*>(weights_bf16));
  } else {
    launch_k(sgd_kernel, grid_for(n, 256, 148 * 8), 256, 0, as_stream(stream), n, master, grad, lr,
             (__nv_bfloat16*)weights_bf16);
  }
  DFX_LAUNCH_CHECK("dfx_sgd_update");
  return DFX_OK;
}

int dfx_scale_f32(int64_t n, float* x, float scale, void* stream) {
  if (n == 0) return DFX_OK;
  launch_k(scale_kernel, grid_for(n, 256, 148 * 8), 256, 0, as_stream(stream), n, x, scale);
  DFX_LAUNCH_CHECK("dfx_scale_f32");
  return DFX_OK;
}

int dfx_cast(int64_t n, int sd, const void* src, int dd, void* dst, void* stream) {
  if (n == 0) return DFX_OK;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(n, 256, 148 * 8);
  if (sd == DFX_F32 && dd == DFX_BF16) launch_k(cast_kernel<float, __nv_bfloat16>, g, 256, 0, st, n, (const float*)src, (__nv_bfloat16*)dst);
  else if (sd == DFX_BF16 && dd == DFX_F32) launch_k(cast_kernel<__nv_bfloat16, float>, g, 256, 0, st, n, (const __nv_bfloat16*)src, (float*)dst);
  else if (sd == DFX_F32 && dd == DFX_F32) launch_k(cast_kernel<float, float>, g, 256, 0, st, n, (const float*)src, (float*)dst);
  else return fail(DFX_ERR_DTYPE, "dfx_cast: unsupported dtype pair");
  DFX_LAUNCH_CHECK("dfx_cast");
  return DFX_OK;
}

int dfx_cast2(int64_t n, int sd, const void* src0, const void* src1, int dd, void* dst0, void* dst1, void* stream) {
  if (n == 0) return DFX_OK;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(2 * n, 256, 148 * 8);
  if (sd == DFX_F32 && dd == DFX_F32)
    launch_k(cast2_kernel<float, float>, g, 256, 0, st, n, (const float*)src0, (const float*)src1, (float*)dst0,
             (float*)dst1);
  else if (sd == DFX_F32 && dd == DFX_BF16)
    launch_k(cast2_kernel<float, __nv_bfloat16>, g, 256, 0, st, n, (const float*)src0, (const float*)src1,
             (__nv_bfloat16*)dst0, (__nv_bfloat16*)dst1);
  else if (sd == DFX_BF16 && dd == DFX_F32)
    launch_k(cast2_kernel<__nv_bfloat16, float>, g, 256, 0, st, n, (const __nv_bfloat16*)src0,
             (const __nv_bfloat16*)src1, (float*)dst0, (float*)dst1);
  else
    return fail(DFX_ERR_DTYPE, "dfx_cast2: unsupported dtype pair");
  DFX_LAUNCH_CHECK("dfx_cast2");
  return DFX_OK;
}

}  // extern "C"

extern "C" __attribute__((visibility("default"))) void dfx_debug_bdrln_trace(void* buf) {
  dfx::g_row_trace = reinterpret_cast<unsigned long long*>(buf);
}
