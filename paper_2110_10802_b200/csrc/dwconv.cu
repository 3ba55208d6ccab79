// dwconv.cu — depthwise KSxKS convolution (stride 1/2), NHWC, sm_100a:
// TMA row ring + register sliding window.
//
// The reference evaluates Conv(group=C) as a 9-tap loop nest with clamped
// reads and ge() padding masks (lowering.py:930-1004; reference semantics
// frontend.py:645-666) and differentiates it through the lowered nest
// (autodiff.py:1623-1629, 1701-1745).  Here one CTA owns (image n, a band of
// R output rows, a tile of Wt output columns, a chunk of Cb channels):
//
//   * a single producer thread streams the band's input rows, each a
//     [Wb = (Wt-1)*s + KS columns][Cb channels] box, into a K-slot shared
//     memory ring with cp.async.bulk.tensor (TMA) + mbarrier tx-counts.  TMA
//     zero-fills everything outside the tensor, so the conv padding costs no
//     predicates and no extra bytes; K = KS + 2s slots keep two output rows of
//     loads in flight per CTA (two CTAs per SM);
//   * threads = (V-channel vector, column segment): each walks its segment of
//     output columns left to right holding a KS x KS window of input vectors in
//     registers, so an output costs KS*s new shared-memory vectors, not KS^2;
//   * outputs go straight from registers to HBM (V-channel vectors, every
//     warp store covers whole pixels).
//
// Three modes share the loop:
//   CONV_STATS (forward): z = conv(x, w), plus the per-CTA BatchNorm partial
//       Welford sets of the unrounded z (frontend.py:558-591), merged in a
//       fixed order (no atomics: bitwise reproducible);
//   DZW (backward): dz = dBN(dswish(dy*s + dpool)) from (dy, z) rows streamed
//       by TMA next to the x ring (the BN VJP autodiff.py:1557-1617 in closed
//       form), dz stored for the dx pass, and dw[t] += window(x)[t] * dz with
//       the UNROUNDED f32 dz — a bf16-rounded dz would break the BN-VJP
//       orthogonality (sum dz = sum dz*z = 0) that dw cancels against;
//   CONV (backward, stride 1): dx = conv(dz, flipped w) with the transposed
//       padding (KS-1-pt, KS-1-pl).  Stride 2 uses a direct gather kernel.
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "dwconv.h"
#include "gemm.h"
#include "tc_ptx.cuh"

namespace dfx {
namespace {

template <int... Is, typename F>
__device__ __forceinline__ void unroll_impl(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}
// f(integral_constant<int, 0..N-1>): compile-time loop index
template <int N, typename F> __device__ __forceinline__ void unroll_for(F&& f) {
  unroll_impl(std::make_integer_sequence<int, N>{}, f);
}

enum { MODE_CONV = 0, MODE_STATS = 1, MODE_DZW = 2 };
constexpr int kMaxThreads = 256;
constexpr size_t kSmemBudget = 110 * 1024;  // two CTAs per SM

template <int KS> struct VecOf { static constexpr int value = KS == 3 ? 4 : 2; };

// V channels of T, raw in registers (bf16 unpacked on use)
template <typename T, int V> struct RV;
template <> struct RV<__nv_bfloat16, 4> {
  uint2 r;
  __device__ __forceinline__ void ld(const __nv_bfloat16* p) { r = *reinterpret_cast<const uint2*>(p); }
  __device__ __forceinline__ void ldg(const __nv_bfloat16* p) { r = __ldg(reinterpret_cast<const uint2*>(p)); }
  __device__ __forceinline__ float get(int i) const {
    const uint32_t w = i < 2 ? r.x : r.y;
    return __uint_as_float((i & 1) ? (w & 0xFFFF0000u) : (w << 16));
  }
};
template <> struct RV<__nv_bfloat16, 2> {
  uint32_t r;
  __device__ __forceinline__ void ld(const __nv_bfloat16* p) { r = *reinterpret_cast<const uint32_t*>(p); }
  __device__ __forceinline__ void ldg(const __nv_bfloat16* p) { r = __ldg(reinterpret_cast<const unsigned int*>(p)); }
  __device__ __forceinline__ float get(int i) const { return __uint_as_float(i ? (r & 0xFFFF0000u) : (r << 16)); }
};
template <> struct RV<float, 4> {
  float4 r;
  __device__ __forceinline__ void ld(const float* p) { r = *reinterpret_cast<const float4*>(p); }
  __device__ __forceinline__ void ldg(const float* p) { r = __ldg(reinterpret_cast<const float4*>(p)); }
  __device__ __forceinline__ float get(int i) const { return i == 0 ? r.x : (i == 1 ? r.y : (i == 2 ? r.z : r.w)); }
};
template <> struct RV<float, 2> {
  float2 r;
  __device__ __forceinline__ void ld(const float* p) { r = *reinterpret_cast<const float2*>(p); }
  __device__ __forceinline__ void ldg(const float* p) { r = __ldg(reinterpret_cast<const float2*>(p)); }
  __device__ __forceinline__ float get(int i) const { return i ? r.y : r.x; }
};

__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <int V> __device__ __forceinline__ void stv(__nv_bfloat16* p, const float (&v)[V]) {
  if constexpr (V == 4)
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]));
  else
    *reinterpret_cast<uint32_t*>(p) = pack_bf2(v[0], v[1]);
}
template <int V> __device__ __forceinline__ void stv(float* p, const float (&v)[V]) {
  if constexpr (V == 4)
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  else
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
}

using F2 = float2;
__device__ __forceinline__ F2 bf2_to_f2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}
// V channels from shared memory, unpacked to V/2 float pairs
template <typename T, int V> __device__ __forceinline__ void ld_f2(const T* p, F2 (&o)[V / 2]);
template <> __device__ __forceinline__ void ld_f2<__nv_bfloat16, 4>(const __nv_bfloat16* p, F2 (&o)[2]) {
  const uint2 r = *reinterpret_cast<const uint2*>(p);
  o[0] = bf2_to_f2(r.x);
  o[1] = bf2_to_f2(r.y);
}
template <> __device__ __forceinline__ void ld_f2<__nv_bfloat16, 2>(const __nv_bfloat16* p, F2 (&o)[1]) {
  o[0] = bf2_to_f2(*reinterpret_cast<const uint32_t*>(p));
}
template <> __device__ __forceinline__ void ld_f2<float, 4>(const float* p, F2 (&o)[2]) {
  const float4 r = *reinterpret_cast<const float4*>(p);
  o[0] = make_float2(r.x, r.y);
  o[1] = make_float2(r.z, r.w);
}
template <> __device__ __forceinline__ void ld_f2<float, 2>(const float* p, F2 (&o)[1]) {
  o[0] = *reinterpret_cast<const float2*>(p);
}
template <int V> __device__ __forceinline__ void st_f2(__nv_bfloat16* p, const F2 (&v)[V / 2]) {
  if constexpr (V == 4)
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf2(v[0].x, v[0].y), pack_bf2(v[1].x, v[1].y));
  else
    *reinterpret_cast<uint32_t*>(p) = pack_bf2(v[0].x, v[0].y);
}
template <int V> __device__ __forceinline__ void st_f2(float* p, const F2 (&v)[V / 2]) {
  if constexpr (V == 4)
    *reinterpret_cast<float4*>(p) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
  else
    *reinterpret_cast<float2*>(p) = v[0];
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// bf16 path: one MUFU op (rel. error ~2^-11, below bf16 rounding); f32 keeps
// the exact form for the 1e-4 parity bar
template <typename T> __device__ __forceinline__ float sigm(float u) {
  if constexpr (sizeof(T) == 2) return fmaf(0.5f, tanh_approx(0.5f * u), 0.5f);
  else return 1.f / (1.f + __expf(-u));
}

struct Welford {
  float n, mean, m2;
};
__device__ __forceinline__ Welford wmerge(Welford a, Welford b) {
  const float n = a.n + b.n;
  if (n == 0.f) return a;
  const float d = b.mean - a.mean;
  const float f = b.n / n;
  return {n, a.mean + d * f, a.m2 + b.m2 + d * d * a.n * f};
}

struct RingP {
  int Ho, Wo, C, pt, pl;
  int Cb, Wt, Wb, R;
  int ncb, nwt, nbands;
  int nseg, L;
  uint32_t in_slot, io_slot;  // bytes per ring slot (128-B multiples)
  int K;                      // ring slots
  int flip;                   // CONV: w[KS*KS-1-t] (transposed conv)
};

template <typename T, int KS, int S, int MODE>
__global__ void __launch_bounds__(kMaxThreads, 2)
    dw_ring_kernel(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap dy_map,
                   const __grid_constant__ CUtensorMap z_map, const RingP p, const float* __restrict__ w,
                   T* __restrict__ out, float* __restrict__ part, const DzConsts dk) {
  constexpr int V = VecOf<KS>::value;
  const int K = p.K;  // ring slots (planner: KS + 2s .. KS + 4s)
  constexpr int T2 = KS * KS;
  constexpr int V2 = V / 2;
  // dynamic shared memory starts the CTA's window (no static smem here), so
  // it is 1024-B aligned; indexing it directly keeps the compiler in the
  // shared state space (LDS, 32-bit addresses) instead of generic loads
  extern __shared__ __align__(1024) uint8_t sm[];
  T* ring = reinterpret_cast<T*>(sm);
  T* dyr = reinterpret_cast<T*>(sm + K * p.in_slot);
  T* zr = reinterpret_cast<T*>(sm + K * p.in_slot + 2 * p.io_slot);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + K * p.in_slot + (MODE == MODE_DZW ? 4 * p.io_slot : 0));

  const int tid = threadIdx.x;
  int b = blockIdx.x;
  const int cb = b % p.ncb;
  b /= p.ncb;
  const int wt = b % p.nwt;
  b /= p.nwt;
  const int band = b % p.nbands;
  const int n = b / p.nbands;
  const int oy0 = band * p.R, nrows = min(p.R, p.Ho - oy0);
  const int ox0 = wt * p.Wt, ncols = min(p.Wt, p.Wo - ox0);
  const int NR = (nrows - 1) * S + KS;
  const int iy0 = oy0 * S - p.pt, ix0 = ox0 * S - p.pl, c0 = cb * p.Cb;
  const uint32_t in_el = p.in_slot / sizeof(T), io_el = p.io_slot / sizeof(T);
  const uint32_t in_bytes = (uint32_t)(p.Wb * p.Cb * sizeof(T)), io_bytes = (uint32_t)(p.Wt * p.Cb * sizeof(T));

  uint32_t* cnts = reinterpret_cast<uint32_t*>(bars + K + 2);  // per-row release counters (r % 16)
  const uint32_t nwarps = (blockDim.x + 31) / 32;
  if (tid == 0) {
    for (int i = 0; i < 16; ++i) cnts[i] = 0;
    for (int i = 0; i < K + 2; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // every input below is produced by the previous kernel
  pdl_trigger();
  auto issue_in = [&](int j) {
    uint64_t* bar = &bars[j % K];
    mbar_expect_tx(bar, in_bytes);
    tma_load_4d_cg<1>(&in_map, smem_u32(bar), ring + (j % K) * in_el, c0, ix0, iy0 + j, n);
  };
  auto issue_io = [&](int r) {
    uint64_t* bar = &bars[K + (r & 1)];
    mbar_expect_tx(bar, 2 * io_bytes);
    tma_load_4d_cg<1>(&dy_map, smem_u32(bar), dyr + (r & 1) * io_el, c0, ox0, oy0 + r, n);
    tma_load_4d_cg<1>(&z_map, smem_u32(bar), zr + (r & 1) * io_el, c0, ox0, oy0 + r, n);
  };
  if (tid == 0) {
    for (int j = 0; j < min(K, NR); ++j) issue_in(j);
    if (MODE == MODE_DZW)
      for (int r = 0; r < min(2, nrows); ++r) issue_io(r);
  }

  const int CVn = p.Cb / V;
  const int cv = tid % CVn, sg = tid / CVn;
  const int xs = sg * p.L, xe = min(xs + p.L, ncols);
  const bool act = xs < xe;
  const int cc = c0 + cv * V;

  // weights / window / accumulators as float2 pairs: FFMA2 (sm_100 packed
  // f32 FMA) does two channels per instruction
  F2 wr[MODE == MODE_DZW ? 1 : T2][V2];
  if constexpr (MODE != MODE_DZW) {
#pragma unroll
    for (int t = 0; t < T2; ++t)
#pragma unroll
      for (int i = 0; i < V2; ++i) {
        const float* wp = w + (size_t)(p.flip ? T2 - 1 - t : t) * p.C + cc + 2 * i;
        wr[t][i] = make_float2(__ldg(wp), __ldg(wp + 1));
      }
  }
  // DZW: dz = P*du + Cz*z + Bc, du = (dy*sv + dp) * swish'(z*P + Q)
  float kP[V], kQ[V], kCz[V], kB[V], kS[V], kD[V];
  if constexpr (MODE == MODE_DZW) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = cc + i;
      const float rs = dk.rstd[c], mu = dk.mean[c];
      kP[i] = dk.gamma[c] * rs;
      kQ[i] = dk.beta[c] - mu * kP[i];
      const float ic = dk.inv_count > 0.f ? dk.inv_count : 1.f / dk.bnsum[2 * p.C + c];  // SyncBN count
      const float mdu = dk.bnsum[c] * ic, mdux = dk.bnsum[p.C + c] * ic;
      kCz[i] = -kP[i] * rs * mdux;
      kB[i] = -kP[i] * mdu - kCz[i] * mu;
      kS[i] = dk.s[(size_t)n * p.C + c];
      kD[i] = dk.dpool[(size_t)n * p.C + c];
    }
  }
  F2 st0[V2], st1[V2], nsh[V2];
  F2 dwa[MODE == MODE_DZW ? T2 : 1][V2];
#pragma unroll
  for (int i = 0; i < V2; ++i) {
    st0[i] = make_float2(0.f, 0.f);
    st1[i] = make_float2(0.f, 0.f);
    nsh[i] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int t = 0; t < (MODE == MODE_DZW ? T2 : 1); ++t)
#pragma unroll
    for (int i = 0; i < V2; ++i) dwa[t][i] = make_float2(0.f, 0.f);
  int cnt = 0;

  if constexpr (MODE == MODE_STATS) {
    if (act) {
#pragma unroll
      for (int ky = 0; ky < KS; ++ky) mbar_wait(&bars[ky], 0);
      F2 acc[V2];
#pragma unroll
      for (int i = 0; i < V2; ++i) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int ky = 0; ky < KS; ++ky)
#pragma unroll
        for (int kx = 0; kx < KS; ++kx) {
          F2 v[V2];
          ld_f2<T, V>(ring + ky * in_el + cv * V + (xs * S + kx) * p.Cb, v);
#pragma unroll
          for (int i = 0; i < V2; ++i) acc[i] = __ffma2_rn(v[i], wr[ky * KS + kx][i], acc[i]);
        }
#pragma unroll
      for (int i = 0; i < V2; ++i) nsh[i] = make_float2(-acc[i].x, -acc[i].y);
    }
  }

  for (int r = 0; r < nrows; ++r) {
#pragma unroll
    for (int ky = 0; ky < KS; ++ky) {
      const int j = r * S + ky;
      mbar_wait(&bars[j % K], (j / K) & 1);
    }
    if (MODE == MODE_DZW) mbar_wait(&bars[K + (r & 1)], (r >> 1) & 1);
    if (act) {
      const T* rows[KS];
#pragma unroll
      for (int ky = 0; ky < KS; ++ky) rows[ky] = ring + ((r * S + ky) % K) * in_el + cv * V;
      T* orow = out + (((size_t)n * p.Ho + oy0 + r) * p.Wo + ox0) * p.C + cc;
      const T* dyrow = dyr + (r & 1) * io_el + cv * V;
      const T* zrow = zr + (r & 1) * io_el + cv * V;
      // window = KS column slots x KS rows; input column q (relative to the
      // segment) lives in slot q % KS.  Unrolling the column walk by KS makes
      // every slot index a compile-time constant: no register shuffling.
      F2 win[KS][KS][V2];
#pragma unroll
      for (int q = 0; q < KS - S; ++q)
#pragma unroll
        for (int ky = 0; ky < KS; ++ky) ld_f2<T, V>(rows[ky] + (xs * S + q) * p.Cb, win[q][ky]);
      auto step = [&](auto uc, int x) {
        constexpr int u = decltype(uc)::value;
#pragma unroll
        for (int jn = 0; jn < S; ++jn)
#pragma unroll
          for (int ky = 0; ky < KS; ++ky)
            ld_f2<T, V>(rows[ky] + (x * S + KS - S + jn) * p.Cb, win[(u * S + KS - S + jn) % KS][ky]);
        if constexpr (MODE != MODE_DZW) {
          // one partial sum per tap row: KS independent FFMA2 chains
          F2 pr[KS][V2];
#pragma unroll
          for (int ky = 0; ky < KS; ++ky)
#pragma unroll
            for (int i = 0; i < V2; ++i) {
              pr[ky][i] = __fmul2_rn(win[(u * S) % KS][ky][i], wr[ky * KS][i]);
#pragma unroll
              for (int kx = 1; kx < KS; ++kx)
                pr[ky][i] = __ffma2_rn(win[(u * S + kx) % KS][ky][i], wr[ky * KS + kx][i], pr[ky][i]);
            }
          F2 acc[V2];
#pragma unroll
          for (int i = 0; i < V2; ++i) {
            acc[i] = pr[0][i];
#pragma unroll
            for (int ky = 1; ky < KS; ++ky) acc[i] = __fadd2_rn(acc[i], pr[ky][i]);
          }
          st_f2<V>(orow + (size_t)x * p.C, acc);
          if constexpr (MODE == MODE_STATS) {
            // shifted sums of the unrounded conv output (shift = the
            // thread's first output, computed before the row loop)
#pragma unroll
            for (int i = 0; i < V2; ++i) {
              const F2 d = __fadd2_rn(acc[i], nsh[i]);
              st0[i] = __fadd2_rn(st0[i], d);
              st1[i] = __ffma2_rn(d, d, st1[i]);
            }
            ++cnt;
          }
        } else {
          F2 dv[V2], zv[V2], dz[V2];
          ld_f2<T, V>(dyrow + x * p.Cb, dv);
          ld_f2<T, V>(zrow + x * p.Cb, zv);
#pragma unroll
          for (int i = 0; i < V; ++i) {
            const float zz = (i & 1) ? zv[i >> 1].y : zv[i >> 1].x;
            const float dd = (i & 1) ? dv[i >> 1].y : dv[i >> 1].x;
            const float u_ = fmaf(zz, kP[i], kQ[i]);
            const float sgm = sigm<T>(u_);
            const float swp = sgm * fmaf(u_, 1.f - sgm, 1.f);
            const float du = fmaf(dd, kS[i], kD[i]) * swp;
            const float o = fmaf(kP[i], du, fmaf(kCz[i], zz, kB[i]));
            if (i & 1) dz[i >> 1].y = o;
            else dz[i >> 1].x = o;
          }
          st_f2<V>(orow + (size_t)x * p.C, dz);
#pragma unroll
          for (int ky = 0; ky < KS; ++ky)
#pragma unroll
            for (int kx = 0; kx < KS; ++kx)
#pragma unroll
              for (int i = 0; i < V2; ++i)
                dwa[ky * KS + kx][i] = __ffma2_rn(win[(u * S + kx) % KS][ky][i], dz[i], dwa[ky * KS + kx][i]);
        }
      };
      // whole groups of KS columns unguarded (the compiler interleaves the
      // independent outputs), then the guarded remainder
      int xb = xs;
      for (; xb + KS <= xe; xb += KS) unroll_for<KS>([&](auto uc) { step(uc, xb + decltype(uc)::value); });
      unroll_for<KS>([&](auto uc) {
        if (xb + decltype(uc)::value < xe) step(uc, xb + decltype(uc)::value);
      });
    }
    // release: the warp is done with the rows leaving the window; the last
    // warp to arrive refills them (no CTA-wide barrier per row)
    __syncwarp();
    if ((tid & 31) == 0) {
      __threadfence_block();
      // a warp leads the slowest by at most (K - KS) / s <= 4 rows: 16 counters never alias
      const uint32_t old = atomicAdd(&cnts[r & 15], 1u);
      if (old == (uint32_t)((r >> 4) + 1) * nwarps - 1) {
#pragma unroll
        for (int q = 0; q < S; ++q) {
          const int jn = r * S + q + K;
          if (jn < NR) issue_in(jn);
        }
        if (MODE == MODE_DZW && r + 2 < nrows) issue_io(r + 2);
      }
    }
  }
  __syncthreads();

  // ------------------------------------------------------------ CTA partials
  // every issued load has been consumed: the ring is free scratch now
  float* red = reinterpret_cast<float*>(sm);
  const size_t tile = ((size_t)n * p.nbands + band) * p.nwt + wt;
  if constexpr (MODE == MODE_STATS) {
    float* s_n = red;
    float* s_mean = red + p.nseg;
    float* s_m2 = s_mean + p.nseg * p.Cb;
    if (cv == 0) s_n[sg] = (float)cnt;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float a0 = (i & 1) ? st0[i >> 1].y : st0[i >> 1].x, a1 = (i & 1) ? st1[i >> 1].y : st1[i >> 1].x;
      const float sh = -((i & 1) ? nsh[i >> 1].y : nsh[i >> 1].x);
      const float m = cnt ? a0 / (float)cnt : 0.f;
      s_mean[sg * p.Cb + cv * V + i] = sh + m;
      s_m2[sg * p.Cb + cv * V + i] = cnt ? fmaxf(a1 - a0 * m, 0.f) : 0.f;
    }
    __syncthreads();
    for (int c = tid; c < p.Cb; c += blockDim.x) {
      Welford acc = {0.f, 0.f, 0.f};
      for (int j = 0; j < p.nseg; ++j) acc = wmerge(acc, Welford{s_n[j], s_mean[j * p.Cb + c], s_m2[j * p.Cb + c]});
      part[(tile * 3 + 0) * p.C + c0 + c] = acc.n;
      part[(tile * 3 + 1) * p.C + c0 + c] = acc.mean;
      part[(tile * 3 + 2) * p.C + c0 + c] = acc.m2;
    }
  } else if constexpr (MODE == MODE_DZW) {
#pragma unroll
    for (int t = 0; t < T2; ++t) {
#pragma unroll
      for (int i = 0; i < V2; ++i) {
        red[sg * p.Cb + cv * V + 2 * i] = dwa[t][i].x;
        red[sg * p.Cb + cv * V + 2 * i + 1] = dwa[t][i].y;
      }
      __syncthreads();
      for (int c = tid; c < p.Cb; c += blockDim.x) {
        float acc = 0.f;
        for (int j = 0; j < p.nseg; ++j) acc += red[j * p.Cb + c];
        part[(tile * T2 + t) * p.C + c0 + c] = acc;
      }
      __syncthreads();
    }
  }
}

// (n, mean, M2) partials [tiles][3][C] -> out [3][C], fixed merge order
__global__ void __launch_bounds__(256) stats_merge_kernel(int ntiles, int C, const float* __restrict__ part,
                                                          float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sn[256], smn[256], sm2[256];
  const int c = blockIdx.x;
  Welford acc = {0.f, 0.f, 0.f};
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x)
    acc = wmerge(acc, Welford{part[((size_t)t * 3) * C + c], part[((size_t)t * 3 + 1) * C + c],
                              part[((size_t)t * 3 + 2) * C + c]});
  sn[threadIdx.x] = acc.n;
  smn[threadIdx.x] = acc.mean;
  sm2[threadIdx.x] = acc.m2;
  __syncthreads();
  for (int sd = blockDim.x / 2; sd > 0; sd >>= 1) {
    if (threadIdx.x < sd) {
      const Welford m = wmerge(Welford{sn[threadIdx.x], smn[threadIdx.x], sm2[threadIdx.x]},
                               Welford{sn[threadIdx.x + sd], smn[threadIdx.x + sd], sm2[threadIdx.x + sd]});
      sn[threadIdx.x] = m.n;
      smn[threadIdx.x] = m.mean;
      sm2[threadIdx.x] = m.m2;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[c] = sn[0];
    out[C + c] = smn[0];
    out[2 * C + c] = sm2[0];
  }
}

// dw[t][c] = sum_b part[b][t][c]: block = 32 channels x 8 part lanes, fixed order
__global__ void __launch_bounds__(256) taps_sum_kernel(int nparts, int taps, int C, const float* __restrict__ part,
                                                       float* __restrict__ dw) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, pl = threadIdx.x >> 5;
  const int t = blockIdx.y, c = blockIdx.x * 32 + lane;
  float acc = 0.f;
  if (c < C) {
#pragma unroll 4
    for (int b = pl; b < nparts; b += 8) acc += part[((size_t)b * taps + t) * C + c];
  }
  red[pl][lane] = acc;
  __syncthreads();
  if (pl == 0 && c < C) {
    float s2 = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s2 += red[j][lane];
    dw[t * C + c] = s2;
  }
}

// dx for stride 2 (a gather: each input pixel receives the taps whose
// output position has the right parity), V channels per thread.  The launch
// keeps (grid x block) a multiple of C/V, so a thread's channel group never
// changes: its KS*KS*V weights are loaded once into registers.
template <typename T, int KS>
__global__ void __launch_bounds__(512) dw_dx_s2_kernel(const DwShape g, const T* __restrict__ dz,
                                                       const float* __restrict__ w, T* __restrict__ dx) {
  constexpr int V = VecOf<KS>::value;
  pdl_wait();
  pdl_trigger();
  const int CVn = g.C / V;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride_pix = (gridDim.x * blockDim.x) / CVn;
  const int cv = tid % CVn;
  const int c = cv * V;
  float wr[KS * KS][V];
#pragma unroll
  for (int t = 0; t < KS * KS; ++t)
#pragma unroll
    for (int i = 0; i < V; ++i) wr[t][i] = __ldg(w + (size_t)t * g.C + c + i);
  const int npix = g.N * g.Hi * g.Wi;
  for (int pix = tid / CVn; pix < npix; pix += stride_pix) {
    const int ix = pix % g.Wi;
    const int t2 = pix / g.Wi;
    const int iy = t2 % g.Hi;
    const int n = t2 / g.Hi;
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    const T* dzn = dz + (size_t)n * g.Ho * g.Wo * g.C + c;
#pragma unroll
    for (int ky = 0; ky < KS; ++ky) {
      const int ty = iy + g.pt - ky;
      if (ty < 0 || (ty & 1) || (ty >> 1) >= g.Ho) continue;
#pragma unroll
      for (int kx = 0; kx < KS; ++kx) {
        const int tx = ix + g.pl - kx;
        if (tx < 0 || (tx & 1) || (tx >> 1) >= g.Wo) continue;
        RV<T, V> v;
        v.ldg(dzn + ((size_t)(ty >> 1) * g.Wo + (tx >> 1)) * g.C);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = fmaf(v.get(i), wr[ky * KS + kx][i], acc[i]);
      }
    }
    stv<V>(dx + (size_t)pix * g.C + c, acc);
  }
}

// dx for stride 2 with the symmetric "same" padding pt = pl = KS/2 (every
// EfficientNet stride-2 block): a thread owns a 2x2 block of input pixels
// (2a..2a+1, 2b..2b+1) and one channel group; with the padding a compile-time
// constant, the tap parities are compile-time too, so the block's dz window
// (2x2 for k3, 3x3 for k5) is loaded once and every tap is one FMA — no
// per-tap parity tests, one index decomposition per 4 outputs.
template <typename T, int KS>
__global__ void __launch_bounds__(512) dw_dx_s2_same_kernel(const DwShape g, const T* __restrict__ dz,
                                                            const float* __restrict__ w, T* __restrict__ dx) {
  constexpr int V = VecOf<KS>::value;
  constexpr int PT = KS / 2;
  constexpr int OMIN = -((KS - 1 - PT) / 2), OMAX = (1 + PT) / 2;  // dz offsets relative to (a, b)
  constexpr int RW = OMAX - OMIN + 1;
  pdl_wait();
  pdl_trigger();
  const int CVn = g.C / V;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride_blk = (gridDim.x * blockDim.x) / CVn;
  const int c = (tid % CVn) * V;
  float wr[KS * KS][V];
#pragma unroll
  for (int t = 0; t < KS * KS; ++t)
#pragma unroll
    for (int i = 0; i < V; ++i) wr[t][i] = __ldg(w + (size_t)t * g.C + c + i);
  const int BH = (g.Hi + 1) / 2, BW = (g.Wi + 1) / 2;
  const int nblk = g.N * BH * BW;
  for (int blk = tid / CVn; blk < nblk; blk += stride_blk) {
    const int b = blk % BW;
    const int t2 = blk / BW;
    const int a = t2 % BH;
    const int n = t2 / BH;
    const T* dzn = dz + (size_t)n * g.Ho * g.Wo * g.C + c;
    float win[RW][RW][V];
#pragma unroll
    for (int oy = 0; oy < RW; ++oy)
#pragma unroll
      for (int ox = 0; ox < RW; ++ox) {
        const int y = a + OMIN + oy, x = b + OMIN + ox;
        RV<T, V> v;
        if (y >= 0 && y < g.Ho && x >= 0 && x < g.Wo) {
          v.ldg(dzn + ((size_t)y * g.Wo + x) * g.C);
#pragma unroll
          for (int i = 0; i < V; ++i) win[oy][ox][i] = v.get(i);
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) win[oy][ox][i] = 0.f;
        }
      }
#pragma unroll
    for (int dyy = 0; dyy < 2; ++dyy)
#pragma unroll
      for (int dxx = 0; dxx < 2; ++dxx) {
        const int iy = 2 * a + dyy, ix = 2 * b + dxx;
        if (iy >= g.Hi || ix >= g.Wi) continue;
        float acc[V];
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = 0.f;
#pragma unroll
        for (int ky = 0; ky < KS; ++ky) {
          if ((dyy + PT - ky) & 1) continue;  // compile-time after unrolling
          const int oy = (dyy + PT - ky) / 2 - OMIN;
#pragma unroll
          for (int kx = 0; kx < KS; ++kx) {
            if ((dxx + PT - kx) & 1) continue;
            const int ox = (dxx + PT - kx) / 2 - OMIN;
#pragma unroll
            for (int i = 0; i < V; ++i) acc[i] = fmaf(win[oy][ox][i], wr[ky * KS + kx][i], acc[i]);
          }
        }
        stv<V>(dx + (((size_t)n * g.Hi + iy) * g.Wi + ix) * g.C + c, acc);
      }
  }
}

// bf16 variant of dw_dx_s2_same_kernel with 16-byte channel vectors (8
// channels): the k5 kernel above moves 4-byte vectors (its 25 weights x V
// channels live in registers, capping V at 2), so it issues 4x the memory
// instructions per byte.  Here the weights sit in shared memory ([KS*KS][C]
// f32, staged once per CTA) and a thread's 2x2 input block reads its dz window
// as uint4 rows.  Same tap arithmetic and order as the generic kernel.
template <int KS>
__global__ void __launch_bounds__(256) dw_dx_s2_v8_kernel(const DwShape g, const __nv_bfloat16* __restrict__ dz,
                                                          const float* __restrict__ w, __nv_bfloat16* __restrict__ dx) {
  constexpr int V = 8;
  constexpr int PT = KS / 2;
  constexpr int OMIN = -((KS - 1 - PT) / 2), OMAX = (1 + PT) / 2;
  constexpr int RW = OMAX - OMIN + 1;
  extern __shared__ float wsm[];  // [KS*KS][C]
  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i < KS * KS * g.C / 4; i += blockDim.x)
    reinterpret_cast<float4*>(wsm)[i] = __ldg(reinterpret_cast<const float4*>(w) + i);
  __syncthreads();
  const int CVn = g.C / V;
  const int BH = (g.Hi + 1) / 2, BW = (g.Wi + 1) / 2;
  const int64_t items = (int64_t)g.N * BH * BW * CVn;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items; it += (int64_t)gridDim.x * blockDim.x) {
    const int cv = (int)(it % CVn);
    int64_t blk = it / CVn;
    const int b = (int)(blk % BW);
    blk /= BW;
    const int a = (int)(blk % BH);
    const int n = (int)(blk / BH);
    const int c = cv * V;
    const __nv_bfloat16* dzn = dz + (size_t)n * g.Ho * g.Wo * g.C + c;
    float win[RW][RW][V];
#pragma unroll
    for (int oy = 0; oy < RW; ++oy)
#pragma unroll
      for (int ox = 0; ox < RW; ++ox) {
        const int y = a + OMIN + oy, x = b + OMIN + ox;
        if (y >= 0 && y < g.Ho && x >= 0 && x < g.Wo) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(dzn + ((size_t)y * g.Wo + x) * g.C));
          unpack4<__nv_bfloat16>(v, win[oy][ox]);
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) win[oy][ox][i] = 0.f;
        }
      }
#pragma unroll
    for (int dyy = 0; dyy < 2; ++dyy)
#pragma unroll
      for (int dxx = 0; dxx < 2; ++dxx) {
        const int iy = 2 * a + dyy, ix = 2 * b + dxx;
        if (iy >= g.Hi || ix >= g.Wi) continue;
        float acc[V];
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = 0.f;
#pragma unroll
        for (int ky = 0; ky < KS; ++ky) {
          if ((dyy + PT - ky) & 1) continue;
          const int oy = (dyy + PT - ky) / 2 - OMIN;
#pragma unroll
          for (int kx = 0; kx < KS; ++kx) {
            if ((dxx + PT - kx) & 1) continue;
            const int ox = (dxx + PT - kx) / 2 - OMIN;
            const float4 w0 = reinterpret_cast<const float4*>(wsm + (ky * KS + kx) * g.C + c)[0];
            const float4 w1 = reinterpret_cast<const float4*>(wsm + (ky * KS + kx) * g.C + c)[1];
            const float wv[V] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int i = 0; i < V; ++i) acc[i] = fmaf(win[oy][ox][i], wv[i], acc[i]);
          }
        }
        *reinterpret_cast<uint4*>(dx + (((size_t)n * g.Hi + iy) * g.Wi + ix) * g.C + c) = pack4<__nv_bfloat16>(acc);
      }
  }
}

// ---------------------------------------------------------------- planning
struct Plan {
  RingP p;
  int threads, grid;
  size_t smem;
};

size_t rnd128(size_t b) { return (b + 127) & ~size_t(127); }

int pick_cb(int C, int V, int esz, int cap = 128) {
  for (int d = std::min(C, cap); d >= V; --d)
    if (C % d == 0 && d % V == 0 && (d * esz) % 16 == 0) return d;
  return 0;
}

bool make_plan_cb(int N, int Ho, int Wo, int C, int ks, int s, int pt, int pl, int esz, int mode, int Cb,
                  Plan* pl_out, long* cost_out);

// in grid (Hi, Wi) -> out grid (Ho, Wo) with (pt, pl): the correlation this launch computes.
// The channel chunk Cb is chosen by the cost model too: narrow maps (EfficientNet's
// 14x14 / 7x7 stages) want wide chunks and whole-row column segments (a 2-column
// segment of a 7-wide row loads a 6-column window: 3x halo), wide maps want
// narrow chunks and many CTAs.
bool make_plan(int N, int Hi, int Wi, int Ho, int Wo, int C, int ks, int s, int pt, int pl, int esz, int mode,
               Plan* pl_out) {
  (void)Hi;
  (void)Wi;
  if (ks != 3 && ks != 5) return false;
  if (s != 1 && s != 2) return false;
  if ((C * esz) % 16 != 0) return false;
  const int V = ks == 3 ? 4 : 2;
  bool found = false;
  long best = 0;
  for (int cap : {128, 192, 256}) {  // a TMA box dimension is at most 256 elements
    const int cb = pick_cb(C, V, esz, cap);
    if (!cb || (cap > 128 && cb <= 128)) continue;  // no new chunk width at this cap
    Plan cand;
    long cost = 0;
    if (!make_plan_cb(N, Ho, Wo, C, ks, s, pt, pl, esz, mode, cb, &cand, &cost)) continue;
    if (!found || cost < best) {
      best = cost;
      *pl_out = cand;
      found = true;
    }
  }
  return found;
}

bool make_plan_cb(int N, int Ho, int Wo, int C, int ks, int s, int pt, int pl, int esz, int mode, int Cb,
                  Plan* pl_out, long* cost_out) {
  const int V = ks == 3 ? 4 : 2;
  if (!Cb) return false;
  const int CVn = Cb / V;
  if (CVn > kMaxThreads) return false;
  auto smem_of = [&](int wt, int k) {
    const size_t in_slot = rnd128((size_t)((wt - 1) * s + ks) * Cb * esz);
    const size_t io_slot = rnd128((size_t)wt * Cb * esz);
    return k * in_slot + (mode == MODE_DZW ? 4 * io_slot : 0) + (k + 2) * 8 + 64;
  };
  // widest tile first (fewer halo columns, fewer per-row overheads): a deeper
  // ring (up to 4 output rows of lookahead) only when the whole row still fits
  const int wmax = std::min(Wo, std::min(256, (256 - ks) / s + 1));
  int K = 0, Wt = 0;
  for (int k = ks + 4 * s; k >= ks + 2 * s && !K; --k) {
    int w = wmax;
    while (w > 1 && smem_of(w, k) > kSmemBudget) --w;
    if (smem_of(w, k) <= kSmemBudget && (w == wmax || k == ks + 2 * s)) {
      K = k;
      Wt = w;
    }
  }
  if (!K) return false;
  const int nwt = (Wo + Wt - 1) / Wt;
  Wt = (Wo + nwt - 1) / nwt;
  const int nseg_max = kMaxThreads / CVn;
  const int L = (Wt + nseg_max - 1) / nseg_max;
  const int nseg = (Wt + L - 1) / L;
  RingP p{};
  p.Ho = Ho;
  p.Wo = Wo;
  p.C = C;
  p.pt = pt;
  p.pl = pl;
  p.Cb = Cb;
  p.Wt = Wt;
  p.Wb = (Wt - 1) * s + ks;
  p.ncb = C / Cb;
  p.nwt = nwt;
  p.nseg = nseg;
  p.L = L;
  p.in_slot = (uint32_t)rnd128((size_t)p.Wb * Cb * esz);
  p.io_slot = (uint32_t)rnd128((size_t)Wt * Cb * esz);
  // reduction scratch must fit in the ring
  p.K = K;
  const size_t red = (size_t)nseg * (1 + 2 * Cb) * 4;
  if (red > (size_t)K * p.in_slot) return false;
  // band height: fewest waves x rows per CTA (2 CTAs per SM)
  const long slots = 2L * num_sms();
  long best = -1;
  int bestR = Ho;
  for (int R = 1; R <= Ho; ++R) {
    const int nb = (Ho + R - 1) / R;
    if ((Ho + nb - 1) / nb != R) continue;
    const long ctas = (long)N * nb * nwt * p.ncb;
    const long waves = (ctas + slots - 1) / slots;
    const long cost = waves * ((long)(R - 1) * s + ks + 4);
    if (best < 0 || cost < best) {
      best = cost;
      bestR = R;
    }
  }
  p.R = bestR;
  p.nbands = (Ho + bestR - 1) / bestR;
  pl_out->p = p;
  pl_out->threads = CVn * nseg;
  pl_out->grid = N * p.nbands * nwt * p.ncb;
  pl_out->smem = smem_of(Wt, K);
  // per-thread work of one output row ~ the window columns a segment loads
  // (L outputs + KS - s halo); wave-quantised over the whole grid
  *cost_out = best * (long)(L * s + ks - s + 2);
  return true;
}

int tmap(CUtensorMap* m, const void* base, int esz, int N, int H, int W, int C, int Cb, int box_w) {
  return make_map(m, base, esz, (uint64_t)C, (uint64_t)W, C, H, (int64_t)W * C, N, (int64_t)H * W * C, (uint32_t)Cb,
                  (uint32_t)box_w, false);
}

template <typename T, int KS, int S, int MODE>
int launch_ring(const Plan& pl, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const float* w,
                void* out, float* part, const DzConsts& dk, cudaStream_t st) {
  auto k = dw_ring_kernel<T, KS, S, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
  launch_k(k, pl.grid, pl.threads, pl.smem, st, a, b, c, pl.p, w, (T*)out, part, dk);
  DFX_LAUNCH_CHECK("dwconv ring kernel");
  return DFX_OK;
}

template <typename T, int MODE>
int dispatch_ring(int ks, int s, const Plan& pl, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                  const float* w, void* out, float* part, const DzConsts& dk, cudaStream_t st) {
  if (ks == 3 && s == 1) return launch_ring<T, 3, 1, MODE>(pl, a, b, c, w, out, part, dk, st);
  if (ks == 3 && s == 2) return launch_ring<T, 3, 2, MODE>(pl, a, b, c, w, out, part, dk, st);
  if (ks == 5 && s == 1) return launch_ring<T, 5, 1, MODE>(pl, a, b, c, w, out, part, dk, st);
  if (ks == 5 && s == 2) return launch_ring<T, 5, 2, MODE>(pl, a, b, c, w, out, part, dk, st);
  return fail(DFX_ERR_UNSUPPORTED, "dwconv: kernel size must be 3 or 5, stride 1 or 2");
}

int esz_of(int dtype) { return dtype == DFX_BF16 ? 2 : 4; }

}  // namespace

bool dw_ring_ok(const DwShape& g, int esz) {
  Plan a, b, c;
  return make_plan(g.N, g.Hi, g.Wi, g.Ho, g.Wo, g.C, g.ks, g.s, g.pt, g.pl, esz, MODE_STATS, &a) &&
         make_plan(g.N, g.Hi, g.Wi, g.Ho, g.Wo, g.C, g.ks, g.s, g.pt, g.pl, esz, MODE_DZW, &b) &&
         (g.s == 2 || make_plan(g.N, g.Ho, g.Wo, g.Hi, g.Wi, g.C, g.ks, 1, g.ks - 1 - g.pt, g.ks - 1 - g.pl, esz,
                                MODE_CONV, &c));
}

size_t dw_stat_tiles(const DwShape& g, int esz) {
  Plan pl;
  if (!make_plan(g.N, g.Hi, g.Wi, g.Ho, g.Wo, g.C, g.ks, g.s, g.pt, g.pl, esz, MODE_STATS, &pl)) return 0;
  return (size_t)g.N * pl.p.nbands * pl.p.nwt;
}

size_t dw_dzw_tiles(const DwShape& g, int esz) {
  Plan pl;
  if (!make_plan(g.N, g.Hi, g.Wi, g.Ho, g.Wo, g.C, g.ks, g.s, g.pt, g.pl, esz, MODE_DZW, &pl)) return 0;
  return (size_t)g.N * pl.p.nbands * pl.p.nwt;
}

int dw_conv_stats(int dtype, const DwShape& g, const void* x, const float* w, void* z, float* part,
                  float* stats_out, cudaStream_t st) {
  const int esz = esz_of(dtype);
  Plan pl;
  if (!make_plan(g.N, g.Hi, g.Wi, g.Ho, g.Wo, g.C, g.ks, g.s, g.pt, g.pl, esz, MODE_STATS, &pl))
    return fail(DFX_ERR_UNSUPPORTED, "dwconv: shape not supported by the TMA ring path");
  CUtensorMap mx;
  if (int rc = tmap(&mx, x, esz, g.N, g.Hi, g.Wi, g.C, pl.p.Cb, pl.p.Wb)) return rc;
  DzConsts none{};
  int rc = dtype == DFX_BF16 ? dispatch_ring<__nv_bfloat16, MODE_STATS>(g.ks, g.s, pl, mx, mx, mx, w, z, part, none, st)
                             : dispatch_ring<float, MODE_STATS>(g.ks, g.s, pl, mx, mx, mx, w, z, part, none, st);
  if (rc) return rc;
  launch_k(stats_merge_kernel, g.C, 256, 0, st, (int)((size_t)g.N * pl.p.nbands * pl.p.nwt), g.C, part, stats_out);
  DFX_LAUNCH_CHECK("dwconv stats merge");
  return DFX_OK;
}

int dw_dz_dw(int dtype, const DwShape& g, const void* x, const void* dy, const void* z, const DzConsts& k, void* dz,
             float* part, float* dw_out, cudaStream_t st) {
  const int esz = esz_of(dtype);
  Plan pl;
  if (!make_plan(g.N, g.Hi, g.Wi, g.Ho, g.Wo, g.C, g.ks, g.s, g.pt, g.pl, esz, MODE_DZW, &pl))
    return fail(DFX_ERR_UNSUPPORTED, "dwconv: shape not supported by the TMA ring path");
  CUtensorMap mx, mdy, mz;
  if (int rc = tmap(&mx, x, esz, g.N, g.Hi, g.Wi, g.C, pl.p.Cb, pl.p.Wb)) return rc;
  if (int rc = tmap(&mdy, dy, esz, g.N, g.Ho, g.Wo, g.C, pl.p.Cb, pl.p.Wt)) return rc;
  if (int rc = tmap(&mz, z, esz, g.N, g.Ho, g.Wo, g.C, pl.p.Cb, pl.p.Wt)) return rc;
  int rc = dtype == DFX_BF16 ? dispatch_ring<__nv_bfloat16, MODE_DZW>(g.ks, g.s, pl, mx, mdy, mz, nullptr, dz, part, k, st)
                             : dispatch_ring<float, MODE_DZW>(g.ks, g.s, pl, mx, mdy, mz, nullptr, dz, part, k, st);
  if (rc) return rc;
  const int taps = g.ks * g.ks;
  launch_k(taps_sum_kernel, dim3((unsigned)((g.C + 31) / 32), (unsigned)taps), 256, 0, st,
           (int)((size_t)g.N * pl.p.nbands * pl.p.nwt), taps, g.C, part, dw_out);
  DFX_LAUNCH_CHECK("dwconv dw sum");
  return DFX_OK;
}

int dw_dx(int dtype, const DwShape& g, const void* dz, const float* w, void* dx, cudaStream_t st) {
  const int esz = esz_of(dtype);
  if (g.s == 2) {
    const int V = g.ks == 3 ? 4 : 2;
    if (g.C % V) return fail(DFX_ERR_UNSUPPORTED, "dwconv dx: channels must be a multiple of the vector width");
    const int CVn = g.C / V;
    const int per_block = CVn <= 256 ? (256 / CVn) * CVn : (CVn <= 512 ? CVn : 0);
    if (!per_block) return fail(DFX_ERR_UNSUPPORTED, "dwconv dx: too many channels for the stride-2 gather");
    const int64_t total = (int64_t)g.N * g.Hi * g.Wi * CVn;
    const int grid = (int)std::min<int64_t>((total + per_block - 1) / per_block, (int64_t)num_sms() * 8);
    const bool same = g.pt == g.ks / 2 && g.pl == g.ks / 2;
    if (same && dtype == DFX_BF16 && g.C % 8 == 0 && (size_t)g.ks * g.ks * g.C * 4 <= 160 * 1024 &&
        getenv("DFX_DW_DX_S2_V2") == nullptr) {
      const size_t wsm = (size_t)g.ks * g.ks * g.C * sizeof(float);
      const int64_t items = (int64_t)g.N * ((g.Hi + 1) / 2) * ((g.Wi + 1) / 2) * (g.C / 8);
      if (g.ks == 3) {
        auto k = dw_dx_s2_v8_kernel<3>;
        if (wsm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, wsm);
        const int grid3 = (int)std::min<int64_t>((items + 255) / 256, (int64_t)num_sms() * std::max(occ, 1));
        launch_k(k, grid3, 256, wsm, st, g, (const __nv_bfloat16*)dz, w, (__nv_bfloat16*)dx);
      } else {
        auto k = dw_dx_s2_v8_kernel<5>;
        if (wsm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, wsm);
        const int grid3 = (int)std::min<int64_t>((items + 255) / 256, (int64_t)num_sms() * std::max(occ, 1));
        launch_k(k, grid3, 256, wsm, st, g, (const __nv_bfloat16*)dz, w, (__nv_bfloat16*)dx);
      }
      DFX_LAUNCH_CHECK("dwconv dx (stride 2, same padding, 16-byte vectors)");
      return DFX_OK;
    }
    if (same) {
      const int64_t blocks = (int64_t)g.N * ((g.Hi + 1) / 2) * ((g.Wi + 1) / 2) * CVn;
      const int grid2 = (int)std::min<int64_t>((blocks + per_block - 1) / per_block, (int64_t)num_sms() * 8);
      if (dtype == DFX_BF16) {
        if (g.ks == 3) launch_k(dw_dx_s2_same_kernel<__nv_bfloat16, 3>, grid2, per_block, 0, st, g, (const __nv_bfloat16*)dz, w, (__nv_bfloat16*)dx);
        else launch_k(dw_dx_s2_same_kernel<__nv_bfloat16, 5>, grid2, per_block, 0, st, g, (const __nv_bfloat16*)dz, w, (__nv_bfloat16*)dx);
      } else {
        if (g.ks == 3) launch_k(dw_dx_s2_same_kernel<float, 3>, grid2, per_block, 0, st, g, (const float*)dz, w, (float*)dx);
        else launch_k(dw_dx_s2_same_kernel<float, 5>, grid2, per_block, 0, st, g, (const float*)dz, w, (float*)dx);
      }
      DFX_LAUNCH_CHECK("dwconv dx (stride 2, same padding)");
      return DFX_OK;
    }
    if (dtype == DFX_BF16) {
      if (g.ks == 3) launch_k(dw_dx_s2_kernel<__nv_bfloat16, 3>, grid, per_block, 0, st, g, (const __nv_bfloat16*)dz, w, (__nv_bfloat16*)dx);
      else launch_k(dw_dx_s2_kernel<__nv_bfloat16, 5>, grid, per_block, 0, st, g, (const __nv_bfloat16*)dz, w, (__nv_bfloat16*)dx);
    } else {
      if (g.ks == 3) launch_k(dw_dx_s2_kernel<float, 3>, grid, per_block, 0, st, g, (const float*)dz, w, (float*)dx);
      else launch_k(dw_dx_s2_kernel<float, 5>, grid, per_block, 0, st, g, (const float*)dz, w, (float*)dx);
    }
    DFX_LAUNCH_CHECK("dwconv dx (stride 2)");
    return DFX_OK;
  }
  Plan pl;
  const int pt = g.ks - 1 - g.pt, pleft = g.ks - 1 - g.pl;
  if (!make_plan(g.N, g.Ho, g.Wo, g.Hi, g.Wi, g.C, g.ks, 1, pt, pleft, esz, MODE_CONV, &pl))
    return fail(DFX_ERR_UNSUPPORTED, "dwconv dx: shape not supported by the TMA ring path");
  pl.p.flip = 1;
  CUtensorMap mdz;
  if (int rc = tmap(&mdz, dz, esz, g.N, g.Ho, g.Wo, g.C, pl.p.Cb, pl.p.Wb)) return rc;
  DzConsts none{};
  return dtype == DFX_BF16 ? dispatch_ring<__nv_bfloat16, MODE_CONV>(g.ks, 1, pl, mdz, mdz, mdz, w, dx, nullptr, none, st)
                           : dispatch_ring<float, MODE_CONV>(g.ks, 1, pl, mdz, mdz, mdz, w, dx, nullptr, none, st);
}

}  // namespace dfx
