// common.cuh — shared device/host helpers for the dfx sm_100a kernels.
#pragma once
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "dfx.h"

namespace dfx {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
void count_launch(int n = 1);
int num_sms();

#define DFX_REQUIRE(cond, code, msg)                     \
  do {                                                   \
    if (!(cond)) return ::dfx::fail((code), (msg));      \
  } while (0)

#define DFX_LAUNCH_CHECK(what)                                                        \
  do {                                                                                \
    cudaError_t e__ = cudaGetLastError();                                             \
    if (e__ != cudaSuccess)                                                           \
      return ::dfx::fail(DFX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e__)); \
    ::dfx::count_launch();                                                            \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
inline bool aligned_n(const void* p, int n) { return (reinterpret_cast<uintptr_t>(p) % n) == 0; }

// ------------------------------------------------- programmatic dependent launch
// Every kernel is launched with programmatic stream serialization: it
// signals `launch_dependents` as soon as it starts (safe — the dependent grid
// is only scheduled once EVERY CTA of this grid has started, so it can never
// starve this grid of SMs) and executes `wait` before its first read of data
// produced by the previous kernel.  Kernel N+1's launch latency and prologue
// (barrier init, TMEM allocation, descriptor prefetch) then overlap kernel N's
// tail, inside CUDA graphs too.  Both are no-ops without a programmatic edge.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  static const bool no_pdl = getenv("DFX_NO_PDL") != nullptr;  // A/B measurements only
  cfg.numAttrs = no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- device
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Vector of V elements of storage type T, loaded/stored as one transaction.
template <typename T, int V> struct Vec;

template <int V> struct Vec<float, V> {
  float v[V];
  __device__ __forceinline__ void load(const float* p) {
    if constexpr (V == 4) {
      float4 t = *reinterpret_cast<const float4*>(p);
      v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else if constexpr (V == 8) {
      float4 a = reinterpret_cast<const float4*>(p)[0];
      float4 b = reinterpret_cast<const float4*>(p)[1];
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = p[i];
    }
  }
  __device__ __forceinline__ void load_nc(const float* p) {
    if constexpr (V == 4) {
      float4 t = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
      load(p);
    }
  }
  __device__ __forceinline__ void store(float* p) const {
    if constexpr (V == 4) {
      *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (V == 8) {
      reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) p[i] = v[i];
    }
  }
};

template <int V> struct Vec<__nv_bfloat16, V> {
  float v[V];
  __device__ __forceinline__ void load(const __nv_bfloat16* p) {
    if constexpr (V == 8) {
      uint4 t = *reinterpret_cast<const uint4*>(p);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x; v[2 * i + 1] = f.y;
      }
    } else if constexpr (V == 4) {
      uint2 t = *reinterpret_cast<const uint2*>(p);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x; v[2 * i + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = __bfloat162float(p[i]);
    }
  }
  __device__ __forceinline__ void load_nc(const __nv_bfloat16* p) { load(p); }
  __device__ __forceinline__ void store(__nv_bfloat16* p) const {
    if constexpr (V == 8) {
      uint4 t;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      *reinterpret_cast<uint4*>(p) = t;
    } else if constexpr (V == 4) {
      uint2 t;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
      for (int i = 0; i < 2; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      *reinterpret_cast<uint2*>(p) = t;
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) p[i] = __float2bfloat16_rn(v[i]);
    }
  }
};

// V keep flags (u8) -> float multipliers {0, scale}.
template <int V>
__device__ __forceinline__ void load_keep(const uint8_t* p, float scale, float (&m)[V]) {
  if constexpr (V == 8) {
    uint2 t = *reinterpret_cast<const uint2*>(p);
    const uint8_t* b = reinterpret_cast<const uint8_t*>(&t);
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = b[i] ? scale : 0.f;
  } else if constexpr (V == 4) {
    uint32_t t = *reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = ((t >> (8 * i)) & 0xff) ? scale : 0.f;
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) m[i] = p[i] ? scale : 0.f;
  }
}

// Bit-packed keep flags (bit e % 8 of byte e / 8 = keep of flat element e,
// the little-endian byte view of kernels.pack_keep_bits' int32 words): the V
// flags of elements e .. e+V-1 (e % V == 0, V <= 8) -> {0, scale}.
template <int V>
__device__ __forceinline__ void load_keep_bits(const uint8_t* kb, size_t e, float scale, float (&m)[V]) {
  const uint32_t bits = (uint32_t)__ldg(kb + (e >> 3)) >> (e & 7);
#pragma unroll
  for (int i = 0; i < V; ++i) m[i] = ((bits >> i) & 1u) ? scale : 0.f;
}

__device__ __forceinline__ float sigmoid_f(float u) { return 1.f / (1.f + __expf(-u)); }

__device__ __forceinline__ float gelu_f(float x) {
  const float c0 = 0.044715f, c1 = 0.7978845608028654f;
  float u = c1 * (x + c0 * x * x * x);
  return 0.5f * x * (1.f + tanhf(u));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float c0 = 0.044715f, c1 = 0.7978845608028654f;
  float u = c1 * (x + c0 * x * x * x);
  float t = tanhf(u);
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c1 * (1.f + 3.f * c0 * x * x);
}

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }


// Fixed-order f64 sum of nparts partial rows (row stride ld floats) at column
// col, for a 1024-thread block whose 32 lanes own 32 consecutive columns: warp
// w takes rows w, w + 32, ... in four independent chains (rows w + 128 i + 32 k
// into chain k), the chains add in order, then warp 0 adds the 32 warps in
// order.  Returns the column total in warp 0 (bitwise reproducible; ~nparts/128
// dependent adds per thread instead of nparts/8).
__device__ __forceinline__ double sum_part_rows(int nparts, const float* __restrict__ part, size_t ld, int col,
                                                bool ok, double (*red)[33]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (ok) {
    int b = w;
    for (; b + 96 < nparts; b += 128) {
      a0 += part[(size_t)b * ld + col];
      a1 += part[(size_t)(b + 32) * ld + col];
      a2 += part[(size_t)(b + 64) * ld + col];
      a3 += part[(size_t)(b + 96) * ld + col];
    }
    for (; b < nparts; b += 32) a0 += part[(size_t)b * ld + col];
  }
  red[w][lane] = ((a0 + a1) + a2) + a3;
  __syncthreads();
  double v = 0.0;
  if (w == 0) {
#pragma unroll 8
    for (int j = 0; j < 32; ++j) v += red[j][lane];
  }
  return v;
}

}  // namespace dfx
