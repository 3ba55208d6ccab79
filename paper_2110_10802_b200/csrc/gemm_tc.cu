// gemm_tc.cu — bf16 contractions on the 5th-generation tensor cores (sm_100a).
//
// Replaces the f64 numpy contractions of the reference (Gemm frontend.py:369-405,
// MatMul 335-366, Einsum 408-481 and their VJPs autodiff.py:1363-1459) for the
// BERT encoder: QKV / out-proj / FFN GEMMs, the batched attention
// contractions, and every dgrad / wgrad of the backward pass, each carrying
// its epilogue (bias, bias+GELU with pre-activation stash, GELU-backward,
// residual add).
//
// Design (persistent, warp-specialised, one CTA per SM):
//   warp 0 (1 thread)  TMA producer: A and B tiles -> 128B-swizzled smem ring
//                      (STAGES deep), completion via mbarrier tx-count.
//   warp 1 (1 thread)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16,
//                      128 x BN x 16 per instruction, fp32 accumulator in TMEM;
//                      tcgen05.commit frees smem stages / publishes accumulators.
//   warps 2-5          epilogue: tcgen05.ld (32 lanes x 32 columns) -> fused
//                      epilogue math in registers -> 16-byte global stores.
//   TMEM holds two BN-column accumulators, so the epilogue of tile i overlaps
//   the MMAs of tile i+1.
// Operands may be K-major or MN-major (the UMMA descriptor's major bit), so
// dgrad and wgrad GEMMs read activations and weights in place without
// transposes.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "gemm.h"

namespace dfx {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle atom row
constexpr int kThreads = 192;

template <int BN> struct TcCfg {
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

struct TcParams {
  int64_t m, n, k;
  int64_t batch2;
  int32_t m_tiles, n_tiles, k_blocks, num_tiles;
  int32_t a_mn, b_mn;  // operand is MN-major
  int32_t epilogue;
  float alpha, beta;
  const float* bias;
  void* d;
  int64_t d_stride_m, d_stride_b1, d_stride_b2;
  const void* aux;
  int64_t aux_stride_m, aux_stride_b1, aux_stride_b2;
  void* aux_out;
  int64_t aux_out_stride_m, aux_out_stride_b1, aux_out_stride_b2;
};

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), sm100 version 1.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: bf16 x bf16 -> f32, M=128, N=BN, majors.
__host__ __device__ constexpr uint32_t make_idesc(int n, int a_mn, int b_mn) {
  return (1u << 4)                      // c_format = F32
         | (1u << 7)                    // a_format = BF16
         | (1u << 10)                   // b_format = BF16
         | ((uint32_t)a_mn << 15)       // a major
         | ((uint32_t)b_mn << 16)       // b major
         | ((uint32_t)(n >> 3) << 17)   // N >> 3
         | ((uint32_t)(BM >> 4) << 24); // M >> 4
}

template <typename TO> __device__ __forceinline__ void store32(TO* dst, const float (&v)[32]);
template <> __device__ __forceinline__ void store32<float>(float* dst, const float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
    reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
template <> __device__ __forceinline__ void store32<__nv_bfloat16>(__nv_bfloat16* dst, const float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 t;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&t);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
    reinterpret_cast<uint4*>(dst)[i] = t;
  }
}
template <typename TO> __device__ __forceinline__ void load32(const TO* src, float (&v)[32]);
template <> __device__ __forceinline__ void load32<float>(const float* src, float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float4 t = reinterpret_cast<const float4*>(src)[i];
    v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
  }
}
template <> __device__ __forceinline__ void load32<__nv_bfloat16>(const __nv_bfloat16* src, float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 t = reinterpret_cast<const uint4*>(src)[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&t);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      v[8 * i + 2 * j] = f.x; v[8 * i + 2 * j + 1] = f.y;
    }
  }
}

template <int BN, typename TO>
__global__ void __launch_bounds__(kThreads, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const TcParams p) {
  using Cfg = TcCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles_mn = p.m_tiles * p.n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      uint32_t it = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const int nb = t % p.n_tiles;
        const int mb = (t / p.n_tiles) % p.m_tiles;
        const int z = t / tiles_mn;
        const int b1 = (int)(z / p.batch2), b2 = (int)(z % p.batch2);
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
          if (p.a_mn) {
            tma_load_4d(&map_a, &full[s], sa, m0, k0, b2, b1);
            tma_load_4d(&map_a, &full[s], sa + 8192, m0 + 64, k0, b2, b1);
          } else {
            tma_load_4d(&map_a, &full[s], sa, k0, m0, b2, b1);
          }
          if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_4d(&map_b, &full[s], sb + j * 8192, n0 + 64 * j, k0, b2, b1);
          } else {
            tma_load_4d(&map_b, &full[s], sb, k0, n0, b2, b1);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      const uint32_t idesc = make_idesc(BN, p.a_mn, p.b_mn);
      // per-UMMA_K (16 elements) descriptor advance, in 16-byte units
      const uint32_t a_step = p.a_mn ? (2048 >> 4) : (32 >> 4);
      const uint32_t b_step = p.b_mn ? (2048 >> 4) : (32 >> 4);
      const uint32_t a_lbo = p.a_mn ? 8192 : 16, b_lbo = p.b_mn ? 8192 : 16;
      uint32_t it = 0, lt = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++lt) {
        const int acc = lt & 1;
        const uint32_t aph = (lt >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
          const uint64_t adesc = make_sdesc(sa, a_lbo, 1024);
          const uint64_t bdesc = make_sdesc(sb, b_lbo, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            tc_mma(tmem_d, adesc + (uint64_t)(kk * a_step), bdesc + (uint64_t)(kk * b_step), idesc,
                   (kb | kk) != 0);
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    uint32_t lt = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++lt) {
      const int nb = t % p.n_tiles;
      const int mb = (t / p.n_tiles) % p.m_tiles;
      const int z = t / tiles_mn;
      const int64_t b1 = z / p.batch2, b2 = z % p.batch2;
      const int acc = lt & 1;
      const uint32_t aph = (lt >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int64_t gm = (int64_t)mb * BM + q * 32 + lane;
      TO* drow = (TO*)p.d + b1 * p.d_stride_b1 + b2 * p.d_stride_b2 + gm * p.d_stride_m;
      const TO* xrow = p.aux ? (const TO*)p.aux + b1 * p.aux_stride_b1 + b2 * p.aux_stride_b2 + gm * p.aux_stride_m : nullptr;
      TO* orow = p.aux_out ? (TO*)p.aux_out + b1 * p.aux_out_stride_b1 + b2 * p.aux_out_stride_b2 + gm * p.aux_out_stride_m : nullptr;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        const int64_t gn = (int64_t)nb * BN + c * 32;
        if (gn >= p.n) break;  // n % 32 == 0 is required on this path
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
        if (p.epilogue == DFX_EPI_BIAS || p.epilogue == DFX_EPI_BIAS_GELU) {
          if (p.bias) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += __ldg(p.bias + gn + i);
          }
          if (p.epilogue == DFX_EPI_BIAS_GELU) {
            if (orow) store32<TO>(orow + gn, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = gelu_f(v[i]);
          }
        } else if (p.epilogue == DFX_EPI_GELU_BWD) {
          float a[32];
          load32<TO>(xrow + gn, a);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_f(a[i]);
        } else if (p.epilogue == DFX_EPI_ADD) {
          float a[32];
          load32<TO>(xrow + gn, a);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += p.beta * a[i];
        }
        store32<TO>(drow + gn, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(Cfg::TMEM_COLS)
                 : "memory");
  }
}

// ----------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// 4-D bf16 tensor map: dims (inner..outer) = {d0, d1, batch2, batch1}.
int make_map(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, int64_t s1, int64_t nb2,
             int64_t sb2, int64_t nb1, int64_t sb1, uint32_t box0, uint32_t box1) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(DFX_ERR_CUDA, "dfx_gemm: cuTensorMapEncodeTiled unavailable");
  const uint64_t esz = 2;
  cuuint64_t dims[4] = {d0, d1, (cuuint64_t)nb2, (cuuint64_t)nb1};
  // unused batch levels get a harmless 16B-multiple stride
  const uint64_t span = ((d1 * (uint64_t)s1 * esz) + 15) & ~uint64_t(15);
  cuuint64_t strides[3] = {(cuuint64_t)(s1 * esz), nb2 > 1 ? (cuuint64_t)(sb2 * esz) : span,
                           nb1 > 1 ? (cuuint64_t)(sb1 * esz) : span};
  cuuint32_t box[4] = {box0, box1, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DFX_ERR_CUDA, "dfx_gemm: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return DFX_OK;
}

int pick_bn(int64_t n) {
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  // minimise padded columns; ties prefer the wider tile
  const int64_t w256 = ((n + 255) / 256) * 256 - n, w128 = ((n + 127) / 128) * 128 - n;
  return w256 <= w128 ? 256 : 128;
}

template <int BN, typename TO>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const TcParams& tp, cudaStream_t st) {
  auto kfn = tc_gemm_kernel<BN, TO>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<BN>::SMEM);
    attr_set = true;
  }
  const int grid = std::min(tp.num_tiles, num_sms());
  kfn<<<grid, kThreads, TcCfg<BN>::SMEM, st>>>(ma, mb, tp);
  DFX_LAUNCH_CHECK("dfx_gemm (tcgen05)");
  return DFX_OK;
}

}  // namespace

bool gemm_tc_supported(const dfx_gemm_args& p) {
  if (p.force_simt || p.in_dtype != DFX_BF16) return false;
  if (p.out_dtype != DFX_BF16 && p.out_dtype != DFX_F32) return false;
  if (p.m <= 0 || p.n <= 0 || p.k <= 0) return false;
  if (p.m % BM || p.k % BK || p.n % 32) return false;
  const bool a_k = p.a_stride_k == 1, a_m = p.a_stride_m == 1;
  const bool b_k = p.b_stride_k == 1, b_n = p.b_stride_n == 1;
  if (!(a_k || a_m) || !(b_k || b_n)) return false;
  const int64_t a_ld = a_k ? p.a_stride_m : p.a_stride_k;
  const int64_t b_ld = b_k ? p.b_stride_n : p.b_stride_k;
  if (a_ld % 8 || b_ld % 8) return false;
  if ((p.batch2 > 1 && (p.a_stride_b2 % 8 || p.b_stride_b2 % 8)) ||
      (p.batch1 > 1 && (p.a_stride_b1 % 8 || p.b_stride_b1 % 8)))
    return false;
  if (!aligned16(p.a) || !aligned16(p.b) || !aligned16(p.d)) return false;
  const int osz = p.out_dtype == DFX_BF16 ? 2 : 4;
  if ((p.d_stride_m * osz) % 16) return false;
  if (p.aux && ((p.aux_stride_m * osz) % 16 || !aligned16(p.aux))) return false;
  if (p.aux_out && ((p.aux_out_stride_m * osz) % 16 || !aligned16(p.aux_out))) return false;
  if (p.batch1 * p.batch2 * (p.m / BM) * ((p.n + 63) / 64) > (1ll << 31)) return false;
  return true;
}

int gemm_tc(const dfx_gemm_args& p, cudaStream_t st) {
  const int bn = pick_bn(p.n);
  const bool a_mn = p.a_stride_k != 1, b_mn = p.b_stride_k != 1;
  CUtensorMap ma, mb;
  int rc;
  if (a_mn)
    rc = make_map(&ma, p.a, p.m, p.k, p.a_stride_k, p.batch2, p.a_stride_b2, p.batch1, p.a_stride_b1, 64, 64);
  else
    rc = make_map(&ma, p.a, p.k, p.m, p.a_stride_m, p.batch2, p.a_stride_b2, p.batch1, p.a_stride_b1, 64, BM);
  if (rc) return rc;
  if (b_mn)
    rc = make_map(&mb, p.b, p.n, p.k, p.b_stride_k, p.batch2, p.b_stride_b2, p.batch1, p.b_stride_b1, 64, 64);
  else
    rc = make_map(&mb, p.b, p.k, p.n, p.b_stride_n, p.batch2, p.b_stride_b2, p.batch1, p.b_stride_b1, 64, bn);
  if (rc) return rc;
  TcParams tp;
  tp.m = p.m; tp.n = p.n; tp.k = p.k; tp.batch2 = p.batch2;
  tp.m_tiles = (int)(p.m / BM);
  tp.n_tiles = (int)((p.n + bn - 1) / bn);
  tp.k_blocks = (int)(p.k / BK);
  tp.num_tiles = (int)(p.batch1 * p.batch2 * tp.m_tiles * tp.n_tiles);
  tp.a_mn = a_mn; tp.b_mn = b_mn;
  tp.epilogue = p.epilogue; tp.alpha = p.alpha; tp.beta = p.beta; tp.bias = p.bias;
  tp.d = p.d; tp.d_stride_m = p.d_stride_m; tp.d_stride_b1 = p.d_stride_b1; tp.d_stride_b2 = p.d_stride_b2;
  tp.aux = p.aux; tp.aux_stride_m = p.aux_stride_m; tp.aux_stride_b1 = p.aux_stride_b1; tp.aux_stride_b2 = p.aux_stride_b2;
  tp.aux_out = p.aux_out; tp.aux_out_stride_m = p.aux_out_stride_m; tp.aux_out_stride_b1 = p.aux_out_stride_b1;
  tp.aux_out_stride_b2 = p.aux_out_stride_b2;
  const bool f32 = p.out_dtype == DFX_F32;
  if (bn == 256) return f32 ? launch_tc<256, float>(ma, mb, tp, st) : launch_tc<256, __nv_bfloat16>(ma, mb, tp, st);
  if (bn == 128) return f32 ? launch_tc<128, float>(ma, mb, tp, st) : launch_tc<128, __nv_bfloat16>(ma, mb, tp, st);
  return f32 ? launch_tc<64, float>(ma, mb, tp, st) : launch_tc<64, __nv_bfloat16>(ma, mb, tp, st);
}

}  // namespace dfx
