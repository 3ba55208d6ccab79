// gemm_tc.cu — bf16 contractions on the 5th-generation tensor cores (sm_100a).
//
// Replaces the f64 numpy contractions of the reference (Gemm frontend.py:369-405,
// MatMul 335-366, Einsum 408-481 and their VJPs autodiff.py:1363-1459) for the
// BERT encoder: QKV / out-proj / FFN GEMMs, the batched attention
// contractions, and every dgrad / wgrad of the backward pass, each carrying
// its epilogue (bias, bias+GELU with pre-activation stash, GELU-backward,
// residual add).
//
// Design (persistent, warp-specialised, one CTA per SM, 10 warps):
//   warp 0 (1 thread)  TMA producer: A and B tiles -> 128B-swizzled smem ring
//                      (STAGES deep), completion via mbarrier tx-count.
//   warp 1 (1 thread)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16,
//                      128 x BN x 16 per instruction, fp32 accumulator in TMEM;
//                      tcgen05.commit frees smem stages / publishes accumulators.
//   warps 2-9          epilogue, two warps per TMEM lane quadrant (each owns
//                      half of the tile's columns): tcgen05.ld (32 lanes x 32
//                      columns) -> fused epilogue math in registers -> staged
//                      in shared memory -> TMA bulk-tensor store (full 32x32
//                      boxes, out-of-range rows/cols clipped by the TMA unit).
//   TMEM holds two BN-column accumulators, so the epilogue of tile i overlaps
//   the MMAs of tile i+1.
// Operands may be K-major or MN-major (the UMMA descriptor's major bit), so
// dgrad and wgrad GEMMs read activations and weights in place without
// transposes.  GEMMs with too few output tiles to fill the 148 SMs (the
// 768-wide weight gradients) split K; fp32 partial tiles go to a workspace and
// a fixed-order reduction writes the result (deterministic, no atomics).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gemm.h"
#include "tc_ptx.cuh"

namespace dfx {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle atom row
constexpr int kEpiWarps = 16;
constexpr int kThreads = (2 + kEpiWarps) * 32;
constexpr int kXfThreads = 256;  // A-operand transform warps of the XF = 1 (excite-folded) instantiation (2 per SMSP)
// Epilogue unit geometry (shared with the host, which builds the bulk-store
// tensor maps): columns per epilogue warp, and bytes per staged unit row.
__host__ __device__ constexpr int epi_wcols(int bn) { return bn <= 128 ? bn : bn / 4; }
__host__ __device__ constexpr int epi_ub(int bn, int esz) {
  return (epi_wcols(bn) * esz) % 64 == 0 ? 64 : ((epi_wcols(bn) * esz) % 32 == 0 ? 32 : 16);
}

template <int BN, int CG = 1> struct TcCfg {
  // epilogue staging (TMA store source) per epilogue warp, and the smem ring
  // depth: both sized so the CTA uses <= 227 KB
  static constexpr int EPI_WARP_BYTES = 4096;  // output unit + aux unit, 32 rows x 64 B each
  static constexpr int STAGES = CG == 2 ? (BN >= 192 ? 5 : 6) : (BN == 256 ? 3 : (BN == 192 ? 4 : (BN == 128 ? 5 : 6)));
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN / CG * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // TMEM accumulator buffers: narrow tiles (BN <= 128) keep FOUR so the
  // mainloop runs up to three tiles ahead of the epilogue, and the 16
  // epilogue warps split into four groups that each drain a whole tile
  // (skinny GEMMs are epilogue-bound); wide tiles keep two.
  static constexpr int NACC = BN <= 128 ? 4 : 2;
  static constexpr int TMEM_COLS = NACC * BN < 32 ? 32 : (BN == 192 ? 512 : NACC * BN);
  static constexpr int EPI_BYTES = kEpiWarps * EPI_WARP_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 512 /*barriers*/;
};

struct TcParams {
  int64_t m, n, k;
  int64_t batch2;
  int32_t m_tiles, n_tiles, k_blocks, num_tiles;
  int32_t splits, kb_per_split;  // split-K (splits > 1 -> fp32 partials to the workspace map)
  int32_t a_mn, b_mn;            // operand is MN-major
  int32_t epilogue;
  int32_t has_aux_out;
  float alpha, beta;
  const float* bias;
  const void* aux;
  int64_t aux_stride_m, aux_stride_b1, aux_stride_b2;
  void* d;
  int64_t d_stride_m, d_stride_b1, d_stride_b2;
  void* aux_out;
  int64_t aux_out_stride_m, aux_out_stride_b1, aux_out_stride_b2;
  float* part;  // split-K partials [split][z][m][n]
  unsigned long long* trace;  // debug timeline (tools/gemm_trace.py), normally null
  // XF = 1 (dfx_gemm_excite): the K-major A operand is a BatchNorm input z;
  // the transform warps turn each landed A stage into
  //   y = swish(z * rstd*gamma + (beta - mean*rstd*gamma)) * gate[row / x_hw][k]
  // in place before the MMA reads it, and (optionally) write y to x_y [m][k]
  const float *x_mean, *x_rstd, *x_gamma, *x_beta;  // [k]
  const float* x_gate;                               // [images][k]
  int64_t x_hw;                                      // A rows per image
  __nv_bfloat16* x_y;                                // [m][k] or null
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot)                                                                       \
  do {                                                                                    \
    if (p.trace) p.trace[(size_t)blockIdx.x * 32 + (slot)] = gtime();                    \
  } while (0)

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// bf16-output epilogues use the hardware tanh (error far below bf16 rounding)
template <typename TO> __device__ __forceinline__ float gelu_epi(float x) {
  if constexpr (sizeof(TO) == 2) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.f + tanh_fast(u));
  } else {
    return gelu_f(x);
  }
}
template <typename TO> __device__ __forceinline__ float gelu_grad_epi(float x) {
  if constexpr (sizeof(TO) == 2) {
    const float c0 = 0.044715f, c1 = 0.7978845608028654f;
    const float t = tanh_fast(c1 * (x + c0 * x * x * x));
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c1 * (1.f + 3.f * c0 * x * x);
  } else {
    return gelu_grad_f(x);
  }
}

// ---- epilogue staging: a warp owns 32 rows; a staging unit is 32 rows x
// UB bytes (UB = 128, or 64 for the narrowest tiles) of one output tensor.
// Thread t writes row t; 16-byte chunk j of row r lives at chunk j ^ (r % L)
// (L = UB / 16 chunks per row) so both the row-wise writes and the
// column-coalesced read-back hit distinct banks.

// Stage this thread's 16 fp32 values (row `lane`, element offset `e0` within
// the unit) as TO / read them back.
// 16-byte chunk permutation of row r: the TMA SWIZZLE_64B (L = 4) / 32B
// (L = 2) pattern, so a staged unit is also a bulk-tensor-store source; both
// the row-per-lane writes and the row-wise reads are bank-conflict free.
template <int L> __device__ __forceinline__ int swz(int r) {
  return L == 4 ? ((r >> 1) & 3) : (L == 2 ? ((r >> 2) & 1) : 0);
}
template <typename TO, int L>
__device__ __forceinline__ void stage16(uint32_t base, int lane, int e0, const float (&v)[16]) {
  constexpr int EPC = 16 / (int)sizeof(TO);
#pragma unroll
  for (int j = 0; j < 16 / EPC; ++j) {
    const int chunk = e0 / EPC + j;
    sts128(base + lane * (L * 16) + ((chunk ^ swz<L>(lane)) * 16), pack4<TO>(&v[j * EPC]));
  }
}
template <typename TO, int L>
__device__ __forceinline__ void unstage16(uint32_t base, int lane, int e0, float (&v)[16]) {
  constexpr int EPC = 16 / (int)sizeof(TO);
#pragma unroll
  for (int j = 0; j < 16 / EPC; ++j) {
    const int chunk = e0 / EPC + j;
    unpack4<TO>(lds128(base + lane * (L * 16) + ((chunk ^ swz<L>(lane)) * 16)), &v[j * EPC]);
  }
}
// Decompose a linear tile index: n fastest, then m, then batch, then split.
struct TileIdx {
  int nb, mb, b1, b2, z, split;
};
__device__ __forceinline__ TileIdx tile_of(int t, const TcParams& p) {
  TileIdx r;
  r.nb = t % p.n_tiles;
  int rest = t / p.n_tiles;
  r.mb = rest % p.m_tiles;
  rest /= p.m_tiles;
  const int nz = p.num_tiles / (p.m_tiles * p.n_tiles * p.splits);
  r.z = rest % nz;
  r.split = rest / nz;
  r.b1 = (int)(r.z / p.batch2);
  r.b2 = (int)(r.z % p.batch2);
  return r;
}

// CG = 1: one CTA per 128 x BN tile.  CG = 2: a CTA pair (cluster of 2) per
// 256 x BN tile: each CTA loads its 128 rows of A and BN/2 columns of B, the
// leader issues tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' shared
// memory, and each CTA's TMEM receives its 128 accumulator rows.  Halving B
// traffic per SM raises the flop-per-L2-byte ratio from 85 to 128.
template <int BN, typename TO, int CG, int XF = 0>
__global__ void __launch_bounds__(kThreads + XF * kXfThreads, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_d, const __grid_constant__ CUtensorMap map_o,
               const __grid_constant__ CUtensorMap map_x, const TcParams p) {
  using Cfg = TcCfg<BN, CG>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int BN_LOAD = BN / CG;  // B columns each CTA loads
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + Cfg::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  constexpr int NACC = Cfg::NACC;
  constexpr int EPI_GROUP_WARPS = NACC == 4 ? 4 : kEpiWarps;  // warps draining one tile
  uint64_t* tfull = empty + STAGES;  // [NACC]
  uint64_t* tempty = tfull + NACC;   // [NACC]
  uint64_t* xbar = tempty + NACC;    // [kEpiWarps]: aux-operand unit landed
  uint64_t* xfull = xbar + kEpiWarps;  // [STAGES] (XF): A stage transformed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfull + (XF ? STAGES : 0));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TRACE(0);
  uint32_t rank = 0;
  if constexpr (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const bool leader = rank == 0;
  const int cluster_id = CG == 2 ? blockIdx.x / 2 : blockIdx.x;
  const int num_clusters = CG == 2 ? gridDim.x / 2 : gridDim.x;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < NACC; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], CG * EPI_GROUP_WARPS); }
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(&xbar[w], 1);
    if constexpr (XF != 0)
      for (int s = 0; s < STAGES; ++s) mbar_init(&xfull[s], kXfThreads / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(Cfg::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(Cfg::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // dependents launch only once this CTA holds its TMEM: a dependent grid's CTA
  // allocating first on this SM would block our alloc while it waits on us
  pdl_trigger();
  pdl_wait();  // setup above overlapped the previous kernel's tail
  if (threadIdx.x == 0) TRACE(1);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      // (CG = 2: both CTAs load their halves; transaction bytes land on the
      //  leader's full barrier, addressed by clearing the peer bit)
      const uint32_t full_addr_mask = CG == 2 ? 0xFEFFFFFFu : 0xFFFFFFFFu;
      uint32_t it = 0;
      for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
        const TileIdx ti = tile_of(t, p);
        const int m0 = ti.mb * BM * CG + (int)rank * BM;
        const int n0 = ti.nb * BN + (int)rank * BN_LOAD;
        const int kb0 = ti.split * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if (leader) mbar_expect_tx(&full[s], CG * Cfg::STAGE_BYTES);
          const uint32_t bar = smem_u32(&full[s]) & full_addr_mask;
          const int k0 = kb * BK;
          if (p.a_mn) {
            tma_load_4d_cg<CG>(&map_a, bar, sa, m0, k0, ti.b2, ti.b1);
            tma_load_4d_cg<CG>(&map_a, bar, sa + 8192, m0 + 64, k0, ti.b2, ti.b1);
          } else {
            tma_load_4d_cg<CG>(&map_a, bar, sa, k0, m0, ti.b2, ti.b1);
          }
          if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN_LOAD / 64; ++j)
              tma_load_4d_cg<CG>(&map_b, bar, sb + j * 8192, n0 + 64 * j, k0, ti.b2, ti.b1);
          } else {
            tma_load_4d_cg<CG>(&map_b, bar, sb, k0, n0, ti.b2, ti.b1);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------------------ MMA issuer
      const uint32_t idesc = make_idesc(BN, BM * CG, p.a_mn, p.b_mn);
      // per-UMMA_K (16 elements) descriptor advance, in 16-byte units
      const uint32_t a_step = p.a_mn ? (2048 >> 4) : (32 >> 4);
      const uint32_t b_step = p.b_mn ? (2048 >> 4) : (32 >> 4);
      const uint32_t a_lbo = p.a_mn ? 8192 : 16, b_lbo = p.b_mn ? 8192 : 16;
      uint32_t it = 0, lt = 0;
      for (int t = cluster_id; t < p.num_tiles; t += num_clusters, ++lt) {
        const TileIdx ti = tile_of(t, p);
        const int kb0 = ti.split * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
        const int acc = (int)(lt % NACC);
        const uint32_t aph = (lt / NACC) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(XF ? &xfull[s] : &full[s], ph);
          tc_fence_after();
          if (it == 0) TRACE(2);
          const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
          const uint64_t adesc = make_sdesc(sa, a_lbo, 1024);
          const uint64_t bdesc = make_sdesc(sb, b_lbo, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            tc_mma_cg<CG>(tmem_d, adesc + (uint64_t)(kk * a_step), bdesc + (uint64_t)(kk * b_step), idesc,
                          (kb != kb0 || kk != 0) ? 1u : 0u);
          tc_commit_cg<CG>(&empty[s]);
        }
        tc_commit_cg<CG>(&tfull[acc]);
        if (lt < 8) TRACE(3 + lt);
      }
    }
  } else if (XF != 0 && warp >= 2 + kEpiWarps) {
    // ------------------------------------------------- A transform (XF = 1)
    // Thread = one 16-byte chunk column (8 channels, fixed per stage) x XIT rows
    // (r0 + XSTEP i) of each landed [128 x 64] A stage: the per-channel BN
    // constants are loaded once per stage, the SE gate per row's image.  Rows
    // past m and channels past k become zeros (TMA zero-fill would otherwise
    // turn into swish(shift) * gate).  Same arithmetic as excite_kernel
    // (mbconv.cu), so y is bitwise the unfused path's.
    constexpr int XSTEP = kXfThreads / 8, XIT = BM / XSTEP;
    const int tt = threadIdx.x - (2 + kEpiWarps) * 32;
    const int ch = tt & 7, r0 = tt >> 3;
    const int hw = (int)p.x_hw;  // rows per image (>= XSTEP: one carry per row step below)
    uint32_t it = 0;
    for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
      const TileIdx ti = tile_of(t, p);
      const int64_t m0 = (int64_t)ti.mb * BM;
      // image of this thread's first row, then carried across its row steps (no divisions per chunk)
      const int first = (int)(m0 + r0);
      const int img0 = first / hw, rem0 = first - img0 * hw;
      for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        const int64_t k = (int64_t)kb * BK + ch * 8;
        const bool kin = k < p.k;  // k % 8 == 0 (host check)
        float sc[8], sh[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          sc[i] = kin ? __ldg(p.x_rstd + k + i) * __ldg(p.x_gamma + k + i) : 0.f;
          sh[i] = kin ? __ldg(p.x_beta + k + i) - __ldg(p.x_mean + k + i) * sc[i] : 0.f;
        }
        mbar_wait(&full[s], ph);
        const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
        int img = img0, rem = rem0;
#pragma unroll
        for (int i = 0; i < XIT; ++i) {
          const int r = r0 + XSTEP * i;
          const int64_t gm = m0 + r;
          if (i > 0) {
            rem += XSTEP;
            if (rem >= hw) { rem -= hw; ++img; }
          }
          const uint32_t addr = sa + r * 128 + ((ch ^ (r & 7)) << 4);
          uint4 out = make_uint4(0u, 0u, 0u, 0u);
          if (kin && gm < p.m) {
            const uint4 zv = lds128(addr);
            const float* gp = p.x_gate + (int64_t)img * p.k + k;
            const float4 g0 = __ldg(reinterpret_cast<const float4*>(gp));
            const float4 g1 = __ldg(reinterpret_cast<const float4*>(gp) + 1);
            const float se[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            float zf[8], yv[8];
            unpack4<__nv_bfloat16>(zv, zf);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float u = fmaf(zf[e], sc[e], sh[e]);
              yv[e] = u * fmaf(0.5f, tanh_fast(0.5f * u), 0.5f) * se[e];
            }
            out = pack4<__nv_bfloat16>(yv);
            if (p.x_y) *reinterpret_cast<uint4*>(p.x_y + gm * p.k + k) = out;
          }
          sts128(addr, out);
        }
        fence_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&xfull[s]);
      }
    }
  } else if (warp >= 2 && warp < 2 + kEpiWarps) {
    // -------------------------------------------------------------- epilogue
    // Four warps per TMEM lane quadrant (32 rows), each owning a quarter of
    // the tile's columns.  Per staging unit (32 rows x 64 bytes):
    // tcgen05.ld -> fused epilogue in registers -> swizzled smem -> coalesced
    // 16-byte global stores (and the mirror path for the aux operand).
    const int ew = warp - 2;          // 0..15
    const int q = warp & 3;           // TMEM lane quadrant this warp may access
    // NACC == 4: group ew>>2 drains every 4th tile, each warp all BN columns
    // of its quadrant; NACC == 2: all 16 warps share a tile, a quarter each
    const int grp = NACC == 4 ? (ew >> 2) : 0;
    const int part = NACC == 4 ? 0 : ew >> 2;
    constexpr int WCOLS = epi_wcols(BN);  // columns per warp
    static_assert(WCOLS == (NACC == 4 ? BN : BN / 4), "epilogue split");
    constexpr int ESZ = (int)sizeof(TO);
    // bytes per row per unit: 64 when the warp's columns tile by it (BN = 192 bf16: 32)
    constexpr int UB = epi_ub(BN, ESZ);
    constexpr int L = UB / 16;
    constexpr int UCOLS = UB / ESZ;   // columns per unit (bf16 32, f32 16)
    static_assert(WCOLS % UCOLS == 0, "warp columns must hold whole units");
    constexpr int UNITS = WCOLS / UCOLS;
    const bool split_out = p.splits > 1;
    const uint32_t st_out = smem_u32(epi_smem + ew * Cfg::EPI_WARP_BYTES);
    const uint32_t st_aux = st_out + 32 * UB;
    const bool unit_alpha = p.alpha == 1.f;
    const bool use_aux = p.splits <= 1 && (p.epilogue == DFX_EPI_GELU_BWD || p.epilogue == DFX_EPI_ADD);
    uint64_t* my_xbar = &xbar[ew];
    uint32_t xph = 0;  // parity of this warp's next aux unit
    // aux unit (32 rows x UB bytes) -> st_aux by bulk tensor load; it lands
    // in the staging layout unstage16 reads
    auto fetch_aux = [&](int64_t n0, int64_t m0, const TileIdx& ti) {
      if (lane == 0) {
        fence_async_smem();  // the slot's previous reads precede the async write
        mbar_expect_tx(my_xbar, 32 * (uint32_t)UB);
        tma_load_4d_cg<1>(&map_x, smem_u32(my_xbar), epi_smem + ew * Cfg::EPI_WARP_BYTES + 32 * UB, (int)n0, (int)m0,
                          ti.b2, ti.b1);
      }
    };
    uint32_t lt = 0, ucount = 0;
    for (int t = cluster_id; t < p.num_tiles; t += num_clusters, ++lt) {
      if (NACC == 4 && (int)(lt & 3) != grp) continue;  // another group's tile
      const TileIdx ti = tile_of(t, p);
      const int acc = (int)(lt % NACC);
      const uint32_t aph = (lt / NACC) & 1;
      // the first aux unit does not depend on the accumulator: fetch it
      // while the tile's MMAs finish
      if (use_aux && (int64_t)ti.nb * BN + part * WCOLS < p.n)
        fetch_aux((int64_t)ti.nb * BN + part * WCOLS, (int64_t)ti.mb * BM * CG + (int)rank * BM + q * 32, ti);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      if (ew == 0 && lane == 0 && lt < 8) TRACE(11 + lt);
      const int64_t m0 = (int64_t)ti.mb * BM * CG + (int)rank * BM + q * 32;
      // bulk-store coordinates beyond (n, m): batch (b2, b1), or (z, split)
      // of the split-K partials [split][z][m][n]
      const int sc2 = split_out ? ti.z : ti.b2, sc3 = split_out ? ti.split : ti.b1;
      const bool gelu = !split_out && p.epilogue == DFX_EPI_BIAS_GELU;
      const bool biased = !split_out && (p.epilogue == DFX_EPI_BIAS || gelu) && p.bias != nullptr;
      const bool store_pre = gelu && p.has_aux_out;
      // output-only units alternate between the warp's two staging slots, so
      // staging unit u+1 overlaps the bulk store of unit u
      const bool dbl = !use_aux && !store_pre;
#pragma unroll 1
      for (int u = 0; u < UNITS; ++u, ++ucount) {
        const int64_t n0 = (int64_t)ti.nb * BN + part * WCOLS + u * UCOLS;
        if (n0 >= p.n) break;
        const uint32_t so = (dbl && (ucount & 1)) ? st_aux : st_out;
        // the unit's accumulator columns: loads issued first, so their latency
        // overlaps the staging-slot wait and the aux fetch
        float vu[UCOLS];
        {
          const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + part * WCOLS + u * UCOLS;
#pragma unroll
          for (int hc = 0; hc < UCOLS / 16; ++hc) tmem_ld16_nowait(ta + hc * 16, vu + hc * 16);
        }
        if (lane == 0) {  // the slot's previous bulk store has read its source
          if (dbl)
            bulk_wait_read<1>();
          else
            bulk_wait_read<0>();
        }
        __syncwarp();
        if (use_aux) {
          mbar_wait(my_xbar, xph);
          xph ^= 1;
        }
        tmem_wait_ld();
#pragma unroll
        for (int hc = 0; hc < UCOLS / 16; ++hc) {
          const int col = part * WCOLS + u * UCOLS + hc * 16;  // column within the tile
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = vu[hc * 16 + i];
          if (!unit_alpha) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] *= p.alpha;
          }
          if (biased) {
            const int64_t gn = (int64_t)ti.nb * BN + col;
            if (gn + 16 <= p.n && (reinterpret_cast<uintptr_t>(p.bias + gn) & 15) == 0) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + gn) + i);
                v[4 * i] += b4.x; v[4 * i + 1] += b4.y; v[4 * i + 2] += b4.z; v[4 * i + 3] += b4.w;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] += (gn + i < p.n) ? __ldg(p.bias + gn + i) : 0.f;
            }
          }
          if (use_aux) {
            float a[16];
            unstage16<TO, L>(st_aux, lane, hc * 16, a);
            if (p.epilogue == DFX_EPI_GELU_BWD) {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] *= gelu_grad_epi<TO>(a[i]);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] += p.beta * a[i];
            }
          }
          if (gelu) {
            if (store_pre) stage16<TO, L>(st_aux, lane, hc * 16, v);  // the aux slot is free in this mode
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = gelu_epi<TO>(v[i]);
          }
          stage16<TO, L>(so, lane, hc * 16, v);
        }
        // staged unit -> one bulk tensor store (the TMA clips rows >= m / cols >= n)
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (store_pre) tma_store_4d(&map_o, st_aux, (int)n0, (int)m0, sc2, sc3);
          tma_store_4d(&map_d, so, (int)n0, (int)m0, sc2, sc3);
          bulk_commit();
        }
        // st_aux has been read: the next unit's aux streams in under this store
        if (use_aux && u + 1 < UNITS && n0 + UCOLS < p.n) fetch_aux(n0 + UCOLS, m0, ti);
      }
      tc_fence_before();
      __syncwarp();
      if (ew == 0 && lane == 0 && lt < 8) TRACE(19 + lt);
      if (lane == 0) {
        if (CG == 2 && !leader)
          mbar_arrive_remote(&tempty[acc], 0);  // the leader's MMA waits for both CTAs
        else
          mbar_arrive(&tempty[acc]);
      }
    }
  }
  if (warp >= 2 && warp < 2 + kEpiWarps && lane == 0) bulk_wait_all();  // this warp's bulk stores are complete
  tc_fence_before();
  if constexpr (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  if (threadIdx.x == 0) TRACE(27);
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg::TMEM_COLS)
                   : "memory");
  }
}

// Fixed-order split-K reduction: D = sum_s part[s] (f32 workspace).  Block =
// 32 output elements x 8 split lanes (warp w sums splits w, w+8, ...; the 8
// lane sums combine in order), so a 148-way split of a tiny weight gradient
// is 19 loads deep per thread instead of 148.
template <typename TO>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(int splits, int64_t Z, int64_t m, int64_t n,
                                                            const float* __restrict__ part, TO* __restrict__ d,
                                                            int64_t d_stride_m, int64_t d_stride_b1,
                                                            int64_t d_stride_b2, int64_t batch2) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8][33];
  const int64_t total = Z * m * n;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < total; base += (int64_t)gridDim.x * 32) {
    const int64_t i = base + lane;
    float acc = 0.f;
    if (i < total) {
#pragma unroll 4
      for (int s = w; s < splits; s += 8) acc += part[s * total + i];
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0 && i < total) {
      float v = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) v += red[j][lane];
      const int64_t col = i % n, row = (i / n) % m, z = i / (n * m);
      d[(z / batch2) * d_stride_b1 + (z % batch2) * d_stride_b2 + row * d_stride_m + col] = from_f<TO>(v);
    }
    __syncthreads();
  }
}

// few splits (the 768-wide BERT weight gradients): one element per thread
template <typename TO>
__global__ void __launch_bounds__(256) splitk_reduce_few_kernel(int splits, int64_t Z, int64_t m, int64_t n,
                                                                const float* __restrict__ part, TO* __restrict__ d,
                                                                int64_t d_stride_m, int64_t d_stride_b1,
                                                                int64_t d_stride_b2, int64_t batch2) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = Z * m * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += part[s * total + i];
    const int64_t col = i % n, row = (i / n) % m, z = i / (n * m);
    d[(z / batch2) * d_stride_b1 + (z % batch2) * d_stride_b2 + row * d_stride_m + col] = from_f<TO>(acc);
  }
}

// few splits, one contiguous f32 output matrix (the BERT / EfficientNet weight
// gradients): 16-byte vectors, 32-bit indices, fixed split order
__global__ void __launch_bounds__(256) splitk_reduce_vec4_kernel(int splits, int total4, int stride4,
                                                                 const float4* __restrict__ part,
                                                                 float4* __restrict__ d) {
  pdl_trigger();
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += gridDim.x * blockDim.x) {
    float4 acc = part[i];
    for (int s = 1; s < splits; ++s) {
      const float4 v = part[(size_t)s * stride4 + i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    d[i] = acc;
  }
}

// ----------------------------------------------------------------- host side
}  // namespace

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

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

// 4-D tensor map: dims (inner..outer) = {d0, d1, nb2, nb1}; strides in elements.
int make_map(CUtensorMap* map, const void* base, int esz, uint64_t d0, uint64_t d1, int64_t s1, int64_t nb2,
             int64_t sb2, int64_t nb1, int64_t sb1, uint32_t box0, uint32_t box1, bool swizzle128) {
  return make_map_sw(map, base, esz, d0, d1, s1, nb2, sb2, nb1, sb1, box0, box1,
                     swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
}

int make_map_sw(CUtensorMap* map, const void* base, int esz, uint64_t d0, uint64_t d1, int64_t s1, int64_t nb2,
                int64_t sb2, int64_t nb1, int64_t sb1, uint32_t box0, uint32_t box1, CUtensorMapSwizzle swz) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(DFX_ERR_CUDA, "dfx_gemm: cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {d0, d1, (cuuint64_t)nb2, (cuuint64_t)nb1};
  // unused batch levels get a harmless 16B-multiple stride
  const uint64_t span = ((d1 * (uint64_t)s1 * esz) + 15) & ~uint64_t(15);
  cuuint64_t strides[3] = {(cuuint64_t)(s1 * esz), nb2 > 1 ? (cuuint64_t)(sb2 * esz) : span,
                           nb1 > 1 ? (cuuint64_t)(sb1 * esz) : span * (uint64_t)std::max<int64_t>(nb2, 1)};
  cuuint32_t box[4] = {box0, box1, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DFX_ERR_CUDA, "dfx_gemm: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return DFX_OK;
}

namespace {

struct Plan {
  int bn, cg, splits, kb_per_split;
  int64_t tiles;  // work units (tiles x splits)
};

// Pick the tile shape by a wave-quantised cost model: time ~ waves x
// (per-SM tile work / relative per-SM throughput).  The 2-CTA 256 x 256 tile
// moves 2/3 of the L2 bytes per flop of a 1-CTA 128 x 256 tile (the GEMMs are
// L2-bandwidth-bound on B200), hence its higher relative throughput.
unsigned long long* g_trace = nullptr;

Plan plan(const dfx_gemm_args& p) {
  const int sms = num_sms();
  const char* force = getenv("DFX_GEMM_FORCE");  // "cg,bn" (tuning / tests only)
  if (force) {
    int fcg = 1, fbn = 256, fsp = 1;
    const int nf = sscanf(force, "%d,%d,%d", &fcg, &fbn, &fsp);
    if (nf >= 2 && (fcg == 1 || fcg == 2) && (fbn == 64 || fbn == 128 || fbn == 192 || fbn == 256) &&
        !(fcg == 2 && fbn == 192 && p.b_stride_k != 1) &&  // pair-192 loads B in 96-row K-major boxes only
        !(fcg == 2 && (fbn == 64 || p.m < 256)) && (fsp == 1 || p.epilogue == DFX_EPI_NONE)) {
      const int64_t z = p.batch1 * p.batch2;
      const int64_t kb = (p.k + BK - 1) / BK;  // K tail: TMA zero-fills past k
      const int64_t units = z * ((p.m + BM * fcg - 1) / (BM * fcg)) * ((p.n + fbn - 1) / fbn);
      Plan f{fbn, fcg, std::max(1, fsp), (int)kb, units};
      f.kb_per_split = (int)((kb + f.splits - 1) / f.splits);
      f.splits = (int)((kb + f.kb_per_split - 1) / f.kb_per_split);
      f.tiles = units * f.splits;
      return f;
    }
  }
  const int64_t z = p.batch1 * p.batch2;
  const int64_t kb = (p.k + BK - 1) / BK;  // K tail: TMA zero-fills past k
  struct Cand { int bn, cg; double thr; };
  // 192-wide single-CTA tiles fill the SMs on the narrow (768-wide) outputs:
  // 32 x 4 = 128 tiles in one wave instead of 16 x 3 pairs on 96 SMs
  // (measured: out 11.2 -> 9.6 us, ffn2 22.4 -> 20.0 us; tools/gemm_force_sweep.sh)
  // relative per-SM throughputs measured on the BERT shapes (tools/gemm_force_sweep.sh,
  // tools/wgrad_sweep.py): the 128-wide pair tile loses to the single-CTA one
  const Cand cands[] = {{256, 2, 1.5}, {128, 2, 0.75}, {256, 1, 1.0}, {192, 1, 1.2}, {128, 1, 0.85}, {64, 1, 0.6}};
  Plan best{64, 1, 1, (int)kb, 0};
  double best_cost = 1e30;
  for (const Cand& c : cands) {
    if (c.cg == 2 && (p.m < 256 || sms < 2)) continue;
    if (c.bn == 192 && p.n > 1024) continue;
    const int64_t units = z * ((p.m + BM * c.cg - 1) / (BM * c.cg)) * ((p.n + c.bn - 1) / c.bn);
    const int64_t slots = sms / c.cg;
    const double waves = (double)((units + slots - 1) / slots);
    // padded columns cost as much as real ones
    const double cost = waves * (double)c.bn / c.thr;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = Plan{c.bn, c.cg, 1, (int)kb, units};
    }
  }
  // one k-block (K <= 64: the EfficientNet expand / stem / project 1x1 convs
  // with 16-40 input channels): the GEMM is a pure epilogue stream, and the
  // pair tile halves the tile count (tools/skinny_sweep.py: 161 -> 107 us on
  // the 1.2M x 96 x 16 expand)
  if (z == 1 && kb == 1 && p.m >= 256 && sms >= 2 && p.epilogue == DFX_EPI_NONE) {
    const int64_t units = (p.m + 255) / 256 * ((p.n + 127) / 128);
    best = Plan{128, 2, 1, (int)kb, units};
  }
  // (tried: split-K-2 one-wave plans for the near-full-wave weight gradients —
  // faster alone, qkv wgrad 24.8 -> 19.6 us, but the BERT step 0.400 -> 0.409 ms
  // and the C5 step 11.17 -> 11.37 ms in context: extra partial traffic and a
  // reduce launch on the forked branch)
  // split K when a 1-CTA plan leaves most SMs idle (the 768-wide wgrads)
  if (best.cg == 1 && p.epilogue == DFX_EPI_NONE && best.tiles * 2 <= sms && kb >= 8) {
    if (best.bn == 256) {
      best.bn = 128;
      best.tiles = z * ((p.m + BM - 1) / BM) * ((p.n + 127) / 128);
    }
    int64_t s = std::min<int64_t>(sms / std::max<int64_t>(best.tiles, 1), kb / 4);
    // few-tile, long-K weight gradients (EfficientNet 1x1 convs: K = N*H*W
    // pixels, a 16..1152-square output) take up to one split per SM; the f32
    // partials stay under 64 MB
    const int64_t cap = std::max<int64_t>(8, (64ll << 20) / std::max<int64_t>(z * p.m * p.n * 4, 1));
    s = std::min<int64_t>(s, cap);
    if (s >= 2) best.splits = (int)s;
  }
  best.kb_per_split = (int)((kb + best.splits - 1) / best.splits);
  best.splits = (int)((kb + best.kb_per_split - 1) / best.kb_per_split);
  best.tiles *= best.splits;
  return best;
}

template <int BN, typename TO, int CG, int XF = 0>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md, const CUtensorMap& mo,
              const CUtensorMap& mx, const TcParams& tp, cudaStream_t st) {
  auto kfn = tc_gemm_kernel<BN, TO, CG, XF>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<BN, CG>::SMEM);
    attr_set = true;
  }
  const int clusters = std::min(tp.num_tiles, num_sms() / CG);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * CG);
  cfg.blockDim = dim3(kThreads + XF * kXfThreads);
  cfg.dynamicSmemBytes = TcCfg<BN, CG>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see common.cuh
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, ma, mb, md, mo, mx, tp);
  if (e != cudaSuccess) return fail(DFX_ERR_CUDA, std::string("dfx_gemm (tcgen05) launch: ") + cudaGetErrorString(e));
  DFX_LAUNCH_CHECK("dfx_gemm (tcgen05)");
  return DFX_OK;
}

template <typename TO>
int launch_tc_any(int bn, int cg, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                  const CUtensorMap& mo, const CUtensorMap& mx, const TcParams& tp, cudaStream_t st) {
  if (cg == 2) {
    if (bn == 256) return launch_tc<256, TO, 2>(ma, mb, md, mo, mx, tp, st);
    if (bn == 192) return launch_tc<192, TO, 2>(ma, mb, md, mo, mx, tp, st);
    return launch_tc<128, TO, 2>(ma, mb, md, mo, mx, tp, st);
  }
  if (bn == 256) return launch_tc<256, TO, 1>(ma, mb, md, mo, mx, tp, st);
  if (bn == 192) return launch_tc<192, TO, 1>(ma, mb, md, mo, mx, tp, st);
  if (bn == 128) return launch_tc<128, TO, 1>(ma, mb, md, mo, mx, tp, st);
  return launch_tc<64, TO, 1>(ma, mb, md, mo, mx, tp, st);
}

}  // namespace

void gemm_tc_set_trace(void* buf) { g_trace = reinterpret_cast<unsigned long long*>(buf); }

// D[m][n] = y · Wᵀ with y = swish(BN(z)) * gate formed on the fly from the
// K-major A operand z (the SE excite folded into the project 1x1 GEMM of an
// MBConv block); y itself is also written when y_out is set (the weight
// gradient reads it).  Single-CTA tiles (the transform warps own one CTA's A).
int gemm_excite(int64_t m, int64_t k, int64_t n, const void* z, int64_t hw, const float* mean, const float* rstd,
                const float* gamma, const float* beta, const float* gate, const void* w, void* d, void* y_out,
                cudaStream_t st) {
  DFX_REQUIRE(m > 0 && n > 0 && k > 0 && hw > 0, DFX_ERR_SHAPE, "dfx_gemm_excite: empty extent");
  DFX_REQUIRE(k % 8 == 0 && n % 8 == 0, DFX_ERR_SHAPE, "dfx_gemm_excite: k and n must be multiples of 8");
  DFX_REQUIRE(hw >= kXfThreads / 8 && m < (1ll << 31), DFX_ERR_UNSUPPORTED,
              "dfx_gemm_excite: needs >= 32 rows per image");
  DFX_REQUIRE(z && w && d && mean && rstd && gamma && beta && gate, DFX_ERR_SHAPE, "dfx_gemm_excite: null operand");
  DFX_REQUIRE(aligned16(z) && aligned16(w) && aligned16(d) && aligned16(gate) && (!y_out || aligned16(y_out)),
              DFX_ERR_ALIGN, "dfx_gemm_excite: operands must be 16-byte aligned");
  dfx_gemm_args g{};
  g.in_dtype = DFX_BF16; g.out_dtype = DFX_BF16; g.epilogue = DFX_EPI_NONE;
  g.m = m; g.n = n; g.k = k; g.batch1 = 1; g.batch2 = 1;
  g.a = z; g.a_stride_m = k; g.a_stride_k = 1;
  g.b = w; g.b_stride_n = k; g.b_stride_k = 1;
  g.d = d; g.d_stride_m = n;
  g.alpha = 1.f;
  Plan pl = plan(g);
  const int bn = pl.cg == 2 ? (n > 128 ? 256 : 128) : pl.bn;  // one CTA per tile
  CUtensorMap ma, mb;
  int rc = make_map(&ma, z, 2, k, m, k, 1, 0, 1, 0, 64, BM, true);
  if (rc) return rc;
  rc = make_map(&mb, w, 2, k, n, k, 1, 0, 1, 0, 64, bn, true);
  if (rc) return rc;
  TcParams tp{};
  tp.m = m; tp.n = n; tp.k = k; tp.batch2 = 1;
  tp.m_tiles = (int)((m + BM - 1) / BM);
  tp.n_tiles = (int)((n + bn - 1) / bn);
  tp.k_blocks = (int)((k + BK - 1) / BK);
  tp.splits = 1; tp.kb_per_split = tp.k_blocks;
  tp.num_tiles = tp.m_tiles * tp.n_tiles;
  tp.a_mn = 0; tp.b_mn = 0;
  tp.epilogue = DFX_EPI_NONE;
  tp.alpha = 1.f; tp.beta = 0.f;
  tp.d = d; tp.d_stride_m = n;
  tp.trace = g_trace;
  tp.x_mean = mean; tp.x_rstd = rstd; tp.x_gamma = gamma; tp.x_beta = beta; tp.x_gate = gate; tp.x_hw = hw;
  tp.x_y = reinterpret_cast<__nv_bfloat16*>(y_out);
  const int ub = epi_ub(bn, 2);
  const CUtensorMapSwizzle oswz =
      ub == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : (ub == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE);
  CUtensorMap md;
  rc = make_map_sw(&md, d, 2, n, m, n, 1, 0, 1, 0, ub / 2, 32, oswz);
  if (rc) return rc;
  using T = __nv_bfloat16;
  if (bn == 256) return launch_tc<256, T, 1, 1>(ma, mb, md, md, md, tp, st);
  if (bn == 192) return launch_tc<192, T, 1, 1>(ma, mb, md, md, md, tp, st);
  if (bn == 128) return launch_tc<128, T, 1, 1>(ma, mb, md, md, md, tp, st);
  return launch_tc<64, T, 1, 1>(ma, mb, md, md, md, tp, st);
}

size_t gemm_tc_workspace(const dfx_gemm_args& p) {
  if (!gemm_tc_supported(p)) return 0;
  const Plan pl = plan(p);
  if (pl.splits <= 1) return 0;
  return (size_t)pl.splits * p.batch1 * p.batch2 * p.m * p.n * sizeof(float) + 256;
}

bool gemm_tc_supported(const dfx_gemm_args& p) {
  if (p.force_simt || p.in_dtype != DFX_BF16) return false;
  if (p.out_dtype != DFX_BF16 && p.out_dtype != DFX_F32) return false;
  if (p.m <= 0 || p.n <= 0 || p.k <= 0) return false;
  // M and K tails: TMA zero-fills out-of-range rows/k, the epilogue clips rows
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
  const int ovec = 16 / osz;
  if (p.n % ovec || p.d_stride_m % ovec) return false;  // TMA store: 16-byte row strides
  if ((p.batch2 > 1 && p.d_stride_b2 % ovec) || (p.batch1 > 1 && p.d_stride_b1 % ovec)) return false;
  if (p.aux && ((p.aux_stride_m * osz) % 16 || !aligned16(p.aux))) return false;
  if (p.aux && ((p.batch2 > 1 && p.aux_stride_b2 % ovec) || (p.batch1 > 1 && p.aux_stride_b1 % ovec)))
    return false;  // bulk-tensor aux loads: 16-byte batch strides
  if (p.aux_out && (p.aux_out_stride_m % ovec || !aligned16(p.aux_out) ||
                    (p.batch2 > 1 && p.aux_out_stride_b2 % ovec) || (p.batch1 > 1 && p.aux_out_stride_b1 % ovec)))
    return false;
  if (p.batch1 * p.batch2 * ((p.m + BM - 1) / BM) * ((p.n + 63) / 64) * 8 > (1ll << 31)) return false;
  return true;
}

int gemm_tc(const dfx_gemm_args& p, cudaStream_t st) {
  const Plan pl = plan(p);
  const int bn = pl.bn;
  const bool a_mn = p.a_stride_k != 1, b_mn = p.b_stride_k != 1;
  DFX_REQUIRE(!(pl.cg == 2 && bn == 192 && b_mn), DFX_ERR_UNSUPPORTED, "dfx_gemm: 2-CTA 192 tile needs K-major B");
  CUtensorMap ma, mb;
  int rc;
  if (a_mn)
    rc = make_map(&ma, p.a, 2, p.m, p.k, p.a_stride_k, p.batch2, p.a_stride_b2, p.batch1, p.a_stride_b1, 64, 64, true);
  else
    rc = make_map(&ma, p.a, 2, p.k, p.m, p.a_stride_m, p.batch2, p.a_stride_b2, p.batch1, p.a_stride_b1, 64, BM, true);
  if (rc) return rc;
  if (b_mn)
    rc = make_map(&mb, p.b, 2, p.n, p.k, p.b_stride_k, p.batch2, p.b_stride_b2, p.batch1, p.b_stride_b1, 64, 64, true);
  else
    rc = make_map(&mb, p.b, 2, p.k, p.n, p.b_stride_n, p.batch2, p.b_stride_b2, p.batch1, p.b_stride_b1, 64,
                  bn / pl.cg, true);
  if (rc) return rc;
  const int64_t Z = p.batch1 * p.batch2;
  float* part = nullptr;
  if (pl.splits > 1) {
    const size_t need = (size_t)pl.splits * Z * p.m * p.n * sizeof(float);
    DFX_REQUIRE(p.workspace && p.workspace_bytes >= need && aligned16(p.workspace), DFX_ERR_WORKSPACE,
                "dfx_gemm: split-K needs dfx_gemm_workspace() bytes of workspace");
    part = (float*)p.workspace;  // partials [split][z][m][n] f32
  }
  TcParams tp;
  tp.m = p.m; tp.n = p.n; tp.k = p.k; tp.batch2 = p.batch2;
  tp.m_tiles = (int)((p.m + BM * pl.cg - 1) / (BM * pl.cg));
  tp.n_tiles = (int)((p.n + bn - 1) / bn);
  tp.k_blocks = (int)((p.k + BK - 1) / BK);
  tp.splits = pl.splits;
  tp.kb_per_split = pl.kb_per_split;
  tp.num_tiles = (int)pl.tiles;
  tp.a_mn = a_mn; tp.b_mn = b_mn;
  tp.epilogue = p.epilogue; tp.has_aux_out = p.aux_out != nullptr;
  tp.alpha = p.alpha; tp.beta = p.beta; tp.bias = p.bias;
  tp.aux = p.aux; tp.aux_stride_m = p.aux_stride_m; tp.aux_stride_b1 = p.aux_stride_b1; tp.aux_stride_b2 = p.aux_stride_b2;
  tp.d = p.d; tp.d_stride_m = p.d_stride_m; tp.d_stride_b1 = p.d_stride_b1; tp.d_stride_b2 = p.d_stride_b2;
  tp.aux_out = p.aux_out; tp.aux_out_stride_m = p.aux_out_stride_m; tp.aux_out_stride_b1 = p.aux_out_stride_b1;
  tp.aux_out_stride_b2 = p.aux_out_stride_b2;
  tp.part = part;
  tp.trace = g_trace;
  const bool f32 = pl.splits > 1 || p.out_dtype == DFX_F32;
  // bulk-store maps of the output (or the split-K partials) and the
  // pre-activation stash: one 32-row x UB-byte unit per box, swizzled like
  // the epilogue's staging
  const int esz = f32 ? 4 : 2;
  const int ub = epi_ub(bn, esz);
  const CUtensorMapSwizzle oswz =
      ub == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : (ub == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE);
  CUtensorMap md, mo;
  if (pl.splits > 1)
    rc = make_map_sw(&md, part, 4, p.n, p.m, p.n, Z, p.m * p.n, pl.splits, Z * p.m * p.n, ub / esz, 32, oswz);
  else
    rc = make_map_sw(&md, p.d, esz, p.n, p.m, p.d_stride_m, p.batch2, p.d_stride_b2, p.batch1, p.d_stride_b1,
                     ub / esz, 32, oswz);
  if (rc) return rc;
  if (p.aux_out) {
    rc = make_map_sw(&mo, p.aux_out, esz, p.n, p.m, p.aux_out_stride_m, p.batch2, p.aux_out_stride_b2, p.batch1,
                     p.aux_out_stride_b1, ub / esz, 32, oswz);
    if (rc) return rc;
  } else {
    mo = md;
  }
  CUtensorMap mx = md;  // aux operand (residual / GELU input), read per unit by bulk tensor loads
  if (p.aux && pl.splits <= 1 && (p.epilogue == DFX_EPI_GELU_BWD || p.epilogue == DFX_EPI_ADD)) {
    rc = make_map_sw(&mx, p.aux, esz, p.n, p.m, p.aux_stride_m, p.batch2, p.aux_stride_b2, p.batch1,
                     p.aux_stride_b1, ub / esz, 32, oswz);
    if (rc) return rc;
  }
  rc = f32 ? launch_tc_any<float>(bn, pl.cg, ma, mb, md, mo, mx, tp, st)
           : launch_tc_any<__nv_bfloat16>(bn, pl.cg, ma, mb, md, mo, mx, tp, st);
  if (rc || pl.splits <= 1) return rc;
  const int64_t total = Z * p.m * p.n;
  if (pl.splits <= 8 && p.out_dtype == DFX_F32 && Z == 1 && p.d_stride_m == p.n && p.n % 4 == 0 &&
      aligned16(p.d) && total / 4 < (1ll << 31)) {
    const int total4 = (int)(total / 4);
    const int grid = (int)std::min<int64_t>((total4 + 255) / 256, (int64_t)num_sms() * 4);
    launch_k(splitk_reduce_vec4_kernel, grid, 256, 0, st, pl.splits, total4, total4, (const float4*)part,
             (float4*)p.d);
  } else if (pl.splits <= 8) {
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
    if (p.out_dtype == DFX_F32)
      launch_k(splitk_reduce_few_kernel<float>, grid, 256, 0, st, pl.splits, Z, p.m, p.n, part, (float*)p.d,
               p.d_stride_m, p.d_stride_b1, p.d_stride_b2, p.batch2);
    else
      launch_k(splitk_reduce_few_kernel<__nv_bfloat16>, grid, 256, 0, st, pl.splits, Z, p.m, p.n, part,
               (__nv_bfloat16*)p.d, p.d_stride_m, p.d_stride_b1, p.d_stride_b2, p.batch2);
  } else {
    const int grid = (int)std::min<int64_t>((total + 31) / 32, (int64_t)num_sms() * 8);
    if (p.out_dtype == DFX_F32)
      launch_k(splitk_reduce_kernel<float>, grid, 256, 0, st, pl.splits, Z, p.m, p.n, part, (float*)p.d,
               p.d_stride_m, p.d_stride_b1, p.d_stride_b2, p.batch2);
    else
      launch_k(splitk_reduce_kernel<__nv_bfloat16>, grid, 256, 0, st, pl.splits, Z, p.m, p.n, part,
               (__nv_bfloat16*)p.d, p.d_stride_m, p.d_stride_b1, p.d_stride_b2, p.batch2);
  }
  DFX_LAUNCH_CHECK("dfx_gemm split-K reduce");
  return DFX_OK;
}

}  // namespace dfx
