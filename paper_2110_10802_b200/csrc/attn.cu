// attn.cu — fused scaled-masked-softmax attention on the 5th-gen tensor cores.
//
// Replaces, for one BERT encoder layer, the chain the reference evaluates as
// separate registry operators:
//     S  = Einsum bsnd,btnd->bnst (Q, K)            frontend.py:408-481
//     P  = Softmax(Div(S, divisor) + mask)          frontend.py:294, 175-188, 493-501
//     Pd = Mul(P, dropout mask)                     frontend.py:293
//     O  = Einsum bnst,btnd->bsnd (Pd, V)
// and its reverse pass (Einsum VJPs autodiff.py:1363-1415, Softmax VJP
// 1465-1484).  The reference recipe itself fuses exactly this into one
// per-query-row map (SURVEY.md §3D kernel 4, §8f.1); here the [B,NH,S,S]
// score / probability tensors never touch HBM.
//
// Work unit: a 128-row strip (128 TMEM lanes) of one (batch, head) against
// all S <= 512 keys.  Warp roles (576 threads): warp 0 = TMA producer, warp 1
// = TMEM allocator + single-thread tcgen05.mma issuer, warps 2..17 = 16
// softmax warps (four per TMEM lane quadrant).  The default forward and
// key-strip backward are persistent: one CTA per SM walks the strips.
//
//   fwd3   per 128-query strip, 128-key chunks: S = Q·Kᵀ (TMEM, double
//          buffered) -> online softmax, P̃d = exp2(S·c·log2e + mask·log2e -
//          m)·keep as bf16 in TMEM (the A operand of the PV MMA) -> O += P̃d·V
//          -> ctx = O·ks / rowsum.  (fwd, DFX_ATTN_FWD_LEGACY: the r01 exact
//          two-pass softmax over the whole 512-column score strip in TMEM.)
//          Also writes lse (log2 domain) and the dropout keep flags packed to
//          bits twice: row-major (for dQ) and transposed (for dK/dV, built
//          with warp ballots) — 2 x 3.1 MB instead of re-reading 25 MB of u8
//          keep flags in each backward kernel.
//   bwd_dq   per 128-query strip, 128-key chunks: S and dPd = dO·Vᵀ in TMEM,
//            dS = P∘(dPd∘M - D)·c in smem, dQ += dS·K.   D = rowsum(dO∘O).
//   bwd_kstrip per 128-key strip, 128-query chunks: Sᵀ = K·Qᵀ, dPdᵀ = V·dOᵀ,
//            dV += Pdᵀ·dO, dK += dSᵀ·Q; dSᵀ tiles to HBM for dQ = dS·K
//            (a tcgen05 GEMM), or dQ from bwd_dq (DFX_ATTN_BWD_LEGACY).
// No cross-CTA reductions: every output element is produced by one CTA in a
// fixed order (bitwise reproducible, no atomics).
#include <cuda.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "gemm.h"
#include "tc_ptx.cuh"

namespace dfx {
namespace {

constexpr int DH = 64;   // head dim = one 128-byte swizzle row of bf16
constexpr int QT = 128;  // rows per strip (TMEM lanes)
constexpr int kSoftWarps = 16;
constexpr int kAttnThreads = (2 + kSoftWarps) * 32;
constexpr int kMaxSeq = 512;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int KB = 1024;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// keep flags: 4 bytes (each 0 or 1) -> 4 bits (byte k -> bit k), no carries
__device__ __forceinline__ uint32_t keep_nibble(uint32_t w) { return (w * 0x01020408u) >> 24; }

// 32x32 bit-matrix transpose across a warp: lane i holds row word r_i on
// entry; on exit lane j holds the column word whose bit i is bit j of r_i.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int j = 16 >> t;
    const uint32_t m = masks[t];
    const uint32_t o = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((o >> j) & m)) : ((x & m) | ((o & m) << j));
  }
  return x;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// keep nibble (4 flags) -> 4 floats {0, v}: the flags enter the packed fp32
// math as multipliers, one LDS.128 per 4 columns instead of a shift / sign /
// AND chain per column
__device__ __forceinline__ void fill_keep_lut(float4* lut, int t, float v) {
  if (t < 16) lut[t] = make_float4(t & 1 ? v : 0.f, t & 2 ? v : 0.f, t & 4 ? v : 0.f, t & 8 ? v : 0.f);
}

// Store 8 consecutive bf16 (16 bytes) of row `r`, 16-byte chunk `ch` (0..7)
// of a [rows x 64] K-major SWIZZLE_128B tile at `tile`.
__device__ __forceinline__ void st_sw128(uint32_t tile, int r, int ch, uint4 v) {
  sts128(tile + r * 128 + ((ch ^ (r & 7)) << 4), v);
}

unsigned long long* g_attn_trace = nullptr;  // debug timeline (tools/attn_trace.py), normally null

__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ATRACE(slot)                                                                   \
  do {                                                                                 \
    if (p.trace) p.trace[(size_t)blockIdx.x * 16 + (slot)] = gtime_ns();              \
  } while (0)

struct AttnFwdParams {
  unsigned long long* trace;
  int B, NH, S, H;
  int64_t ld_ctx;
  const float* add_mask;  // [B, S] or null
  const uint8_t* keep;    // [B, NH, S, S] u8 or null
  float ks;               // keep scale 1/(1-p) (1 when keep is null)
  float sc2;              // inv_divisor * log2(e)
  __nv_bfloat16* ctx;
  float* lse;             // [B, NH, S], log2 domain
  uint32_t* kb_row;       // [B, NH, S, S/32] or null (written, or READ when kb_in)
  uint32_t* kb_col;       // [B, NH, S(key), S/32] or null
  int kb_in;              // keep flags arrive packed (kb_row is the input, keep is null)
};

// shared-memory plan of the forward kernel (bytes from a 1024-aligned base)
struct FwdSmem {
  static constexpr int Q = 0;
  static constexpr int K = Q + QT * 128;            // S keys x 128 B
  static constexpr int V = K + kMaxSeq * 128;
  static constexpr int P2 = V + kMaxSeq * 128;      // P chunks 4..7 (0..3 reuse K)
  static constexpr int MASK = P2 + 4 * QT * 128;    // S floats
  static constexpr int RED = MASK + kMaxSeq * 4;    // [2][4][128] floats
  static constexpr int LUT = RED + 2 * 4 * QT * 4;  // keep byte -> 4 bf16-pair masks
  static constexpr int BAR = LUT + 256 * 16;        // mbarriers
  static constexpr int TOTAL = BAR + 128 + KB;      // + alignment slack
};
static_assert(FwdSmem::TOTAL <= 227 * 1024, "attention forward exceeds shared memory");

__device__ __forceinline__ uint32_t p_chunk(uint32_t base, int c) {
  return c < 4 ? base + FwdSmem::K + c * (QT * 128) : base + FwdSmem::P2 + (c - 4) * (QT * 128);
}

__global__ void __launch_bounds__(kAttnThreads, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap map_qkv, const AttnFwdParams p) {
  // dynamic smem opens the CTA's window (no static smem in this kernel): it is
  // 1024-B aligned, and indexing it directly keeps every access LDS/STS
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + FwdSmem::BAR);
  // bar_p[j]: P of key chunk j (128 keys) complete in smem -> PV MMA of chunk j
  uint64_t *bar_qk = bar, *bar_v = bar + 1, *bar_s = bar + 2, *bar_o = bar + 4, *bar_p = bar + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);
  float* mask2 = reinterpret_cast<float*>(smem + FwdSmem::MASK);
  float* red_max = reinterpret_cast<float*>(smem + FwdSmem::RED);
  float* red_sum = red_max + 4 * QT;

  const int S = p.S;
  const int qblocks = S / QT;
  const int qb = blockIdx.x % qblocks;
  const int bh = blockIdx.x / qblocks;
  const int b = bh / p.NH, h = bh % p.NH;
  const int q0 = qb * QT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(bar_qk, 1);
    mbar_init(bar_v, 1);
    mbar_init(bar_s, 1);
    for (int j = 0; j < 4; ++j) mbar_init(&bar_p[j], kSoftWarps);
    mbar_init(bar_o, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_qkv)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dependents launch only once this CTA holds its TMEM: a dependent grid's CTA
  // allocating first on this SM would block our alloc while it waits on us
  pdl_trigger();
  pdl_wait();  // setup above overlapped the previous kernel's tail
  if (threadIdx.x == 0) ATRACE(0);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer
      const int row0 = b * S;
      mbar_expect_tx(bar_qk, (QT + S) * 128);
      const uint32_t bqk = smem_u32(bar_qk), bv = smem_u32(bar_v);
      tma_load_4d_cg<1>(&map_qkv, bqk, smem + FwdSmem::Q, h * DH, row0 + q0, 0, 0);
      tma_load_4d_cg<1>(&map_qkv, bqk, smem + FwdSmem::Q + 8 * KB, h * DH, row0 + q0 + 64, 0, 0);
      for (int j = 0; j < S / 64; ++j)
        tma_load_4d_cg<1>(&map_qkv, bqk, smem + FwdSmem::K + j * 8 * KB, p.H + h * DH, row0 + 64 * j, 0, 0);
      mbar_expect_tx(bar_v, S * 128);
      for (int j = 0; j < S / 64; ++j)
        tma_load_4d_cg<1>(&map_qkv, bv, smem + FwdSmem::V + j * 8 * KB, 2 * p.H + h * DH, row0 + 64 * j, 0, 0);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      mbar_wait(bar_qk, 0);
      tc_fence_after();
      ATRACE(1);
      const uint32_t idesc_s = make_idesc(128, QT, 0, 0);
      const uint64_t qdesc = make_sdesc(sbase + FwdSmem::Q, 16, 1024);
      for (int nb = 0; nb < S / 128; ++nb) {
        const uint64_t kdesc = make_sdesc(sbase + FwdSmem::K + nb * 16 * KB, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          tc_mma_cg<1>(tmem + nb * 128, qdesc + 2 * kk, kdesc + 2 * kk, idesc_s, kk > 0 ? 1u : 0u);
      }
      tc_commit_cg<1>(bar_s);
      mbar_wait(bar_v, 0);
      // O = P·V chunk by chunk as the softmax warps finish each 128-key chunk:
      // the PV MMAs of chunk j overlap the exp pass of chunk j+1.  O lives in
      // TMEM columns [0, 64) — S chunk 0, consumed before bar_p[0] fires.
      const uint32_t idesc_o = make_idesc(DH, QT, 0, 1);
      const uint64_t vdesc = make_sdesc(sbase + FwdSmem::V, 8 * KB, 1024);
      for (int j = 0; j < S / 128; ++j) {
        mbar_wait(&bar_p[j], 0);
        tc_fence_after();
#pragma unroll
        for (int kc = j * 8; kc < j * 8 + 8; ++kc) {
          const uint64_t pdesc = make_sdesc(p_chunk(sbase, kc >> 2), 16, 1024);
          tc_mma_cg<1>(tmem, pdesc + 2 * (kc & 3), vdesc + (uint64_t)(kc * (2048 >> 4)), idesc_o, kc > 0 ? 1u : 0u);
        }
      }
      ATRACE(5);
      tc_commit_cg<1>(bar_o);
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int sw = warp - 2;
    const int q = warp & 3;          // TMEM lane quadrant
    const int part = sw >> 2;        // 32-column slice of every 128-key chunk
    // chunk j of this thread's row: columns j*128 + part*32 .. +31 (all 16
    // warps finish chunk j together, so its PV MMA can start early)
    auto colof = [part](int j) { return j * 128 + part * 32; };
    const int rl = q * 32 + lane;    // row within the strip
    const int grow = q0 + rl;        // query index
    const int st = threadIdx.x - 64; // 0..511
    for (int i = st; i < S; i += kSoftWarps * 32)
      mask2[i] = p.add_mask ? p.add_mask[(size_t)b * S + i] * kLog2e : 0.f;
    // packed keep byte (8 columns) -> AND masks of its 4 bf16 pairs: one
    // LDS.128 expands 8 flags (instead of per-bit shift/select chains)
    uint4* klut = reinterpret_cast<uint4*>(smem + FwdSmem::LUT);
    if (st < 256) {
      uint32_t m[4];
#pragma unroll
      for (int w = 0; w < 4; ++w)
        m[w] = (((st >> (2 * w)) & 1) ? 0x0000FFFFu : 0u) | (((st >> (2 * w + 1)) & 1) ? 0xFFFF0000u : 0u);
      klut[st] = make_uint4(m[0], m[1], m[2], m[3]);
    }
    // dropout keep flags of this thread's row segment, 32 bytes per chunk
    const size_t rowoff = ((size_t)bh * S + grow) * S;
    const uint4* kp = reinterpret_cast<const uint4*>(p.keep + rowoff);  // 16 columns per uint4
    const uint4 ones = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    uint4 kv0 = p.keep ? __ldg(kp + colof(0) / 16) : ones, kv1 = p.keep ? __ldg(kp + colof(0) / 16 + 1) : ones;
    // packed keep flags (one word per 32-column chunk slice): all of this
    // thread's words are fetched up front, off the exp pass's critical path
    uint32_t kbw[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
    if (p.kb_in) {
      const uint32_t* kr = p.kb_row + ((size_t)bh * S + grow) * (S / 32);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < S / 128) kbw[j] = __ldg(kr + colof(j) / 32);
    }
    named_bar(1, kSoftWarps * 32);
    const float4* mask4 = reinterpret_cast<const float4*>(mask2);
    if (sw == 0 && lane == 0) ATRACE(2);
    mbar_wait(bar_s, 0);
    tc_fence_after();
    if (sw == 0 && lane == 0) ATRACE(3);
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    // pass 1: row max of t = S*c*log2e + mask*log2e (TMEM load of chunk j+1
    // in flight while chunk j is reduced)
    float mx = -INFINITY;
    const int nj = S / 128;
    {
      float v[2][32];
      tmem_ld32(trow + colof(0), v[0]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= nj) break;
        if (j + 1 < nj) tmem_ld32_nowait(trow + colof(j + 1), v[(j + 1) & 1]);
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 m = mask4[(colof(j) + i) >> 2];
          const float* w = v[j & 1];
          mx = fmax3(mx, fmaf(w[i], p.sc2, m.x), fmaf(w[i + 1], p.sc2, m.y));
          mx = fmax3(mx, fmaf(w[i + 2], p.sc2, m.z), fmaf(w[i + 3], p.sc2, m.w));
        }
        tmem_wait_ld();
      }
    }
    red_max[part * QT + rl] = mx;
    if (sw == 0 && lane == 0) ATRACE(4);
    named_bar(1, kSoftWarps * 32);
    mx = fmaxf(fmaxf(red_max[rl], red_max[QT + rl]), fmaxf(red_max[2 * QT + rl], red_max[3 * QT + rl]));
    // pass 2: e = exp2(t - max); rowsum; P̃d = e * keep (the 1/(1-p) scale is
    // applied to O) -> bf16 swizzled smem; keep flags -> packed bits
    float sum = 0.f;
    const int words = S / 32;
    // the keep-flag format is a compile-time branch: a uniform branch inside
    // the column loop would split it into basic blocks the scheduler cannot
    // interleave (each MUFU result then stalls its own block)
    auto pass2 = [&](auto kbin_c) {
    constexpr bool KBIN = decltype(kbin_c)::value;
#pragma unroll 1
    for (int j = 0; j < nj; ++j) {
      float w[32];
      tmem_ld32_nowait(trow + colof(j), w);
      const uint32_t kw[8] = {kv0.x, kv0.y, kv0.z, kv0.w, kv1.x, kv1.y, kv1.z, kv1.w};
      if (!KBIN && j + 1 < nj && p.keep) {  // next chunk's keep flags
        kv0 = __ldg(kp + colof(j + 1) / 16);
        kv1 = __ldg(kp + colof(j + 1) / 16 + 1);
      }
      tmem_wait_ld();
      uint32_t pk[16];
      uint32_t bits = 0;
      const uint32_t kbj = j == 0 ? kbw[0] : (j == 1 ? kbw[1] : (j == 2 ? kbw[2] : kbw[3]));
      // packed fp32 (FFMA2 / FADD2): t = s*c*log2e + (mask*log2e - max), two
      // columns per instruction; the exps stay on the MUFU pipe
      const float2 sc2x2 = make_float2(p.sc2, p.sc2), nmx2 = make_float2(-mx, -mx);
      float2 sacc = make_float2(0.f, 0.f);
      uint4 lm;  // masks of the current keep byte (KBIN)
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // 4 columns per keep word
        const float4 m = mask4[(colof(j) + 4 * u) >> 2];
        const float2 ta = __ffma2_rn(make_float2(w[4 * u], w[4 * u + 1]), sc2x2, __fadd2_rn(make_float2(m.x, m.y), nmx2));
        const float2 tb = __ffma2_rn(make_float2(w[4 * u + 2], w[4 * u + 3]), sc2x2, __fadd2_rn(make_float2(m.z, m.w), nmx2));
        const float e0 = ex2(ta.x), e1 = ex2(ta.y), e2 = ex2(tb.x), e3 = ex2(tb.y);
        sacc = __fadd2_rn(sacc, __fadd2_rn(make_float2(e0, e1), make_float2(e2, e3)));
        if constexpr (KBIN) {
          if ((u & 1) == 0) lm = klut[(kbj >> (8 * (u >> 1))) & 0xFFu];
          pk[2 * u] = pack_bf16x2(e0, e1) & ((u & 1) ? lm.z : lm.x);
          pk[2 * u + 1] = pack_bf16x2(e2, e3) & ((u & 1) ? lm.w : lm.y);
        } else {
          const uint32_t ff = kw[u] * 0xFFu;  // bytes 0x00 / 0xFF
          pk[2 * u] = pack_bf16x2(e0, e1) & __byte_perm(ff, 0, 0x1100);
          pk[2 * u + 1] = pack_bf16x2(e2, e3) & __byte_perm(ff, 0, 0x3322);
          bits |= keep_nibble(kw[u]) << (4 * u);
        }
      }
      if constexpr (KBIN) bits = kbj;
      sum += sacc.x + sacc.y;
      const int col = colof(j);
      const uint32_t tile = p_chunk(sbase, col >> 6);
      const int ch0 = (col & 63) >> 3;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        st_sw128(tile, rl, ch0 + u, make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]));
      if (p.kb_row) {
        if constexpr (!KBIN) p.kb_row[((size_t)bh * S + grow) * words + (col >> 5)] = bits;
        // transposed: bit i of word [key][q/32] = keep of query (32-row group base + i)
        const uint32_t colword = warp_transpose32(bits, lane);
        p.kb_col[((size_t)bh * S + col + lane) * words + (grow >> 5)] = colword;
      }
      // chunk j of P̃d complete in smem -> the MMA warp may issue its PV MMAs
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_p[j]);
    }
    };
    if (p.kb_in)
      pass2(std::true_type{});
    else
      pass2(std::false_type{});
    red_sum[part * QT + rl] = sum;
    named_bar(1, kSoftWarps * 32);
    const float tot = red_sum[rl] + red_sum[QT + rl] + red_sum[2 * QT + rl] + red_sum[3 * QT + rl];
    const float inv = p.ks / tot;
    if (part == 0) p.lse[(size_t)bh * S + grow] = mx + __log2f(tot);
    if (sw == 0 && lane == 0) ATRACE(6);
    mbar_wait(bar_o, 0);
    tc_fence_after();
    if (sw == 0 && lane == 0) ATRACE(7);
    float o[16];
    tmem_ld16(trow + part * 16, o);
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = pack_bf16x2(o[2 * i] * inv, o[2 * i + 1] * inv);
    uint4* dst = reinterpret_cast<uint4*>(p.ctx + ((size_t)b * S + grow) * p.ld_ctx + h * DH + part * 16);
    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ATRACE(8);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------ persistent forward, online softmax
// One CTA per SM walks the (b, h, 128-query) strips blockIdx.x, + grid, ...
// (384 strips at C2 are 1.3 waves of two-per-SM CTAs: the last 88 ran alone).
// Sixteen softmax warps, four per TMEM lane quadrant, 32 key columns each of a
// 128-key chunk; S is double-buffered in TMEM so the next chunk's Q·Kᵀ runs
// under this chunk's exp pass, and P̃d (bf16, the A operand of the PV MMA read
// from TMEM) is double-buffered so the exp pass of chunk j + 1 overlaps
// PV_j.  Online softmax with a lazily rescaled reference max: the O
// accumulator and the row sum are rescaled only when a chunk max exceeds the
// reference by more than 2^8, so P = exp2(t - m) <= 256 always fits bf16 (the
// rescale branch is warp-uniform: tcgen05.ld/st are .sync.aligned).  The row
// max of a chunk meets over the four warps of a lane quadrant only.  Q and the
// key-mask row are double-buffered per strip; ctx leaves by TMA from a bf16
// staging tile.  TMEM: S0 | S1 | P0 | P1 | O.
struct F3Smem {
  static constexpr int Q = 0;                        // two strip buffers
  static constexpr int NST = 3;
  static constexpr int STAGE = 2 * 128 * 128;        // K_j | V_j
  static constexpr int RING = Q + 2 * QT * 128;
  static constexpr int MASK = RING + NST * STAGE;    // two strip buffers of S floats (log2 domain)
  static constexpr int RED = MASK + 2 * kMaxSeq * 4; // [2 chunk parities][4 parts][128] chunk max
  static constexpr int SUM = RED + 2 * 4 * QT * 4;   // [4][128] row sums
  static constexpr int OST = SUM + 4 * QT * 4;       // ctx staging tile [128 x 64] bf16 SW128
  static constexpr int LUT = OST + QT * 128;         // keep byte -> 4 bf16-pair AND masks
  static constexpr int BAR = LUT + 256 * 16;
  static constexpr int TOTAL = BAR + 256 + KB;
};
static_assert(F3Smem::TOTAL <= 227 * 1024, "persistent forward exceeds shared memory");

__global__ void __launch_bounds__(kAttnThreads, 1)
attn_fwd3_kernel(const __grid_constant__ CUtensorMap map_qkv, const __grid_constant__ CUtensorMap map_ctx,
                 const AttnFwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + F3Smem::BAR);
  uint64_t* bar_q = bar;            // [2] Q of the strip (parity it & 1) landed
  uint64_t* q_free = bar + 2;       // [2] its last Q·Kᵀ completed
  uint64_t* bar_m = bar + 4;        // [2] key-mask row landed
  uint64_t* m_free = bar + 6;       // [2] its last read
  uint64_t* bar_s = bar + 8;        // [2] S_J in buffer J & 1
  uint64_t* bar_sfree = bar + 10;   // [2] S_J read
  uint64_t* bar_p = bar + 12;       // [2] P̃d_J written
  uint64_t* bar_pv = bar + 14;      // [2] PV_J completed
  constexpr int NST = F3Smem::NST;
  static_assert((16 + 2 * NST) * 8 + 4 <= 256, "forward barriers exceed their smem slot");
  uint64_t* full = bar + 16;          // [NST]
  uint64_t* empty = bar + 16 + NST;   // [NST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16 + 2 * NST);
  float* red_max = reinterpret_cast<float*>(smem + F3Smem::RED);
  float* red_sum = reinterpret_cast<float*>(smem + F3Smem::SUM);

  const int S = p.S, nch = S / 128;
  const int nstrips = p.B * p.NH * (S / QT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto strip = [&](int sidx, int& bh, int& b, int& h, int& q0) {
    const int nqb = S / QT;
    bh = sidx / nqb; q0 = (sidx % nqb) * QT; b = bh / p.NH; h = bh % p.NH;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_q[i], 1);
      mbar_init(&q_free[i], 1);
      mbar_init(&bar_m[i], 1);
      mbar_init(&m_free[i], kSoftWarps);
      mbar_init(&bar_s[i], 1);
      mbar_init(&bar_sfree[i], kSoftWarps);
      mbar_init(&bar_p[i], kSoftWarps);
      mbar_init(&bar_pv[i], 1);
    }
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_qkv)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dependents launch only once this CTA holds its TMEM: a dependent grid's CTA
  // allocating first on this SM would block our alloc while it waits on us
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 64) ATRACE(0);
  constexpr uint32_t T_P = 256, T_O = 384;  // S_J at 128 (J & 1); P̃d_J at T_P + 64 (J & 1)

  if (warp == 0) {
    if (lane == 0) {
      int J = 0, it = 0;
      for (int sidx = blockIdx.x; sidx < nstrips; sidx += gridDim.x, ++it) {
        int bh, b, h, q0;
        strip(sidx, bh, b, h, q0);
        const int qb = it & 1;
        if (it >= 2) mbar_wait(&q_free[qb], ((it - 2) >> 1) & 1);
        mbar_expect_tx(&bar_q[qb], QT * 128);
        for (int u = 0; u < 2; ++u)
          tma_load_4d_cg<1>(&map_qkv, smem_u32(&bar_q[qb]), smem + F3Smem::Q + qb * QT * 128 + u * 8 * KB, h * DH,
                            b * S + q0 + 64 * u, 0, 0);
        if (p.add_mask) {
          if (it >= 2) mbar_wait(&m_free[qb], ((it - 2) >> 1) & 1);
          mbar_expect_tx(&bar_m[qb], S * 4);
          bulk_g2s(smem + F3Smem::MASK + qb * kMaxSeq * 4, p.add_mask + (size_t)b * S, S * 4, smem_u32(&bar_m[qb]));
        }
        for (int j = 0; j < nch; ++j, ++J) {
          const int s = J % NST;
          mbar_wait(&empty[s], ((J / NST) & 1) ^ 1);
          mbar_expect_tx(&full[s], F3Smem::STAGE);
          const uint32_t bf = smem_u32(&full[s]);
          uint8_t* stg = smem + F3Smem::RING + s * F3Smem::STAGE;
          for (int u = 0; u < 2; ++u) {
            tma_load_4d_cg<1>(&map_qkv, bf, stg + u * 8 * KB, p.H + h * DH, b * S + j * 128 + 64 * u, 0, 0);
            tma_load_4d_cg<1>(&map_qkv, bf, stg + 16 * KB + u * 8 * KB, 2 * p.H + h * DH, b * S + j * 128 + 64 * u,
                              0, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_s = make_idesc(128, QT, 0, 0);
      const uint32_t idesc_o = make_idesc(DH, QT, 0, 1);  // A = P̃d from TMEM, B = V_j MN-major
      auto issue_pv = [&](int J, int j) {
        mbar_wait(&bar_p[J & 1], (J >> 1) & 1);
        tc_fence_after();
        const uint32_t stg = sbase + F3Smem::RING + (J % NST) * F3Smem::STAGE;
        const uint64_t vdesc = make_sdesc(stg + 16 * KB, 8 * KB, 1024);
        const uint32_t tp = tmem + T_P + 64 * (J & 1);
#pragma unroll
        for (int kc = 0; kc < 8; ++kc)
          tc_mma_ts(tmem + T_O, tp + kc * 8, vdesc + (uint64_t)(kc * (2048 >> 4)), idesc_o, (j > 0 || kc > 0) ? 1u : 0u);
        tc_commit_cg<1>(&empty[J % NST]);
        tc_commit_cg<1>(&bar_pv[J & 1]);
      };
      int J = 0, it = 0;
      for (int sidx = blockIdx.x; sidx < nstrips; sidx += gridDim.x, ++it) {
        const int qb = it & 1;
        mbar_wait(&bar_q[qb], (it >> 1) & 1);
        if (it == 0) ATRACE(1);
        const uint64_t qdesc = make_sdesc(sbase + F3Smem::Q + qb * QT * 128, 16, 1024);
        for (int j = 0; j < nch; ++j, ++J) {
          mbar_wait(&full[J % NST], (J / NST) & 1);
          if (J >= 2) mbar_wait(&bar_sfree[J & 1], ((J - 2) >> 1) & 1);
          tc_fence_after();
          const uint32_t stg = sbase + F3Smem::RING + (J % NST) * F3Smem::STAGE;
          const uint64_t kdesc = make_sdesc(stg, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            tc_mma_cg<1>(tmem + 128 * (J & 1), qdesc + 2 * kk, kdesc + 2 * kk, idesc_s, kk > 0 ? 1u : 0u);
          tc_commit_cg<1>(&bar_s[J & 1]);
          if (j == nch - 1) tc_commit_cg<1>(&q_free[qb]);
          if (j > 0) issue_pv(J - 1, j - 1);
        }
        // the strip's last PV before the next strip's first Q·Kᵀ (which waits for its Q)
        issue_pv(J - 1, nch - 1);
      }
    }
  } else {
    // -------------------------------------------------------------- softmax
    const int sw = warp - 2, qd = warp & 3, part = sw >> 2;  // part: key columns [32 part, 32 part + 32) of a chunk
    const int rl = qd * 32 + lane;
    const int st = threadIdx.x - 64;  // 0..511
    // keep-bit pair -> AND mask of a bf16 pair: four words, so a warp's lookups
    // hit at most four banks (a 256-entry byte table of uint4 masks cost ~1.5 M
    // bank-conflict wavefronts per launch)
    uint32_t* klut = reinterpret_cast<uint32_t*>(smem + F3Smem::LUT);
    if (st < 4) klut[st] = (st & 1 ? 0x0000FFFFu : 0u) | (st & 2 ? 0xFFFF0000u : 0u);
    named_bar(1, kSoftWarps * 32);
    const int words = S / 32;
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const float2 sc2x2 = make_float2(p.sc2, p.sc2);
    int J = 0, it = 0;
    for (int sidx = blockIdx.x; sidx < nstrips; sidx += gridDim.x, ++it) {
      int bh, b, h, q0;
      strip(sidx, bh, b, h, q0);
      const int qb = it & 1;
      const int grow = q0 + rl;
      const size_t rowi = (size_t)bh * S + grow;
      const float* mask2 = reinterpret_cast<const float*>(smem + F3Smem::MASK + qb * kMaxSeq * 4);
      if (p.add_mask) mbar_wait(&bar_m[qb], (it >> 1) & 1);
      float mref = 0.f, lsum = 0.f;  // reference max (log2 domain) and this thread's partial row sum
      // packed keep words one chunk ahead (their latency stays off the exp pass)
      uint32_t kw_n = p.kb_in ? __ldg(p.kb_row + rowi * words + part) : 0xFFFFFFFFu;
      for (int j = 0; j < nch; ++j, ++J) {
        const int col = j * 128 + part * 32;  // first key column of this thread's slice
        const uint32_t kw = kw_n;
        if (p.kb_in && j + 1 < nch) kw_n = __ldg(p.kb_row + rowi * words + 4 * (j + 1) + part);
        uint4 kv[2];
        if (p.keep) {
          const uint4* kp = reinterpret_cast<const uint4*>(p.keep + rowi * S + col);
          kv[0] = __ldg(kp);
          kv[1] = __ldg(kp + 1);
        }
        mbar_wait(&bar_s[J & 1], (J >> 1) & 1);
        if (it == 0 && sw == 0 && lane == 0 && j < 4) ATRACE(2 + j);
        tc_fence_after();
        float t[32];
        tmem_ld32(trow + 128 * (J & 1) + part * 32, t);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_sfree[J & 1]);  // S_J is in registers
        // t = s * c + mask (log2 domain), and its max over the slice
        const float4* mask4 = reinterpret_cast<const float4*>(mask2 + col);
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 m = p.add_mask ? mask4[i >> 2] : make_float4(0.f, 0.f, 0.f, 0.f);
          const float2 a = __ffma2_rn(make_float2(t[i], t[i + 1]), sc2x2, make_float2(m.x, m.y));
          const float2 c2 = __ffma2_rn(make_float2(t[i + 2], t[i + 3]), sc2x2, make_float2(m.z, m.w));
          t[i] = a.x; t[i + 1] = a.y; t[i + 2] = c2.x; t[i + 3] = c2.y;
          mx = fmax3(mx, fmaxf(a.x, a.y), fmaxf(c2.x, c2.y));
        }
        // the row's max over the four parts: only the quadrant's four warps meet
        float* rm = red_max + (J & 1) * 4 * QT;
        rm[part * QT + rl] = mx;
        named_bar(2 + qd, 4 * 32);
        const float cmax = fmaxf(fmaxf(rm[rl], rm[QT + rl]), fmaxf(rm[2 * QT + rl], rm[3 * QT + rl]));
        if (j == nch - 1 && p.add_mask) {  // the strip's mask row is no longer read
          __syncwarp();
          if (lane == 0) mbar_arrive(&m_free[qb]);
        }
        if (j == 0) {
          mref = cmax;
        } else if (__any_sync(0xffffffffu, cmax > mref + 8.f)) {
          // rare: a row's reference max moves up; O (after PV_{J-1}) and the
          // row sum rescale (warp-uniform branch: tcgen05.ld/st are .sync.aligned)
          const bool up = cmax > mref + 8.f;
          const float f = up ? ex2(mref - cmax) : 1.f;
          mbar_wait(&bar_pv[(J - 1) & 1], ((J - 1) >> 1) & 1);
          tc_fence_after();
          float o[16];
          tmem_ld16(trow + T_O + part * 16, o);
          uint32_t ou[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) ou[i] = __float_as_uint(o[i] * f);
          tmem_st16(trow + T_O + part * 16, ou);
          tmem_wait_st();
          lsum *= f;
          if (up) mref = cmax;
        }
        // P = exp2(t - mref); P̃d = P ∘ keep -> bf16 pairs -> TMEM (A of the PV MMA)
        float2 sacc = make_float2(0.f, 0.f);
        uint32_t bits = 0u;
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // 4 columns per step
          const float e0 = ex2(t[4 * u] - mref), e1 = ex2(t[4 * u + 1] - mref);
          const float e2 = ex2(t[4 * u + 2] - mref), e3 = ex2(t[4 * u + 3] - mref);
          sacc = __fadd2_rn(sacc, __fadd2_rn(make_float2(e0, e1), make_float2(e2, e3)));
          uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu;
          if (p.kb_in) {
            m0 = klut[(kw >> (4 * u)) & 3u];
            m1 = klut[(kw >> (4 * u + 2)) & 3u];
          } else if (p.keep) {
            const uint4 q4 = kv[u >> 2];
            const uint32_t w = (u & 3) == 0 ? q4.x : ((u & 3) == 1 ? q4.y : ((u & 3) == 2 ? q4.z : q4.w));
            const uint32_t ff = w * 0xFFu;
            m0 = __byte_perm(ff, 0, 0x1100);
            m1 = __byte_perm(ff, 0, 0x3322);
            bits |= keep_nibble(w) << (4 * u);
          }
          pk[2 * u] = pack_bf16x2(e0, e1) & m0;
          pk[2 * u + 1] = pack_bf16x2(e2, e3) & m1;
        }
        lsum += sacc.x + sacc.y;
        if (J >= 2) mbar_wait(&bar_pv[J & 1], ((J - 2) >> 1) & 1);  // P buffer J & 1 free once PV_{J-2} read it
        tc_fence_after();
        tmem_st16(trow + T_P + 64 * (J & 1) + part * 16, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_p[J & 1]);
        if (it == 0 && sw == 0 && lane == 0 && j < 4) ATRACE(6 + j);
        if (p.kb_col) {
          if (p.kb_in) bits = kw;
          else p.kb_row[rowi * words + (col >> 5)] = bits;
          const uint32_t colword = warp_transpose32(bits, lane);
          p.kb_col[((size_t)bh * S + col + lane) * words + (grow >> 5)] = colword;
        }
      }
      // ---- epilogue: ctx = O / rowsum, lse
      if (st == 0) bulk_wait_read<0>();  // the previous strip's ctx tile left the staging buffer
      red_sum[part * QT + rl] = lsum;
      named_bar(1, kSoftWarps * 32);
      const float tot = ((red_sum[rl] + red_sum[QT + rl]) + red_sum[2 * QT + rl]) + red_sum[3 * QT + rl];
      if (part == 0) p.lse[rowi] = mref + __log2f(tot);
      const float inv = p.ks / tot;
      mbar_wait(&bar_pv[(J - 1) & 1], ((J - 1) >> 1) & 1);  // O complete
      if (it < 3 && sw == 0 && lane == 0) ATRACE(10 + it);
      tc_fence_after();
      float o[16];
      tmem_ld16(trow + T_O + part * 16, o);
      const uint32_t ost = sbase + F3Smem::OST;
#pragma unroll
      for (int u = 0; u < 2; ++u)
        st_sw128(ost, rl, part * 2 + u,
                 make_uint4(pack_bf16x2(o[8 * u] * inv, o[8 * u + 1] * inv),
                            pack_bf16x2(o[8 * u + 2] * inv, o[8 * u + 3] * inv),
                            pack_bf16x2(o[8 * u + 4] * inv, o[8 * u + 5] * inv),
                            pack_bf16x2(o[8 * u + 6] * inv, o[8 * u + 7] * inv)));
      fence_async_smem();
      tc_fence_before();  // O is read: the next strip's first PV may overwrite it
      named_bar(1, kSoftWarps * 32);
      if (st == 0) {
        tma_store_4d(&map_ctx, ost, h * DH, b * S + q0, 0, 0);
        bulk_commit();
      }
    }
    if (st == 0) bulk_wait_read<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 64) ATRACE(15);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// qkv bias gradient: out[col] (+)= sum over the strip partials, fixed order
__global__ void __launch_bounds__(256) attn_bias_reduce_kernel(int nparts, int cols, const float* __restrict__ part,
                                                               float* __restrict__ out, int accumulate) {
  pdl_trigger();
  pdl_wait();
  const int col = blockIdx.x * 256 + threadIdx.x;
  if (col >= cols) return;
  float t = 0.f;
  int r = 0;
  for (; r + 8 <= nparts; r += 8) {  // eight partial rows in flight (not one L2 round trip per row)
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(part + (size_t)(r + u) * cols + col);
#pragma unroll
    for (int u = 0; u < 8; ++u) t += v[u];
  }
  for (; r < nparts; ++r) t += __ldg(part + (size_t)r * cols + col);
  out[col] = accumulate ? out[col] + t : t;
}

// --------------------------------------------------------------------- backward
struct AttnBwdParams {
  unsigned long long* trace;
  int B, NH, S, H;
  int64_t ld_ctx, ld_dqkv;
  const __nv_bfloat16* ctx;   // O   [T, ld_ctx]
  const __nv_bfloat16* dctx;  // dO  [T, ld_ctx]
  const float* add_mask;      // [B, S] or null
  const float* lse;           // [B, NH, S] log2 domain
  float* delta;               // [B, NH, S]  D = rowsum(dO∘O) (written by dq / the delta pre-pass, read by kstrip)
  const uint32_t* kb_row;     // or null (no dropout)
  const uint32_t* kb_col;
  float ks, sc2, scale;       // keep scale, inv_divisor*log2e, inv_divisor
  __nv_bfloat16* dqkv;        // [T, ld_dqkv]: dQ | dK | dV column blocks
  float* bias_part;           // [B*S/128][3H]: per-strip column sums of dQ | dK | dV (qkv bias gradient)
  int ds_store;               // kstrip: also store dSᵀ (map_ds) and the strip's dQ column sums (dQ = dS·K GEMM path)
  const __nv_bfloat16* qkv;   // Q | K | V [T, ld_qkv] (the key-strip kernel reads K rows for dQ's column sums)
  int64_t ld_qkv;
};

constexpr int CH = 128;  // keys (dq) / queries (kstrip) per chunk

struct DqSmem {
  static constexpr int Q = 0;
  static constexpr int DO = Q + QT * 128;
  static constexpr int K = DO + QT * 128;
  static constexpr int V = K + kMaxSeq * 128;
  static constexpr int DS = V + kMaxSeq * 128;      // [128 x 128] bf16 as 2 x [128 x 64]
  static constexpr int MASK = DS + QT * CH * 2;
  static constexpr int RED = MASK + kMaxSeq * 4;
  static constexpr int LUT = RED + 4 * QT * 4;   // keep nibble -> 4 x {0, ks}
  static constexpr int BAR = LUT + 16 * 16;
  static constexpr int TOTAL = BAR + 256 + KB;
};
static_assert(DqSmem::TOTAL <= 227 * 1024, "attention dq exceeds shared memory");


// Write 32 consecutive columns (col0 % 32 == 0, within a 128-column chunk) of
// row r of a [128 x 128] bf16 operand stored as two [128 x 64] SW128 tiles.
__device__ __forceinline__ void st_row32(uint32_t buf, int r, int col0, const uint32_t (&pk)[16]) {
  const uint32_t tile = buf + (col0 >> 6) * (QT * 128);
  const int ch0 = (col0 & 63) >> 3;
#pragma unroll
  for (int u = 0; u < 4; ++u) st_sw128(tile, r, ch0 + u, make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]));
}

// Column sums of NT [128 x 64] fp32 tiles held one row slice per softmax
// thread (warp quarter q: rows 32 q + lane; part: columns 16 part .. + 15), in a
// fixed order: a halving butterfly over the warp's 32 rows (16 shuffles per
// tile; lane l ends with column (l >> 1) & 15), then the four quarters in
// order q = 0..3 through smem (red: NT x 4 x 64 floats) -> out_t[0..63].
template <int NT>
__device__ __forceinline__ void strip_colsum(float (&v)[NT][16], int lane, int q, int part, int st, float* red,
                                             float* const (&out)[NT]) {
#pragma unroll
  for (int t = 0; t < NT; ++t) {
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1) {
      const bool hi = lane & (2 * w);
#pragma unroll
      for (int i = 0; i < w; ++i) {
        const float send = hi ? v[t][i] : v[t][i + w];
        const float keep = hi ? v[t][i + w] : v[t][i];
        v[t][i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * w);
      }
    }
    v[t][0] += __shfl_xor_sync(0xffffffffu, v[t][0], 1);
    if (!(lane & 1)) red[(t * 4 + q) * 64 + part * 16 + ((lane >> 1) & 15)] = v[t][0];
  }
  named_bar(1, kSoftWarps * 32);
  if (st < NT * 64) {
    const int t = st >> 6, col = st & 63;
    const float* r = red + t * 256 + col;
    float* o = out[0];  // (selects, not an indexed local array)
#pragma unroll
    for (int u = 1; u < NT; ++u) o = t == u ? out[u] : o;
    o[col] = ((r[0] + r[64]) + r[128]) + r[192];
  }
}

// Column sums of NT 128 x 64 fp32 tiles whose rows are spread one 16-column
// slice per softmax thread (row rl, columns c0..c0+15), in a fixed order:
// staged in smem, 8 groups of 16 rows, then the 8 group sums -> out_t[0..63].
// 16-byte chunk c of row r lives at chunk c ^ (r & 15): the row-per-lane
// writes and the column reads are both bank-conflict free.
template <int NT>
__device__ __forceinline__ void tile_colsum_128x64(float* const (&stage)[NT], float* const (&scratch)[NT], int rl,
                                                   int c0, const float (&v)[NT][16], int st,
                                                   float* const (&out)[NT]) {
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    float4* d = reinterpret_cast<float4*>(stage[t] + rl * 64);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      d[((c0 >> 2) + i) ^ (rl & 15)] = make_float4(v[t][4 * i], v[t][4 * i + 1], v[t][4 * i + 2], v[t][4 * i + 3]);
  }
  named_bar(1, kSoftWarps * 32);
  const int col = st & 63, grp = st >> 6;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int row = grp * 16 + r;
      acc += stage[t][row * 64 + (((col >> 2) ^ (row & 15)) << 2) + (col & 3)];
    }
    scratch[t][grp * 64 + col] = acc;
  }
  named_bar(1, kSoftWarps * 32);
  if (st < 64) {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      float u = 0.f;
#pragma unroll
      for (int g = 0; g < 8; ++g) u += scratch[t][g * 64 + st];
      out[t][st] = u;
    }
  }
}

__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* g, const float (&o)[16]) {
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = pack_bf16x2(o[2 * i], o[2 * i + 1]);
  uint4* dst = reinterpret_cast<uint4*>(g);
  dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
  dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// dQ strip: CTA = (b, h, 128-query block); loops over 128-key chunks.
__global__ void __launch_bounds__(kAttnThreads, 1)
attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap map_qkv, const __grid_constant__ CUtensorMap map_do,
                   const __grid_constant__ CUtensorMap map_o, const AttnBwdParams p) {
  // dynamic smem opens the CTA's window (no static smem in this kernel): it is
  // 1024-B aligned, and indexing it directly keeps every access LDS/STS
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + DqSmem::BAR);
  uint64_t *bar_q = bar, *bar_s = bar + 1, *bar_tfree = bar + 2, *bar_ds = bar + 3, *bar_dsfree = bar + 4;
  uint64_t* bar_kv = bar + 8;  // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);
  float* mask2 = reinterpret_cast<float*>(smem + DqSmem::MASK);
  float* red = reinterpret_cast<float*>(smem + DqSmem::RED);

  const int S = p.S, nch = S / CH;
  const int qb = blockIdx.x % (S / QT);
  const int bh = blockIdx.x / (S / QT);
  const int b = bh / p.NH, h = bh % p.NH;
  const int q0 = qb * QT, row0 = b * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_tfree, kSoftWarps);
    mbar_init(bar_ds, kSoftWarps);
    mbar_init(bar_dsfree, 1);
    for (int j = 0; j < 4; ++j) mbar_init(&bar_kv[j], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dependents launch only once this CTA holds its TMEM: a dependent grid's CTA
  // allocating first on this SM would block our alloc while it waits on us
  pdl_trigger();
  pdl_wait();  // setup above overlapped the previous kernel's tail
  if (threadIdx.x == 0) ATRACE(0);
  constexpr uint32_t T_S = 0, T_DP = 128, T_DQ = 256;

  if (warp == 0) {
    if (lane == 0) {
      // Q, dO, and O (parked in the dS buffer until D = rowsum(dO∘O) is formed)
      mbar_expect_tx(bar_q, 3 * QT * 128);
      const uint32_t bq = smem_u32(bar_q);
      for (int u = 0; u < 2; ++u) {
        tma_load_4d_cg<1>(&map_qkv, bq, smem + DqSmem::Q + u * 8 * KB, h * DH, row0 + q0 + 64 * u, 0, 0);
        tma_load_4d_cg<1>(&map_do, bq, smem + DqSmem::DO + u * 8 * KB, h * DH, row0 + q0 + 64 * u, 0, 0);
        tma_load_4d_cg<1>(&map_o, bq, smem + DqSmem::DS + u * 8 * KB, h * DH, row0 + q0 + 64 * u, 0, 0);
      }
      for (int j = 0; j < nch; ++j) {
        // at most two K/V chunks in flight: the first chunk is not slowed by
        // the rest of the strip's loads (every SM fetches at once at start)
        if (j >= 2) mbar_wait(&bar_kv[j - 2], 0);
        mbar_expect_tx(&bar_kv[j], 2 * CH * 128);
        const uint32_t bk = smem_u32(&bar_kv[j]);
        for (int u = 0; u < 2; ++u) {
          const int r = row0 + j * CH + 64 * u;
          tma_load_4d_cg<1>(&map_qkv, bk, smem + DqSmem::K + (j * 2 + u) * 8 * KB, p.H + h * DH, r, 0, 0);
          tma_load_4d_cg<1>(&map_qkv, bk, smem + DqSmem::V + (j * 2 + u) * 8 * KB, 2 * p.H + h * DH, r, 0, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_s = make_idesc(CH, QT, 0, 0);
      const uint32_t idesc_q = make_idesc(DH, QT, 0, 1);
      const uint64_t qdesc = make_sdesc(sbase + DqSmem::Q, 16, 1024);
      const uint64_t dodesc = make_sdesc(sbase + DqSmem::DO, 16, 1024);
      mbar_wait(bar_q, 0);
      tc_fence_after();
      ATRACE(1);
      auto issue_dq = [&](int j) {  // dQ += dS_j · K_j   (K_j read MN-major)
        mbar_wait(bar_ds, j & 1);
        tc_fence_after();
        const uint64_t kdesc = make_sdesc(sbase + DqSmem::K + j * 16 * KB, 8 * KB, 1024);
#pragma unroll
        for (int kc = 0; kc < CH / 16; ++kc) {
          const uint64_t adesc = make_sdesc(sbase + DqSmem::DS + (kc >> 2) * 16 * KB, 16, 1024);
          tc_mma_cg<1>(tmem + T_DQ, adesc + 2 * (kc & 3), kdesc + (uint64_t)(kc * (2048 >> 4)), idesc_q,
                       (j > 0 || kc > 0) ? 1u : 0u);
        }
        tc_commit_cg<1>(bar_dsfree);
      };
      for (int j = 0; j < nch; ++j) {
        mbar_wait(&bar_kv[j], 0);
        if (j > 0) mbar_wait(bar_tfree, (j - 1) & 1);
        tc_fence_after();
        const uint64_t kdesc = make_sdesc(sbase + DqSmem::K + j * 16 * KB, 16, 1024);
        const uint64_t vdesc = make_sdesc(sbase + DqSmem::V + j * 16 * KB, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          tc_mma_cg<1>(tmem + T_S, qdesc + 2 * kk, kdesc + 2 * kk, idesc_s, kk > 0 ? 1u : 0u);
          tc_mma_cg<1>(tmem + T_DP, dodesc + 2 * kk, vdesc + 2 * kk, idesc_s, kk > 0 ? 1u : 0u);
        }
        tc_commit_cg<1>(bar_s);
        if (j > 0) issue_dq(j - 1);
      }
      issue_dq(nch - 1);
    }
  } else {
    const int sw = warp - 2, q = warp & 3, part = sw >> 2;
    const int rl = q * 32 + lane, grow = q0 + rl;
    const int st = threadIdx.x - 64;
    const size_t rowi = (size_t)bh * S + grow;
    const int words = S / 32;
    // this thread's packed keep words for every chunk, issued first: their
    // latency overlaps the prologue (not a global-latency stall per chunk)
    uint32_t kbw[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
    if (p.kb_row) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nch) kbw[j] = __ldg(p.kb_row + rowi * words + ((j * CH + part * 32) >> 5));
    }
    const float lse_c = p.lse[rowi] - __log2f(p.scale);  // folds the 1/divisor into P
    for (int i = st; i < S; i += kSoftWarps * 32)
      mask2[i] = p.add_mask ? p.add_mask[(size_t)b * S + i] * kLog2e : 0.f;
    const float4* klut = reinterpret_cast<const float4*>(smem + DqSmem::LUT);
    fill_keep_lut(reinterpret_cast<float4*>(smem + DqSmem::LUT), st, p.ks);
    // D = rowsum(dO ∘ O) from the TMA-staged tiles (SW128 rows): each of the
    // 4 warps of a quadrant sums 16 of the 64 columns (chunks 2*part, +1)
    mbar_wait(bar_q, 0);
    {
      float dsum = 0.f;
#pragma unroll
      for (int c = 2 * part; c < 2 * part + 2; ++c) {
        const uint32_t off = rl * 128 + ((c ^ (rl & 7)) << 4);
        const uint4 x = lds128(sbase + DqSmem::DO + off), y = lds128(sbase + DqSmem::DS + off);
        const __nv_bfloat162* hx = reinterpret_cast<const __nv_bfloat162*>(&x);
        const __nv_bfloat162* hy = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 fx = __bfloat1622float2(hx[i]), fy = __bfloat1622float2(hy[i]);
          dsum = fmaf(fx.x, fy.x, dsum);
          dsum = fmaf(fx.y, fy.y, dsum);
        }
      }
      red[part * QT + rl] = dsum;
    }
    named_bar(1, kSoftWarps * 32);
    const float D = red[rl] + red[QT + rl] + red[2 * QT + rl] + red[3 * QT + rl];
    if (part == 0) p.delta[rowi] = D;
    if (sw == 0 && lane == 0) ATRACE(12);
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    for (int j = 0; j < nch; ++j) {
      mbar_wait(bar_s, j & 1);
      tc_fence_after();
      if (sw == 0 && lane == 0 && j < 4) ATRACE(2 + j);
      float s[32], dp[32];
      tmem_ld32(trow + T_S + part * 32, s);
      tmem_ld32(trow + T_DP + part * 32, dp);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_tfree);
      const int key0 = j * CH + part * 32;
      const uint32_t bits = j == 0 ? kbw[0] : (j == 1 ? kbw[1] : (j == 2 ? kbw[2] : kbw[3]));
      uint32_t pk[16];
      // packed fp32 pairs: P' = exp2(s*c + mask - lse') ; dS = P' * (dPd*keep*ks - D)
      const float2 sc2x2 = make_float2(p.sc2, p.sc2), nl2 = make_float2(-lse_c, -lse_c);
      const float2 nD2 = make_float2(-D, -D);
      float4 kf;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float2 m = reinterpret_cast<const float2*>(mask2 + key0)[i >> 1];
        const float2 t = __ffma2_rn(make_float2(s[i], s[i + 1]), sc2x2, __fadd2_rn(m, nl2));
        const float2 P = make_float2(ex2(t.x), ex2(t.y));
        // dPd * keep * ks - D with keep*ks in {0, ks} (dropped: 0 - D = -D)
        if ((i & 3) == 0) kf = klut[(bits >> i) & 15u];
        const float2 kk = (i & 3) ? make_float2(kf.z, kf.w) : make_float2(kf.x, kf.y);
        const float2 d = __fmul2_rn(P, __ffma2_rn(make_float2(dp[i], dp[i + 1]), kk, nD2));
        pk[i >> 1] = pack_bf16x2(d.x, d.y);
      }
      if (j > 0) mbar_wait(bar_dsfree, (j - 1) & 1);
      st_row32(sbase + DqSmem::DS, rl, part * 32, pk);
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_ds);
      if (sw == 0 && lane == 0 && j < 4) ATRACE(6 + j);
    }
    mbar_wait(bar_dsfree, (nch - 1) & 1);
    if (sw == 0 && lane == 0) ATRACE(10);
    tc_fence_after();
    float o[16];
    tmem_ld16(trow + T_DQ + part * 16, o);
    store_bf16x16(p.dqkv + (size_t)(row0 + grow) * p.ld_dqkv + h * DH + part * 16, o);
    if (p.bias_part) {  // this strip's dQ column sums (the dS buffer is free now)
      float* const stg[1] = {reinterpret_cast<float*>(smem + DqSmem::DS)};
      float* const scr[1] = {red};
      float* const dst[1] = {p.bias_part + (size_t)(b * (S / QT) + qb) * 3 * p.H + h * DH};
      const float (&vv)[1][16] = *reinterpret_cast<const float(*)[1][16]>(&o);
      tile_colsum_128x64<1>(stg, scr, rl, part * 16, vv, st, dst);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ATRACE(11);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ----------------------------------------------- persistent key-strip backward
// One CTA per SM walks the (b, h, 128-key) strips blockIdx.x, + grid, ...: the
// Q / dO ring, the S / dPd TMEM buffers and the chunk barriers run on one
// chunk sequence across strips, so the next strip's K / V / lse / D loads and
// its first Sᵀ / dPdᵀ MMAs overlap this strip's last chunk and epilogue (the
// next strip's first dK / dV MMA follows its first Pd / dS tiles, which the
// softmax warps write only after reading this strip's dK / dV).  Per chunk:
// P and dS = P∘(dPd∘keep·ks − D) in packed fp32 from Sᵀ / dPdᵀ, Pdᵀ / dSᵀ as
// SW128 bf16 tiles, dV += Pdᵀ·dO_j and dK += dSᵀ·Q_j.  A 19th warp TMA-stores
// each dSᵀ tile (so the MMA thread never waits on a bulk read), the epilogue stores dK / dV by TMA
// from bf16 tiles staged in the Pd buffer and reduces the bias column sums by
// shuffles.
constexpr int kKsThreads = kAttnThreads + 32;
struct KsSmem {
  static constexpr int K = 0;
  static constexpr int V = K + QT * 128;
  static constexpr int NST = 3;
  static constexpr int RING = V + QT * 128;
  static constexpr int STAGE = 2 * CH * 128;         // Q_j | dO_j
  static constexpr int PD = RING + NST * STAGE;      // Pdᵀ tile; the dK | dV bf16 tiles in the epilogue
  static constexpr int DS = PD + QT * CH * 2;
  static constexpr int ROWS = DS + QT * CH * 2;      // two buffers (strip parity) of lse | D | key mask
  static constexpr int ROWB = 2 * kMaxSeq * 4 + QT * 4;
  static constexpr int LUT = ROWS + 2 * ROWB;
  static constexpr int CS = LUT + 16 * 16;           // [4][128] per-part Σ_q dS
  static constexpr int RED = CS + 4 * QT * 4;        // [3][4][64] column-sum quarters
  static constexpr int KROW = RED + 3 * 4 * 64 * 4;  // the strip's K rows (SW128), kept for dQ's column sums
  static constexpr int BAR = KROW + QT * 128;
  static constexpr int TOTAL = BAR + 256 + KB;
};
static_assert(KsSmem::TOTAL <= 227 * 1024, "attention key-strip kernel exceeds shared memory");

struct StripIdx {
  int bh, b, h, k0, row0;
};
__device__ __forceinline__ StripIdx strip_idx(int sidx, const AttnBwdParams& p) {
  const int nkb = p.S / QT, kb = sidx % nkb, bh = sidx / nkb;
  return {bh, bh / p.NH, bh % p.NH, kb * QT, (bh / p.NH) * p.S};
}

__global__ void __launch_bounds__(kKsThreads, 1)
attn_bwd_kstrip_kernel(const __grid_constant__ CUtensorMap map_qkv, const __grid_constant__ CUtensorMap map_do,
                       const __grid_constant__ CUtensorMap map_ds, const __grid_constant__ CUtensorMap map_dkv,
                       const AttnBwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + KsSmem::BAR);
  uint64_t *bar_kv = bar, *bar_s = bar + 1, *bar_tfree = bar + 2, *bar_pds = bar + 3, *bar_pdsfree = bar + 4;
  uint64_t* kv_free = bar + 5;
  uint64_t* bar_rows = bar + 6;   // [2]
  uint64_t* rows_free = bar + 8;  // [2]
  uint64_t* ds_free = bar + 10;   // the dSᵀ tile's store has read it
  constexpr int NST = KsSmem::NST;
  static_assert((11 + 2 * NST) * 8 + 4 <= 256, "key-strip barriers exceed their smem slot");
  uint64_t* full = bar + 11;              // [NST]
  uint64_t* empty = bar + 11 + NST;       // [NST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 11 + 2 * NST);
  auto rows = [&](int it) { return reinterpret_cast<float*>(smem + KsSmem::ROWS + (it & 1) * KsSmem::ROWB); };

  const int S = p.S, nch = S / CH;
  const int nstrips = p.B * p.NH * (S / QT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_tfree, kSoftWarps);
    mbar_init(bar_pds, kSoftWarps);
    mbar_init(bar_pdsfree, 1);
    mbar_init(kv_free, kSoftWarps);  // every softmax warp saw the strip's last Sᵀ / dPdᵀ (and copied its K rows)
    mbar_init(ds_free, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_rows[b], 1);
      mbar_init(&rows_free[b], kSoftWarps);  // every softmax warp's last lse / D read of the buffer's strip
    }
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dependents launch only once this CTA holds its TMEM: a dependent grid's CTA
  // allocating first on this SM would block our alloc while it waits on us
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) ATRACE(0);
  constexpr uint32_t T_S = 0, T_DP = 128, T_DK = 256, T_DV = 320;

  if (warp == 0) {
    if (lane == 0) {
      int J = 0, it = 0;
      for (int sidx = blockIdx.x; sidx < nstrips; sidx += gridDim.x, ++it) {
        const StripIdx t = strip_idx(sidx, p);
        // K / V once the previous strip's Sᵀ / dPdᵀ MMAs are done; lse / D /
        // mask rows into the buffer the strip two back released
        if (it > 0) mbar_wait(kv_free, (it - 1) & 1);
        mbar_expect_tx(bar_kv, 2 * QT * 128);
        const uint32_t ba = smem_u32(bar_kv);
        for (int u = 0; u < 2; ++u) {
          tma_load_4d_cg<1>(&map_qkv, ba, smem + KsSmem::K + u * 8 * KB, p.H + t.h * DH, t.row0 + t.k0 + 64 * u, 0, 0);
          tma_load_4d_cg<1>(&map_qkv, ba, smem + KsSmem::V + u * 8 * KB, 2 * p.H + t.h * DH, t.row0 + t.k0 + 64 * u, 0,
                            0);
        }
        if (it >= 2) mbar_wait(&rows_free[it & 1], ((it - 2) >> 1) & 1);
        mbar_expect_tx(&bar_rows[it & 1], 2 * S * 4 + (p.add_mask ? QT * 4 : 0));
        const uint32_t br = smem_u32(&bar_rows[it & 1]);
        float* rw = rows(it);
        bulk_g2s(rw, p.lse + (size_t)t.bh * S, S * 4, br);
        bulk_g2s(rw + kMaxSeq, p.delta + (size_t)t.bh * S, S * 4, br);
        if (p.add_mask) bulk_g2s(rw + 2 * kMaxSeq, p.add_mask + (size_t)t.b * S + t.k0, QT * 4, br);
        for (int j = 0; j < nch; ++j, ++J) {
          const int s = J % NST;
          mbar_wait(&empty[s], ((J / NST) & 1) ^ 1);
          mbar_expect_tx(&full[s], KsSmem::STAGE);
          const uint32_t bf = smem_u32(&full[s]);
          uint8_t* stq = smem + KsSmem::RING + s * KsSmem::STAGE;
          for (int u = 0; u < 2; ++u) {
            tma_load_4d_cg<1>(&map_qkv, bf, stq + u * 8 * KB, t.h * DH, t.row0 + j * CH + 64 * u, 0, 0);
            tma_load_4d_cg<1>(&map_do, bf, stq + CH * 128 + u * 8 * KB, t.h * DH, t.row0 + j * CH + 64 * u, 0, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_s = make_idesc(CH, QT, 0, 0);
      const uint32_t idesc_g = make_idesc(DH, QT, 0, 1);
      const uint64_t kdesc = make_sdesc(sbase + KsSmem::K, 16, 1024);
      const uint64_t vdesc = make_sdesc(sbase + KsSmem::V, 16, 1024);
      // dV += Pdᵀ·dO_j ; dK += dSᵀ·Q_j for chunk J = chunk j of the it-th strip
      auto issue_grads = [&](int J, int j) {
        mbar_wait(bar_pds, J & 1);
        tc_fence_after();
        const uint32_t dsb = sbase + KsSmem::DS;
        const uint32_t stq = sbase + KsSmem::RING + (J % NST) * KsSmem::STAGE;
        const uint64_t qmn = make_sdesc(stq, 8 * KB, 1024);
        const uint64_t domn = make_sdesc(stq + CH * 128, 8 * KB, 1024);
#pragma unroll
        for (int kc = 0; kc < CH / 16; ++kc) {
          const uint64_t pd = make_sdesc(sbase + KsSmem::PD + (kc >> 2) * 16 * KB, 16, 1024);
          const uint64_t ds = make_sdesc(dsb + (kc >> 2) * 16 * KB, 16, 1024);
          const uint32_t acc = (j > 0 || kc > 0) ? 1u : 0u;
          tc_mma_cg<1>(tmem + T_DV, pd + 2 * (kc & 3), domn + (uint64_t)(kc * (2048 >> 4)), idesc_g, acc);
          tc_mma_cg<1>(tmem + T_DK, ds + 2 * (kc & 3), qmn + (uint64_t)(kc * (2048 >> 4)), idesc_g, acc);
        }
        tc_commit_cg<1>(&empty[J % NST]);
        tc_commit_cg<1>(bar_pdsfree);
      };
      int J = 0, it = 0;
      for (int sidx = blockIdx.x; sidx < nstrips; sidx += gridDim.x, ++it) {
        mbar_wait(bar_kv, it & 1);
        if (it == 0) ATRACE(1);
        for (int j = 0; j < nch; ++j, ++J) {
          mbar_wait(&full[J % NST], (J / NST) & 1);
          if (J > 0) mbar_wait(bar_tfree, (J - 1) & 1);
          tc_fence_after();
          const uint32_t stq = sbase + KsSmem::RING + (J % NST) * KsSmem::STAGE;
          const uint64_t qdesc = make_sdesc(stq, 16, 1024);
          const uint64_t dodesc = make_sdesc(stq + CH * 128, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            tc_mma_cg<1>(tmem + T_S, kdesc + 2 * kk, qdesc + 2 * kk, idesc_s, kk > 0 ? 1u : 0u);
            tc_mma_cg<1>(tmem + T_DP, vdesc + 2 * kk, dodesc + 2 * kk, idesc_s, kk > 0 ? 1u : 0u);
          }
          tc_commit_cg<1>(bar_s);
          if (j > 0) issue_grads(J - 1, j - 1);
        }
        // the strip's last gradients before the next strip's first Sᵀ / dPdᵀ,
        // which wait for its K / V: the epilogue needs the former, not the latter
        issue_grads(J - 1, nch - 1);
      }
    }
  } else if (warp == 2 + kSoftWarps) {
    if (lane == 0) {  // dSᵀ tiles (two 64-query SW128 halves) -> HBM, the dQ GEMM's A operand
      int J = 0;
      for (int sidx = blockIdx.x; sidx < nstrips; sidx += gridDim.x) {
        const StripIdx t = strip_idx(sidx, p);
        for (int j = 0; j < nch; ++j, ++J) {
          mbar_wait(bar_pds, J & 1);
          if (p.ds_store) {
            tma_store_4d(&map_ds, sbase + KsSmem::DS, j * CH, t.bh * S + t.k0, 0, 0);
            tma_store_4d(&map_ds, sbase + KsSmem::DS + 16 * KB, j * CH + 64, t.bh * S + t.k0, 0, 0);
            bulk_commit();
            bulk_wait_read<0>();
          }
          mbar_arrive(ds_free);
        }
      }
    }
  } else {
    const int sw = warp - 2, q = warp & 3, part = sw >> 2;
    const int rl = q * 32 + lane;
    const int st = threadIdx.x - 64;
    const int words = S / 32;
    // keep-bit pair -> {0, 1} multipliers of a column pair: four float2, so a
    // warp's lookups hit at most eight banks (a 16-entry float4 table of
    // nibbles cost ~1.5 M bank-conflict wavefronts per launch)
    const float2* klut = reinterpret_cast<const float2*>(smem + KsSmem::LUT);
    if (st < 4) reinterpret_cast<float2*>(smem + KsSmem::LUT)[st] = make_float2(st & 1 ? 1.f : 0.f, st & 2 ? 1.f : 0.f);
    named_bar(1, kSoftWarps * 32);
    const float lsc = __log2f(p.scale);
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const float2 sc2x2 = make_float2(p.sc2, p.sc2), ks2 = make_float2(p.ks, p.ks);
    int J = 0, it = 0;
    for (int sidx = blockIdx.x; sidx < nstrips; sidx += gridDim.x, ++it) {
      const StripIdx t = strip_idx(sidx, p);
      const size_t keyi = (size_t)t.bh * S + t.k0 + rl;
      const uint32_t* kbp = p.kb_col ? p.kb_col + keyi * words + part : nullptr;  // chunk j's word: kbp[4 j]
      uint32_t bits_n = kbp ? __ldg(kbp) : 0xFFFFFFFFu;
      const float* lse_s = rows(it);
      const float* del_s = lse_s + kMaxSeq;
      mbar_wait(&bar_rows[it & 1], (it >> 1) & 1);  // lse / D / mask rows landed
      // P' = P / divisor: the divisor's log2 folds into the row mask term
      const float mrow = (p.add_mask ? lse_s[2 * kMaxSeq + rl] * kLog2e : 0.f) + lsc;
      const float2 mrow2 = make_float2(mrow, mrow);
      float cs = 0.f;  // Σ_q dS[q, key] over this thread's columns (ds_store: the dQ column sums)
      for (int j = 0; j < nch; ++j, ++J) {
        const uint32_t bits = bits_n;
        if (kbp && j + 1 < nch) bits_n = __ldg(kbp + 4 * (j + 1));
        mbar_wait(bar_s, J & 1);
        if (it == 0 && sw == 0 && lane == 0 && j < 4) ATRACE(2 + j);
        if (j == nch - 1) {  // the strip's last Sᵀ / dPdᵀ are done: K / V are free once K's rows are kept
          if (p.bias_part && p.ds_store) {
            mbar_wait(bar_kv, it & 1);  // (observed by this thread too: the TMA writes are visible to it)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int off = rl * 128 + (((part * 2 + u) ^ (rl & 7)) << 4);
              sts128(sbase + KsSmem::KROW + off, *reinterpret_cast<const uint4*>(smem + KsSmem::K + off));
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(kv_free);
        }
        tc_fence_after();
        float sv[32], dp[32];
        tmem_ld32(trow + T_S + part * 32, sv);
        tmem_ld32(trow + T_DP + part * 32, dp);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_tfree);
        const int qc0 = j * CH + part * 32;
        uint32_t pkp[16], pks[16];
        float2 csum = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 l = reinterpret_cast<const float2*>(lse_s + qc0)[i >> 1];
          const float2 dd = reinterpret_cast<const float2*>(del_s + qc0)[i >> 1];
          const float2 tt = __ffma2_rn(make_float2(sv[i], sv[i + 1]), sc2x2, __fadd2_rn(mrow2, make_float2(-l.x, -l.y)));
          const float2 P = make_float2(ex2(tt.x), ex2(tt.y));
          const float2 kk = klut[(bits >> i) & 3u];  // keep in {0, 1}
          const float2 pd = __fmul2_rn(P, kk);
          const float2 dpm = __fmul2_rn(make_float2(dp[i], dp[i + 1]), kk);
          const float2 ds = __fmul2_rn(P, __ffma2_rn(dpm, ks2, make_float2(-dd.x, -dd.y)));
          csum = __fadd2_rn(csum, ds);
          pkp[i >> 1] = pack_bf16x2(pd.x, pd.y);
          pks[i >> 1] = pack_bf16x2(ds.x, ds.y);
        }
        cs += csum.x + csum.y;
        if (j == nch - 1) {  // the strip's lse / D / mask rows are no longer read
          __syncwarp();
          if (lane == 0) mbar_arrive(&rows_free[it & 1]);
        }
        if (J > 0) {  // the previous Pd / dS tiles: MMAs done, dS stored
          mbar_wait(bar_pdsfree, (J - 1) & 1);
          mbar_wait(ds_free, (J - 1) & 1);
        }
        st_row32(sbase + KsSmem::PD, rl, part * 32, pkp);
        st_row32(sbase + KsSmem::DS, rl, part * 32, pks);
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_pds);
      }
      // ---- epilogue
      float g2[3][16];  // dK, dV rows of this thread (and dQ's bias terms)
      const bool dq_sums = p.bias_part && p.ds_store;
      if (dq_sums) {
        // dQ = dS·K comes from the GEMM over the stored dSᵀ; its column sums
        // over this strip's keys are Σ_k cs[k] K[k][:] with cs[k] = Σ_q dS[q, k]
        // (prepared while the last gradient MMAs run)
        float* cs_s = reinterpret_cast<float*>(smem + KsSmem::CS);
        cs_s[part * QT + rl] = cs;
        named_bar(1, kSoftWarps * 32);
        const float c = ((cs_s[rl] + cs_s[QT + rl]) + cs_s[2 * QT + rl]) + cs_s[3 * QT + rl];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint4 kv = *reinterpret_cast<const uint4*>(smem + KsSmem::KROW + rl * 128 +
                                                            (((part * 2 + u) ^ (rl & 7)) << 4));
          const uint32_t w4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            g2[2][8 * u + 2 * i] = c * __uint_as_float(w4[i] << 16);
            g2[2][8 * u + 2 * i + 1] = c * __uint_as_float(w4[i] & 0xFFFF0000u);
          }
        }
      }
      // the strip's gradient MMAs are done once the last chunk's Pd / dS are released
      mbar_wait(bar_pdsfree, (J - 1) & 1);
      if (it < 3 && sw == 0 && lane == 0) ATRACE(6 + it);
      tc_fence_after();
      tmem_ld16(trow + T_DK + part * 16, g2[0]);
      tmem_ld16(trow + T_DV + part * 16, g2[1]);
      const float dvs = p.ks / p.scale;
#pragma unroll
      for (int i = 0; i < 16; ++i) g2[1][i] *= dvs;
      // bf16 dK / dV strips through SW128 tiles in the (released) Pd buffer, out by TMA
      const uint32_t tdk = sbase + KsSmem::PD, tdv = tdk + QT * 128;
#pragma unroll
      for (int tt = 0; tt < 2; ++tt)
#pragma unroll
        for (int u = 0; u < 2; ++u)
          st_sw128(tt ? tdv : tdk, rl, part * 2 + u,
                   make_uint4(pack_bf16x2(g2[tt][8 * u], g2[tt][8 * u + 1]),
                              pack_bf16x2(g2[tt][8 * u + 2], g2[tt][8 * u + 3]),
                              pack_bf16x2(g2[tt][8 * u + 4], g2[tt][8 * u + 5]),
                              pack_bf16x2(g2[tt][8 * u + 6], g2[tt][8 * u + 7])));
      fence_async_smem();
      named_bar(1, kSoftWarps * 32);
      if (st == 0) {
        tma_store_4d(&map_dkv, tdk, p.H + t.h * DH, t.row0 + t.k0, 0, 0);
        tma_store_4d(&map_dkv, tdv, 2 * p.H + t.h * DH, t.row0 + t.k0, 0, 0);
        bulk_commit();
      }
      if (p.bias_part) {  // column sums of dK, dV (and dQ) over this key strip
        float* bp = p.bias_part + (size_t)(t.b * (S / QT) + t.k0 / QT) * 3 * p.H + t.h * DH;
        float* red = reinterpret_cast<float*>(smem + KsSmem::RED);
        if (p.ds_store) {
          float* const dst[3] = {bp + p.H, bp + 2 * p.H, bp};
          strip_colsum<3>(g2, lane, q, part, st, red, dst);
        } else {
          float* const dst[2] = {bp + p.H, bp + 2 * p.H};
          strip_colsum<2>(reinterpret_cast<float(&)[2][16]>(g2), lane, q, part, st, red, dst);
        }
      }
      if (st == 0) bulk_wait_read<0>();  // the dK / dV tiles are read: Pd is free for the next strip
      named_bar(1, kSoftWarps * 32);
      if (it < 3 && sw == 0 && lane == 0) ATRACE(10 + it);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 64) ATRACE(15);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// D = rowsum(dO ∘ O) for the key-strip backward when no dq strip kernel runs
// first: four threads per (row, head) slice of 64, a 4-lane shuffle reduction
__global__ void __launch_bounds__(256) attn_bwd_delta_kernel(const __nv_bfloat16* __restrict__ o,
                                                             const __nv_bfloat16* __restrict__ dout, int64_t ld,
                                                             int T, int S, int NH, float* __restrict__ delta) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int slice = t >> 2, qtr = t & 3;
  const bool live = slice < T * NH;
  const int row = live ? slice / NH : 0, h = live ? slice - row * NH : 0;
  float2 acc = make_float2(0.f, 0.f);
  if (live) {
    const uint4* a = reinterpret_cast<const uint4*>(o + (size_t)row * ld + h * DH + qtr * 16);
    const uint4* g = reinterpret_cast<const uint4*>(dout + (size_t)row * ld + h * DH + qtr * 16);
    const uint4 va0 = __ldg(a), va1 = __ldg(a + 1), vg0 = __ldg(g), vg1 = __ldg(g + 1);
    const __nv_bfloat162* x0 = reinterpret_cast<const __nv_bfloat162*>(&va0);
    const __nv_bfloat162* x1 = reinterpret_cast<const __nv_bfloat162*>(&va1);
    const __nv_bfloat162* y0 = reinterpret_cast<const __nv_bfloat162*>(&vg0);
    const __nv_bfloat162* y1 = reinterpret_cast<const __nv_bfloat162*>(&vg1);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc = __ffma2_rn(__bfloat1622float2(x0[e]), __bfloat1622float2(y0[e]), acc);
      acc = __ffma2_rn(__bfloat1622float2(x1[e]), __bfloat1622float2(y1[e]), acc);
    }
  }
  float v = acc.x + acc.y;
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  if (live && qtr == 0) {
    const int b = row / S, srow = row - b * S;
    delta[((size_t)b * NH + h) * S + srow] = v;
  }
}

int check_common(int64_t B, int64_t NH, int64_t S, int64_t dh, const void* qkv, int64_t ld_qkv) {
  DFX_REQUIRE(B >= 1 && NH >= 1, DFX_ERR_SHAPE, "dfx_attn: batch and heads must be >= 1");
  DFX_REQUIRE(dh == DH, DFX_ERR_UNSUPPORTED, "dfx_attn: head_dim must be 64");
  DFX_REQUIRE(S >= 128 && S <= kMaxSeq && S % 128 == 0, DFX_ERR_UNSUPPORTED,
              "dfx_attn: seq must be a multiple of 128 in [128, 512]");
  DFX_REQUIRE(ld_qkv >= 3 * NH * DH && ld_qkv % 8 == 0, DFX_ERR_SHAPE, "dfx_attn: ld_qkv must be >= 3*H, %8");
  DFX_REQUIRE(aligned16(qkv), DFX_ERR_ALIGN, "dfx_attn: qkv must be 16-byte aligned");
  return DFX_OK;
}

}  // namespace
}  // namespace dfx

using namespace dfx;

extern "C" int dfx_attn_fwd(int64_t batch, int64_t heads, int64_t seq, int64_t head_dim, const void* qkv,
                            int64_t ld_qkv, const float* add_mask, const uint8_t* keep, float keep_scale,
                            float inv_divisor, void* ctx, int64_t ld_ctx, float* lse, uint32_t* keep_bits_row,
                            uint32_t* keep_bits_col, void* stream) {
  int rc = check_common(batch, heads, seq, head_dim, qkv, ld_qkv);
  if (rc) return rc;
  DFX_REQUIRE(ctx && lse, DFX_ERR_SHAPE, "dfx_attn_fwd: ctx and lse are required");
  DFX_REQUIRE(ld_ctx >= heads * DH && ld_ctx % 8 == 0 && aligned16(ctx), DFX_ERR_ALIGN,
              "dfx_attn_fwd: ctx rows must be 16-byte aligned, ld >= H");
  DFX_REQUIRE(!keep || aligned16(keep), DFX_ERR_ALIGN, "dfx_attn_fwd: keep must be 16-byte aligned");
  DFX_REQUIRE((keep_bits_row == nullptr) == (keep_bits_col == nullptr), DFX_ERR_SHAPE,
              "dfx_attn_fwd: pass both packed keep-bit outputs or neither");
  // keep == NULL with keep_bits_row set: the keep flags arrive PACKED in
  // keep_bits_row (input; only keep_bits_col is written)
  const bool kb_in = !keep && keep_bits_row;
  CUtensorMap map;
  const int64_t T = batch * seq;
  rc = make_map(&map, qkv, 2, (uint64_t)ld_qkv, (uint64_t)T, ld_qkv, 1, 0, 1, 0, 64, 64, true);
  if (rc) return rc;
  AttnFwdParams p;
  p.trace = g_attn_trace;
  p.B = (int)batch; p.NH = (int)heads; p.S = (int)seq; p.H = (int)(heads * DH);
  p.ld_ctx = ld_ctx;
  p.add_mask = add_mask;
  p.keep = keep;
  p.ks = (keep || kb_in) ? keep_scale : 1.f;
  p.kb_in = kb_in ? 1 : 0;
  p.sc2 = inv_divisor * kLog2e;
  p.ctx = reinterpret_cast<__nv_bfloat16*>(ctx);
  p.lse = lse;
  p.kb_row = keep_bits_row;
  p.kb_col = keep_bits_col;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem::TOTAL);
    cudaFuncSetAttribute(attn_fwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F3Smem::TOTAL);
    attr = true;
  }
  const int grid = (int)(batch * heads * (seq / QT));
  static const bool legacy = getenv("DFX_ATTN_FWD_LEGACY") != nullptr;  // A/B: exact two-pass, 1 CTA / SM
  if (legacy) {
    launch_k(attn_fwd_kernel, grid, kAttnThreads, FwdSmem::TOTAL, as_stream(stream), map, p);
  } else {
    CUtensorMap mctx;  // ctx strips: [128 rows x 64] boxes
    rc = make_map(&mctx, ctx, 2, (uint64_t)ld_ctx, (uint64_t)T, ld_ctx, 1, 0, 1, 0, 64, 128, true);
    if (rc) return rc;
    launch_k(attn_fwd3_kernel, std::min(grid, num_sms()), kAttnThreads, F3Smem::TOTAL, as_stream(stream), map, mctx,
             p);
  }
  DFX_LAUNCH_CHECK("dfx_attn_fwd");
  return DFX_OK;
}

// delta D [B, NH, S] f32, then (256-byte aligned) the qkv-bias column partials
// [B*S/128][3*NH*64] f32 that dfx_attn_bwd_bias_grad reduces
static size_t attn_delta_bytes(int64_t batch, int64_t heads, int64_t seq) {
  return ((size_t)(batch * heads * seq) * sizeof(float) + 255) & ~(size_t)255;
}
static size_t attn_part_bytes(int64_t batch, int64_t heads, int64_t seq) {
  return ((size_t)(batch * (seq / QT)) * 3 * heads * DH * sizeof(float) + 255) & ~(size_t)255;
}
static size_t attn_ds_bytes(int64_t batch, int64_t heads, int64_t seq) {
  return ((size_t)(batch * heads) * seq * seq * 2 + 255) & ~(size_t)255;
}
// dQ[b, h] = dS[b, h] · K[b, h]: A = the stored dSᵀ read MN-major, B = K read MN-major from qkv
static dfx_gemm_args dq_gemm_args(int64_t batch, int64_t heads, int64_t seq, const void* qkv, int64_t ld_qkv,
                                  const void* dsT, void* dqkv, int64_t ld_dqkv) {
  dfx_gemm_args g{};
  g.in_dtype = DFX_BF16; g.out_dtype = DFX_BF16; g.epilogue = DFX_EPI_NONE;
  g.m = seq; g.n = DH; g.k = seq; g.batch1 = batch; g.batch2 = heads;
  g.a = dsT; g.a_stride_m = 1; g.a_stride_k = seq; g.a_stride_b2 = seq * seq; g.a_stride_b1 = heads * seq * seq;
  g.b = reinterpret_cast<const __nv_bfloat16*>(qkv) + heads * DH;
  g.b_stride_n = 1; g.b_stride_k = ld_qkv; g.b_stride_b2 = DH; g.b_stride_b1 = seq * ld_qkv;
  g.d = dqkv; g.d_stride_m = ld_dqkv; g.d_stride_b2 = DH; g.d_stride_b1 = seq * ld_dqkv;
  g.alpha = 1.f; g.beta = 0.f;
  return g;
}
// delta [B, NH, S] f32 | qkv-bias column partials [B*S/128][3*NH*64] f32 |
// dSᵀ [B, NH, S(key), S(query)] bf16 | the dQ GEMM's split-K partials (few heads)
extern "C" size_t dfx_attn_bwd_workspace(int64_t batch, int64_t heads, int64_t seq) {
  const dfx_gemm_args g = dq_gemm_args(batch, heads, seq, nullptr, 3 * heads * DH, nullptr, nullptr, 3 * heads * DH);
  return attn_delta_bytes(batch, heads, seq) + attn_part_bytes(batch, heads, seq) + attn_ds_bytes(batch, heads, seq) +
         gemm_tc_workspace(g) + 256;
}

extern "C" int dfx_attn_bwd(int64_t batch, int64_t heads, int64_t seq, int64_t head_dim, const void* qkv,
                            int64_t ld_qkv, const void* ctx, const void* dctx, int64_t ld_ctx, const float* add_mask,
                            const float* lse, const uint32_t* keep_bits_row, const uint32_t* keep_bits_col,
                            float keep_scale, float inv_divisor, void* dqkv, int64_t ld_dqkv, void* workspace,
                            size_t ws_bytes, void* stream) {
  int rc = check_common(batch, heads, seq, head_dim, qkv, ld_qkv);
  if (rc) return rc;
  DFX_REQUIRE(ctx && dctx && lse && dqkv, DFX_ERR_SHAPE, "dfx_attn_bwd: ctx, dctx, lse, dqkv are required");
  DFX_REQUIRE(ld_ctx >= heads * DH && ld_ctx % 8 == 0 && aligned16(ctx) && aligned16(dctx), DFX_ERR_ALIGN,
              "dfx_attn_bwd: ctx/dctx rows must be 16-byte aligned, ld >= H");
  DFX_REQUIRE(ld_dqkv >= 3 * heads * DH && ld_dqkv % 8 == 0 && aligned16(dqkv), DFX_ERR_ALIGN,
              "dfx_attn_bwd: dqkv rows must be 16-byte aligned, ld >= 3H");
  DFX_REQUIRE((keep_bits_row == nullptr) == (keep_bits_col == nullptr), DFX_ERR_SHAPE,
              "dfx_attn_bwd: pass both packed keep-bit tensors or neither");
  DFX_REQUIRE(workspace && ws_bytes >= dfx_attn_bwd_workspace(batch, heads, seq) && aligned16(workspace),
              DFX_ERR_WORKSPACE, "dfx_attn_bwd: needs dfx_attn_bwd_workspace() bytes of workspace");
  const int64_t T = batch * seq;
  CUtensorMap mqkv, mdo, mo;
  rc = make_map(&mqkv, qkv, 2, (uint64_t)ld_qkv, (uint64_t)T, ld_qkv, 1, 0, 1, 0, 64, 64, true);
  if (rc) return rc;
  rc = make_map(&mdo, dctx, 2, (uint64_t)ld_ctx, (uint64_t)T, ld_ctx, 1, 0, 1, 0, 64, 64, true);
  if (rc) return rc;
  rc = make_map(&mo, ctx, 2, (uint64_t)ld_ctx, (uint64_t)T, ld_ctx, 1, 0, 1, 0, 64, 64, true);
  if (rc) return rc;
  CUtensorMap mdkv;  // dK / dV strips: [128 keys x 64] boxes of dqkv
  rc = make_map(&mdkv, dqkv, 2, (uint64_t)ld_dqkv, (uint64_t)T, ld_dqkv, 1, 0, 1, 0, 64, 128, true);
  if (rc) return rc;
  AttnBwdParams p;
  p.trace = nullptr;
  p.B = (int)batch; p.NH = (int)heads; p.S = (int)seq; p.H = (int)(heads * DH);
  p.ld_ctx = ld_ctx; p.ld_dqkv = ld_dqkv;
  p.qkv = reinterpret_cast<const __nv_bfloat16*>(qkv); p.ld_qkv = ld_qkv;
  p.ctx = reinterpret_cast<const __nv_bfloat16*>(ctx);
  p.dctx = reinterpret_cast<const __nv_bfloat16*>(dctx);
  p.add_mask = add_mask; p.lse = lse;
  p.delta = reinterpret_cast<float*>(workspace);
  p.bias_part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(workspace) + attn_delta_bytes(batch, heads, seq));
  p.kb_row = keep_bits_row; p.kb_col = keep_bits_col;
  p.ks = keep_bits_row ? keep_scale : 1.f;
  p.sc2 = inv_divisor * kLog2e;
  p.scale = inv_divisor;
  p.dqkv = reinterpret_cast<__nv_bfloat16*>(dqkv);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_bwd_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DqSmem::TOTAL);
    cudaFuncSetAttribute(attn_bwd_kstrip_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, KsSmem::TOTAL);
    attr = true;
  }
  const int grid = (int)(batch * heads * (seq / QT));
  static const bool legacy = getenv("DFX_ATTN_BWD_LEGACY") != nullptr;  // A/B: the dq strip kernel for dQ
  if (!legacy) {
    // D pre-pass -> key-strip kernel (dK, dV, dSᵀ to HBM, bias sums) -> dQ = dS·K GEMM
    uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
    __nv_bfloat16* dsT = reinterpret_cast<__nv_bfloat16*>(ws + attn_delta_bytes(batch, heads, seq) +
                                                          attn_part_bytes(batch, heads, seq));
    CUtensorMap mds;
    rc = make_map(&mds, dsT, 2, (uint64_t)seq, (uint64_t)(batch * heads * seq), seq, 1, 0, 1, 0, 64, 128, true);
    if (rc) return rc;
    const int nthr = (int)(T * heads * 4);
    launch_k(attn_bwd_delta_kernel, (nthr + 255) / 256, 256, 0, as_stream(stream), p.ctx, p.dctx, ld_ctx, (int)T,
             (int)seq, (int)heads, p.delta);
    DFX_LAUNCH_CHECK("dfx_attn_bwd (delta)");
    p.ds_store = 1;
    p.trace = g_attn_trace;
    launch_k(attn_bwd_kstrip_kernel, std::min(grid, num_sms()), kKsThreads, KsSmem::TOTAL, as_stream(stream), mqkv,
             mdo, mds, mdkv, p);
    DFX_LAUNCH_CHECK("dfx_attn_bwd (dk, dv, dS)");
    dfx_gemm_args g = dq_gemm_args(batch, heads, seq, qkv, ld_qkv, dsT, dqkv, ld_dqkv);
    g.workspace = reinterpret_cast<uint8_t*>(dsT) + attn_ds_bytes(batch, heads, seq);
    g.workspace_bytes = gemm_tc_workspace(g);
    DFX_REQUIRE(gemm_tc_supported(g), DFX_ERR_UNSUPPORTED, "dfx_attn_bwd: dQ GEMM shape not on the tcgen05 path");
    return gemm_tc(g, as_stream(stream));
  }
  p.ds_store = 0;
  // debug timeline of the dq kernel, or of kstrip with DFX_ATTN_TRACE_KSTRIP set (tools/attn_trace.py)
  const bool trace_ks = getenv("DFX_ATTN_TRACE_KSTRIP") != nullptr;
  p.trace = trace_ks ? nullptr : g_attn_trace;
  launch_k(attn_bwd_dq_kernel, grid, kAttnThreads, DqSmem::TOTAL, as_stream(stream), mqkv, mdo, mo, p);
  DFX_LAUNCH_CHECK("dfx_attn_bwd (dq)");
  p.trace = trace_ks ? g_attn_trace : nullptr;
  launch_k(attn_bwd_kstrip_kernel, std::min(grid, num_sms()), kKsThreads, KsSmem::TOTAL, as_stream(stream), mqkv, mdo,
           mqkv, mdkv, p);
  DFX_LAUNCH_CHECK("dfx_attn_bwd (dk, dv)");
  return DFX_OK;
}

extern "C" int dfx_attn_bwd_bias_grad(int64_t batch, int64_t heads, int64_t seq, const void* workspace,
                                      size_t ws_bytes, float* dbias, int accumulate, void* stream) {
  DFX_REQUIRE(dbias && workspace && ws_bytes >= dfx_attn_bwd_workspace(batch, heads, seq), DFX_ERR_WORKSPACE,
              "dfx_attn_bwd_bias_grad: pass the workspace of the preceding dfx_attn_bwd");
  DFX_REQUIRE(seq % QT == 0, DFX_ERR_SHAPE, "dfx_attn_bwd_bias_grad: seq must be a multiple of 128");
  const int cols = (int)(3 * heads * DH);
  const float* part = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(workspace) +
                                                     attn_delta_bytes(batch, heads, seq));
  launch_k(attn_bias_reduce_kernel, (cols + 255) / 256, 256, 0, as_stream(stream), (int)(batch * (seq / QT)), cols,
           part, dbias, accumulate);
  DFX_LAUNCH_CHECK("dfx_attn_bwd_bias_grad");
  return DFX_OK;
}

extern "C" __attribute__((visibility("default"))) void dfx_debug_attn_trace(void* buf) {
  dfx::g_attn_trace = reinterpret_cast<unsigned long long*>(buf);
}
