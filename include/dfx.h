/*
 * dfx.h — C ABI of the B200 (sm_100a) fused training hot path.
 *
 * This is the drop-in boundary that replaces the CPU execution of the fused
 * memory-bound subgraphs of a training step in the reference `dfir` package
 * (arXiv 2110.10802 re-specification, /root/reference/pkg/src/dfir).  The
 * reference executes these subgraphs through
 *
 *     interp.execute(g, inputs, bindings, library_eval)      interp.py:1301-1317
 *       -> _Execution.run_library -> library_eval(op, attrs, inputs)
 *                                                             interp.py:337-368
 *       -> frontend.reference_apply(op, attrs, inputs)        frontend.py:146-150
 *
 * and through the manual VJPs of autodiff.py (1363-1617).  The Python host
 * layer (paper_2110_10802_b200/library_eval.py) binds every entry point below
 * with ctypes and exposes the same `library_eval(op, attrs, inputs)` seam;
 * INTEGRATION.md shows the binding.  Each function cites the reference
 * operator(s) whose semantics it implements.
 *
 * Conventions
 *  - Plain pointers to DEVICE memory, element counts and element strides; no
 *    framework types.  `stream` is a cudaStream_t passed as void*.
 *  - Calls are asynchronous and stream-ordered; no host synchronisation, no
 *    allocation.  Callers own every buffer (interp.py:206-212 ownership rule).
 *  - Reductions are fixed-order (no float atomics): results are bitwise
 *    reproducible run to run (the reference's determinism, autodiff.py:19-25).
 *  - Return value: DFX_OK (0) or a DFX_ERR_* code; dfx_last_error() returns a
 *    thread-local message (mirrors ShapeError / ExecError text).
 *  - dtype codes extend the DTNS codes (dtns.py:30-45): 0=f32 1=f64 2=i64
 *    3=bool, plus 4=bf16 and 5=u8.  Activation tensors are f32 or bf16;
 *    parameter vectors (bias, gamma, beta) and statistics are always f32.
 *  - Dropout masks are u8 keep flags (0/1) plus keep_scale = 1/(1-p): the
 *    reference's explicit float mask tensor equals keep * keep_scale
 *    (no Dropout op exists in the reference).
 */
#ifndef DFX_H_
#define DFX_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

enum dfx_dtype { DFX_F32 = 0, DFX_F64 = 1, DFX_I64 = 2, DFX_BOOL = 3, DFX_BF16 = 4, DFX_U8 = 5 };

enum dfx_status {
  DFX_OK = 0,
  DFX_ERR_SHAPE = 1,       /* frontend.ShapeError analogue */
  DFX_ERR_DTYPE = 2,
  DFX_ERR_ALIGN = 3,       /* pointer/stride alignment the kernel needs */
  DFX_ERR_CUDA = 4,        /* launch or runtime failure */
  DFX_ERR_UNSUPPORTED = 5, /* frontend.UnsupportedOp analogue */
  DFX_ERR_WORKSPACE = 6
};

/* ---- library ------------------------------------------------------------ */
const char* dfx_last_error(void);
int dfx_version(void);
/* DFX_OK iff the current device is an sm_100 part the cubins were built for. */
int dfx_device_check(void);
/* Number of kernel launches issued by this thread since the last reset. */
int64_t dfx_launch_count(void);
void dfx_reset_launch_count(void);

/* ---- a1/a2: bias + dropout + residual + LayerNorm (forward) --------------
 * s = (h + bias) * keep * keep_scale + residual ; y = LN(s) over the last axis
 * Replaces Add (frontend.py:291) + Mul (293) + Add + LayerNormalization
 * (frontend.py:519-529; biased variance).  keep may be NULL (no dropout),
 * bias may be NULL, residual may be NULL.  s_stash, mean, rstd may be NULL;
 * the backward needs s_stash (or recomputes nothing else). */
int dfx_bdrln_fwd(int dtype, int64_t rows, int64_t cols, const void* h, const float* bias,
                  const uint8_t* keep, float keep_scale, const void* residual,
                  const float* gamma, const float* beta, float eps, void* y, void* s_stash,
                  float* mean, float* rstd, void* stream);

/* Same, with the keep flags bit-packed: bit e % 32 of keep_bits[e / 32] is the
 * keep flag of flat element e = row * cols + col (kernels.pack_keep_bits over
 * the last axis; rows * cols % 32 == 0).  8x fewer mask bytes over PCIe and
 * HBM than the u8 form; results are identical. */
int dfx_bdrln_fwd_kb(int dtype, int64_t rows, int64_t cols, const void* h, const float* bias,
                     const uint32_t* keep_bits, float keep_scale, const void* residual,
                     const float* gamma, const float* beta, float eps, void* y, void* s_stash,
                     float* mean, float* rstd, void* stream);

/* ---- a3: backward of the above -------------------------------------------
 * LN VJP (autodiff.py:1490-1545): ds = rstd*(dy*g - mean(dy*g) - xhat*mean(dy*g*xhat))
 * dh = ds * keep * keep_scale ; dgamma = sum_rows dy*xhat ; dbeta = sum_rows dy ;
 * dbias = sum_rows dh.  ds is also the gradient of `residual`.  Any of dh,
 * dgamma, dbeta, dbias may be NULL.  Workspace: dfx_bdrln_bwd_workspace(). */
size_t dfx_bdrln_bwd_workspace(int64_t rows, int64_t cols);
int dfx_bdrln_bwd(int dtype, int64_t rows, int64_t cols, const void* dy, const void* s_stash,
                  const float* gamma, const uint8_t* keep, float keep_scale, float eps,
                  void* ds, void* dh, float* dgamma, float* dbeta, float* dbias, void* workspace,
                  size_t ws_bytes, void* stream);
/* dfx_bdrln_bwd with bit-packed keep flags (layout as dfx_bdrln_fwd_kb). */
int dfx_bdrln_bwd_kb(int dtype, int64_t rows, int64_t cols, const void* dy, const void* s_stash,
                     const float* gamma, const uint32_t* keep_bits, float keep_scale, float eps,
                     void* ds, void* dh, float* dgamma, float* dbeta, float* dbias, void* workspace,
                     size_t ws_bytes, void* stream);
/* The parameter-gradient half of dfx_bdrln_bwd as its own launch: call
 * dfx_bdrln_bwd with dgamma = dbeta = dbias = NULL (it leaves the per-block
 * partial sums in `workspace`), then this — possibly on another stream, after
 * an event — to reduce them (fixed order) into dgamma / dbeta / dbias. */
int dfx_bdrln_bwd_finalize(int dtype, int64_t rows, int64_t cols, const void* workspace, size_t ws_bytes,
                           float* dgamma, float* dbeta, float* dbias, void* stream);

/* ---- a4/a5: scaled + masked softmax + dropout (forward) -------------------
 * rows are [batch, heads, q] (row-major), cols = k.
 * p  = softmax(scores * inv_divisor + add_mask[b, :])     (Div frontend.py:294,
 *      Add 175-188, Softmax 493-501)
 * pd = p * keep * keep_scale                               (Mul 293)
 * add_mask is f32 [batch, cols] or NULL; keep/pd may be NULL. */
int dfx_softmax_fwd(int dtype, int64_t batch, int64_t heads, int64_t q, int64_t cols,
                    const void* scores, float inv_divisor, const float* add_mask,
                    const uint8_t* keep, float keep_scale, void* p, void* pd, void* stream);

/* ---- a6: backward (autodiff.py:1465-1484, stashes the forward output p) ----
 * g = dpd * keep * keep_scale ; dscores = (g - sum(g*p)) * p * inv_divisor */
int dfx_softmax_bwd(int dtype, int64_t rows, int64_t cols, const void* dpd, const void* p,
                    const uint8_t* keep, float keep_scale, float inv_divisor, void* dscores,
                    void* stream);

/* ---- a4-a6 + a8 fused: scaled-masked-softmax attention (bf16, tcgen05) -----
 * The QKᵀ Einsum (frontend.py:408-481), Div by `divisor` (294), additive mask
 * (175-188), Softmax (493-501), dropout Mul (293) and the PV Einsum of one
 * encoder layer in one kernel, the [B,NH,S,S] scores never leaving the SM
 * (the reference recipe's per-query-row attention map).
 * qkv: bf16 [B*S, ld_qkv] holding Q | K | V column blocks of NH*64 columns
 * (head h = columns h*64..h*64+63 of each block); head_dim must be 64,
 * seq a multiple of 128 and <= 512.
 *   ctx[b*S+s, h*64+d] = sum_t Pd[b,h,s,t] V[b*S+t, h*64+d]   (bf16)
 *   lse[b,h,s]          = log2 sum_t exp2(log2e*(S/divisor + mask))  (f32)
 *   keep_bits_row[b,h,s,t/32] bit t%32 = keep[b,h,s,t]; keep_bits_col[b,h,t,s/32]
 *   bit s%32 = keep[b,h,s,t] — the packed dropout masks the backward reads
 *   (each [B,NH,S,S/32] u32; pass both or neither; keep may be NULL = no dropout).
 *   keep == NULL with keep_bits_row != NULL: the keep flags are supplied
 *   PACKED in keep_bits_row (an input, 1/8 of the u8 bytes); only
 *   keep_bits_col is written. */
int dfx_attn_fwd(int64_t batch, int64_t heads, int64_t seq, int64_t head_dim, const void* qkv,
                 int64_t ld_qkv, const float* add_mask, const uint8_t* keep, float keep_scale,
                 float inv_divisor, void* ctx, int64_t ld_ctx, float* lse, uint32_t* keep_bits_row,
                 uint32_t* keep_bits_col, void* stream);
/* Backward of the above (Einsum VJPs autodiff.py:1363-1415, Softmax VJP
 * 1465-1484, dropout Mul VJP): writes dQ | dK | dV into dqkv [B*S, ld_dqkv]
 * (bf16, same column layout as qkv).  ctx is the forward output, dctx its
 * gradient (both [B*S, ld_ctx] bf16).  Workspace: dfx_attn_bwd_workspace(). */
size_t dfx_attn_bwd_workspace(int64_t batch, int64_t heads, int64_t seq);
int dfx_attn_bwd(int64_t batch, int64_t heads, int64_t seq, int64_t head_dim, const void* qkv,
                 int64_t ld_qkv, const void* ctx, const void* dctx, int64_t ld_ctx,
                 const float* add_mask, const float* lse, const uint32_t* keep_bits_row,
                 const uint32_t* keep_bits_col, float keep_scale, float inv_divisor, void* dqkv,
                 int64_t ld_dqkv, void* workspace, size_t ws_bytes, void* stream);
/* The qkv bias gradient dbias[3*NH*64] (+)= column sums of dQ | dK | dV, from
 * the per-strip partial sums dfx_attn_bwd leaves in its workspace (fixed
 * order; the unrounded fp32 gradients).  Replaces a column-sum pass over the
 * [B*S, 3H] dqkv tensor (Gemm C-input VJP, autodiff.py:1416-1459). */
int dfx_attn_bwd_bias_grad(int64_t batch, int64_t heads, int64_t seq, const void* workspace,
                           size_t ws_bytes, float* dbias, int accumulate, void* stream);

/* ---- a7: bias + tanh-GELU -------------------------------------------------
 * pre = f + bias ; y = 0.5*pre*(1+tanh(0.7978845608*(pre+0.044715*pre^3)))
 * (Pow/Mul/Add/Tanh chain, frontend.py:223-295).  pre may be NULL. */
int dfx_bias_gelu_fwd(int dtype, int64_t rows, int64_t cols, const void* f, const float* bias,
                      void* pre, void* y, void* stream);
/* dpre = dy * gelu'(pre) (symexpr.py:672-738 derivative); dbias = colsum(dpre)
 * (NULL to skip).  Workspace: dfx_colsum_workspace(rows, cols). */
int dfx_bias_gelu_bwd(int dtype, int64_t rows, int64_t cols, const void* dy, const void* pre,
                      void* dpre, float* dbias, void* workspace, size_t ws_bytes, void* stream);

/* ---- column sums (bias gradients; Gemm VJP of C, autodiff.py:1452-1458) ---- */
size_t dfx_colsum_workspace(int64_t rows, int64_t cols);
int dfx_colsum(int dtype, int64_t rows, int64_t cols, const void* x, int64_t ld, float* out,
               int accumulate, void* workspace, size_t ws_bytes, void* stream);

/* ---- a8: contractions -------------------------------------------------------
 * D[b1,b2][m,n] = epilogue( alpha * sum_k A[b1,b2](m,k) * B[b1,b2](n,k) )
 * Gemm (frontend.py:369-405) / MatMul (335-366) / Einsum (408-481) with their
 * VJPs (autodiff.py:1363-1459).  A and B are each either K-contiguous
 * (stride_k == 1) or M/N-contiguous (stride_m/stride_n == 1); D is
 * N-contiguous.  bf16 inputs run on tcgen05 tensor cores (TMA-fed, TMEM
 * accumulator) when the shape tiles (m%128, k%64, 16B-aligned rows/strides);
 * everything else (and f32) runs on the CUDA-core FP32 path so f32 results
 * meet the 1e-4 parity bar. */
enum dfx_epilogue {
  DFX_EPI_NONE = 0,      /* D = alpha*acc                                     */
  DFX_EPI_BIAS = 1,      /* D = alpha*acc + bias[n]                           */
  DFX_EPI_BIAS_GELU = 2, /* pre = alpha*acc + bias[n]; aux_out = pre; D = gelu(pre) */
  DFX_EPI_GELU_BWD = 3,  /* D = alpha*acc * gelu'(aux)                        */
  DFX_EPI_ADD = 4        /* D = alpha*acc + beta*aux                          */
};

typedef struct dfx_gemm_args {
  int32_t in_dtype;   /* DFX_F32 or DFX_BF16 (A and B)                */
  int32_t out_dtype;  /* DFX_F32 or DFX_BF16 (D, aux, aux_out)         */
  int32_t epilogue;   /* enum dfx_epilogue                             */
  int32_t force_simt; /* 1: skip the tensor-core path (testing)        */
  int64_t m, n, k;
  int64_t batch1, batch2; /* >= 1 */
  const void* a;
  int64_t a_stride_m, a_stride_k, a_stride_b1, a_stride_b2;
  const void* b;
  int64_t b_stride_n, b_stride_k, b_stride_b1, b_stride_b2;
  void* d;
  int64_t d_stride_m, d_stride_b1, d_stride_b2;
  float alpha, beta;
  const float* bias; /* [n] */
  const void* aux;
  int64_t aux_stride_m, aux_stride_b1, aux_stride_b2;
  void* aux_out;
  int64_t aux_out_stride_m, aux_out_stride_b1, aux_out_stride_b2;
  void* workspace; /* split-K partials (tensor-core path); see dfx_gemm_workspace */
  size_t workspace_bytes;
} dfx_gemm_args;

int dfx_gemm(const dfx_gemm_args* args, void* stream);
/* Workspace bytes dfx_gemm needs for these args (0 when none). */
size_t dfx_gemm_workspace(const dfx_gemm_args* args);
/* 1 if the call would take the tcgen05 path. */
int dfx_gemm_uses_tensor_cores(const dfx_gemm_args* args);
/* SE excite folded into an MBConv block's project 1x1 conv (bf16 only):
 *   d[m][n] = sum_k y[m][k] w[n][k],
 *   y[m][k] = swish(z[m][k] * rstd[k]*gamma[k] + beta[k] - mean[k]*rstd[k]*gamma[k]) * gate[m / hw][k]
 * with y formed in shared memory from the TMA-loaded z tiles (tcgen05 GEMM with
 * A-transform warps); y is also written to y_out when non-NULL (the weight
 * gradient's operand).  Replaces excite (dfx_mbconv_fwd_se's last pass) +
 * the project dfx_gemm: one read of z instead of read z, write y, read y.
 * Reference: Conv 1x1 (frontend.py:598-678) of Mul(a, Sigmoid(...)) (frontend.py:293). */
int dfx_gemm_excite(int64_t m, int64_t k, int64_t n, const void* z, int64_t hw, const float* mean,
                    const float* rstd, const float* gamma, const float* beta, const float* gate,
                    const void* w, void* d, void* y_out, void* stream);

/* ---- a9-a13: EfficientNet-B0 MBConv block, NHWC ---------------------------
 * x [N,H,W,C] (f32 or bf16, C % 4 (f32) / C % 8 (bf16) == 0); depthwise
 * ksize x ksize (3 or 5; EfficientNet-B0 uses both) weight stored [k][k][C]
 * f32 (the reference's (C,1,k,k) transposed); pads = {top, left, bottom,
 * right} in [0, ksize-1]; stride 1 or 2.
 *   Conv group=C (frontend.py:598-678; depthwise check 608-635)
 *   BatchNormalization, training mode (frontend.py:544-591): biased variance,
 *     running = running*momentum + batch*(1-momentum)
 *   swish = Mul(u, Sigmoid(u)) (frontend.py:229, 293)
 *   SE: GlobalAveragePool (681-706) -> Gemm(Wr [SE,C], transB) -> swish ->
 *       Gemm(We [C,SE], transB) -> Sigmoid -> broadcast Mul
 * Backward: BN VJP autodiff.py:1557-1617, depthwise conv VJP of the lowered
 * loop nest (lowering.py:930-1004 + tasklet VJPs, autodiff.py:1623-1629).
 * One workspace (dfx_mbconv_workspace) serves every call of a step. */
size_t dfx_mbconv_workspace(int64_t N, int64_t H, int64_t W, int64_t C, int stride, int ksize,
                            const int* pads, int SE);
/* z = dwconv(x); bn_local[3][C] = per-channel (count, mean, M2) of z on this
 * rank (Welford, fixed order).  SyncBN gathers bn_local of every rank. */
int dfx_mbconv_fwd_stats(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int stride,
                         int ksize, const int* pads, const void* x, const float* w_dw, void* z, float* bn_local,
                         void* workspace, size_t ws_bytes, void* stream);
/* Merge nsets (count, mean, M2) sets in order -> mean, var (biased), rstd and
 * the running-statistic update (any output but rstd may be NULL). */
int dfx_bn_finalize(int64_t C, int nsets, const float* sets, float eps, float momentum, float* mean,
                    float* var, float* rstd, float* run_mean, float* run_var, void* stream);
/* pooled[N][C] = mean_hw swish(BN(z)); r[N][SE] = Wr pooled + br;
 * s[N][C] = sigmoid(We swish(r) + be); y = swish(BN(z)) * s.  y == NULL
 * skips the excite pass (its consumer, dfx_gemm_excite, forms y itself). */
int dfx_mbconv_fwd_se(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int stride,
                      int ksize, const int* pads, int64_t SE, const void* z, const float* mean, const float* rstd,
                      const float* gamma, const float* beta, const float* w_r, const float* b_r,
                      const float* w_e, const float* b_e, float* pooled, float* r, float* s, void* y,
                      void* workspace, size_t ws_bytes, void* stream);
/* Backward part 1 (given dy): SE-MLP gradients dw_e [C][SE], db_e [C],
 * dw_r [SE][C], db_r [SE]; dpool[N][C] (per-pixel gradient reaching a from
 * the pool); bnsum[2][C] = (sum du, sum du*xhat) = (dbeta, dgamma) of this
 * rank — SyncBN allreduces bnsum before part 2. */
int dfx_mbconv_bwd_reduce(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int stride,
                          int ksize, const int* pads, int64_t SE, const void* dy, const void* z,
                          const float* mean, const float* rstd, const float* gamma,
                          const float* beta, const float* s, const float* r, const float* pooled,
                          const float* w_r, const float* w_e, float* dw_e, float* db_e, float* dw_r,
                          float* db_r, float* dpool, float* bnsum, void* workspace, size_t ws_bytes,
                          void* stream);
/* Backward part 2: dx and dw_dw [3][3][C]; count = number of elements each
 * BN channel normalises over (all ranks), or 0 for SyncBN: bnsum is then
 * [3][C] and bnsum[2][c] holds the allreduced per-channel count (each rank
 * contributes its own local count, so unequal per-rank batches normalise
 * exactly as the forward's merged statistics do). */
int dfx_mbconv_bwd_dx(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int stride,
                      int ksize, const int* pads, const void* dy, const void* z, const void* x,
                      const float* w_dw, const float* mean, const float* rstd, const float* gamma,
                      const float* beta, const float* s, const float* dpool, const float* bnsum,
                      double count, void* dx, float* dw_dw, void* workspace, size_t ws_bytes,
                      void* stream);

/* ---- C4: normalisation sweep (LayerNorm vs BatchNorm fused with an activation)
 * act: 0 = none, 1 = swish (Mul(u, Sigmoid(u)), frontend.py:229, 293).
 * LayerNorm over the last axis (frontend.py:519-529; VJP autodiff.py:1490-1545):
 * rows x cols, y = act(LN(x)); the backward recomputes the statistics from x.
 * Workspace: dfx_bdrln_bwd_workspace(rows, cols). */
int dfx_layernorm_act_fwd(int dtype, int64_t rows, int64_t cols, const void* x, const float* gamma,
                          const float* beta, float eps, int act, void* y, void* stream);
int dfx_layernorm_act_bwd(int dtype, int64_t rows, int64_t cols, const void* dy, const void* x,
                          const float* gamma, const float* beta, float eps, int act, void* dx,
                          float* dgamma, float* dbeta, void* workspace, size_t ws_bytes,
                          void* stream);
/* BatchNorm over the channel axis, channels-last [rows, C] (rows = N x spatial),
 * training mode (frontend.py:544-591; VJP autodiff.py:1557-1617).
 *   stats: local[3][C] = (count, mean, M2) — finalize with dfx_bn_finalize
 *          (nsets = #ranks for SyncBN)
 *   apply: y = act((x - mean) * rstd * gamma + beta)
 *   bwd_reduce: bnsum[2][C] = (sum du, sum du*xhat) = (dbeta, dgamma)
 *   bwd_dx: dx = gamma*rstd*(du - bnsum[0]/count - xhat*bnsum[1]/count);
 *           count = 0 (SyncBN): per-channel count read from bnsum[2][C] */
size_t dfx_batchnorm_workspace(int64_t rows, int64_t C);
int dfx_batchnorm_stats(int dtype, int64_t rows, int64_t C, const void* x, float* local,
                        void* workspace, size_t ws_bytes, void* stream);
int dfx_batchnorm_act_apply(int dtype, int64_t rows, int64_t C, const void* x, const float* mean,
                            const float* rstd, const float* gamma, const float* beta, int act,
                            void* y, void* stream);
int dfx_batchnorm_act_bwd_reduce(int dtype, int64_t rows, int64_t C, const void* dy, const void* x,
                                 const float* mean, const float* rstd, const float* gamma,
                                 const float* beta, int act, float* bnsum, void* workspace,
                                 size_t ws_bytes, void* stream);
int dfx_batchnorm_act_bwd_dx(int dtype, int64_t rows, int64_t C, const void* dy, const void* x,
                             const float* mean, const float* rstd, const float* gamma,
                             const float* beta, int act, const float* bnsum, double count, void* dx,
                             void* stream);
/* Single-replica fusions of the calls above (one launch fewer each):
 *   stats_finalize = dfx_batchnorm_stats + dfx_bn_finalize(nsets = 1) — the
 *     statistics of the one set written by the merge (local as before);
 *   bwd_reduce_grads = dfx_batchnorm_act_bwd_reduce that also writes the local
 *     parameter gradients dbeta = bnsum[0], dgamma = bnsum[1] (either may be NULL). */
int dfx_batchnorm_stats_finalize(int dtype, int64_t rows, int64_t C, const void* x, float* local,
                                 float eps, float momentum, float* mean, float* var, float* rstd,
                                 float* run_mean, float* run_var, void* workspace, size_t ws_bytes,
                                 void* stream);
int dfx_batchnorm_act_bwd_reduce_grads(int dtype, int64_t rows, int64_t C, const void* dy,
                                       const void* x, const float* mean, const float* rstd,
                                       const float* gamma, const float* beta, int act, float* bnsum,
                                       float* dbeta, float* dgamma, void* workspace, size_t ws_bytes,
                                       void* stream);

/* ---- C5: EfficientNet-B0 training-step glue (NHWC) ------------------------
 * stem im2col for a 3x3 conv (frontend.py:598-678): cols [N*Ho*Wo, Kp] with
 *   k = (ky*3 + kx)*Cin + c, zeros for padding taps and k >= 9*Cin;
 * GlobalAveragePool (frontend.py:681-706) and its VJP over [N, HW, C];
 * softmax cross-entropy: loss = mean_n(logsumexp(z_n) - z_n[label_n]) (the
 *   Softmax of frontend.py:488-501 + the log-likelihood of the label),
 *   dlogits = (softmax(z) - onehot) / N;
 * residual Add (frontend.py:291): out = a + b (out may alias a or b). */
int dfx_im2col3x3(int dtype, int64_t N, int64_t H, int64_t W, int64_t Cin, int stride, const int* pads,
                  int64_t Kp, const void* x, void* cols, void* stream);
int dfx_avgpool_fwd(int dtype, int64_t N, int64_t HW, int64_t C, const void* x, void* pooled, void* stream);
int dfx_avgpool_bwd(int dtype, int64_t N, int64_t HW, int64_t C, const void* dpooled, void* dx, void* stream);
int dfx_softmax_xent(int64_t N, int64_t classes, const float* logits, const int32_t* labels, float* loss,
                     float* loss_rows, int grad_dtype, void* dlogits, void* stream);
int dfx_add(int dtype, int64_t n, const void* a, const void* b, void* out, void* stream);

/* ---- optimizer (the user-written SGD step of the training loop) --
 * master -= lr * grad (f32); if weights_bf16 != NULL also refresh the bf16 copy. */
int dfx_sgd_update(int64_t n, float* master, const float* grad, float lr, void* weights_bf16,
                   void* stream);
/* y = x * scale (f32, in place allowed) — gradient averaging after allreduce. */
int dfx_scale_f32(int64_t n, float* x, float scale, void* stream);
/* bf16 <-> f32 casts of flat buffers. */
int dfx_cast(int64_t n, int src_dtype, const void* src, int dst_dtype, void* dst, void* stream);
/* dst0 = cast(src0), dst1 = cast(src1) (n elements each) in one launch. */
int dfx_cast2(int64_t n, int src_dtype, const void* src0, const void* src1, int dst_dtype, void* dst0,
              void* dst1, void* stream);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* DFX_H_ */
