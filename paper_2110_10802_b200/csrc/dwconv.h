// dwconv.h — internal entry points of the TMA row-ring depthwise convolution
// (dwconv.cu), used by the MBConv block (mbconv.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace dfx {

// One depthwise correlation, NHWC: out[n,oy,ox,c] =
//   sum_{ky,kx} in[n, oy*s+ky-pt, ox*s+kx-pl, c] * w[ky*KS+kx][c]
// (the Conv group=C reference, frontend.py:645-666; zero padding = reads
// outside the input grid, lowering.py:949-971).
struct DwShape {
  int N, Hi, Wi, Ho, Wo, C;
  int ks, s, pt, pl;
};

// BN-VJP constants for the fused dz = dBN(dswish(dy*s + dpool)) (autodiff.py:1557-1617)
struct DzConsts {
  const float *mean, *rstd, *gamma, *beta;  // [C]
  const float *s, *dpool;                   // [N][C]
  const float* bnsum;                       // [2][C]: sum du, sum du*xhat
  float inv_count;
};

// true when the TMA ring path covers the shape (else the caller uses the generic kernels)
bool dw_ring_ok(const DwShape& g, int esz);
// number of spatial CTA tiles of each mode: partial buffers are [tiles][3][C] (stats) / [tiles][ks*ks][C] (dw)
size_t dw_stat_tiles(const DwShape& g, int esz);
size_t dw_dzw_tiles(const DwShape& g, int esz);

// z = conv(x, w) + per-tile BN partial (n, mean, M2) sets -> merged into stats_out [3][C]
int dw_conv_stats(int dtype, const DwShape& g, const void* x, const float* w, void* z, float* part,
                  float* stats_out, cudaStream_t st);
// dz (stored, dtype) and dw (f32, fixed-order reduced into dw_out [ks*ks][C]) from
// (x window, dy, z): dw uses the unrounded f32 dz
int dw_dz_dw(int dtype, const DwShape& g, const void* x, const void* dy, const void* z, const DzConsts& k,
             void* dz, float* part, float* dw_out, cudaStream_t st);
// dx = transposed conv of dz (the VJP of the forward loop nest, lowering.py:930-1004)
int dw_dx(int dtype, const DwShape& g, const void* dz, const float* w, void* dx, cudaStream_t st);

}  // namespace dfx
