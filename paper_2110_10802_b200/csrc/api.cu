// api.cu — library-level entry points of the dfx C ABI: error reporting,
// device check, launch accounting and the contraction dispatcher.
#include <atomic>
#include <string>

#include "common.cuh"
#include "gemm.h"

namespace dfx {

static thread_local std::string g_last_error;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
void count_launch(int n) { g_launches += n; }

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

static int check_gemm_args(const dfx_gemm_args& p) {
  DFX_REQUIRE(p.m >= 0 && p.n >= 0 && p.k >= 0, DFX_ERR_SHAPE, "dfx_gemm: negative extent");
  DFX_REQUIRE(p.batch1 >= 1 && p.batch2 >= 1, DFX_ERR_SHAPE, "dfx_gemm: batch counts must be >= 1");
  DFX_REQUIRE(p.a && p.b && p.d, DFX_ERR_SHAPE, "dfx_gemm: null operand");
  DFX_REQUIRE(p.in_dtype == DFX_F32 || p.in_dtype == DFX_BF16, DFX_ERR_DTYPE,
              "dfx_gemm: in_dtype must be f32 or bf16");
  DFX_REQUIRE(p.out_dtype == DFX_F32 || p.out_dtype == DFX_BF16, DFX_ERR_DTYPE,
              "dfx_gemm: out_dtype must be f32 or bf16");
  switch (p.epilogue) {
    case DFX_EPI_NONE: break;
    case DFX_EPI_BIAS: DFX_REQUIRE(p.bias, DFX_ERR_SHAPE, "dfx_gemm: BIAS epilogue needs bias"); break;
    case DFX_EPI_BIAS_GELU: break;
    case DFX_EPI_GELU_BWD:
    case DFX_EPI_ADD: DFX_REQUIRE(p.aux, DFX_ERR_SHAPE, "dfx_gemm: epilogue needs aux"); break;
    default: return fail(DFX_ERR_UNSUPPORTED, "dfx_gemm: unknown epilogue");
  }
  return DFX_OK;
}

}  // namespace dfx

using namespace dfx;

extern "C" {

const char* dfx_last_error(void) { return g_last_error.c_str(); }
int dfx_version(void) { return 1; }
int64_t dfx_launch_count(void) { return g_launches; }
void dfx_reset_launch_count(void) { g_launches = 0; }

int dfx_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(DFX_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(DFX_ERR_UNSUPPORTED, "dfx: built for sm_100a (B200); device is sm_" +
                                         std::to_string(major) + std::to_string(minor));
  return DFX_OK;
}

int dfx_gemm_uses_tensor_cores(const dfx_gemm_args* args) {
  return args && gemm_tc_supported(*args) ? 1 : 0;
}

/* debug: per-CTA timeline of the tensor-core GEMM (32 u64 per CTA; NULL = off). */
__attribute__((visibility("default"))) void dfx_debug_gemm_trace(void* buf) { gemm_tc_set_trace(buf); }

size_t dfx_gemm_workspace(const dfx_gemm_args* args) {
  if (!args) return 0;
  return gemm_tc_supported(*args) ? gemm_tc_workspace(*args) : gemm_simt_workspace(*args);
}

int dfx_gemm_excite(int64_t m, int64_t k, int64_t n, const void* z, int64_t hw, const float* mean,
                    const float* rstd, const float* gamma, const float* beta, const float* gate, const void* w,
                    void* d, void* y_out, void* stream) {
  return gemm_excite(m, k, n, z, hw, mean, rstd, gamma, beta, gate, w, d, y_out, as_stream(stream));
}

int dfx_gemm(const dfx_gemm_args* args, void* stream) {
  DFX_REQUIRE(args, DFX_ERR_SHAPE, "dfx_gemm: null args");
  if (int rc = check_gemm_args(*args)) return rc;
  if (args->m == 0 || args->n == 0) return DFX_OK;
  if (gemm_tc_supported(*args)) return gemm_tc(*args, as_stream(stream));
  return gemm_simt(*args, as_stream(stream));
}

}  // extern "C"
