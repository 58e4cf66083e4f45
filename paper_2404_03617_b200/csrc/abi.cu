// abi.cu — the C ABI of libwlfuse.so (include/wlfuse.h): descriptor checks,
// launch planning, weight packing from the reference's float32 tensors,
// tensor-map encoding and kernel launches.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/wlfuse.h"
#include "launch.h"
#include "gemm.h"

namespace wl {

static thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return WL_OK;
  return set_error(WL_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ------------------------------------------------------------ driver entry
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled_t g_encode = nullptr;
static std::once_flag g_encode_once;

int encode_tmap(CUtensorMap* tm, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                const uint32_t* box, bool swizzle128) {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_encodeTiled_t>(fn);
  });
  if (!g_encode) return set_error(WL_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) s[i] = strides_bytes[i];
  }
  CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rank, const_cast<void*>(base), d, s, b, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(WL_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return WL_OK;
}

// --------------------------------------------------------------- helpers
static inline uint16_t f2h(float v) {
  __half h = __float2half_rn(v);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
static inline uint16_t f2bf(float v) {
  __nv_bfloat16 h = __float2bfloat16_rn(v);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
void put_h(uint8_t* base, size_t off, float v) {
  uint16_t u = f2h(v);
  memcpy(base + off, &u, 2);
}
void put_v(uint8_t* base, size_t off, float v, int dtype) {
  uint16_t u = dtype == WL_DTYPE_BF16 ? f2bf(v) : f2h(v);
  memcpy(base + off, &u, 2);
}

}  // namespace wl

using namespace wl;

// =================================================================== ABI
extern "C" {

int wl_version(void) { return WL_ABI_VERSION; }

void wl_debug_set_trace(void* dev_ptr) {
  wl::mb_set_trace(dev_ptr);
  wl::cf2_set_trace(dev_ptr);
  wl::cf_set_trace(dev_ptr);
  wl::ffn_set_trace(dev_ptr);
}

const char* wl_last_error(void) { return g_last_error.c_str(); }

int wl_init(int device) {
  if (check_cuda(cudaSetDevice(device), "cudaSetDevice")) return WL_ECUDA;
  cudaDeviceProp prop;
  if (check_cuda(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties")) return WL_ECUDA;
  if (prop.major != 10) return set_error(WL_EUNSUPPORTED, "libwlfuse targets sm_100a; device is sm_%d%d", prop.major, prop.minor);
  return init_kernels();
}

int wl_validate(const wl_block_desc* d) {
  if (!d) return set_error(WL_EINVAL, "null descriptor");
  return validate_desc(*d);
}

int wl_weight_count(const wl_block_desc* d) {
  if (int e = wl_validate(d)) return e;
  return weight_count(*d);
}

int64_t wl_weight_numel(const wl_block_desc* d, int i) {
  if (int e = wl_validate(d)) return e;
  return weight_numel(*d, i);
}

int64_t wl_packed_bytes(const wl_block_desc* d) {
  if (int e = wl_validate(d)) return e;
  return packed_bytes(*d);
}

int wl_pack_weights(const wl_block_desc* d, const float* const* w, int count, void* packed_host) {
  if (int e = wl_validate(d)) return e;
  if (count != weight_count(*d))
    return set_error(WL_EINVAL, "expected %d weight tensors, got %d", weight_count(*d), count);
  for (int i = 0; i < count; ++i)
    if (!w[i]) return set_error(WL_EINVAL, "weight tensor %d is null", i);
  return pack_weights(*d, w, reinterpret_cast<uint8_t*>(packed_host));
}

int64_t wl_workspace_bytes(const wl_block_desc* d) {
  if (int e = wl_validate(d)) return e;
  return workspace_bytes(*d);
}

int wl_kernel_launches(const wl_block_desc* d) {
  if (int e = wl_validate(d)) return e;
  return kernel_launches(*d);
}

int wl_output_dims(const wl_block_desc* d, int32_t* n, int32_t* h, int32_t* w, int32_t* c) {
  if (int e = wl_validate(d)) return e;
  output_dims(*d, n, h, w, c);
  return WL_OK;
}

int wl_block_forward(const wl_block_desc* d, const void* x, const void* packed, void* z, void* ws, void* stream) {
  if (int e = wl_validate(d)) return e;
  if (!x || !packed || !z) return set_error(WL_EINVAL, "null tensor pointer");
  if (workspace_bytes(*d) > 0 && !ws) return set_error(WL_EINVAL, "workspace required");
  return forward(*d, x, packed, z, ws, reinterpret_cast<cudaStream_t>(stream));
}

static int fwd_kind(int kind, const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  if (!d) return set_error(WL_EINVAL, "null descriptor");
  if (d->kind != kind) return set_error(WL_EINVAL, "descriptor kind %d does not match entry point (%d)", d->kind, kind);
  return wl_block_forward(d, x, p, z, ws, s);
}
int wl_convfirst_fwd(const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  return fwd_kind(WL_KIND_CONVFIRST, d, x, p, z, ws, s);
}
int wl_mbconv_fwd(const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  return fwd_kind(WL_KIND_MBCONV, d, x, p, z, ws, s);
}
int wl_stem_fwd(const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  return fwd_kind(WL_KIND_STEM, d, x, p, z, ws, s);
}
int wl_head_fwd(const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  return fwd_kind(WL_KIND_HEAD, d, x, p, z, ws, s);
}

int wl_ffn_fwd(const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  return fwd_kind(WL_KIND_FFN, d, x, p, z, ws, s);
}
int wl_patch_stem_fwd(const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  return fwd_kind(WL_KIND_PATCH_STEM, d, x, p, z, ws, s);
}
int wl_downsample_fwd(const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  return fwd_kind(WL_KIND_DOWNSAMPLE, d, x, p, z, ws, s);
}
int wl_ln_head_fwd(const wl_block_desc* d, const void* x, const void* p, void* z, void* ws, void* s) {
  return fwd_kind(WL_KIND_LN_HEAD, d, x, p, z, ws, s);
}

int wl_stage_forward(const wl_block_desc* d, int nblocks, const void* x, const void* const* packed, void* z, void* ws,
                     void* stream) {
  if (int e = wl_validate(d)) return e;
  if (!x || !packed || !z || !ws) return set_error(WL_EINVAL, "null tensor pointer");
  if (d->kind != WL_KIND_MBCONV) return set_error(WL_EUNSUPPORTED, "stage launches cover MBConv blocks");
  return mb1_stage_forward(*d, nblocks, x, packed, z, ws, reinterpret_cast<cudaStream_t>(stream));
}

int wl_pair_supported(const wl_block_desc* d0, const wl_block_desc* d1) {
  if (!d0 || !d1 || validate_desc(*d0) != WL_OK || validate_desc(*d1) != WL_OK) return 0;
  return stem_cf_supported(*d0, *d1) ? 1 : 0;
}
int64_t wl_pair_packed_bytes(const wl_block_desc* d0, const wl_block_desc* d1) {
  if (!wl_pair_supported(d0, d1)) return set_error(WL_EUNSUPPORTED, "no fused kernel for this unit pair");
  return stem_cf_packed_bytes();
}
int wl_pair_pack(const wl_block_desc* d0, const wl_block_desc* d1, const float* const* w0, int n0,
                 const float* const* w1, int n1, void* packed_host) {
  if (!wl_pair_supported(d0, d1)) return set_error(WL_EUNSUPPORTED, "no fused kernel for this unit pair");
  if (n0 != weight_count(*d0) || n1 != weight_count(*d1))
    return set_error(WL_EINVAL, "expected %d + %d weight tensors", weight_count(*d0), weight_count(*d1));
  return stem_cf_pack(w0, w1, reinterpret_cast<uint8_t*>(packed_host));
}
int wl_pair_forward(const wl_block_desc* d0, const wl_block_desc* d1, const void* x, const void* packed, void* z,
                    void* stream) {
  if (!x || !packed || !z) return set_error(WL_EINVAL, "null tensor pointer");
  if (!wl_pair_supported(d0, d1)) return set_error(WL_EUNSUPPORTED, "no fused kernel for this unit pair");
  return stem_cf_forward(*d0, *d1, x, packed, z, reinterpret_cast<cudaStream_t>(stream));
}

int wl_stage_max_blocks(const wl_block_desc* d) {
  if (!d || validate_desc(*d) != WL_OK || d->kind != WL_KIND_MBCONV) return 0;
  return mb1_stage_max(*d);
}

int wl_gemm(const void* a, int m, int k, int lda, const void* b, int n, int ldb, void* d, int ldd, const float* bias,
            int act, const void* res, int ldr, int dtype, void* stream) {
  if (dtype != WL_DTYPE_F16 && dtype != WL_DTYPE_BF16) return set_error(WL_EINVAL, "unknown dtype %d", dtype);
  if (!a || !b || !d) return set_error(WL_EINVAL, "null tensor pointer");
  if (act < 0 || act > 4) return set_error(WL_EINVAL, "unknown activation %d", act);
  int dev = 0;
  cudaGetDevice(&dev);
  if (int e = init_kernels()) return e;
  GemmEpi e;
  e.bias = bias;
  e.act = act;
  e.res = reinterpret_cast<const __half*>(res);
  e.ldr = ldr;
  return gemm_run(a, m, k, lda, b, n, ldb, d, ldd, e, reinterpret_cast<cudaStream_t>(stream), dtype);
}

int wl_execute_numeric(const wl_block_desc* d, const float* x_host, const float* const* weights, int count,
                       float* z_host) {
  if (int e = wl_validate(d)) return e;
  if (!x_host || !z_host) return set_error(WL_EINVAL, "null host buffer");
  int dev = 0;
  cudaGetDevice(&dev);
  if (int e = wl_init(dev)) return e;
  const int64_t pbytes = packed_bytes(*d);
  std::vector<uint8_t> packed((size_t)pbytes);
  if (int e = wl_pack_weights(d, weights, count, packed.data())) return e;
  int32_t on, oh, ow, oc;
  output_dims(*d, &on, &oh, &ow, &oc);
  const size_t nx = (size_t)d->n * d->h * d->w * d->c, nz = (size_t)on * oh * ow * oc;
  std::vector<uint16_t> xh(nx), zh(nz);
  const bool bf = d->dtype == WL_DTYPE_BF16;
  for (size_t i = 0; i < nx; ++i) xh[i] = bf ? f2bf(x_host[i]) : f2h(x_host[i]);
  void *dx = nullptr, *dz = nullptr, *dp = nullptr, *dws = nullptr;
  const int64_t wsb = workspace_bytes(*d);
  int rc = WL_OK;
  cudaStream_t st = nullptr;
  do {
    if ((rc = check_cuda(cudaMalloc(&dx, nx * 2), "cudaMalloc"))) break;
    if ((rc = check_cuda(cudaMalloc(&dz, nz * 2), "cudaMalloc"))) break;
    if ((rc = check_cuda(cudaMalloc(&dp, pbytes), "cudaMalloc"))) break;
    if (wsb > 0 && (rc = check_cuda(cudaMalloc(&dws, wsb), "cudaMalloc"))) break;
    if (wsb > 0 && (rc = check_cuda(cudaMemset(dws, 0, wsb), "cudaMemset"))) break;
    if ((rc = check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate"))) break;
    if ((rc = check_cuda(cudaMemcpyAsync(dx, xh.data(), nx * 2, cudaMemcpyHostToDevice, st), "H2D"))) break;
    if ((rc = check_cuda(cudaMemcpyAsync(dp, packed.data(), pbytes, cudaMemcpyHostToDevice, st), "H2D"))) break;
    if ((rc = forward(*d, dx, dp, dz, dws, st))) break;
    if ((rc = check_cuda(cudaMemcpyAsync(zh.data(), dz, nz * 2, cudaMemcpyDeviceToHost, st), "D2H"))) break;
    if ((rc = check_cuda(cudaStreamSynchronize(st), "sync"))) break;
  } while (0);
  if (st) cudaStreamDestroy(st);
  cudaFree(dx);
  cudaFree(dz);
  cudaFree(dp);
  cudaFree(dws);
  if (rc) return rc;
  for (size_t i = 0; i < nz; ++i) {
    if (bf) {
      __nv_bfloat16 h;
      memcpy(&h, &zh[i], 2);
      z_host[i] = __bfloat162float(h);
    } else {
      __half h;
      memcpy(&h, &zh[i], 2);
      z_host[i] = __half2float(h);
    }
  }
  return WL_OK;
}

}  // extern "C"
