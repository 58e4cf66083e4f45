// blocks.cu — dispatch of the C ABI over block families.
#include <mutex>
#include "launch.h"

namespace wl {

static const Family* family_of(const wl_block_desc& d) {
  if (d.scheme == WL_SCHEME_LAYER_WISE) return &kLayerwiseFamily;
  switch (d.kind) {
    case WL_KIND_CONVFIRST: return &kCfFamily;
    case WL_KIND_MBCONV: return &kMbFamily;
    case WL_KIND_STEM: return &kStemFamily;
    case WL_KIND_HEAD: return &kHeadFamily;
    case WL_KIND_FFN: return &kFfnFamily;
    case WL_KIND_PATCH_STEM: return &kPatchStemFamily;
    case WL_KIND_DOWNSAMPLE: return &kDownsampleFamily;
    case WL_KIND_LN_HEAD: return &kLnHeadFamily;
  }
  return nullptr;
}

// kernel attributes (max dynamic shared memory) are per device context: run
// the family init once per device ordinal, thread-safely
int init_kernels() {
  constexpr int kMaxDevices = 64;
  static std::once_flag once[kMaxDevices];
  static int status[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return set_error(WL_ECUDA, "no current CUDA device");
  std::call_once(once[dev], [dev] {
    status[dev] = WL_OK;
    for (const Family* f :
         {&kCfFamily, &kCf2Family, &kMbFamily, &kStemFamily, &kHeadFamily, &kFfnFamily, &kLayerwiseFamily})
      if (f->init && (status[dev] = f->init()) != WL_OK) break;
  });
  return status[dev];
}

int validate_desc(const wl_block_desc& d) {
  const Family* f = family_of(d);
  if (!f) return set_error(WL_EINVAL, "unknown block kind %d", d.kind);
  if (d.dtype != WL_DTYPE_F16 && d.dtype != WL_DTYPE_BF16) return set_error(WL_EINVAL, "unknown dtype %d", d.dtype);
  if (d.scheme != WL_SCHEME_FUSED && d.scheme != WL_SCHEME_LAYER_WISE)
    return set_error(WL_EINVAL, "unknown scheme %d", d.scheme);
  if (d.scheme == WL_SCHEME_LAYER_WISE) return f->validate(d);
  if (d.dtype == WL_DTYPE_BF16) {
    const bool ok = d.kind == WL_KIND_FFN || d.kind == WL_KIND_PATCH_STEM || d.kind == WL_KIND_DOWNSAMPLE ||
                    d.kind == WL_KIND_LN_HEAD || cnx_wide(d);
    if (!ok) return set_error(WL_EUNSUPPORTED, "bf16 storage is built for the FFN and ConvNeXt-T units only");
  }
  return f->validate(d);
}
int weight_count(const wl_block_desc& d) { return family_of(d)->weight_count(d); }
int64_t weight_numel(const wl_block_desc& d, int i) { return family_of(d)->weight_numel(d, i); }
int64_t packed_bytes(const wl_block_desc& d) { return family_of(d)->packed_bytes(d); }
int pack_weights(const wl_block_desc& d, const float* const* w, uint8_t* out) { return family_of(d)->pack(d, w, out); }
int64_t workspace_bytes(const wl_block_desc& d) { return family_of(d)->workspace_bytes(d); }
int kernel_launches(const wl_block_desc& d) {
  if (d.scheme == WL_SCHEME_LAYER_WISE) return lw_launches(d);
  if (d.kind == WL_KIND_HEAD || d.kind == WL_KIND_PATCH_STEM || d.kind == WL_KIND_DOWNSAMPLE ||
      d.kind == WL_KIND_LN_HEAD)
    return 2;
  if (d.kind == WL_KIND_FFN) return ffn_launches(d, true);
  if (cnx_wide(d)) return 1 + ffn_launches(d, true);  // packed blob carries the fused kernel's weight images
  if (cf_wide(d)) return 1 + ffn_launches(d, false);
  if (d.kind == WL_KIND_MBCONV) return mb_kernel_launches(d);
  return 1;
}
int forward(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  return family_of(d)->forward(d, x, p, z, ws, st);
}

void output_dims(const wl_block_desc& d, int32_t* n, int32_t* h, int32_t* w, int32_t* c) {
  *n = d.n;
  if (d.kind == WL_KIND_HEAD || d.kind == WL_KIND_LN_HEAD) {
    *h = 1;
    *w = 1;
    *c = d.classes;
    return;
  }
  int s = d.kind == WL_KIND_STEM ? 2 : d.kind == WL_KIND_PATCH_STEM ? d.ksize : d.kind == WL_KIND_DOWNSAMPLE ? 2 : d.stride;
  if (d.kind == WL_KIND_FFN || s < 1) s = 1;  // FFN rows keep their geometry
  *h = d.h / s;
  *w = d.w / s;
  *c = d.k;
}

}  // namespace wl
