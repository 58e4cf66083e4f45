// launch.h — host-side interface between the C ABI and the block families.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <utility>
#include "../../include/wlfuse.h"

namespace wl {

int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
int encode_tmap(CUtensorMap* tm, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                const uint32_t* box, bool swizzle128 = false);
void put_h(uint8_t* base, size_t off, float v);
void put_v(uint8_t* base, size_t off, float v, int dtype);  // fp16 or bf16 by WL_DTYPE_*
static inline size_t core_off_h(int row, int k, int lbo) {
  return (size_t)(k / 8) * lbo + (size_t)(row / 8) * 128 + (size_t)(row % 8) * 16 + (size_t)(k % 8) * 2;
}

// launch with programmatic stream serialization (PDL): the kernel's prologue
// may overlap the previous kernel on the stream; kernels call pdl_wait()
// before reading what that kernel produced (sm100.cuh)
template <typename... KArgs, typename... Args>
int launch_pdl_cluster(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, const char* what,
                       int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cluster;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = cluster > 1 ? 2 : 1;
  return check_cuda(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), what);
}
template <typename... KArgs, typename... Args>
int launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, const char* what,
               Args&&... args) {
  return launch_pdl_cluster(kernel, grid, block, smem, st, what, 1, std::forward<Args>(args)...);
}

// dispatch over block kinds (blocks.cu)
int init_kernels();
int validate_desc(const wl_block_desc& d);
int weight_count(const wl_block_desc& d);
int64_t weight_numel(const wl_block_desc& d, int i);
int64_t packed_bytes(const wl_block_desc& d);
int pack_weights(const wl_block_desc& d, const float* const* w, uint8_t* out);
int64_t workspace_bytes(const wl_block_desc& d);
int kernel_launches(const wl_block_desc& d);
int mb_kernel_launches(const wl_block_desc& d);
void output_dims(const wl_block_desc& d, int32_t* n, int32_t* h, int32_t* w, int32_t* c);
int forward(const wl_block_desc& d, const void* x, const void* packed, void* z, void* ws, cudaStream_t st);

// one family = one set of these (cf_fused.cu, cf_s2.cu, mbconv.cu, stem_head.cu)
struct Family {
  int (*validate)(const wl_block_desc&);
  int (*weight_count)(const wl_block_desc&);
  int64_t (*weight_numel)(const wl_block_desc&, int);
  int64_t (*packed_bytes)(const wl_block_desc&);
  int (*pack)(const wl_block_desc&, const float* const*, uint8_t*);
  int64_t (*workspace_bytes)(const wl_block_desc&);
  int (*forward)(const wl_block_desc&, const void*, const void*, void*, void*, cudaStream_t);
  int (*init)();
};
extern const Family kCfFamily;
extern const Family kCf2Family;
extern const Family kMbFamily;
extern const Family kStemFamily;
extern const Family kHeadFamily;
extern const Family kFfnFamily;
extern const Family kPatchStemFamily;
extern const Family kDownsampleFamily;
extern const Family kLnHeadFamily;
extern const Family kLayerwiseFamily;  // the reference's LAYER_WISE schedules (layerwise.cu)
int lw_launches(const wl_block_desc& d);
// wide ConvNeXt block (C > 128): dwln + two GEMMs (cnx.cu), reached through the conv-first family
bool cnx_wide(const wl_block_desc& d);
int cnx_wide_validate(const wl_block_desc& d);
int64_t cnx_wide_pb(const wl_block_desc& d);
int cnx_wide_pack(const wl_block_desc& d, const float* const* w, uint8_t* out);
int64_t cnx_wide_ws(const wl_block_desc& d);
int cnx_wide_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st);
// wide conv-first blocks without LayerNorm (C > 128, beyond the fused kernel's TMEM
// plan): grouped conv kernel -> xc in the workspace, then the FFN rows (cnx.cu)
bool cf_wide(const wl_block_desc& d);
int cf_wide_validate(const wl_block_desc& d);
int64_t cf_wide_pb(const wl_block_desc& d);
int cf_wide_pack(const wl_block_desc& d, const float* const* w, uint8_t* out);
int64_t cf_wide_ws(const wl_block_desc& d);
int cf_wide_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st);
int lw_gconv(const wl_block_desc& d, int C, const void* x, const float* w, const float* b, void* y, int act,
             cudaStream_t st);  // fp16 x / y
int ffn_row_batches(const wl_block_desc& d);
int ffn_launches(const wl_block_desc& d, bool images);
// fused FFN (ffn.cu): hidden kept on chip
bool ffn_fused_ok(int64_t M, int C, int hid);
int ffn_fused_run(const void* x, int64_t M, int C, int hid, const void* wimg, const float* abias, const float* bbias,
                  int act, const void* res, void* z, cudaStream_t st, int dtype);
int64_t ffn_images_bytes(int C, int hid);
void ffn_pack_images(int C, int hid, const float* u, const float* v, uint8_t* out, int dtype);
int ffn_fused_init();
// stride-1 MBConv stage launch (mb_s1.cu)
int mb1_stage_max(const wl_block_desc& d);
// stem + first ConvFirst block (stem_cf.cu)
bool stem_cf_supported(const wl_block_desc& d0, const wl_block_desc& d1);
int64_t stem_cf_packed_bytes();
int stem_cf_pack(const float* const* w0, const float* const* w1, uint8_t* out);
int stem_cf_forward(const wl_block_desc& d0, const wl_block_desc& d1, const void* x, const void* packed, void* z,
                    cudaStream_t st);
int mb1_stage_forward(const wl_block_desc& d, int nblk, const void* x, const void* const* packed, void* z, void* ws,
                      cudaStream_t st);
void mb_set_trace(void* p);
void cf2_set_trace(void* p);
void cf_set_trace(void* p);
void ffn_set_trace(void* p);

}  // namespace wl
