/* wlfuse.h — C ABI of the B200 (sm_100a) block-fusion library libwlfuse.so.
 *
 * The reference (`waterline`, /root/reference/pkg/src/waterline) is pure
 * Python with no FFI; its hot-path interface is
 *     machine.execute_numeric(schedule, inputs: dict[str, ndarray]) -> ndarray
 *       (machine.py:1053-1061; schedules from build_schedule, machine.py:736)
 * driven per block by core.plan_blocks (core.py:362-398). Every entry point
 * below names the reference interface it replaces. All pointers are plain
 * device (or, where stated, host) pointers; no torch types cross the ABI.
 *
 * Tensors: activations are NHWC fp16, contiguous. Weights are packed once
 * (wl_pack_weights) from the reference's float32 tensors, in the reference
 * tensor-table order and layouts (machine.py:402-415, 572-590).
 *
 * Errors: every int-returning function returns WL_OK (0) or a negative
 * status; wl_last_error() (thread-local) describes the last failure.
 * Launches are stream-ordered, never synchronise, never allocate, and are
 * CUDA-graph capturable once wl_init() has run.
 */
#ifndef WLFUSE_H
#define WLFUSE_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define WL_API __attribute__((visibility("default")))
#else
#define WL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define WL_ABI_VERSION 1

/* status codes; the Python wrapper maps them to the reference exceptions */
#define WL_OK 0
#define WL_EINVAL (-1)       /* invalid descriptor        -> ValueError     */
#define WL_EUNSUPPORTED (-2) /* valid but not executable  -> ScheduleError  */
#define WL_ECUDA (-3)        /* CUDA launch/runtime error -> RuntimeError   */

/* block kinds (core.py:92-155) */
#define WL_KIND_CONVFIRST 1 /* ConvFirst / ConvNeXt-style conv-first block */
#define WL_KIND_MBCONV 2    /* MBConv + squeeze-excite                      */
#define WL_KIND_FFN 3       /* FFN z = phi(xU + a)V + b over pixels (core.py:125-132) */
#define WL_KIND_STEM 4      /* dense 3x3 stride-2 stem                      */
#define WL_KIND_HEAD 5      /* 1x1 conv + pool + linear classifier          */
/* ConvNeXt-T units (BASELINE config 4; no reference constructor) */
#define WL_KIND_PATCH_STEM 6 /* p x p stride-p conv (ksize = p) + LayerNorm   */
#define WL_KIND_DOWNSAMPLE 7 /* LayerNorm + 2x2 stride-2 conv c -> k          */
#define WL_KIND_LN_HEAD 8    /* global average pool + LayerNorm + linear      */

/* activations (machine.py:178-188, plus GELU) */
#define WL_ACT_IDENTITY 0
#define WL_ACT_RELU 1
#define WL_ACT_SILU 2
#define WL_ACT_SIGMOID 3
#define WL_ACT_GELU 4

/* storage types (fp32 accumulation either way). bf16 covers the FFN block,
 * the ConvNeXt-T units (patchify stem, ConvNeXt blocks with C >= 96,
 * downsample, LN head) and wl_gemm; the other families are fp16 only. */
#define WL_DTYPE_F16 0
#define WL_DTYPE_BF16 1

/* execution scheme (core.py:15-17 ExecutionScheme): the fused block kernels,
 * or the reference's LAYER_WISE schedule — one launch per layer, every
 * intermediate through HBM (ConvFirst / MBConv stride 1, FFN; fp16) — the
 * baseline block fusion is measured against */
#define WL_SCHEME_FUSED 0
#define WL_SCHEME_LAYER_WISE 1

/* normalisation after the conv of a conv-first block */
#define WL_NORM_NONE 0
#define WL_NORM_LAYERNORM 1

typedef struct wl_block_desc {
  int32_t kind;
  int32_t n, h, w, c;    /* block input, NHWC                             */
  int32_t k;             /* output channels (== c for stride 1)           */
  int32_t expansion;     /* hidden = expansion * c                        */
  int32_t group_width;   /* T of the grouped conv (1 = depthwise)         */
  int32_t ksize;         /* conv kernel size (3 or 7)                     */
  int32_t stride;        /* 1 or 2                                        */
  int32_t se_sq;         /* MBConv squeeze width int(se_ratio * c)        */
  int32_t norm;          /* WL_NORM_*                                     */
  int32_t act;           /* WL_ACT_*                                      */
  float ln_eps;          /* LayerNorm epsilon                             */
  int32_t embed;         /* head: embedding width                         */
  int32_t classes;       /* head: classifier width                        */
  int32_t dtype;         /* WL_DTYPE_*: activation / weight storage type  */
  int32_t scheme;        /* WL_SCHEME_*: fused block or the layer-wise baseline */
  int32_t reserved[2];
} wl_block_desc;

/* library / device ------------------------------------------------------ */
WL_API int wl_version(void);
WL_API const char* wl_last_error(void);
/* one-time per-device setup (kernel attributes, driver entry points); call
 * outside stream capture. Idempotent. */
WL_API int wl_init(int device);

/* descriptor checks mirroring core.validate_network (core.py:300-347) and
 * build_schedule's executability rules (machine.py:753-758, 1055-1059) */
WL_API int wl_validate(const wl_block_desc* d);

/* number of reference weight tensors consumed by wl_pack_weights, and the
 * expected element count of tensor i (reference layouts) */
WL_API int wl_weight_count(const wl_block_desc* d);
WL_API int64_t wl_weight_numel(const wl_block_desc* d, int i);
/* packed (device-format) weight blob size in bytes */
WL_API int64_t wl_packed_bytes(const wl_block_desc* d);
/* pack reference float32 HOST tensors into the device format (HOST output;
 * copy it to the device once). Replaces the per-call weight handling of
 * machine._Executor.__init__ (machine.py:915-929). */
WL_API int wl_pack_weights(const wl_block_desc* d, const float* const* weights, int count, void* packed_host);
/* device workspace the forward needs (0 for fully fused blocks). The caller
 * zeroes it once before the first forward; the library keeps its arrival-
 * counter header zeroed across calls, so one workspace can serve many blocks
 * launched in stream order. */
WL_API int64_t wl_workspace_bytes(const wl_block_desc* d);

/* number of kernels one wl_block_forward launches for this descriptor (1 for
 * every fused block; 2 for the head, and for MBConv when it falls back to its
 * two-launch form); negative status on an invalid descriptor. */
WL_API int wl_kernel_launches(const wl_block_desc* d);

/* forward: z = block(x). x, packed, z, workspace are DEVICE pointers.
 * Replaces execute_numeric(build_schedule(block, dims, BLOCK_FUSION), ...)
 * (machine.py:1053) for one block. */
WL_API int wl_block_forward(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
                     void* stream);
/* per-family aliases (same contract, kind checked) */
WL_API int wl_convfirst_fwd(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
                     void* stream);
WL_API int wl_mbconv_fwd(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
                  void* stream);
WL_API int wl_stem_fwd(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
                void* stream);
WL_API int wl_head_fwd(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
                void* stream);
/* FFN block: replaces execute_numeric on an FFN schedule (machine.py:339-365) */
WL_API int wl_ffn_fwd(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
               void* stream);
WL_API int wl_patch_stem_fwd(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
                      void* stream);
WL_API int wl_downsample_fwd(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
                      void* stream);
WL_API int wl_ln_head_fwd(const wl_block_desc* d, const void* x, const void* packed, void* z, void* workspace,
                   void* stream);

/* A stage: nblocks consecutive blocks with the SAME descriptor (stride 1,
 * channels kept) in one launch; block i+1 consumes block i's output without
 * it leaving the SM (the per-stage persistent kernel of machine.py:1091-1120,
 * PAPER.md:1328-1347). packed: HOST array of nblocks DEVICE pointers to each
 * block's packed weights; x / z: the stage's input / output; workspace as
 * for one block. Currently the stride-1 T=8 MBConv (W <= 14, <= 20 blocks);
 * WL_EUNSUPPORTED otherwise (launch the blocks one by one). */
WL_API int wl_stage_forward(const wl_block_desc* d, int nblocks, const void* x, const void* const* packed, void* z,
                            void* workspace, void* stream);
/* most blocks one wl_stage_forward may run for this descriptor (0: no stage
 * kernel for it) */
WL_API int wl_stage_max_blocks(const wl_block_desc* d);

/* Two consecutive units fused into one launch, the intermediate activation
 * kept on chip: currently the dense 3x3 stride-2 stem (3 -> 16, ReLU) with the
 * first stride-1 ConvFirst block (T = 8, C = 16, expansion 3) — ConvFirstNet-
 * Pico's stem + s1b0. d0 / d1 are the
 * two units' descriptors; weights in each unit's reference order; packed:
 * wl_pair_packed_bytes bytes. */
WL_API int wl_pair_supported(const wl_block_desc* d0, const wl_block_desc* d1);
WL_API int64_t wl_pair_packed_bytes(const wl_block_desc* d0, const wl_block_desc* d1);
WL_API int wl_pair_pack(const wl_block_desc* d0, const wl_block_desc* d1, const float* const* w0, int n0,
                        const float* const* w1, int n1, void* packed_host);
WL_API int wl_pair_forward(const wl_block_desc* d0, const wl_block_desc* d1, const void* x, const void* packed,
                           void* z, void* stream);

/* The pointwise contraction of the layer-wise units (1x1 conv / linear),
 * exposed for the layer-wise FFN schedule and for direct testing:
 * D[M][N] = act(A[M][K] . B[N][K]^T + bias[N]) (+ res[M][N]); fp16 storage,
 * fp32 accumulation in TMEM. A, B, D, res: DEVICE pointers with leading
 * dimensions lda/ldb/ldd/ldr (elements, multiples of 8); bias: DEVICE fp32
 * or null; res: null for none. Replaces the float64 `x @ w` of the
 * reference executor (machine.py:1017) on the device. */
WL_API int wl_gemm(const void* a, int m, int k, int lda, const void* b, int n, int ldb, void* d, int ldd,
                   const float* bias, int act, const void* res, int ldr, int dtype, void* stream);

/* Host-buffer convenience with execute_numeric's exact contract
 * (machine.py:1053): float32 HOST input x (NHWC) and float32 HOST weights in
 * reference order, float32 HOST output. Allocates, copies, runs, copies
 * back, frees; synchronous. Output extent: n * out_h * out_w * k (head:
 * n * classes). */
WL_API int wl_execute_numeric(const wl_block_desc* d, const float* x_host, const float* const* weights, int count,
                       float* z_host);

/* debug only: when dev_ptr (>= 512 bytes of device memory) is non-null,
 * CTA 0 of the MBConv front kernel records clock64() phase stamps there */
WL_API void wl_debug_set_trace(void* dev_ptr);

/* output geometry of a block */
WL_API int wl_output_dims(const wl_block_desc* d, int32_t* n, int32_t* h, int32_t* w, int32_t* c);

#ifdef __cplusplus
}
#endif
#endif /* WLFUSE_H */
