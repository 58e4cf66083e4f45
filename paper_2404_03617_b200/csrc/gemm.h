// gemm.h — the pointwise (1x1 conv / linear) contraction of the layer-wise
// units: D = epilogue(A . B^T), tcgen05 + TMA, used by the ConvNeXt-T units
// (patchify stem, LN + 2x2 downsample, the wide blocks' expand / project, the
// classifier) and by the layer-wise FFN schedule (machine.py:339-365).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/wlfuse.h"

namespace wl {

// epilogue, applied per output element in this order:
//   v = acc + bias[n];  v = act(v);  v = LayerNorm_row(v) (gamma, beta);  v += res[m][n]
struct GemmEpi {
  const float* bias = nullptr;   // [N] fp32 (device) or null
  int act = 0;                   // wl::Act
  const float* ln_g = nullptr;   // [N] fp32: LayerNorm over the whole output row (N <= 256)
  const float* ln_b = nullptr;
  float ln_eps = 1e-6f;
  const __half* res = nullptr;   // residual [M][ldr] fp16 or null
  int ldr = 0;
};

// A: [M][lda] fp16 (K contiguous), B: [N][ldb] fp16 (K contiguous, the
// weight stored output-major), D: [M][ldd] fp16. K, lda, ldb, ldd, ldr
// multiples of 8; M, N >= 1. Stream-ordered, graph-capturable.
int gemm_run(const void* A, int M, int K, int lda, const void* B, int N, int ldb, void* D, int ldd,
             const GemmEpi& e, cudaStream_t st, int dtype = 0);  // dtype: WL_DTYPE_*
int gemm_init();

}  // namespace wl
