// cnx.cu — the units that ConvNeXt-T (BASELINE config 4) needs beyond the
// fused conv-first kernel, and the FFN block of the reference
// (core.py:125-132; machine.py:228-252, 339-365):
//
//   WL_KIND_FFN         z = phi(x U + a) V + b over the rows of x
//   ConvNeXt block, C > 128 (WL_KIND_CONVFIRST, LayerNorm, depthwise k x k):
//                       x^ = LN(dwconv(x) + b_dw)        dwln_kernel (CUDA cores)
//                       z  = x + GELU(x^ U + a) V + b    two tcgen05 GEMMs, hidden
//                                                         in L2-sized row batches
//   WL_KIND_PATCH_STEM  z = LN(conv_pxp/stride p(x) + b) patchify + GEMM (LN epilogue)
//   WL_KIND_DOWNSAMPLE  z = conv_2x2/s2(LN(x)) + b      ln_s2d_kernel + GEMM
//   WL_KIND_LN_HEAD     z = LN(mean_hw(x)) W + b        pool_ln_kernel + GEMM
//
// The wide block is the reference's "scaling variant" problem
// (machine.py:528-569): at C = 384..768 one CTA can hold neither the whole
// hidden nor the whole output row (TMEM is 512 fp32 columns), so the hidden
// goes through the GLOBAL tier as the reference's partitioned schedule does,
// sized so that a row batch of it stays L2-resident (126 MB L2).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <algorithm>
#include <cstring>
#include "common.cuh"
#include "gemm.h"
#include "launch.h"
#include "plan.h"

namespace wl {

constexpr int kWsHdr = 4096;                     // the arrival-counter header every family leaves alone
constexpr int64_t kHiddenBatchBytes = 80 << 20;  // hidden row batch kept L2-resident (126 MB L2)

__device__ __forceinline__ void ld8f(const float* p, float* o) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}

// ================================================================= kernels
// patchify: x (n, H, W, cin) -> A (n * H/p * W/p, p * p * cin), column
// (dy * p + dx) * cin + ci (the weight layout (k, p, p, cin)). Generic path:
// one element per thread; p * cin % 4 == 0 (the 4x4 x 3 stem): thread per
// (patch, dy) moving p * cin halves as 8-byte words.
__global__ void patchify_kernel(const __half* __restrict__ x, __half* __restrict__ A, int n, int H, int W, int cin,
                                int p) {
  const int Ho = H / p, Wo = W / p, kk = p * p * cin, seg = p * cin;
  pdl_wait();
  if (seg % 4 == 0) {
    const int64_t total = (int64_t)n * Ho * Wo * p;
    const int words = seg / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int dy = (int)(i % p);
      const int64_t m = i / p;
      const int ox = (int)(m % Wo);
      const int64_t rest = m / Wo;
      const int oy = (int)(rest % Ho), img = (int)(rest / Ho);
      const uint2* src = reinterpret_cast<const uint2*>(x + (((int64_t)img * H + oy * p + dy) * W + ox * p) * cin);
      uint2* dst = reinterpret_cast<uint2*>(A + m * kk + dy * seg);
      for (int w = 0; w < words; ++w) dst[w] = __ldg(src + w);
    }
  } else {
    const int64_t total = (int64_t)n * Ho * Wo * kk;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int k = (int)(i % kk);
      const int64_t m = i / kk;
      const int ox = (int)(m % Wo), oy = (int)((m / Wo) % Ho), img = (int)(m / ((int64_t)Wo * Ho));
      const int ci = k % cin, dx = (k / cin) % p, dy = k / (cin * p);
      A[i] = x[(((int64_t)img * H + oy * p + dy) * W + ox * p + dx) * cin + ci];
    }
  }
  pdl_trigger();
}

// depthwise KS x KS conv + bias + channel LayerNorm. Persistent CTAs walk
// work items (image, vertical segment of SR rows) and slide a ring of padded
// input rows down the segment: each step computes RB output rows from the
// window [y0 - R, y0 + RB + R) while cp.async brings in the next RB rows, so
// every input row is read from L2/HBM about once and the loads overlap the
// stencil. Thread item = (output row, kDwPx pixels, 8 channels); the KS x KS
// taps accumulate in packed half (HFMA2) and are widened once; the pre-norm
// result is kept in shared memory (fp16) for the two-pass, fixed-order
// per-pixel LayerNorm statistics.
constexpr int kDwPx = 4;
constexpr int kDwThreads = 384;
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// CT: the channel count as a compile-time constant (0: runtime C) so every
// shared-memory and weight offset of the stencil folds into an immediate
template <int KS, typename T, int CT>
__global__ void __launch_bounds__(kDwThreads, 1)
    dwln_kernel(const T* __restrict__ x, const T* __restrict__ wdw, const float* __restrict__ bdw,
                const float* __restrict__ g, const float* __restrict__ be, T* __restrict__ y, int N, int H, int W,
                int C_rt, float eps, int RB, int nseg) {
  const int C = CT ? CT : C_rt;
  constexpr bool kF16 = Dt<T>::kIdescAB == 0;  // fp16: taps in packed half; bf16: fp32 FMAs
  constexpr int R = KS / 2, PX = kDwPx, NI = PX + 2 * R;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int C8 = C / 8, WG = (W + PX - 1) / PX, rowh = W * C;
  const int NR = 2 * RB + 2 * R;                 // ring rows
  const int WP = WG * PX + 2 * R;                // padded row width (zero columns both sides + tail)
  const int prowh = WP * C;                      // padded row (halves)
  T* s_in = reinterpret_cast<T*>(dsm);  // [NR][W + 2R][C]
  T* s_y = s_in + (size_t)NR * prowh;   // [RB][W][C] pre-norm
  float* s_sum = reinterpret_cast<float*>(s_y + (size_t)RB * rowh);  // [RB * W] mean
  float* s_sq = s_sum + RB * W;                                       // [RB * W] rstd
  float* s_part = s_sq + RB * W;                                      // [RB * W][C8]
  const int tid = threadIdx.x, nt = blockDim.x;
  const int SR = (H + nseg - 1) / nseg;
  // the pad columns of every ring row stay zero
  for (int i = tid; i < NR * WP * C8; i += nt) reinterpret_cast<uint4*>(s_in)[i] = make_uint4(0, 0, 0, 0);
  pdl_wait();
  __syncthreads();
  const int per_row = rowh / 8;
  for (int item = blockIdx.x; item < N * nseg; item += gridDim.x) {
    const int img = item / nseg, ys = (item % nseg) * SR, ye = min(H, ys + SR);
    if (ys >= ye) continue;
    const int base = ys - R;  // ring slot of input row iy: (iy - base) % NR
    auto load_rows = [&](int lo, int hi) {
      lo = max(lo, ys - R);
      hi = min(hi, ye + R);
      for (int i = tid; i < (hi - lo) * per_row; i += nt) {
        const int iy = lo + i / per_row, off = i % per_row;
        T* dst = s_in + (size_t)((iy - base) % NR) * prowh + R * C + off * 8;
        if (iy >= 0 && iy < H)
          cp_async16(dst, x + ((size_t)img * H + iy) * rowh + off * 8);
        else
          *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    load_rows(ys - R, ys + RB + R);  // the first window
    for (int y0 = ys; y0 < ye; y0 += RB) {
      load_rows(y0 + RB + R, y0 + 2 * RB + R);  // the next step's new rows (overlap this step)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncthreads();
      const int rows = min(RB, ye - y0);
      const int items = rows * WG * C8;
      for (int it = tid; it < items; it += nt) {
        const int c8 = it % C8, rest = it / C8, pg = rest % WG, ry = rest / WG;
        const int x0 = pg * PX;
        __half2 h[PX][4];
#pragma unroll
        for (int p = 0; p < PX; ++p)
#pragma unroll
          for (int i = 0; i < 4; ++i) h[p][i] = __float2half2_rn(0.f);
        float acc[PX][8];
#pragma unroll
        for (int p = 0; p < PX; ++p)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[p][i] = 0.f;
        int slot = (y0 + ry - R - base) % NR;  // ring slot of the window's first row
#pragma unroll
        for (int dy = 0; dy < KS; ++dy) {
          const T* row = s_in + (size_t)slot * prowh + (size_t)x0 * C + c8 * 8;
          slot = slot + 1 == NR ? 0 : slot + 1;
          uint4 in[NI];
#pragma unroll
          for (int j = 0; j < NI; ++j) in[j] = lds128(row + (size_t)j * C);
#pragma unroll
          for (int dx = 0; dx < KS; ++dx) {
            const uint4 wv = __ldg(reinterpret_cast<const uint4*>(wdw + (size_t)(dy * KS + dx) * C + c8 * 8));
            if constexpr (kF16) {
              const __half2* w2 = reinterpret_cast<const __half2*>(&wv);
#pragma unroll
              for (int p = 0; p < PX; ++p) {
                const __half2* i2 = reinterpret_cast<const __half2*>(&in[p + dx]);
#pragma unroll
                for (int i = 0; i < 4; ++i) h[p][i] = __hfma2(i2[i], w2[i], h[p][i]);
              }
            } else {
              float wf[8];
              unpack8t<T>(wv, wf);
#pragma unroll
              for (int p = 0; p < PX; ++p) {
                float xf[8];
                unpack8t<T>(in[p + dx], xf);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[p][i] = fmaf(xf[i], wf[i], acc[p][i]);
              }
            }
          }
          if (kF16 && (dy == R || dy == KS - 1)) {  // widen to fp32 twice per window (<= 4 rows of taps in half)
#pragma unroll
            for (int p = 0; p < PX; ++p)
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 f = __half22float2(h[p][i]);
                acc[p][2 * i] += f.x;
                acc[p][2 * i + 1] += f.y;
                h[p][i] = __float2half2_rn(0.f);
              }
          }
        }
        float b[8];
        ld8f(bdw + c8 * 8, b);
#pragma unroll
        for (int p = 0; p < PX; ++p) {
          if (x0 + p >= W) break;
          float s = 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            acc[p][i] += b[i];
            s += acc[p][i];
          }
          s_part[(ry * W + x0 + p) * C8 + c8] = s;
          *reinterpret_cast<uint4*>(s_y + ((size_t)ry * W + x0 + p) * C + c8 * 8) = pack8t<T>(acc[p]);
        }
      }
      __syncthreads();
      const int npix = rows * W, pitems = npix * C8;
      for (int pix = tid; pix < npix; pix += nt) {
        float t = 0.f;
        for (int j = 0; j < C8; ++j) t += s_part[pix * C8 + j];
        s_sum[pix] = t / (float)C;
      }
      __syncthreads();
      for (int it = tid; it < pitems; it += nt) {
        const int c8 = it % C8, pix = it / C8;
        const float mean = s_sum[pix];
        float v[8];
        unpack8t<T>(lds128(s_y + (size_t)pix * C + c8 * 8), v);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += (v[i] - mean) * (v[i] - mean);
        s_part[it] = s;
      }
      __syncthreads();
      for (int pix = tid; pix < npix; pix += nt) {
        float t = 0.f;
        for (int j = 0; j < C8; ++j) t += s_part[pix * C8 + j];
        s_sq[pix] = rsqrtf(t / (float)C + eps);
      }
      __syncthreads();
      for (int it = tid; it < pitems; it += nt) {
        const int c8 = it % C8, pix = it / C8;
        const float mean = s_sum[pix], rstd = s_sq[pix];
        float v[8], gg[8], bb[8];
        unpack8t<T>(lds128(s_y + (size_t)pix * C + c8 * 8), v);
        ld8f(g + c8 * 8, gg);
        ld8f(be + c8 * 8, bb);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (v[i] - mean) * rstd * gg[i] + bb[i];
        *reinterpret_cast<uint4*>(y + ((size_t)img * H + y0) * rowh + (size_t)pix * C + c8 * 8) = pack8t<T>(v);
      }
      __syncthreads();  // the ring rows of this window may be overwritten by the next prefetch
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  pdl_trigger();
}
int dwln_smem_rb(int KS, int W, int C, int RB) {
  const int WP = (W + kDwPx - 1) / kDwPx * kDwPx + KS - 1;
  return (2 * RB + KS - 1) * WP * C * 2 + RB * W * C * 2 + 2 * RB * W * 4 + RB * W * (C / 8) * 4;
}
int dwln_rows(int KS, int W, int C) {
  for (int rb : {4, 2, 1})
    if (dwln_smem_rb(KS, W, C, rb) <= 232448) return rb;
  return 0;
}
int dwln_smem(int KS, int W, int C) { return dwln_smem_rb(KS, W, C, dwln_rows(KS, W, C)); }
int dwln_segments(int N, int H, int RB) {
  int nseg = (3 * kNumSMs + N - 1) / N;
  const int cap = H / (2 * RB);
  if (nseg > cap) nseg = cap;
  return nseg < 1 ? 1 : nseg;
}

// 7x7 depthwise + LayerNorm for W % 7 == 0 (every ConvNeXt-T stage: 56, 28,
// 14, 7). Same ring of padded input rows as dwln_kernel, but the block has
// exactly one item per thread per band step — (output row, 7-pixel group,
// 8 channels) — so the 56 accumulators stay in registers through the norm:
//   pixel sums      -> segmented shuffle reduction over the lanes of a pixel
//                      group; each warp's segment head stores its partial in
//                      its own slot (no shared atomics: fp32 ones are CAS loops)
//   mean            -> sum of (v - mean)^2 from the fp32 registers (the
//                      reference's two-pass variance, no E[x^2] - mean^2)
//   normalise       -> straight from registers to the output row
// Three block barriers per step (the ring, the sums, the squares) and no
// pre-norm round trip through shared memory.
constexpr int kDw7Px = 7;
constexpr int kDw7MaxThreads = 384;
template <typename T, int CT>
__global__ void __launch_bounds__(kDw7MaxThreads, 1)
    dwln7_kernel(const T* __restrict__ x, const T* __restrict__ wdw, const float* __restrict__ bdw,
                 const float* __restrict__ g, const float* __restrict__ be, T* __restrict__ y, int N, int H, int W,
                 int C_rt, float eps, int RB, int nseg) {
  constexpr int KS = 7, R = 3, PX = kDw7Px, NI = PX + 2 * R;
  constexpr bool kF16 = Dt<T>::kIdescAB == 0;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int C = CT ? CT : C_rt;
  const int C8 = C / 8, WG = W / PX, rowh = W * C;
  const int NR = 2 * RB + 2 * R, WP = W + 2 * R, prowh = WP * C;
  // NH: the most warps one pixel group's C8 lanes can span (a compile-time bound when C is)
  constexpr int kNH = CT ? (CT / 8 + 30) / 32 + 1 : 4;
  const int npx = RB * W, NH = CT ? kNH : (C8 + 30) / 32 + 1;
  const float invC = 1.f / (float)C;
  T* s_in = reinterpret_cast<T*>(dsm);                           // [NR][WP][C]
  float* s_S = reinterpret_cast<float*>(s_in + (size_t)NR * prowh);  // [RB * W][NH] partial sums
  float* s_Q = s_S + npx * NH;                                        // [RB * W][NH] partial squares
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_Q + npx * NH);      // [2] ring-row groups (bulk copies)
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  const int c8 = tid % C8, rest = tid / C8, pg = rest % WG, ry = rest / WG;  // ry >= RB: padding thread
  // lanes l and l + 2^k hold the same pixel group: the segmented reduction's adds
  uint32_t seg = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k)
    if (lane + (1 << k) < 32 && (tid + (1 << k)) / C8 == rest) seg |= 1u << k;
  const bool head = lane == 0 || (tid - 1) / C8 != rest;
  // the group's lanes span warps w0 .. w0 + nw - 1; this head's slot is warp - w0
  const int w0 = rest * C8 / 32, nw = (rest * C8 + C8 - 1) / 32 - w0 + 1, hslot = tid / 32 - w0;
  auto seg_sum = [&](float v) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const float o = __shfl_down_sync(0xffffffffu, v, 1 << k);
      if (seg >> k & 1) v += o;
    }
    return v;
  };
  for (int i = tid; i < NR * WP * C8; i += nt) reinterpret_cast<uint4*>(s_in)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  pdl_wait();
  __syncthreads();
  const int SR = (H + nseg - 1) / nseg, per_row = rowh / 8;
  uint32_t grp = 0;  // ring-row groups issued so far (group g completes on s_bar[g & 1], phase (g >> 1) & 1)
  for (int item = blockIdx.x; item < N * nseg; item += gridDim.x) {
    const int img = item / nseg, ys = (item % nseg) * SR, ye = min(H, ys + SR);
    if (ys >= ye) continue;
    const int base = ys - R;
    // one group of ring rows: each image row is one contiguous bulk copy (thread 0);
    // rows outside the image are zero-filled by the block (ordered by the next barrier)
    auto load_rows = [&](int lo, int hi) {
      lo = max(lo, ys - R);
      hi = min(hi, ye + R);
      const int vlo = max(lo, 0), vhi = min(hi, H);
      if (tid == 0) {
        uint64_t* bar = &s_bar[grp & 1];
        mbar_arrive_expect_tx(bar, vhi > vlo ? (uint32_t)((vhi - vlo) * rowh * (int)sizeof(T)) : 0u);
        for (int iy = vlo; iy < vhi; ++iy)
          bulk_g2s(s_in + (size_t)((iy - base) % NR) * prowh + R * C, x + ((size_t)img * H + iy) * rowh,
                   rowh * (int)sizeof(T), bar);
      }
      for (int iy = lo; iy < hi; ++iy)
        if (iy < 0 || iy >= H) {
          T* dst = s_in + (size_t)((iy - base) % NR) * prowh + R * C;
          for (int off = tid; off < per_row; off += nt) *reinterpret_cast<uint4*>(dst + off * 8) = make_uint4(0, 0, 0, 0);
        }
      ++grp;
    };
    load_rows(ys - R, ys + RB + R);
    for (int y0 = ys; y0 < ye; y0 += RB) {
      // (the rows this prefetch overwrites were last read by the previous
      // step's stencil, which every thread finished before its sum barrier)
      const uint32_t need = grp - 1;  // the group holding this step's newest rows
      load_rows(y0 + RB + R, y0 + 2 * RB + R);
      mbar_wait(&s_bar[need & 1], (need >> 1) & 1);
      __syncthreads();
      const bool act = ry < min(RB, ye - y0);
      float acc[PX][8];
      {
        float bias[8];
        ld8f(bdw + c8 * 8, bias);
#pragma unroll
        for (int p = 0; p < PX; ++p)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[p][i] = bias[i];
      }
      if (act) {
        __half2 h[PX][4];
#pragma unroll
        for (int p = 0; p < PX; ++p)
#pragma unroll
          for (int i = 0; i < 4; ++i) h[p][i] = __float2half2_rn(0.f);
        int slot = (y0 + ry - R - base) % NR;
#pragma unroll
        for (int dy = 0; dy < KS; ++dy) {
          const T* row = s_in + (size_t)slot * prowh + (size_t)pg * PX * C + c8 * 8;
          slot = slot + 1 == NR ? 0 : slot + 1;
          uint4 in[NI];
#pragma unroll
          for (int j = 0; j < NI; ++j) in[j] = lds128(row + (size_t)j * C);
#pragma unroll
          for (int dx = 0; dx < KS; ++dx) {
            const uint4 wv = __ldg(reinterpret_cast<const uint4*>(wdw + (size_t)(dy * KS + dx) * C + c8 * 8));
            if constexpr (kF16) {
              const __half2* w2 = reinterpret_cast<const __half2*>(&wv);
#pragma unroll
              for (int p = 0; p < PX; ++p) {
                const __half2* i2 = reinterpret_cast<const __half2*>(&in[p + dx]);
#pragma unroll
                for (int i = 0; i < 4; ++i) h[p][i] = __hfma2(i2[i], w2[i], h[p][i]);
              }
            } else {
              float wf[8];
              unpack8t<T>(wv, wf);
#pragma unroll
              for (int p = 0; p < PX; ++p) {
                float xf[8];
                unpack8t<T>(in[p + dx], xf);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[p][i] = fmaf(xf[i], wf[i], acc[p][i]);
              }
            }
          }
          if (kF16 && (dy == R || dy == KS - 1)) {  // widen twice per window (<= 4 rows of taps in half)
#pragma unroll
            for (int p = 0; p < PX; ++p)
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 f = __half22float2(h[p][i]);
                acc[p][2 * i] += f.x;
                acc[p][2 * i + 1] += f.y;
                h[p][i] = __float2half2_rn(0.f);
              }
          }
        }
      }
      const int pix0 = ry * W + pg * PX;
      // pixel sums (the padding / idle threads add zeros to their own segments)
#pragma unroll
      for (int p = 0; p < PX; ++p) {
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += acc[p][i];
        s = seg_sum(act ? s : 0.f);
        if (act && head) s_S[(pix0 + p) * NH + hslot] = s;
      }
      __syncthreads();
      float mean[PX];
#pragma unroll
      for (int p = 0; p < PX; ++p) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < kNH; ++k)
          if (k < nw) t += s_S[(pix0 + p) * NH + k];
        mean[p] = act ? t * invC : 0.f;
        float q = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) q += (acc[p][i] - mean[p]) * (acc[p][i] - mean[p]);
        q = seg_sum(act ? q : 0.f);
        if (act && head) s_Q[(pix0 + p) * NH + hslot] = q;
      }
      __syncthreads();
      if (act) {
        float gg[8], bb[8];
        ld8f(g + c8 * 8, gg);
        ld8f(be + c8 * 8, bb);
        T* yrow = y + ((size_t)img * H + y0 + ry) * rowh + (size_t)pg * PX * C + c8 * 8;
#pragma unroll
        for (int p = 0; p < PX; ++p) {
          float t = 0.f;
#pragma unroll
          for (int k = 0; k < kNH; ++k)
            if (k < nw) t += s_Q[(pix0 + p) * NH + k];
          const float rstd = rsqrtf(t * invC + eps);
          float v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = (acc[p][i] - mean[p]) * rstd * gg[i] + bb[i];
          *reinterpret_cast<uint4*>(yrow + (size_t)p * C) = pack8t<T>(v);
        }
      }
    }
    // the item's last (possibly empty) prefetch group must land before the ring is reused
    mbar_wait(&s_bar[(grp - 1) & 1], ((grp - 1) >> 1) & 1);
    __syncthreads();
  }
  pdl_trigger();
}
int dwln7_smem(int W, int C, int RB) {
  return (2 * RB + 6) * (W + 6) * C * 2 + 2 * RB * W * ((C / 8 + 30) / 32 + 1) * 4 + 16;
}
int dwln7_threads(int W, int C, int RB) { return (RB * (W / kDw7Px) * (C / 8) + 31) / 32 * 32; }
// segments per image: waves of (image, segment) items x (band steps + ~0.75 of
// a step for the window a segment loads before its first step) — at b128 one
// segment per image (128 CTAs) beats four ragged ones on 148 SMs
int dwln7_segments(int N, int H, int RB) {
  int best = 1;
  double best_cost = 1e30;
  for (int nseg = 1; nseg * RB <= H; ++nseg) {
    const int SR = (H + nseg - 1) / nseg, steps = (SR + RB - 1) / RB;
    const int waves = (N * nseg + kNumSMs - 1) / kNumSMs;
    const double cost = waves * (steps + 0.75);
    if (cost < best_cost - 1e-9) best = nseg, best_cost = cost;
  }
  return best;
}
// rows per band step for the 7-pixel kernel (0: not eligible)
int dwln7_rows(int KS, int W, int C) {
  if (KS != 7 || W % kDw7Px || C % 8) return 0;
  for (int rb : {4, 3, 2, 1})
    if (dwln7_threads(W, C, rb) <= kDw7MaxThreads && dwln7_smem(W, C, rb) <= 232448) return rb;
  return 0;
}

// LayerNorm per pixel; S2D: the output row is written in 2x2 space-to-depth
// order A[(img, y/2, x/2)][((y%2) 2 + x%2) C + c]. CTA = P pixels x C/8
// threads; one 16-byte chunk per thread, two-pass statistics over shared sums.
template <typename T>
__global__ void __launch_bounds__(256) ln_s2d_kernel(const T* __restrict__ x, const float* __restrict__ g,
                                                     const float* __restrict__ be, T* __restrict__ A, int n,
                                                     int H, int W, int C, float eps) {
  // fixed-order (deterministic) reductions: per-thread partials, then the
  // pixel's first thread sums its C/8 partials in channel order
  __shared__ float s_part[256], s_mean[256], s_rstd[256];
  const int C8 = C / 8, P = 256 / C8, tid = threadIdx.x;
  const int pl = tid / C8, c8 = tid - pl * C8;
  const int64_t pix = (int64_t)blockIdx.x * P + pl;
  const int64_t npix = (int64_t)n * H * W;
  const bool on = pl < P && pix < npix;
  pdl_wait();
  float v[8];
  float s = 0.f;
  if (on) {
    unpack8t<T>(__ldg(reinterpret_cast<const uint4*>(x + pix * C) + c8), v);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
  }
  s_part[tid] = s;
  __syncthreads();
  if (on && c8 == 0) {
    float t = 0.f;
    for (int j = 0; j < C8; ++j) t += s_part[tid + j];
    s_mean[pl] = t / (float)C;
  }
  __syncthreads();
  const float mean = on ? s_mean[pl] : 0.f;
  s = 0.f;
  if (on) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s += (v[i] - mean) * (v[i] - mean);
  }
  s_part[tid] = s;
  __syncthreads();
  if (on && c8 == 0) {
    float t = 0.f;
    for (int j = 0; j < C8; ++j) t += s_part[tid + j];
    s_rstd[pl] = rsqrtf(t / (float)C + eps);
  }
  __syncthreads();
  if (on) {
    const float rstd = s_rstd[pl];
    float gg[8], bb[8];
    ld8f(g + c8 * 8, gg);
    ld8f(be + c8 * 8, bb);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (v[i] - mean) * rstd * gg[i] + bb[i];
    const int xx = (int)(pix % W), yy = (int)((pix / W) % H);
    const int64_t img = pix / ((int64_t)W * H);
    T* dst = A + (((img * (H / 2) + yy / 2) * (W / 2) + xx / 2) * 4 + (yy % 2) * 2 + xx % 2) * C;
    reinterpret_cast<uint4*>(dst)[c8] = pack8t<T>(v);
  }
  pdl_trigger();
}

// global average pool + LayerNorm: one CTA per image, thread = channel pair
template <typename T>
__global__ void __launch_bounds__(512) pool_ln_kernel(const T* __restrict__ x, const float* __restrict__ g,
                                                      const float* __restrict__ be, T* __restrict__ f, int HW,
                                                      int C, float eps) {
  __shared__ float red[2][32];
  const int img = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool on = 2 * tid < C;
  pdl_wait();
  float m0 = 0.f, m1 = 0.f;
  if (on) {
    const uint32_t* px = reinterpret_cast<const uint32_t*>(x + (size_t)img * HW * C) + tid;
    for (int p = 0; p < HW; ++p) {
      const float2 v = Dt<T>::unpack2(px[(size_t)p * (C / 2)]);
      m0 += v.x;
      m1 += v.y;
    }
    m0 /= (float)HW;
    m1 /= (float)HW;
  }
  auto block_sum = [&](float v, int slot) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[slot][warp] = v;
    __syncthreads();
    float t = 0.f;
    for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) t += red[slot][i];
    return t;
  };
  const float mean = block_sum(on ? m0 + m1 : 0.f, 0) / (float)C;
  const float d0 = m0 - mean, d1 = m1 - mean;
  const float var = block_sum(on ? d0 * d0 + d1 * d1 : 0.f, 1) / (float)C;
  const float rstd = rsqrtf(var + eps);
  if (on)
    reinterpret_cast<uint32_t*>(f + (size_t)img * C)[tid] =
        Dt<T>::pack2(d0 * rstd * g[2 * tid] + be[2 * tid], d1 * rstd * g[2 * tid + 1] + be[2 * tid + 1]);
  pdl_trigger();
}

// ============================================================ host helpers
namespace {

template <typename Kern, typename... Args>
int launch_simple(Kern k, int grid, int block, cudaStream_t st, const char* what, Args... args) {
  return launch_pdl(k, grid, block, 0, st, what, args...);
}

int64_t a128(int64_t v) { return (v + 127) / 128 * 128; }

void put_f32(uint8_t* base, int64_t off, const float* src, int64_t count) {
  memcpy(base + off, src, (size_t)count * 4);
}
// B operand (N rows of K fp16, K contiguous) from a reference (K, N) matrix
void put_t16(uint8_t* base, int64_t off, const float* src, int K, int N, int dtype) {
  for (int nn = 0; nn < N; ++nn)
    for (int k = 0; k < K; ++k) put_v(base, off + ((int64_t)nn * K + k) * 2, src[(int64_t)k * N + nn], dtype);
}

// row batch of the two-GEMM FFN so that the hidden stays L2-resident
int64_t hidden_rows(int64_t M, int hid) {
  int64_t r = kHiddenBatchBytes / ((int64_t)hid * 2);
  r = r / 128 * 128;
  if (r < 128) r = 128;
  return r < M ? r : M;
}

// z = phi(x U + a) V + b (+ res): the fused kernel (hidden on chip, ffn.cu)
// when its TMEM plan fits (C <= 384), else two GEMMs per row batch with the
// hidden in the L2-resident workspace
// the fused FFN kernel (hidden on chip) up to C = 256 when its weight images exist
bool ffn_fused_route(int64_t M, int C, int hid) {
  return C <= 256 && ffn_images_bytes(C, hid) > 0 && ffn_fused_ok(M, C, hid);
}
int ffn_rows(const __half* x, int64_t M, int C, int hid, int K, const __half* ut, const float* a, const __half* vt,
             const float* b, int act, const __half* res, __half* z, __half* hbuf, const uint8_t* wimg,
             cudaStream_t st, int dtype) {
  // the fused kernel (hidden on chip) up to C = 256; above, the two GEMMs with an
  // L2-resident hidden (ConvNeXt-T b128 per block, after the FFN issuer rework:
  // 28x28x192 180 vs 212 us fused vs GEMMs, 14x14x384 195 vs 121 us)
  if (K == C && wimg && ffn_fused_route(M, C, hid))
    return ffn_fused_run(x, M, C, hid, wimg, a, b, act, res, z, st, dtype);
  const int64_t rb = hidden_rows(M, hid);
  for (int64_t r0 = 0; r0 < M; r0 += rb) {
    const int rows = (int)(M - r0 < rb ? M - r0 : rb);
    GemmEpi e1;
    e1.bias = a;
    e1.act = act;
    if (int e = gemm_run(x + r0 * C, rows, C, C, ut, hid, C, hbuf, hid, e1, st, dtype)) return e;
    GemmEpi e2;
    e2.bias = b;
    if (res) {
      e2.res = res + r0 * K;
      e2.ldr = K;
    }
    if (int e = gemm_run(hbuf, rows, hid, hid, vt, K, hid, z + r0 * K, K, e2, st, dtype)) return e;
  }
  return WL_OK;
}

int common_dims(const wl_block_desc& d) {
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c < 1) return set_error(WL_EINVAL, "dims must be positive");
  if (d.c % 8) return set_error(WL_EUNSUPPORTED, "channel count %d must be a multiple of 8", d.c);
  return WL_OK;
}

// ------------------------------------------------------------------ FFN
// weights (reference order, machine.py:345-351): u (C, hid), a (hid), v (hid, C), b (C)
struct FfnLayout {
  int64_t o_a, o_b, o_u, o_v, o_img, total;
};
FfnLayout ffn_layout(const wl_block_desc& d) {
  const int64_t C = d.c, hid = (int64_t)d.expansion * d.c;
  FfnLayout L;
  L.o_a = 0;
  L.o_b = a128(hid * 4);
  L.o_u = L.o_b + a128(C * 4 + 64);
  L.o_v = L.o_u + a128(hid * C * 2);
  L.o_img = L.o_v + a128(hid * C * 2);  // fused-kernel weight images (0 bytes when it has no plan)
  L.total = L.o_img + a128(ffn_images_bytes((int)C, (int)hid));
  return L;
}
int ffn_validate(const wl_block_desc& d) {
  if (int e = common_dims(d)) return e;
  if (d.expansion < 1) return set_error(WL_EINVAL, "expansion must be at least 1");
  if (d.k != d.c) return set_error(WL_EINVAL, "FFN blocks keep their channel count");
  if (d.act < 0 || d.act > 4) return set_error(WL_EINVAL, "unknown activation");
  return WL_OK;
}
int ffn_wc(const wl_block_desc&) { return 4; }
int64_t ffn_wn(const wl_block_desc& d, int i) {
  const int64_t C = d.c, hid = (int64_t)d.expansion * d.c;
  switch (i) {
    case 0: return C * hid;
    case 1: return hid;
    case 2: return hid * C;
    case 3: return C;
  }
  return set_error(WL_EINVAL, "weight index out of range");
}
int64_t ffn_pb(const wl_block_desc& d) { return ffn_layout(d).total; }
int ffn_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  const FfnLayout L = ffn_layout(d);
  const int C = d.c, hid = d.expansion * d.c;
  memset(out, 0, (size_t)L.total);
  put_f32(out, L.o_a, w[1], hid);
  put_f32(out, L.o_b, w[3], C);
  put_t16(out, L.o_u, w[0], C, hid, d.dtype);  // U^T: (hid, C)
  put_t16(out, L.o_v, w[2], hid, C, d.dtype);  // V^T: (C, hid)
  ffn_pack_images(C, hid, w[0], w[2], out + L.o_img, d.dtype);
  return WL_OK;
}
int64_t ffn_ws(const wl_block_desc& d) {
  const int64_t M = (int64_t)d.n * d.h * d.w, hid = (int64_t)d.expansion * d.c;
  return kWsHdr + a128(hidden_rows(M, (int)hid) * hid * 2);
}
int ffn_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  const FfnLayout L = ffn_layout(d);
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(p);
  const int64_t M = (int64_t)d.n * d.h * d.w;
  return ffn_rows(reinterpret_cast<const __half*>(x), M, d.c, d.expansion * d.c, d.c,
                  reinterpret_cast<const __half*>(pk + L.o_u), reinterpret_cast<const float*>(pk + L.o_a),
                  reinterpret_cast<const __half*>(pk + L.o_v), reinterpret_cast<const float*>(pk + L.o_b), d.act,
                  nullptr, reinterpret_cast<__half*>(z), reinterpret_cast<__half*>((uint8_t*)ws + kWsHdr),
                  L.o_img < L.total ? pk + L.o_img : nullptr, st, d.dtype);
}

// ------------------------------------------------- wide ConvNeXt block
// weights (cf_weight_numel order): w_conv (C, k, k, 1), b_conv (C), ln_gamma, ln_beta,
// u (C, hid), a (hid), v (hid, C), b (C)
struct WideLayout {
  int64_t o_wdw, o_bdw, o_g, o_be, o_a, o_b, o_u, o_v, o_img, total;
};
WideLayout wide_layout(const wl_block_desc& d) {
  const int64_t C = d.c, hid = (int64_t)d.expansion * d.c, taps = (int64_t)d.ksize * d.ksize;
  WideLayout L;
  L.o_wdw = 0;  // [tap][C] fp16
  L.o_bdw = a128(taps * C * 2);
  L.o_g = L.o_bdw + a128(C * 4 + 64);
  L.o_be = L.o_g + a128(C * 4 + 64);
  L.o_a = L.o_be + a128(C * 4 + 64);
  L.o_b = L.o_a + a128(hid * 4 + 64);
  L.o_u = L.o_b + a128(C * 4 + 64);
  L.o_v = L.o_u + a128(hid * C * 2);
  L.o_img = L.o_v + a128(hid * C * 2);
  L.total = L.o_img + a128(ffn_images_bytes((int)C, (int)hid));
  return L;
}
}  // namespace

int ffn_row_batches(const wl_block_desc& d) {
  const int64_t M = (int64_t)d.n * d.h * d.w, rb = hidden_rows(M, d.expansion * d.c);
  return (int)((M + rb - 1) / rb);
}
int ffn_launches(const wl_block_desc& d, bool images) {
  const int64_t M = (int64_t)d.n * d.h * d.w;
  return images && ffn_fused_route(M, d.c, d.expansion * d.c) ? 1 : 2 * ffn_row_batches(d);
}

bool cnx_wide(const wl_block_desc& d) {
  // C > 128: only this path. C = 96..128 with a 7x7 stencil: this path for large
  // batches (ConvNeXt-T b128 56x56 stage: 453 vs 544 us per block), the single
  // fused conv-first kernel for small ones (BASELINE config 1, b8: 50 vs 63 us)
  const bool big = (int64_t)d.n * d.h * d.w >= 65536;
  return d.kind == WL_KIND_CONVFIRST && d.norm == WL_NORM_LAYERNORM && d.group_width == 1 && d.stride == 1 &&
         (d.c > 128 || (d.c >= 96 && d.ksize == 7 && (big || d.dtype == WL_DTYPE_BF16)));
}
int cnx_wide_validate(const wl_block_desc& d) {
  if (int e = common_dims(d)) return e;
  if (d.ksize != 7 && d.ksize != 3) return set_error(WL_EUNSUPPORTED, "wide ConvNeXt block: 3x3 or 7x7 only");
  if (d.c > 1024) return set_error(WL_EUNSUPPORTED, "wide ConvNeXt block: C <= 1024");
  if (dwln_rows(d.ksize, d.w, d.c) == 0 || d.w > 128)
    return set_error(WL_EUNSUPPORTED, "wide ConvNeXt block: a %d-row band of %dx%d does not fit shared memory",
                     d.ksize, d.w, d.c);
  return WL_OK;
}
int64_t cnx_wide_pb(const wl_block_desc& d) { return wide_layout(d).total; }
int cnx_wide_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  const WideLayout L = wide_layout(d);
  const int C = d.c, hid = d.expansion * d.c, taps = d.ksize * d.ksize;
  memset(out, 0, (size_t)L.total);
  for (int c = 0; c < C; ++c)
    for (int t = 0; t < taps; ++t) put_v(out, L.o_wdw + ((int64_t)t * C + c) * 2, w[0][(size_t)c * taps + t], d.dtype);
  put_f32(out, L.o_bdw, w[1], C);
  put_f32(out, L.o_g, w[2], C);
  put_f32(out, L.o_be, w[3], C);
  put_f32(out, L.o_a, w[5], hid);
  put_f32(out, L.o_b, w[7], C);
  put_t16(out, L.o_u, w[4], C, hid, d.dtype);
  put_t16(out, L.o_v, w[6], hid, C, d.dtype);
  ffn_pack_images(C, hid, w[4], w[6], out + L.o_img, d.dtype);
  return WL_OK;
}
int64_t cnx_wide_ws(const wl_block_desc& d) {
  const int64_t M = (int64_t)d.n * d.h * d.w, hid = (int64_t)d.expansion * d.c;
  return kWsHdr + a128(M * d.c * 2) + a128(hidden_rows(M, (int)hid) * hid * 2);
}
int cnx_wide_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  const WideLayout L = wide_layout(d);
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(p);
  const int64_t M = (int64_t)d.n * d.h * d.w;
  __half* xh = reinterpret_cast<__half*>((uint8_t*)ws + kWsHdr);
  __half* hb = reinterpret_cast<__half*>((uint8_t*)ws + kWsHdr + a128(M * d.c * 2));
  const float eps = d.ln_eps > 0 ? d.ln_eps : 1e-6f;
  const int rb7 = dwln7_rows(d.ksize, d.w, d.c);
  auto dw7 = [&]() {
    const int nseg = dwln7_segments(d.n, d.h, rb7), grid = std::min(d.n * nseg, kNumSMs);
    auto run7 = [&](auto kern, auto tag) {
      using T = decltype(tag);
      return launch_pdl(kern, grid, dwln7_threads(d.w, d.c, rb7), dwln7_smem(d.w, d.c, rb7), st, "dwln7 launch",
                        reinterpret_cast<const T*>(x), reinterpret_cast<const T*>(pk + L.o_wdw),
                        reinterpret_cast<const float*>(pk + L.o_bdw), reinterpret_cast<const float*>(pk + L.o_g),
                        reinterpret_cast<const float*>(pk + L.o_be), reinterpret_cast<T*>(xh), d.n, d.h, d.w, d.c,
                        eps, rb7, nseg);
    };
    auto pick7 = [&](auto tag) {
      using T = decltype(tag);
      switch (d.c) {
        case 96: return run7(dwln7_kernel<T, 96>, tag);
        case 192: return run7(dwln7_kernel<T, 192>, tag);
        case 384: return run7(dwln7_kernel<T, 384>, tag);
        case 768: return run7(dwln7_kernel<T, 768>, tag);
      }
      return run7(dwln7_kernel<T, 0>, tag);
    };
    return d.dtype == WL_DTYPE_BF16 ? pick7(__nv_bfloat16{}) : pick7(__half{});
  };
  const int rb = dwln_rows(d.ksize, d.w, d.c), nseg = dwln_segments(d.n, d.h, rb);
  const int grid = std::min(d.n * nseg, kNumSMs);
  auto run_dw = [&](auto kern, auto tag) {
    using T = decltype(tag);
    return launch_pdl(kern, grid, kDwThreads, dwln_smem(d.ksize, d.w, d.c), st, "dwln launch",
                      reinterpret_cast<const T*>(x), reinterpret_cast<const T*>(pk + L.o_wdw),
                      reinterpret_cast<const float*>(pk + L.o_bdw), reinterpret_cast<const float*>(pk + L.o_g),
                      reinterpret_cast<const float*>(pk + L.o_be), reinterpret_cast<T*>(xh), d.n, d.h, d.w, d.c, eps,
                      rb, nseg);
  };
  auto pick = [&](auto tag) {
    using T = decltype(tag);
    if (d.ksize == 3) return run_dw(dwln_kernel<3, T, 0>, tag);
    switch (d.c) {
      case 96: return run_dw(dwln_kernel<7, T, 96>, tag);
      case 192: return run_dw(dwln_kernel<7, T, 192>, tag);
      case 384: return run_dw(dwln_kernel<7, T, 384>, tag);
      case 768: return run_dw(dwln_kernel<7, T, 768>, tag);
    }
    return run_dw(dwln_kernel<7, T, 0>, tag);
  };
  const int e = rb7 ? dw7() : d.dtype == WL_DTYPE_BF16 ? pick(__nv_bfloat16{}) : pick(__half{});
  if (e) return e;
  return ffn_rows(xh, M, d.c, d.expansion * d.c, d.c, reinterpret_cast<const __half*>(pk + L.o_u),
                  reinterpret_cast<const float*>(pk + L.o_a), reinterpret_cast<const __half*>(pk + L.o_v),
                  reinterpret_cast<const float*>(pk + L.o_b), d.act, reinterpret_cast<const __half*>(x),
                  reinterpret_cast<__half*>(z), hb, L.o_img < L.total ? pk + L.o_img : nullptr, st, d.dtype);
}

// ------------------------------------------------------- wide ConvFirst (no LayerNorm)
// The reference's channel-partitioned schedule (machine.py:528-569) lets the
// partial hidden sums meet in the GLOBAL tier; past one CTA's TMEM (C > 128)
// the block runs as: grouped k x k conv + b_conv (CUDA cores, layerwise.cu) ->
// xc (workspace) -> z = x + b + phi(xc U + a) V through the FFN rows (two
// tcgen05 GEMMs per L2-sized row batch).
// weights: w_conv (C,k,k,T), b_conv (C), u (C,hid), a (hid), v (hid,C), b (C)
namespace {
struct CfWideLayout {
  int64_t o_conv, o_bconv, o_a, o_b, o_u, o_v, total;
};
CfWideLayout cf_wide_layout(const wl_block_desc& d) {
  const int64_t C = d.c, hid = (int64_t)d.expansion * d.c, taps = (int64_t)d.ksize * d.ksize;
  CfWideLayout L;
  L.o_conv = 0;
  L.o_bconv = a128(C * taps * d.group_width * 4);
  L.o_a = L.o_bconv + a128(C * 4 + 64);
  L.o_b = L.o_a + a128(hid * 4 + 64);
  L.o_u = L.o_b + a128(C * 4 + 64);
  L.o_v = L.o_u + a128(hid * C * 2);
  L.total = L.o_v + a128(hid * C * 2);
  return L;
}
}  // namespace

bool cf_wide(const wl_block_desc& d) {
  return d.kind == WL_KIND_CONVFIRST && d.norm == WL_NORM_NONE && d.stride == 1 && d.c > 128;
}
int cf_wide_validate(const wl_block_desc& d) {
  if (int e = common_dims(d)) return e;
  if (d.dtype != WL_DTYPE_F16) return set_error(WL_EUNSUPPORTED, "wide conv-first block: fp16");
  if (d.c % 8) return set_error(WL_EUNSUPPORTED, "wide conv-first block: C %% 8 == 0");
  if (d.group_width != 8 && d.group_width != 1)
    return set_error(WL_EUNSUPPORTED, "wide conv-first block: T = 8 or 1 (got %d)", d.group_width);
  if (d.ksize != 3 && !(d.ksize == 7 && d.group_width == 1))
    return set_error(WL_EUNSUPPORTED, "wide conv-first block: 3x3, or 7x7 depthwise");
  if (d.act != kRelu && d.act != kSilu && d.act != kGelu)
    return set_error(WL_EUNSUPPORTED, "wide conv-first block supports relu/silu/gelu");
  return WL_OK;
}
int64_t cf_wide_pb(const wl_block_desc& d) { return cf_wide_layout(d).total; }
int cf_wide_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  const CfWideLayout L = cf_wide_layout(d);
  const int C = d.c, hid = d.expansion * d.c;
  memset(out, 0, (size_t)L.total);
  put_f32(out, L.o_conv, w[0], (int64_t)C * d.ksize * d.ksize * d.group_width);
  put_f32(out, L.o_bconv, w[1], C);
  put_f32(out, L.o_a, w[3], hid);
  put_f32(out, L.o_b, w[5], C);
  put_t16(out, L.o_u, w[2], C, hid, d.dtype);
  put_t16(out, L.o_v, w[4], hid, C, d.dtype);
  return WL_OK;
}
int64_t cf_wide_ws(const wl_block_desc& d) {
  const int64_t M = (int64_t)d.n * d.h * d.w, hid = (int64_t)d.expansion * d.c;
  return kWsHdr + a128(M * d.c * 2) + a128(hidden_rows(M, (int)hid) * hid * 2);
}
int cf_wide_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  const CfWideLayout L = cf_wide_layout(d);
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(p);
  const int64_t M = (int64_t)d.n * d.h * d.w;
  __half* xc = reinterpret_cast<__half*>((uint8_t*)ws + kWsHdr);
  __half* hb = reinterpret_cast<__half*>((uint8_t*)ws + kWsHdr + a128(M * d.c * 2));
  if (int e = lw_gconv(d, d.c, reinterpret_cast<const __half*>(x), reinterpret_cast<const float*>(pk + L.o_conv),
                       reinterpret_cast<const float*>(pk + L.o_bconv), xc, kIdentity, st))
    return e;
  return ffn_rows(xc, M, d.c, d.expansion * d.c, d.c, reinterpret_cast<const __half*>(pk + L.o_u),
                  reinterpret_cast<const float*>(pk + L.o_a), reinterpret_cast<const __half*>(pk + L.o_v),
                  reinterpret_cast<const float*>(pk + L.o_b), d.act, reinterpret_cast<const __half*>(x),
                  reinterpret_cast<__half*>(z), hb, nullptr, st, d.dtype);
}

namespace {
// ------------------------------------------------------- patchify stem
// desc: c = input channels, k = output channels, ksize = patch = stride
// weights: w (k, p, p, c), b (k), ln_gamma (k), ln_beta (k)
struct PsLayout {
  int64_t o_b, o_g, o_be, o_w, total;
  int kk;
};
PsLayout ps_layout(const wl_block_desc& d) {
  PsLayout L;
  L.kk = d.ksize * d.ksize * d.c;
  L.o_b = 0;
  L.o_g = a128(d.k * 4 + 64);
  L.o_be = L.o_g + a128(d.k * 4 + 64);
  L.o_w = L.o_be + a128(d.k * 4 + 64);
  L.total = L.o_w + a128((int64_t)d.k * L.kk * 2);
  return L;
}
int ps_validate(const wl_block_desc& d) {
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c < 1 || d.k < 1) return set_error(WL_EINVAL, "dims must be positive");
  if (d.ksize < 1 || d.h % d.ksize || d.w % d.ksize)
    return set_error(WL_EINVAL, "patch %d must divide the input %dx%d", d.ksize, d.h, d.w);
  if ((d.ksize * d.ksize * d.c) % 8 || d.k % 8 || d.k > 256)
    return set_error(WL_EUNSUPPORTED, "patchify stem: p*p*c and k multiples of 8, k <= 256");
  return WL_OK;
}
int ps_wc(const wl_block_desc& d) { return d.norm == WL_NORM_LAYERNORM ? 4 : 2; }
int64_t ps_wn(const wl_block_desc& d, int i) {
  switch (i) {
    case 0: return (int64_t)d.k * d.ksize * d.ksize * d.c;
    case 1:
    case 2:
    case 3: return d.k;
  }
  return set_error(WL_EINVAL, "weight index out of range");
}
int64_t ps_pb(const wl_block_desc& d) { return ps_layout(d).total; }
int ps_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  const PsLayout L = ps_layout(d);
  memset(out, 0, (size_t)L.total);
  put_f32(out, L.o_b, w[1], d.k);
  if (d.norm == WL_NORM_LAYERNORM) {
    put_f32(out, L.o_g, w[2], d.k);
    put_f32(out, L.o_be, w[3], d.k);
  }
  for (int64_t i = 0; i < (int64_t)d.k * L.kk; ++i) put_v(out, L.o_w + i * 2, w[0][i], d.dtype);  // (k, p, p, c) = B rows
  return WL_OK;
}
int64_t ps_ws(const wl_block_desc& d) {
  const int64_t M = (int64_t)d.n * (d.h / d.ksize) * (d.w / d.ksize);
  return kWsHdr + a128(M * ps_layout(d).kk * 2);
}
int ps_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  const PsLayout L = ps_layout(d);
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(p);
  const int64_t M = (int64_t)d.n * (d.h / d.ksize) * (d.w / d.ksize);
  __half* A = reinterpret_cast<__half*>((uint8_t*)ws + kWsHdr);
  const int64_t total = (d.ksize * d.c) % 4 == 0 ? M * d.ksize : M * L.kk;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, kNumSMs * 32);
  if (int e = launch_simple(patchify_kernel, grid, 256, st, "patchify launch", reinterpret_cast<const __half*>(x), A,
                            d.n, d.h, d.w, d.c, d.ksize))
    return e;
  GemmEpi ep;
  ep.bias = reinterpret_cast<const float*>(pk + L.o_b);
  ep.act = d.act;
  if (d.norm == WL_NORM_LAYERNORM) {
    ep.ln_g = reinterpret_cast<const float*>(pk + L.o_g);
    ep.ln_b = reinterpret_cast<const float*>(pk + L.o_be);
    ep.ln_eps = d.ln_eps > 0 ? d.ln_eps : 1e-6f;
  }
  return gemm_run(A, (int)M, L.kk, L.kk, pk + L.o_w, d.k, L.kk, z, d.k, ep, st, d.dtype);
}

// ----------------------------------------------------------- downsample
// desc: c -> k, stride 2 (2x2 patches); weights ln_gamma (c), ln_beta (c), w (k, 2, 2, c), b (k)
struct DsLayout {
  int64_t o_g, o_be, o_b, o_w, total;
};
DsLayout ds_layout(const wl_block_desc& d) {
  DsLayout L;
  L.o_g = 0;
  L.o_be = a128(d.c * 4 + 64);
  L.o_b = L.o_be + a128(d.c * 4 + 64);
  L.o_w = L.o_b + a128(d.k * 4 + 64);
  L.total = L.o_w + a128((int64_t)d.k * 4 * d.c * 2);
  return L;
}
int ds_validate(const wl_block_desc& d) {
  if (int e = common_dims(d)) return e;
  if (d.k < 8 || d.k % 8) return set_error(WL_EUNSUPPORTED, "downsample: k must be a multiple of 8");
  if (d.h % 2 || d.w % 2) return set_error(WL_EINVAL, "downsample needs an even resolution (%dx%d)", d.h, d.w);
  if (d.c > 2048) return set_error(WL_EUNSUPPORTED, "downsample: C <= 2048");
  return WL_OK;
}
int ds_wc(const wl_block_desc&) { return 4; }
int64_t ds_wn(const wl_block_desc& d, int i) {
  switch (i) {
    case 0:
    case 1: return d.c;
    case 2: return (int64_t)d.k * 4 * d.c;
    case 3: return d.k;
  }
  return set_error(WL_EINVAL, "weight index out of range");
}
int64_t ds_pb(const wl_block_desc& d) { return ds_layout(d).total; }
int ds_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  const DsLayout L = ds_layout(d);
  memset(out, 0, (size_t)L.total);
  put_f32(out, L.o_g, w[0], d.c);
  put_f32(out, L.o_be, w[1], d.c);
  put_f32(out, L.o_b, w[3], d.k);
  for (int64_t i = 0; i < (int64_t)d.k * 4 * d.c; ++i) put_v(out, L.o_w + i * 2, w[2][i], d.dtype);
  return WL_OK;
}
int64_t ds_ws(const wl_block_desc& d) { return kWsHdr + a128((int64_t)d.n * d.h * d.w * d.c * 2); }
int ds_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  const DsLayout L = ds_layout(d);
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(p);
  __half* A = reinterpret_cast<__half*>((uint8_t*)ws + kWsHdr);
  const int64_t npix = (int64_t)d.n * d.h * d.w;
  const float eps = d.ln_eps > 0 ? d.ln_eps : 1e-6f;
  const int P = 256 / (d.c / 8);
  const int grid = (int)((npix + P - 1) / P);
  const float* g = reinterpret_cast<const float*>(pk + L.o_g);
  const float* be = reinterpret_cast<const float*>(pk + L.o_be);
  const int e = d.dtype == WL_DTYPE_BF16
                    ? launch_simple(ln_s2d_kernel<__nv_bfloat16>, grid, 256, st, "ln_s2d launch",
                                    reinterpret_cast<const __nv_bfloat16*>(x), g, be,
                                    reinterpret_cast<__nv_bfloat16*>(A), d.n, d.h, d.w, d.c, eps)
                    : launch_simple(ln_s2d_kernel<__half>, grid, 256, st, "ln_s2d launch",
                                    reinterpret_cast<const __half*>(x), g, be, A, d.n, d.h, d.w, d.c, eps);
  if (e) return e;
  GemmEpi ep;
  ep.bias = reinterpret_cast<const float*>(pk + L.o_b);
  return gemm_run(A, (int)(npix / 4), 4 * d.c, 4 * d.c, pk + L.o_w, d.k, 4 * d.c, z, d.k, ep, st, d.dtype);
}

// -------------------------------------------------------------- LN head
// desc: c, classes; weights ln_gamma (c), ln_beta (c), w_cls (c, classes), b_cls (classes)
struct LhLayout {
  int64_t o_g, o_be, o_b, o_w, total;
};
LhLayout lh_layout(const wl_block_desc& d) {
  LhLayout L;
  L.o_g = 0;
  L.o_be = a128(d.c * 4 + 64);
  L.o_b = L.o_be + a128(d.c * 4 + 64);
  L.o_w = L.o_b + a128(d.classes * 4 + 64);
  L.total = L.o_w + a128((int64_t)d.classes * d.c * 2);
  return L;
}
int lh_validate(const wl_block_desc& d) {
  if (int e = common_dims(d)) return e;
  if (d.classes < 8 || d.classes % 8) return set_error(WL_EUNSUPPORTED, "LN head: classes must be a multiple of 8");
  if (d.c > 1024) return set_error(WL_EUNSUPPORTED, "LN head: C <= 1024");
  return WL_OK;
}
int lh_wc(const wl_block_desc&) { return 4; }
int64_t lh_wn(const wl_block_desc& d, int i) {
  switch (i) {
    case 0:
    case 1: return d.c;
    case 2: return (int64_t)d.c * d.classes;
    case 3: return d.classes;
  }
  return set_error(WL_EINVAL, "weight index out of range");
}
int64_t lh_pb(const wl_block_desc& d) { return lh_layout(d).total; }
int lh_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  const LhLayout L = lh_layout(d);
  memset(out, 0, (size_t)L.total);
  put_f32(out, L.o_g, w[0], d.c);
  put_f32(out, L.o_be, w[1], d.c);
  put_f32(out, L.o_b, w[3], d.classes);
  put_t16(out, L.o_w, w[2], d.c, d.classes, d.dtype);
  return WL_OK;
}
int64_t lh_ws(const wl_block_desc& d) { return kWsHdr + a128((int64_t)d.n * d.c * 2); }
int lh_fwd(const wl_block_desc& d, const void* x, const void* p, void* z, void* ws, cudaStream_t st) {
  const LhLayout L = lh_layout(d);
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(p);
  __half* f = reinterpret_cast<__half*>((uint8_t*)ws + kWsHdr);
  const float eps = d.ln_eps > 0 ? d.ln_eps : 1e-6f;
  const int threads = align_up(d.c / 2, 32);
  const float* g = reinterpret_cast<const float*>(pk + L.o_g);
  const float* be = reinterpret_cast<const float*>(pk + L.o_be);
  const int e = d.dtype == WL_DTYPE_BF16
                    ? launch_simple(pool_ln_kernel<__nv_bfloat16>, d.n, threads, st, "pool_ln launch",
                                    reinterpret_cast<const __nv_bfloat16*>(x), g, be,
                                    reinterpret_cast<__nv_bfloat16*>(f), d.h * d.w, d.c, eps)
                    : launch_simple(pool_ln_kernel<__half>, d.n, threads, st, "pool_ln launch",
                                    reinterpret_cast<const __half*>(x), g, be, f, d.h * d.w, d.c, eps);
  if (e) return e;
  GemmEpi ep;
  ep.bias = reinterpret_cast<const float*>(pk + L.o_b);
  return gemm_run(f, d.n, d.c, d.c, pk + L.o_w, d.classes, d.c, z, d.classes, ep, st, d.dtype);
}

int cnx_init() {
  if (int e = gemm_init()) return e;
  if (int e = ffn_fused_init()) return e;
  auto set = [](auto k) {
    return check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448),
                      "cudaFuncSetAttribute(dwln)");
  };
  for (int e : {set(dwln_kernel<3, __half, 0>), set(dwln_kernel<7, __half, 0>), set(dwln_kernel<7, __half, 96>),
                set(dwln_kernel<7, __half, 192>), set(dwln_kernel<7, __half, 384>), set(dwln_kernel<7, __half, 768>),
                set(dwln_kernel<3, __nv_bfloat16, 0>), set(dwln_kernel<7, __nv_bfloat16, 0>),
                set(dwln_kernel<7, __nv_bfloat16, 96>), set(dwln_kernel<7, __nv_bfloat16, 192>),
                set(dwln_kernel<7, __nv_bfloat16, 384>), set(dwln_kernel<7, __nv_bfloat16, 768>),
                set(dwln7_kernel<__half, 0>), set(dwln7_kernel<__half, 96>), set(dwln7_kernel<__half, 192>),
                set(dwln7_kernel<__half, 384>), set(dwln7_kernel<__half, 768>), set(dwln7_kernel<__nv_bfloat16, 0>),
                set(dwln7_kernel<__nv_bfloat16, 96>), set(dwln7_kernel<__nv_bfloat16, 192>),
                set(dwln7_kernel<__nv_bfloat16, 384>), set(dwln7_kernel<__nv_bfloat16, 768>)})
    if (e) return e;
  return WL_OK;
}
int no_init() { return WL_OK; }

}  // namespace

const Family kFfnFamily = {ffn_validate, ffn_wc, ffn_wn, ffn_pb, ffn_pack, ffn_ws, ffn_fwd, cnx_init};
const Family kPatchStemFamily = {ps_validate, ps_wc, ps_wn, ps_pb, ps_pack, ps_ws, ps_fwd, no_init};
const Family kDownsampleFamily = {ds_validate, ds_wc, ds_wn, ds_pb, ds_pack, ds_ws, ds_fwd, no_init};
const Family kLnHeadFamily = {lh_validate, lh_wc, lh_wn, lh_pb, lh_pack, lh_ws, lh_fwd, no_init};

}  // namespace wl
