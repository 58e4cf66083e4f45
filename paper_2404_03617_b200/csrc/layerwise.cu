// layerwise.cu — the reference's LAYER_WISE schedules on the device: every
// layer its own launch, every intermediate through HBM (machine.py:418-459
// ConvFirst, 593-646 MBConv, 339-365 FFN; core.py:401-429 expand_network).
// It is the baseline the block-fusion kernels are measured against (the
// paper's fused-vs-unfused comparison) and makes
// execute_numeric(build_schedule(..., LAYER_WISE)) executable on the GPU.
//
//   ConvFirst   xc = conv(x) + b_conv         gconv_kernel (CUDA cores)
//               H  = phi(xc U + a)            tcgen05 GEMM (gemm.cu)
//               z  = H V + b + x              tcgen05 GEMM, residual epilogue
//   MBConv      h1 = phi(x W_exp + b_exp)     GEMM
//               h2 = phi(conv(h1) + b_conv)   gconv_kernel
//               g  = SE(h2)                   se_kernel (pool, squeeze, excite)
//               h2 = h2 * g                   gate_kernel
//               z  = h2 W_prj + b_prj + x     GEMM
//   FFN         H = phi(x U + a); z = H V + b  two GEMMs
#include <cuda.h>
#include <cuda_fp16.h>
#include <algorithm>
#include <cstdint>
#include <cstring>
#include "common.cuh"
#include "gemm.h"
#include "launch.h"
#include "plan.h"

namespace wl {

namespace {
constexpr int kLwHdr = 4096;

// grouped KS x KS conv, stride 1, zero pad KS/2, NHWC, C -> C with groups of T
// input channels (T = 8 or 1). CTA = (pixel range, slice of up to 64
// channels); warp = one 8-channel group (warp-uniform weights: shared-memory
// broadcasts), lane = pixel; the slice's fp32 weights [co][tap][t] staged in
// shared memory (<= 18 KB)
constexpr int kSlice = 64;
template <int KS, int T, int ACT>
__global__ void __launch_bounds__(256) gconv_kernel(const __half* __restrict__ x, const float* __restrict__ w,
                                                    const float* __restrict__ b, __half* __restrict__ y, int N, int H,
                                                    int W, int C) {
  constexpr int R = KS / 2, TAPS = KS * KS;
  __shared__ float s_w[kSlice * TAPS * T];
  const int c0 = blockIdx.y * kSlice;
  const int S8 = min(kSlice, C - c0) / 8;  // 8-channel groups in this slice (1..8)
  for (int i = threadIdx.x; i < S8 * 8 * TAPS * T; i += blockDim.x) s_w[i] = w[(size_t)c0 * TAPS * T + i];
  pdl_wait();
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpg = 8 / S8;                  // warps per channel group (S8 divides 8: C % 64 or C in {8,16,32})
  if (warp >= S8 * wpg) return;
  const int cl = warp % S8, c8 = c0 / 8 + cl;
  const int64_t M = (int64_t)N * H * W;
  const int64_t step = (int64_t)gridDim.x * wpg * 32;
  for (int64_t p = ((int64_t)blockIdx.x * wpg + warp / S8) * 32 + lane; p < M; p += step) {
    const int px = (int)(p % W), py = (int)((p / W) % H);
    const int64_t img = p / ((int64_t)W * H);
    float acc[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) acc[o] = __ldg(b + c8 * 8 + o);
    for (int dy = -R; dy <= R; ++dy) {
      const int iy = py + dy;
      if (iy < 0 || iy >= H) continue;
#pragma unroll
      for (int dx = -R; dx <= R; ++dx) {
        const int ix = px + dx;
        if (ix < 0 || ix >= W) continue;
        float in[8];
        unpack8(__ldg(reinterpret_cast<const uint4*>(x + ((img * H + iy) * W + ix) * C + c8 * 8)), in);
        const int tap = (dy + R) * KS + (dx + R);
#pragma unroll
        for (int o = 0; o < 8; ++o) {
          const float* wo = s_w + ((cl * 8 + o) * TAPS + tap) * T;
          if constexpr (T == 8) {
#pragma unroll
            for (int t = 0; t < 8; ++t) acc[o] = fmaf(wo[t], in[t], acc[o]);
          } else {
            acc[o] = fmaf(wo[0], in[o], acc[o]);
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < 8; ++o) acc[o] = act<ACT>(acc[o]);
    *reinterpret_cast<uint4*>(y + p * C + c8 * 8) = pack8(acc);
  }
  pdl_trigger();
}

// squeeze-excite gates of one image (machine.py:700-723): pool over the
// pixels, squeeze + ReLU, excite + sigmoid; one CTA per image. Pool: thread =
// (8-channel group, pixel lane of 8), fixed-order partial sums; squeeze: warp
// per output, lanes over the hidden channels (W_sq stored [sq][hid]).
constexpr int kSeThreads = 256;
constexpr int kSeSmemMax = 200 * 1024;
__global__ void __launch_bounds__(kSeThreads) se_kernel(const __half* __restrict__ h2, const __half* __restrict__ wsqt,
                                                        const float* __restrict__ bsq, const __half* __restrict__ wex,
                                                        const float* __restrict__ bex, float* __restrict__ gates,
                                                        int HW, int hid, int sq) {
  extern __shared__ float s_se[];  // pool[hid] | s[sq] | part[8][hid]
  float* pool = s_se;
  float* sv = pool + hid;
  float* part = sv + sq;
  const int img = blockIdx.x, H8 = hid / 8;
  pdl_wait();
  for (int i = threadIdx.x; i < H8 * 8; i += kSeThreads) {
    const int g = i % H8, pl = i / H8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int p = pl; p < HW; p += 8) {
      float v[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(h2 + ((size_t)img * HW + p) * hid) + g), v);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += v[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) part[pl * hid + g * 8 + k] = acc[k];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < hid; c += kSeThreads) {
    float a = 0.f;
#pragma unroll
    for (int pl = 0; pl < 8; ++pl) a += part[pl * hid + c];
    pool[c] = a / (float)HW;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int o = warp; o < sq; o += kSeThreads / 32) {
    float a = 0.f;
    for (int c = lane; c < hid; c += 32) a = fmaf(pool[c], __half2float(wsqt[(size_t)o * hid + c]), a);
#pragma unroll
    for (int m = 16; m; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
    if (lane == 0) sv[o] = fmaxf(a + bsq[o], 0.f);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < hid; c += kSeThreads) {
    float a = bex[c];
    for (int o = 0; o < sq; ++o) a = fmaf(sv[o], __half2float(wex[(size_t)o * hid + c]), a);
    gates[(size_t)img * hid + c] = act<kSigmoid>(a);
  }
  pdl_trigger();
}

__global__ void gate_kernel(__half* __restrict__ h2, const float* __restrict__ gates, int64_t HW, int hid,
                            int64_t total8) {
  pdl_wait();
  const int H8 = hid / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total8; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % H8);
    const int64_t img = (i / H8) / HW;
    float v[8];
    uint4* p = reinterpret_cast<uint4*>(h2) + i;
    unpack8(*p, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] *= gates[img * hid + c8 * 8 + k];
    *p = pack8(v);
  }
  pdl_trigger();
}

int64_t a128l(int64_t v) { return (v + 127) / 128 * 128; }

// ---------------------------------------------------------------- layouts
struct LwLayout {
  int64_t o_conv, o_bconv, o_a, o_b, o_ut, o_vt;  // ConvFirst / FFN
  int64_t o_bexp, o_wexp, o_wsq, o_bsq, o_wex, o_bex, o_wprj, o_bprj;  // MBConv
  int64_t total;
};
LwLayout lw_layout(const wl_block_desc& d) {
  LwLayout L;
  memset(&L, 0, sizeof(L));
  const int64_t C = d.c, hid = (int64_t)d.expansion * d.c, taps = (int64_t)d.ksize * d.ksize;
  int64_t o = 0;
  if (d.kind == WL_KIND_MBCONV) {
    const int64_t sq = d.se_sq;
    L.o_bexp = o; o += a128l(hid * 4);
    L.o_wexp = o; o += a128l(hid * C * 2);               // W_exp^T [hid][C]
    L.o_conv = o; o += a128l(hid * taps * d.group_width * 4);
    L.o_bconv = o; o += a128l(hid * 4);
    L.o_wsq = o; o += a128l(hid * sq * 2);               // W_sq^T [sq][hid]
    L.o_bsq = o; o += a128l(sq * 4);
    L.o_wex = o; o += a128l(sq * hid * 2);               // [sq][hid]
    L.o_bex = o; o += a128l(hid * 4);
    L.o_wprj = o; o += a128l(C * hid * 2);               // W_prj^T [C][hid]
    L.o_bprj = o; o += a128l(C * 4);
  } else {
    if (d.kind == WL_KIND_CONVFIRST) {
      L.o_conv = o; o += a128l(C * taps * d.group_width * 4);
      L.o_bconv = o; o += a128l(C * 4);
    }
    L.o_a = o; o += a128l(hid * 4);
    L.o_b = o; o += a128l(C * 4);
    L.o_ut = o; o += a128l(hid * C * 2);                 // U^T [hid][C]
    L.o_vt = o; o += a128l(C * hid * 2);                 // V^T [C][hid]
  }
  L.total = o;
  return L;
}
void put_f(uint8_t* base, int64_t off, const float* src, int64_t n) { memcpy(base + off, src, (size_t)n * 4); }
void put_tr(uint8_t* base, int64_t off, const float* src, int K, int N) {  // (K, N) -> [N][K] fp16
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) put_h(base, off + ((int64_t)n * K + k) * 2, src[(int64_t)k * N + n]);
}
void put_hv(uint8_t* base, int64_t off, const float* src, int64_t n) {
  for (int64_t i = 0; i < n; ++i) put_h(base, off + i * 2, src[i]);
}

int lw_validate(const wl_block_desc& d) {
  if (d.kind != WL_KIND_CONVFIRST && d.kind != WL_KIND_MBCONV && d.kind != WL_KIND_FFN)
    return set_error(WL_EUNSUPPORTED, "layer-wise execution covers ConvFirst, MBConv and FFN blocks");
  if (d.dtype != WL_DTYPE_F16) return set_error(WL_EUNSUPPORTED, "layer-wise execution is fp16");
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c < 8 || d.c % 8) return set_error(WL_EUNSUPPORTED, "C % 8 == 0 required");
  if (d.expansion < 1) return set_error(WL_EINVAL, "expansion must be at least 1");
  if (d.kind == WL_KIND_FFN) return WL_OK;
  // the reference's layer-wise schedules are stride 1 (machine.py:423-425, 599-600)
  if (d.stride != 1) return set_error(WL_EUNSUPPORTED, "the layer-wise schedule models stride-1 blocks only");
  if (d.k != d.c) return set_error(WL_EINVAL, "stride-1 blocks keep their channel count");
  if (d.group_width != 8 && d.group_width != 1)
    return set_error(WL_EUNSUPPORTED, "layer-wise grouped conv: T = 8 or 1");
  if (d.ksize != 3 && !(d.ksize == 7 && d.group_width == 1)) return set_error(WL_EUNSUPPORTED, "3x3 or 7x7 dw");
  if (d.kind == WL_KIND_CONVFIRST && d.norm != WL_NORM_NONE)
    return set_error(WL_EUNSUPPORTED, "the layer-wise schedule is the reference's (no LayerNorm)");
  if (d.kind == WL_KIND_MBCONV && (d.se_sq < 1 || (d.expansion * d.c) % 8))
    return set_error(WL_EUNSUPPORTED, "MBConv layer-wise: hidden % 8 == 0, se_sq >= 1");
  if (d.kind == WL_KIND_MBCONV && (9 * d.expansion * d.c + d.se_sq) * 4 > kSeSmemMax)
    return set_error(WL_EUNSUPPORTED, "MBConv layer-wise: SE partial sums exceed shared memory");
  return WL_OK;
}
int lw_wc(const wl_block_desc& d) {
  if (d.kind == WL_KIND_FFN) return kFfnFamily.weight_count(d);
  return d.kind == WL_KIND_MBCONV ? kMbFamily.weight_count(d) : kCfFamily.weight_count(d);
}
int64_t lw_wn(const wl_block_desc& d, int i) {
  if (d.kind == WL_KIND_FFN) return kFfnFamily.weight_numel(d, i);
  return d.kind == WL_KIND_MBCONV ? kMbFamily.weight_numel(d, i) : kCfFamily.weight_numel(d, i);
}
int64_t lw_pb(const wl_block_desc& d) { return lw_layout(d).total; }
int lw_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  const LwLayout L = lw_layout(d);
  memset(out, 0, (size_t)L.total);
  const int C = d.c, hid = d.expansion * d.c, taps = d.ksize * d.ksize;
  if (d.kind == WL_KIND_MBCONV) {
    // w_exp (C,hid), b_exp, w_conv (hid,k,k,T), b_conv, w_sq (hid,sq), b_sq, w_ex (sq,hid), b_ex, w_prj (hid,C), b_prj
    put_f(out, L.o_bexp, w[1], hid);
    put_tr(out, L.o_wexp, w[0], C, hid);
    put_f(out, L.o_conv, w[2], (int64_t)hid * taps * d.group_width);
    put_f(out, L.o_bconv, w[3], hid);
    put_tr(out, L.o_wsq, w[4], hid, d.se_sq);
    put_f(out, L.o_bsq, w[5], d.se_sq);
    put_hv(out, L.o_wex, w[6], (int64_t)d.se_sq * hid);
    put_f(out, L.o_bex, w[7], hid);
    put_tr(out, L.o_wprj, w[8], hid, C);
    put_f(out, L.o_bprj, w[9], C);
    return WL_OK;
  }
  int o = 0;
  if (d.kind == WL_KIND_CONVFIRST) {  // w_conv (C,k,k,T), b_conv, u, a, v, b
    put_f(out, L.o_conv, w[0], (int64_t)C * taps * d.group_width);
    put_f(out, L.o_bconv, w[1], C);
    o = 2;
  }
  put_tr(out, L.o_ut, w[o + 0], C, hid);
  put_f(out, L.o_a, w[o + 1], hid);
  put_tr(out, L.o_vt, w[o + 2], hid, C);
  put_f(out, L.o_b, w[o + 3], C);
  return WL_OK;
}
int64_t lw_ws(const wl_block_desc& d) {
  const int64_t M = (int64_t)d.n * d.h * d.w, C = d.c, hid = (int64_t)d.expansion * d.c;
  if (d.kind == WL_KIND_MBCONV) return kLwHdr + 2 * a128l(M * hid * 2) + a128l((int64_t)d.n * hid * 4);
  if (d.kind == WL_KIND_CONVFIRST) return kLwHdr + a128l(M * C * 2) + a128l(M * hid * 2);
  return kLwHdr + a128l(M * hid * 2);
}

using GconvK = void (*)(const __half*, const float*, const float*, __half*, int, int, int, int);
template <int ACT>
GconvK gconv_pick(int ks, int t) {
  if (t == 8) return gconv_kernel<3, 8, ACT>;
  return ks == 7 ? gconv_kernel<7, 1, ACT> : gconv_kernel<3, 1, ACT>;
}
GconvK gconv_for(int ks, int t, int act) {
  switch (act) {
    case kRelu: return gconv_pick<kRelu>(ks, t);
    case kSilu: return gconv_pick<kSilu>(ks, t);
    case kGelu: return gconv_pick<kGelu>(ks, t);
    case kSigmoid: return gconv_pick<kSigmoid>(ks, t);
  }
  return gconv_pick<kIdentity>(ks, t);
}
int gconv_run(const wl_block_desc& d, int C, const __half* x, const float* w, const float* b, __half* y, int act,
              cudaStream_t st) {
  const int slices = (C + kSlice - 1) / kSlice;
  const int ppc = 8 / (std::min(C, kSlice) / 8) * 32;  // pixels per CTA iteration
  const int64_t M = (int64_t)d.n * d.h * d.w;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((M + ppc - 1) / ppc, kNumSMs * 8 / slices));
  void (*k)(const __half*, const float*, const float*, __half*, int, int, int, int) =
      gconv_for(d.ksize, d.group_width, act);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gx, slices);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return check_cuda(cudaLaunchKernelEx(&cfg, k, x, w, b, y, d.n, d.h, d.w, C), "gconv launch");
}

int lw_fwd(const wl_block_desc& d, const void* xv, const void* p, void* zv, void* ws, cudaStream_t st) {
  const LwLayout L = lw_layout(d);
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(p);
  const __half* x = reinterpret_cast<const __half*>(xv);
  __half* z = reinterpret_cast<__half*>(zv);
  const int64_t M = (int64_t)d.n * d.h * d.w;
  const int C = d.c, hid = d.expansion * d.c;
  uint8_t* w0 = reinterpret_cast<uint8_t*>(ws) + kLwHdr;
  auto F = [&](int64_t off) { return reinterpret_cast<const float*>(pk + off); };
  if (d.kind == WL_KIND_MBCONV) {
    __half* h1 = reinterpret_cast<__half*>(w0);
    __half* h2 = reinterpret_cast<__half*>(w0 + a128l(M * hid * 2));
    float* gates = reinterpret_cast<float*>(w0 + 2 * a128l(M * hid * 2));
    GemmEpi e1;
    e1.bias = F(L.o_bexp);
    e1.act = d.act;
    if (int e = gemm_run(x, (int)M, C, C, pk + L.o_wexp, hid, C, h1, hid, e1, st)) return e;
    if (int e = gconv_run(d, hid, h1, F(L.o_conv), F(L.o_bconv), h2, d.act, st)) return e;
    if (int e = launch_pdl(se_kernel, d.n, kSeThreads, (size_t)(9 * hid + d.se_sq) * 4, st, "se launch",
                           (const __half*)h2, reinterpret_cast<const __half*>(pk + L.o_wsq), F(L.o_bsq),
                           reinterpret_cast<const __half*>(pk + L.o_wex), F(L.o_bex), gates, d.h * d.w, hid, d.se_sq))
      return e;
    const int64_t t8 = M * hid / 8;
    if (int e = launch_pdl(gate_kernel, (int)std::min<int64_t>((t8 + 255) / 256, kNumSMs * 16), 256, 0, st,
                           "gate launch", h2, (const float*)gates, (int64_t)d.h * d.w, hid, t8))
      return e;
    GemmEpi e2;
    e2.bias = F(L.o_bprj);
    e2.res = x;
    e2.ldr = C;
    return gemm_run(h2, (int)M, hid, hid, pk + L.o_wprj, C, hid, z, C, e2, st);
  }
  const __half* src = x;
  __half* hb;
  if (d.kind == WL_KIND_CONVFIRST) {
    __half* xc = reinterpret_cast<__half*>(w0);
    hb = reinterpret_cast<__half*>(w0 + a128l(M * C * 2));
    if (int e = gconv_run(d, C, x, F(L.o_conv), F(L.o_bconv), xc, kIdentity, st)) return e;  // machine.py:496
    src = xc;
  } else {
    hb = reinterpret_cast<__half*>(w0);
  }
  GemmEpi e1;
  e1.bias = F(L.o_a);
  e1.act = d.act;
  if (int e = gemm_run(src, (int)M, C, C, pk + L.o_ut, hid, C, hb, hid, e1, st)) return e;
  GemmEpi e2;
  e2.bias = F(L.o_b);
  if (d.kind == WL_KIND_CONVFIRST) {
    e2.res = x;
    e2.ldr = C;
  }
  return gemm_run(hb, (int)M, hid, hid, pk + L.o_vt, C, hid, z, C, e2, st);
}
int lw_init() {
  if (int e = gemm_init()) return e;
  return check_cuda(cudaFuncSetAttribute(se_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSeSmemMax),
                    "cudaFuncSetAttribute(se)");
}
}  // namespace

// the grouped conv on its own (the wide ConvFirst route, cnx.cu: cf_wide_fwd)
int lw_gconv(const wl_block_desc& d, int C, const void* x, const float* w, const float* b, void* y, int act,
             cudaStream_t st) {
  return gconv_run(d, C, reinterpret_cast<const __half*>(x), w, b, reinterpret_cast<__half*>(y), act, st);
}

int lw_launches(const wl_block_desc& d) {
  if (d.kind == WL_KIND_MBCONV) return 5;
  return d.kind == WL_KIND_CONVFIRST ? 3 : 2;
}

const Family kLayerwiseFamily = {lw_validate, lw_wc, lw_wn, lw_pb, lw_pack, lw_ws, lw_fwd, lw_init};

}  // namespace wl
