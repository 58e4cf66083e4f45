// mbconv.cu — MBConv + squeeze-excite on sm_100a (core.py:112-122; fused
// schedule machine.py:649-733; layer-wise numerics machine.py:593-646).
//
// Two launches per block; the expanded activation never reaches HBM by
// design — the conv output h2 passes between the launches through the
// 126 MB L2 (the tensor machine's GLOBAL tier, machine.py:667-687):
//   front : one CTA per (image group, hidden range). Whole image(s) stacked in
//           a flat padded layout (row pitch >= W+1: the left pad column of row
//           y+1 doubles as the right pad of row y), so every 3x3 tap is a
//           constant shift of the flat index and an M=128 conv tile is 16
//           consecutive 8-pixel core-matrix rows. Per hidden chunk:
//             expand (SS MMA, x smem x U_j)                 -> TMEM E (x2)
//             E + b_exp, phi (packed half), pads -> 0       -> smem h1 planes
//             grouped 3x3 conv (block-diagonal MMAs T=8, CUDA cores T=1)
//             + b_conv, phi [-> BlurPool 3x3 stride 2]      -> smem staging
//             staging -> h2 (TMA store), column sums -> pool (deterministic)
//           The last CTA of an image group (threadfence + counter) runs the
//           squeeze-excite once: gates = sigmoid(relu(pool W_sq + b_sq) W_ex + b_ex).
//   back  : one CTA per (128 consecutive output pixels, output-channel range):
//           h2 tiles arrive by TMA, are gated in shared memory (packed half),
//           the projection accumulates in TMEM; z = Z + b_prj (+ x, stride 1).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include "common.cuh"
#include "plan.h"

namespace wl {

struct MbFrontArgs {
  int C, hid, sq, HR, HC, nch;  // nch: chunks per hidden range
  int T8, stride;
  int H, W, Wp, imgs, groups;
  int total_rows, n_et, n_ct, conv_base, flat_h1, x_alloc;  // conv_base = Wp + 1
  int Ho, Wo, ranges;
  // row bands: a cluster pair splits ONE image by output rows when its whole
  // tile does not fit (H/Ho above are then the band's conv / output rows);
  // the pair meets once, to sum the SE pool over DSMEM
  int bands, H_img, Ho_img;
  int P_out, P_full;       // dense output / full-res pixels per CTA
  int st_rows, st_stores;  // TMA store box rows, stores per chunk
  int e_bufs, c_bufs, h1_bufs, x_tmem;
  int h1_bytes, st_bytes, full_bytes;
  int hdr_bytes, chunk_bytes, u_bytes;  // per-range hdr = [b_exp | b_conv | (T1) convw fp32 [9][HR]]
  int o_bconv, o_convw;
  int o_wsq, o_bsq, o_wex, o_bex, se_bytes;  // SE section (fp32) at the front of the blob
  int s_x, s_h1, s_st, s_full, s_hdr, s_ring, s_pool, s_map, s_bar, smem;
  int ring_stages;
  int t_x, t_e, t_c, tmem_cols, s_h1b;
  const uint8_t* wpack;  // front blob: [SE][range hdrs][chunks]
  float* pool;           // (n, hid) spatial mean
  float* gates;          // (n, hid) SE gates
  int* counters;         // (groups) zero-initialised arrival counters
  long long* trace;      // debug: per-phase clock64 stamps of CTA 0 (null = off)
  // fused projection (one launch per block): gated h2 (re-read from L2) x W_prj
  int fused, K, n_pt, HCb, nchb, vchunk_bytes, residual, sa, SQP;
  // bulk mode (fused, single-store staging): h2 lives chunk-major in global,
  // [group][hidden/8][P_out][8], so every conv chunk leaves and every
  // projection chunk (HCb = lcm(HC, 64) channels) returns as ONE bulk copy
  int bulk, a_stage_b;
  int xsw;  // x staged as 128-byte-swizzled pixel rows of 64 channels (one 128 B TMA row per pixel)
  int se_pref, se_off;  // squeeze-excite weights prefetched into the tail of the (then idle) weight ring
  // z staged in shared memory (128B-swizzled 64-channel rows, over the dead SE
  // weights): residual rows arrive by TMA during the projection, z leaves by TMA
  int zst, zst_rows;
  __half* h2;
  int s_pa, s_pv, s_gate, t_z;
  const uint8_t* wback;  // back blob: [b_prj fp32][V chunks]
  const __half* x;       // residual source (n, H, W, C)
  __half* z;             // (n, Ho, Wo, K)
};

struct MbBackArgs {
  int hid, K, KR, HCb, nchb, stride;
  int P, pix_per_img;
  int kranges, residual;
  int vchunk_bytes, o_bprj;
  int s_a, s_gate, s_ring, s_bar, smem, ring_stages;
  int t_z, tmem_cols;
  const uint8_t* wpack;  // back blob: [b_prj fp32][V chunks per (krange, j)]
  const float* gates;
  const __half* x;  // residual (n, H, W, K)
  __half* z;        // (n, Ho, Wo, K)
};

namespace mbk {
constexpr int kThreads = 640;
struct FrontBars {
  uint64_t hdr_full, x_full;
  uint64_t w_full[4], w_empty[4];
  uint64_t e_full[2], c_full[2], c_empty[2];
  uint64_t h1_full[2], h1_empty[2], x_ready;
  uint64_t pa_full[4], pa_ready[4], pa_empty[4], pv_full[3], pv_empty[3], z_full;
  uint64_t se_full, res_full;
  uint32_t tmem_base;
  int last;
};
struct BackBars {
  uint64_t a_full[2], a_empty[2], a_ready[2];
  uint64_t v_full[4], v_empty[4];
  uint64_t z_full;
  uint32_t tmem_base;
};
}  // namespace mbk

// flat position f holds a real pixel (not a pad row / pad column)
__device__ __forceinline__ bool mb_real(int f, int Wp, int W, int H, int total_rows) {
  const int row = f / Wp, col = f - row * Wp;
  return col >= 1 && col <= W && row < total_rows - 1 && (row % (H + 1)) != 0;
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
// thread-block-cluster pair (two CTAs split one image group's hidden channels)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t peer_smem(const void* p, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
__device__ __forceinline__ void st_peer_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_peer_v4(uint32_t addr, const uint32_t* v) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3])
               : "memory");
}

__device__ __forceinline__ void tma_store_3d(const void* tmap, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// staging offset (bytes) of 8-channel group g of dense pixel p: stores of
// st_rows rows, each [HC/8][st_rows][8] (the TMA store box)
__device__ __forceinline__ int st_off(int p, int g, int st_rows, int groups8) {
  const int k = p / st_rows, r = p - k * st_rows;
  return ((k * groups8 + g) * st_rows + r) * 16;
}

#define WL_TRACE(slot)                                                  \
  do {                                                                  \
    if (a.trace && blockIdx.x == 0) a.trace[(slot)] = clock64();        \
  } while (0)

// SE pool of one chunk when a single image's h2 staging spans several store
// blocks [k][G8][st_rows][8]: warps take (channel group, block) pairs and walk
// contiguous rows; the per-block partials meet in the (idle until the squeeze)
// pool-vector scratch in a fixed order. Out of line: the common single-block
// path keeps its register allocation.
__device__ __noinline__ void mb_pool_split_stores(const MbFrontArgs& a, uint8_t* smem, const uint8_t* s_st, float* s_pool,
                                                   int j, int HC, int G8, int wi, int lane, int tid) {
  float* scr = reinterpret_cast<float*>(smem + a.s_gate) + a.hid;
  const int i = lane >> 2, w = lane & 3;
  for (int pr = wi; pr < G8 * a.st_stores; pr += 8) {
    const int g = pr % G8, k = pr / G8;
    const uint8_t* base = s_st + ((size_t)(k * G8 + g) * a.st_rows) * 16 + w * 4;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int r = i;
    for (; r + 8 < a.st_rows; r += 16) {
      const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(base + r * 16));
      const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(base + (r + 8) * 16));
      s0 += f0.x;
      s1 += f0.y;
      s2 += f1.x;
      s3 += f1.y;
    }
    if (r < a.st_rows) {
      const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(base + r * 16));
      s0 += f0.x;
      s1 += f0.y;
    }
    s0 += s2;
    s1 += s3;
#pragma unroll
    for (int m = 4; m < 32; m <<= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, m);
      s1 += __shfl_xor_sync(0xffffffffu, s1, m);
    }
    if (i == 0) {
      scr[k * HC + g * 8 + w * 2] = s0;
      scr[k * HC + g * 8 + w * 2 + 1] = s1;
    }
  }
  asm volatile("bar.sync 1, 256;" ::: "memory");
  for (int c = tid; c < HC; c += 256) {
    float acc = 0.f;
    for (int k = 0; k < a.st_stores; ++k) acc += scr[k * HC + c];
    s_pool[j * HC + c] += acc;
  }
}

// T8 / S2 / FUSED are compile-time so each instantiation carries only the
// code its configuration executes (a smaller hot instruction footprint)
template <int ACT, bool T8, bool S2, bool FUSED>
__global__ void __launch_bounds__(mbk::kThreads, 1)
    mb_front_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_h2,
                    const __grid_constant__ CUtensorMap tmap_h2l, const __grid_constant__ MbFrontArgs a) {
  using namespace mbk;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_x = smem + a.s_x;
  uint8_t* s_h1 = smem + a.s_h1;
  uint8_t* s_st = smem + a.s_st;      // final h2 staging (dense output pixels)
  uint8_t* s_full = smem + a.s_full;  // stride 2: full-resolution staging
  uint8_t* s_hdr = smem + a.s_hdr;
  uint8_t* s_ring = smem + a.s_ring;
  float* s_pool = reinterpret_cast<float*>(smem + a.s_pool);  // [imgs][HR]
  int* s_cmap = reinterpret_cast<int*>(smem + a.s_map);            // conv tile row -> dense pixel / -1
  uint8_t* s_emap = smem + a.s_map + a.n_ct * 128 * 4;              // expand tile row -> real?
  FrontBars& B = *reinterpret_cast<FrontBars*>(smem + a.s_bar);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int group = blockIdx.x / a.ranges, range = blockIdx.x % a.ranges;
  if ((smem_u32(smem) & 1023) != 0) __trap();  // swizzled tiles need 1024-byte alignment
  // row bands (a.bands == 2): CTA pair (group = 2 n + band) splits image n;
  // the band's first conv row c0 and the image row of its first x row xr0
  const int band = a.bands > 1 ? group % 2 : 0;
  const int n0 = a.bands > 1 ? group / 2 : group * a.imgs;
  const int c0 = !band ? 0 : (a.stride == 1 ? a.H : 2 * a.Ho - 1);
  const int xr0 = c0 - 1;
  const int h0 = range * a.HR;
  const int S = a.ring_stages, HC = a.HC, nch = a.nch, G8 = HC / 8;
  // T=8 with two or more conv tiles: warp 3 issues the odd tiles' conv MMAs so
  // the single issuing thread (which shares its SMSP with busy epilogue warps)
  // is not the bottleneck of the 16-wide grouped-conv instructions
  // conv (tile, pair) items are dealt round-robin to NIS issuing threads
  // (warps 1, 3, 2): warp 1 also issues the expansions
  // T=8: warp 1 issues only the expansions; the grouped conv's (tile, pair)
  // items go round-robin to NIS dedicated issuing threads (warps 3, 2), so the
  // conv never queues behind an expansion waiting for its weight chunk
  const int NIS = T8 ? min(2, a.n_ct * (HC / 16)) : 1;
  const int img_flat = (a.bands > 1 ? a.H + 2 : a.H + 1) * a.Wp;
  const int x_valid = a.imgs * img_flat;
  if (threadIdx.x == 0) WL_TRACE(0);
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {  // plan snapshot for the trace reader
    a.trace[14] = a.se_pref * 10000 + a.sa * 1000 + a.ring_stages * 100 + a.h1_bufs * 10 + a.e_bufs;
    a.trace[15] = a.c_bufs * 100000 + a.x_tmem * 10000 + a.HC * 10 + a.n_pt;
  }

  for (int i = threadIdx.x; i < a.h1_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(s_h1)[i] = make_uint4(0, 0, 0, 0);
  if (a.h1_bufs > 1 && !a.x_tmem)
    for (int i = threadIdx.x; i < G8 * a.flat_h1; i += blockDim.x)
      reinterpret_cast<uint4*>(smem + a.s_h1b)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < a.imgs * a.HR; i += blockDim.x) s_pool[i] = 0.f;
  {
    const int conv_end = (a.total_rows - 1) * a.Wp;
    for (int i = threadIdx.x; i < a.n_ct * 128; i += blockDim.x) {
      const int f = a.conv_base + i;
      int p = -1;
      if (f < conv_end && mb_real(f, a.Wp, a.W, a.H, a.total_rows)) {
        const int row = f / a.Wp, img = row / (a.H + 1);
        p = (img * a.H + row - img * (a.H + 1) - 1) * a.W + (f - row * a.Wp - 1);
      }
      s_cmap[i] = p;
    }
    for (int f = threadIdx.x; f < a.n_et * 128; f += blockDim.x) {
      bool real;
      if (a.bands > 1) {  // halo rows are real image rows unless past the image border
        const int row = f / a.Wp, col = f - row * a.Wp;
        real = f < x_valid && col >= 1 && col <= a.W && xr0 + row >= 0 && xr0 + row < a.H_img;
      } else {
        real = f < x_valid && mb_real(f, a.Wp, a.W, a.H, a.total_rows);
      }
      s_emap[f] = real ? 1 : 0;
    }
  }
  {
    const int tail = a.x_alloc - x_valid, planes = a.C / 8;
    for (int i = threadIdx.x; i < planes * tail; i += blockDim.x) {
      const int pl = i / tail, f = x_valid + i % tail;
      *reinterpret_cast<uint4*>(s_x + ((size_t)pl * a.x_alloc + f) * 16) = make_uint4(0, 0, 0, 0);
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&B.hdr_full, 1);
    mbar_init(&B.x_full, 1);
    for (int i = 0; i < S; ++i) {
      mbar_init(&B.w_full[i], 1);
      mbar_init(&B.w_empty[i], T8 ? NIS + 1 : 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.e_full[i], 1);
      mbar_init(&B.c_full[i], NIS);
      mbar_init(&B.c_empty[i], 256);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.h1_full[i], 256);
      mbar_init(&B.h1_empty[i], T8 ? NIS : 256);
    }
    mbar_init(&B.x_ready, 256);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&B.pa_full[i], 1);
      mbar_init(&B.pa_ready[i], 256);
      mbar_init(&B.pa_empty[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&B.pv_full[i], 1);
      mbar_init(&B.pv_empty[i], 1);
    }
    mbar_init(&B.z_full, 1);
    mbar_init(&B.se_full, 1);
    mbar_init(&B.res_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_n(&B.tmem_base, a.tmem_cols);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // cluster pairs exchange partial pools / squeezes / Z over DSMEM: a CTA may
  // only write its peer's shared memory once the peer is known to have
  // started (compute-sanitizer racecheck flagged the unsynchronised first
  // store, profiles/r02_sanitizer.txt)
  if (FUSED && (a.ranges == 2 || a.bands == 2)) cluster_sync_all();
  if (FUSED) pdl_trigger();  // single-wave persistent grid: let the next kernel stage its prologue
  pdl_wait();
  const uint32_t tmem = B.tmem_base;
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {  // per-CTA span (global ns): start
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.trace[512 + 2 * blockIdx.x] = (long long)gt;
  }

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmap_x);
      WL_TRACE(1);
      mbar_arrive_expect_tx(&B.hdr_full, a.hdr_bytes);
      bulk_g2s(s_hdr, a.wpack + a.se_bytes + (size_t)range * a.hdr_bytes, a.hdr_bytes, &B.hdr_full);
      const int planes = a.C / 8;
      if (a.xsw) {
        // 64-channel blocks, box {64 ch, Wp, H+1, imgs}: 128-byte rows per
        // pixel (SWIZZLE_128B) — 8x fewer TMA rows than 16-byte planes
        mbar_arrive_expect_tx(&B.x_full, img_flat * 128 * (a.C / 64) * a.imgs);
        for (int cb = 0; cb < a.C / 64; ++cb)
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
              "%4, %5}], [%6];" ::"r"(smem_u32(s_x + (size_t)cb * a.n_et * 128 * 128)),
              "l"(&tmap_x), "r"(cb * 64), "r"(-1), "r"(xr0), "r"(n0), "r"(smem_u32(&B.x_full))
              : "memory");
      } else {
        // the whole x tile in ONE tensor-map load: box {8 ch, Wp, H+1, imgs, C/8}
        // lands as [plane][image][row][col][8] (plane stride = x_alloc rows)
        mbar_arrive_expect_tx(&B.x_full, img_flat * 16 * planes * a.imgs);
        tma_load_5d(s_x, &tmap_x, 0, -1, xr0, n0, 0, &B.x_full);
      }
      const uint8_t* chunks = a.wpack + a.se_bytes + (size_t)a.ranges * a.hdr_bytes;
      for (int j = 0; j < nch; ++j) {
        const int slot = j % S, use = j / S;
        mbar_wait(&B.w_empty[slot], (use & 1) ^ 1);
        if (j < 10) WL_TRACE(16 + 8 * j + 7);
        mbar_arrive_expect_tx(&B.w_full[slot], a.chunk_bytes);
        bulk_g2s(s_ring + slot * a.chunk_bytes, chunks + (size_t)(range * nch + j) * a.chunk_bytes, a.chunk_bytes,
                 &B.w_full[slot]);
      }
      if (FUSED && a.se_pref) {
        // squeeze-excite weights into the weight ring once its last chunks
        // are consumed: they land while the final conv epilogue runs
        for (int j = nch - S; j < nch; ++j)
          if (j >= 0) mbar_wait(&B.w_empty[j % S], (j / S) & 1);
        mbar_arrive_expect_tx(&B.se_full, a.se_bytes);
        bulk_g2s(smem + a.se_off, a.wpack, a.se_bytes, &B.se_full);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_e = make_idesc_f16(128, HC);
      const uint32_t idesc_c = make_idesc_f16(128, 16);
      const uint32_t x0 = smem_u32(s_x), ring0 = smem_u32(s_ring);
      mbar_wait(&B.x_full, 0);
      if (a.x_tmem) mbar_wait(&B.x_ready, 0);
      WL_TRACE(2);
      // ring positions as counters (see the conv issuers)
      int x_slot = 0, x_sph = 0, x_eb = 0;  // the next expansion's weight stage, its phase, its E buffer
      auto issue_expand = [&](int j) {  // called for j = 0, 1, 2, ... in order
        const int slot = x_slot, eb = x_eb;
        if (j < 20) WL_TRACE(232 + j);
        mbar_wait(&B.w_full[slot], x_sph & 1);
        if (++x_slot == S) x_slot = 0, ++x_sph;
        if (++x_eb == a.e_bufs) x_eb = 0;
        WL_TRACE(16 + 8 * j + 0);
        tc_fence_after();
        const uint32_t ub = ring0 + slot * a.chunk_bytes;
        const uint64_t b_base = make_sdesc(ub, HC * 16, 128);
        for (int t = 0; t < a.n_et; ++t) {
          const uint32_t d = tmem + a.t_e + (eb * a.n_et + t) * HC;
          if (a.x_tmem) {  // A = x tile in TMEM: only B streams from shared memory
            for (int kk = 0; kk < a.C / 16; ++kk)
              mma_ts(d, tmem + a.t_x + t * (a.C / 2) + kk * 8, b_base + (uint64_t)(kk * 2 * HC), idesc_e, kk > 0);
          } else {
            const uint64_t a_base = make_sdesc(x0 + t * 128 * 16, a.x_alloc * 16, 128);
            for (int kk = 0; kk < a.C / 16; ++kk)
              mma_ss(d, a_base + (uint64_t)(kk * 2 * a.x_alloc), b_base + (uint64_t)(kk * 2 * HC), idesc_e, kk > 0);
          }
        }
        mma_commit(&B.e_full[eb]);
      };
      issue_expand(0);
      int m_slot = 0, m_hb = 0, m_hph = 0;  // chunk j's weight stage, h1 buffer and its phase
      int d_hb = 0, d_hph = 0;             // the same for chunk jd = j + 1 - e_bufs (once jd >= 0)
      for (int j = 0; j < nch; ++j) {
        const int slot = m_slot, hb = m_hb, hph = m_hph;
        if (++m_slot == S) m_slot = 0;
        if (++m_hb == a.h1_bufs) m_hb = 0, ++m_hph;
        if (T8) {
          // expansion j+1 reuses the E buffer of chunk j+1-e_bufs: wait for its drain
          const int jd = j + 1 - a.e_bufs;
          if (j + 1 < nch) {
            if (jd >= 0) {
              mbar_wait(&B.h1_full[d_hb], d_hph & 1);
              if (++d_hb == a.h1_bufs) d_hb = 0, ++d_hph;
            }
            issue_expand(j + 1);
          }
          mma_commit(&B.w_empty[slot]);
          continue;
        }
        if (a.e_bufs == 1) mbar_wait(&B.h1_full[hb], hph & 1);  // E of chunk j consumed
        if (j + 1 < nch) issue_expand(j + 1);
        if (T8) {
          const int cb = j % a.c_bufs;
          if (a.e_bufs != 1) mbar_wait(&B.h1_full[hb], hph & 1);
          if (j >= a.c_bufs) mbar_wait(&B.c_empty[cb], ((j / a.c_bufs) & 1) ^ 1);
          WL_TRACE(16 + 8 * j + 1);
          tc_fence_after();
          // descriptors advance by constant 16-byte steps from the (dy, dx) = (-1, -1) tap
          const uint32_t h1a = smem_u32(hb ? smem + a.s_h1b : s_h1);
          const uint64_t a_base = make_sdesc(h1a + (a.conv_base - a.Wp - 1) * 16, a.flat_h1 * 16, 128);
          // block-diagonal B tiles, compact: entry e = pr*9+tap keeps its two 8x8
          // diagonal blocks at Z -/+ (e+1)*128 around one shared zero block Z,
          // addressed with LBO = SBO = (e+1)*128 (both off-diagonal blocks hit Z)
          const int E = (HC / 16) * 9;
          const uint32_t zaddr = ring0 + slot * a.chunk_bytes + a.u_bytes + E * 128;
          const uint64_t b_base = make_sdesc(zaddr - 128, 128, 128);
          const uint64_t b_step = (8ull << 16) + (8ull << 32) - 8ull;
          for (int k = 0; k < a.n_ct * (HC / 16); k += NIS) {
            const int t = k / (HC / 16), pr = k - t * (HC / 16);
            {
              const uint32_t d = tmem + a.t_c + (cb * a.n_ct + t) * HC + 16 * pr;
              const uint64_t ap = a_base + (uint64_t)(2 * pr * a.flat_h1 + t * 128);
              // incremental descriptors: one 64-bit add each between MMAs keeps
              // the single issuing thread off the critical path
              uint64_t ad = ap, bd = b_base + (uint64_t)(pr * 9) * b_step;
#pragma unroll
              for (int tap = 0; tap < 9; ++tap) {
                mma_ss(d, ad, bd, idesc_c, tap > 0);
                ad += (tap % 3 == 2) ? (uint64_t)(a.Wp - 2) : 1ull;
                bd += b_step;
              }
            }
          }
          mma_commit(&B.c_full[cb]);
          mma_commit(&B.h1_empty[hb]);
          WL_TRACE(16 + 8 * j + 2);
        }
        mma_commit(&B.w_empty[slot]);
      }
    }
  } else if (warp == 3 || warp == 2) {
    const int isx = warp == 3 ? 0 : 1;  // conv issuer index
    if (T8 && isx < NIS && lane == 0) {
      const uint32_t idesc_c = make_idesc_f16(128, 16);
      const uint32_t ring0 = smem_u32(s_ring);
      // ring positions as counters (an integer division is a MUFU.RCP queued
      // behind the epilogues' SiLU)
      const int npr = HC / 16;
      int slot = 0, hb = 0, cb = 0, hph = 0, cph = 0;
      for (int j = 0; j < nch; ++j) {
        mbar_wait(&B.h1_full[hb], hph & 1);  // h1 ready implies the chunk's weights landed
        if (j >= a.c_bufs) mbar_wait(&B.c_empty[cb], (cph & 1) ^ 1);
        if (isx == 0) WL_TRACE(16 + 8 * j + 1);
        tc_fence_after();
        const uint32_t h1a = smem_u32(hb ? smem + a.s_h1b : s_h1);
        const uint64_t a_base = make_sdesc(h1a + (a.conv_base - a.Wp - 1) * 16, a.flat_h1 * 16, 128);
        const int E = (HC / 16) * 9;
        const uint32_t zaddr = ring0 + slot * a.chunk_bytes + a.u_bytes + E * 128;
        const uint64_t b_base = make_sdesc(zaddr - 128, 128, 128);
        const uint64_t b_step = (8ull << 16) + (8ull << 32) - 8ull;
        int t = 0, pr = isx;  // k = t * npr + pr
        while (pr >= npr) pr -= npr, ++t;
        for (int k = isx; k < a.n_ct * npr; k += NIS) {
          {
            const uint32_t d = tmem + a.t_c + (cb * a.n_ct + t) * HC + 16 * pr;
            uint64_t ad = a_base + (uint64_t)(2 * pr * a.flat_h1 + t * 128), bd = b_base + (uint64_t)(pr * 9) * b_step;
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
              mma_ss(d, ad, bd, idesc_c, tap > 0);
              ad += (tap % 3 == 2) ? (uint64_t)(a.Wp - 2) : 1ull;
              bd += b_step;
            }
          }
          pr += NIS;
          while (pr >= npr) pr -= npr, ++t;
        }
        mma_commit(&B.c_full[cb]);
        mma_commit(&B.h1_empty[hb]);
        mma_commit(&B.w_empty[slot]);
        if (isx == 0) WL_TRACE(16 + 8 * j + 2);
        if (++slot == S) slot = 0;
        if (++hb == a.h1_bufs) hb = 0, ++hph;
        if (++cb == a.c_bufs) cb = 0, ++cph;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ------------- expand epilogue: E + b_exp -> phi -> pads 0 -> h1 planes
    const int q = warp % 4, eh = (warp - 4) / 4;  // TMEM quadrant, 16-column parity
    const float* s_bexp = reinterpret_cast<const float*>(s_hdr);
    if (a.x_tmem) {
      // move the x tile into TMEM (A operand of the expansion), then recycle
      // its shared-memory region as the second h1 buffer
      mbar_wait(&B.x_full, 0);
      for (int t = 0; t < a.n_et; ++t) {
        const int f = t * 128 + q * 32 + lane;
        for (int pg = eh; pg < a.C / 16; pg += 2) {
          uint4 lo, hi;
          if (a.xsw) {  // pixel row f of 64-channel block pg/4, 16-byte chunk c at (c ^ f%8)
            const uint8_t* row = s_x + ((size_t)(pg / 4) * a.n_et * 128 + f) * 128;
            const int c = (pg % 4) * 2;
            lo = lds128(row + ((c ^ (f & 7)) << 4));
            hi = lds128(row + (((c + 1) ^ (f & 7)) << 4));
          } else {
            lo = lds128(s_x + ((size_t)(2 * pg) * a.x_alloc + f) * 16);
            hi = lds128(s_x + ((size_t)(2 * pg + 1) * a.x_alloc + f) * 16);
          }
          const uint32_t r8[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
          WL_TMEM_ST8(tmem_lane_addr(tmem, q, a.t_x + t * (a.C / 2) + pg * 8), r8);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      named_bar(2, 256);
      if (a.h1_bufs > 1) {
        for (int i = (warp - 4) * 32 + lane; i < G8 * a.flat_h1; i += 256)
          reinterpret_cast<uint4*>(smem + a.s_h1b)[i] = make_uint4(0, 0, 0, 0);
        fence_async_smem();
      }
      mbar_arrive(&B.x_ready);
    }
    mbar_wait(&B.hdr_full, 0);
    for (int j = 0; j < nch; ++j) {
      const int eb = j % a.e_bufs, hb = j % a.h1_bufs;
      uint8_t* h1 = hb ? smem + a.s_h1b : s_h1;
      mbar_wait(&B.e_full[eb], (j / a.e_bufs) & 1);
      if (j >= a.h1_bufs) mbar_wait(&B.h1_empty[hb], ((j / a.h1_bufs) & 1) ^ 1);
      if (warp == 4 && lane == 0) WL_TRACE(16 + 8 * j + 3);
      tc_fence_after();
      // (tile, 16-column block) items dealt round-robin to the two warps of a quadrant
      for (int it = eh; it < a.n_et * (HC / 16); it += 2) {
        const int t = it / (HC / 16), c0 = (it - t * (HC / 16)) * 16;
        const int f = t * 128 + q * 32 + lane;
        const bool real = s_emap[f] != 0;
        {
          uint32_t v[16];
          WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_e + (eb * a.n_et + t) * HC + c0), v);
          tmem_ld_wait();
          uint4 lo = bias_act8<ACT>(v, s_bexp + j * HC + c0);
          uint4 hi = bias_act8<ACT>(v + 8, s_bexp + j * HC + c0 + 8);
          if (!real) lo = hi = make_uint4(0, 0, 0, 0);
          if (f < a.flat_h1) {
            *reinterpret_cast<uint4*>(h1 + ((size_t)(c0 / 8) * a.flat_h1 + f) * 16) = lo;
            *reinterpret_cast<uint4*>(h1 + ((size_t)(c0 / 8 + 1) * a.flat_h1 + f) * 16) = hi;
          }
        }
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&B.h1_full[hb]);
      if (warp == 4 && lane == 0) WL_TRACE(16 + 8 * j + 4);
    }
  } else if (warp >= 12) {
    // ------------- conv epilogue -> staging -> h2 (TMA store) + pool.
    // 8 warps: TMEM quadrant q = warp % 4, 16-column blocks split by parity hh.
    const int q = warp % 4, hh = (warp - 12) / 4;
    const int tid = (warp - 12) * 32 + lane;  // 0..255
    const int wi = warp - 12;
    const int lrow = q * 32 + lane;
    const float* s_bconv = reinterpret_cast<const float*>(s_hdr + a.o_bconv);
    const float* s_cw = reinterpret_cast<const float*>(s_hdr + a.o_convw);  // [9][HR] (T1)
    mbar_wait(&B.hdr_full, 0);
    uint8_t* dst_stage = !S2 ? s_st : s_full;
    const int dst_rows = !S2 ? a.st_rows : a.P_full;
    const bool one_store = S2 || a.st_stores == 1;
    for (int j = 0; j < nch; ++j) {
      const int cb = j % a.c_bufs;
      if (T8) {
        mbar_wait(&B.c_full[cb], (j / a.c_bufs) & 1);
        tc_fence_after();
      } else {
        mbar_wait(&B.h1_full[j % a.h1_bufs], (j / a.h1_bufs) & 1);
      }
      const uint8_t* h1c = (j % a.h1_bufs) ? smem + a.s_h1b : s_h1;
      if (tid == 0) WL_TRACE(16 + 8 * j + 5);
      // staging may still be read by the previous chunk's TMA store
      if (tid == 0) bulk_wait_read0();
      named_bar(1, 256);
      for (int it = hh; it < a.n_ct * (HC / 16); it += 2) {  // (tile, 16-column block) round-robin
        const int t = it / (HC / 16), c0 = (it - t * (HC / 16)) * 16;
        const int f = a.conv_base + t * 128 + lrow;
        const int p = s_cmap[t * 128 + lrow];  // dense full-resolution pixel, -1 = pad
        {
          uint32_t v[16];
          if (T8) {
            WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_c + (cb * a.n_ct + t) * HC + c0), v);
            tmem_ld_wait();
          } else {
            float fv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) fv[i] = 0.f;
            if (p >= 0) {
              for (int tap = 0; tap < 9; ++tap) {
                const int ff = f + (tap / 3 - 1) * a.Wp + (tap % 3 - 1);
                float hv[16];
                unpack8(lds128(h1c + ((size_t)(c0 / 8) * a.flat_h1 + ff) * 16), hv);
                unpack8(lds128(h1c + ((size_t)(c0 / 8 + 1) * a.flat_h1 + ff) * 16), hv + 8);
                const float* w = s_cw + tap * a.HR + j * HC + c0;
#pragma unroll
                for (int i = 0; i < 16; ++i) fv[i] += hv[i] * w[i];
              }
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(fv[i]);
          }
          if (p >= 0) {
            const uint4 lo = bias_act8<ACT>(v, s_bconv + j * HC + c0);
            const uint4 hi = bias_act8<ACT>(v + 8, s_bconv + j * HC + c0 + 8);
            if (one_store) {
              *reinterpret_cast<uint4*>(dst_stage + ((c0 / 8) * dst_rows + p) * 16) = lo;
              *reinterpret_cast<uint4*>(dst_stage + ((c0 / 8 + 1) * dst_rows + p) * 16) = hi;
            } else {
              *reinterpret_cast<uint4*>(dst_stage + st_off(p, c0 / 8, dst_rows, G8)) = lo;
              *reinterpret_cast<uint4*>(dst_stage + st_off(p, c0 / 8 + 1, dst_rows, G8)) = hi;
            }
          }
        }
      }
      if (T8) {
        tc_fence_before();
        mbar_arrive(&B.c_empty[cb]);
      } else {
        mbar_arrive(&B.h1_empty[j % a.h1_bufs]);
      }
      named_bar(1, 256);
      if (tid == 0 && j < 20) WL_TRACE(300 + j);
      if (S2) {
        // BlurPool Triangle-3 x Triangle-3 / 16, stride 2, reflect pad (-1 -> 1),
        // separable: a thread owns (image, channel group, output column, segment
        // of kRB output rows) and slides down it, so each output row costs two
        // horizontal row-blurs (6 loads) and the row above is reused
        constexpr int kRB = 4;
        const int nseg = (a.Ho + kRB - 1) / kRB;
        const int nitems = a.imgs * G8 * a.Wo * nseg;
        for (int it = tid; it < nitems; it += 256) {
          int r = it;
          const int xo = r % a.Wo;
          r /= a.Wo;
          const int g = r % G8;
          r /= G8;
          const int seg = r % nseg, im = r / nseg;
          const int x0 = 2 * xo - 1 < 0 ? 1 : 2 * xo - 1;
          const uint8_t* plane = s_full + ((size_t)g * a.P_full + (size_t)im * a.H * a.W + 2 * xo) * 16;
          const int dxm = (x0 - 2 * xo) * 16;  // -16, or +16 at the reflected left edge
          auto hrow = [&](int cr, float (&o)[8]) {  // horizontal [1 2 1]/4 of band conv row cr
            const uint8_t* p0 = plane + (size_t)cr * a.W * 16;
            float h0[8], h1[8], h2[8];
            unpack8(lds128(p0 + dxm), h0);  // explicit 16-byte loads (no 4x split)
            unpack8(lds128(p0), h1);
            unpack8(lds128(p0 + 16), h2);
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = 0.25f * (h0[k] + h2[k]) + 0.5f * h1[k];
          };
          const int yo0 = seg * kRB, yo1 = min(yo0 + kRB, a.Ho);
          float prev[8];
          {
            const int yg = yo0 + band * a.Ho;
            hrow((2 * yg - 1 < 0 ? 1 : 2 * yg - 1) - c0, prev);
          }
          for (int yo = yo0; yo < yo1; ++yo) {
            const int yg = yo + band * a.Ho;
            float mid[8], nxt[8], acc[8];
            hrow(2 * yg - c0, mid);
            hrow(2 * yg + 1 - c0, nxt);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              acc[k] = 0.25f * (prev[k] + nxt[k]) + 0.5f * mid[k];
              prev[k] = nxt[k];
            }
            const int qp = (im * a.Ho + yo) * a.Wo + xo;
            const int off = a.st_stores == 1 ? (g * a.st_rows + qp) * 16 : st_off(qp, g, a.st_rows, G8);
            *reinterpret_cast<uint4*>(s_st + off) = pack8(acc);
          }
        }
        named_bar(1, 256);
        if (tid == 0 && j < 20) WL_TRACE(320 + j);
      }
      // h2 chunk -> global (TMA store of the dense staging)
      fence_async_smem();
      named_bar(1, 256);
      if (tid == 0) WL_TRACE(16 + 8 * j + 6);
      if (tid == 0) {
        if (a.bulk) {
          const size_t off = ((size_t)group * a.hid + h0 + j * HC) * a.P_out;  // halves
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.h2 + off),
                       "r"(smem_u32(s_st)), "r"(a.P_out * HC * 2)
                       : "memory");
        } else {
          for (int k = 0; k < a.st_stores; ++k)
            tma_store_3d(&tmap_h2, s_st + (size_t)k * G8 * a.st_rows * 16, 0, group * a.P_out + k * a.st_rows,
                         (h0 + j * HC) / 8);
        }
        bulk_commit();
      }
      // pool: deterministic column sums of the staged (fp16) h2 values.
      // warp wi sums channel groups g = wi, wi+8, ...; lane = (pixel offset i, word w)
      const int pix_img = a.Ho * a.Wo;
      // multi-block staging (P_out > 256) only arises in the two-launch plans of
      // large stride-1 images; compiled out of the fused kernels so their
      // register allocation is untouched
      constexpr bool kSplitPool = !S2 && !FUSED;
      if (kSplitPool && a.imgs == 1 && a.st_stores > 1 && a.st_stores * HC <= a.hid)
        mb_pool_split_stores(a, smem, s_st, s_pool, j, HC, G8, wi, lane, tid);
      for (int g = wi; g < G8 && !(kSplitPool && a.imgs == 1 && a.st_stores > 1 && a.st_stores * HC <= a.hid); g += 8) {
        const int i = lane >> 2, w = lane & 3;
        for (int im = 0; im < a.imgs; ++im) {
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
          int pp = im * pix_img + i;
          const int pe = (im + 1) * pix_img;
          if (a.st_stores == 1) {
            const uint8_t* base = s_st + g * a.st_rows * 16 + w * 4;
            for (; pp + 8 < pe; pp += 16) {
              const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(base + pp * 16));
              const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(base + (pp + 8) * 16));
              s0 += f0.x;
              s1 += f0.y;
              s2 += f1.x;
              s3 += f1.y;
            }
            if (pp < pe) {
              const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(base + pp * 16));
              s0 += f0.x;
              s1 += f0.y;
            }
          } else {
            for (; pp < pe; pp += 8) {
              const uint32_t hv = *reinterpret_cast<const uint32_t*>(s_st + st_off(pp, g, a.st_rows, G8) + w * 4);
              const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&hv));
              s0 += f2.x;
              s1 += f2.y;
            }
          }
          s0 += s2;
          s1 += s3;
#pragma unroll
          for (int m = 4; m < 32; m <<= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, m);
            s1 += __shfl_xor_sync(0xffffffffu, s1, m);
          }
          if (i == 0) {
            s_pool[im * a.HR + j * HC + g * 8 + w * 2] += s0;
            s_pool[im * a.HR + j * HC + g * 8 + w * 2 + 1] += s1;
          }
        }
      }
      if (tid == 0 && j < 20) WL_TRACE(160 + j);
    }
    named_bar(1, 256);
    if (tid == 0) WL_TRACE(8);
    if (tid == 0) bulk_wait0();
    const float inv = 1.f / (float)(a.Ho_img * a.Wo);
    if (FUSED && a.bands > 1) {
      // row bands: each CTA pooled its band; the partial sums cross to the
      // peer's (still unused) gate region over DSMEM; they are summed below,
      // after the cluster barrier every thread of both CTAs passes
      float* s_gt = reinterpret_cast<float*>(smem + a.s_gate);
      const uint32_t peer = band ? 0u : 1u;
      for (int i = tid; i < a.hid; i += 256) st_peer_f32(peer_smem(s_gt + i, peer), s_pool[i]);
    } else if (FUSED) {  // ranges == 1: the squeeze-excite below reads the pool straight from shared memory
      float* s_vec = reinterpret_cast<float*>(smem + a.s_gate) + a.imgs * a.hid;
      for (int i = tid; i < a.imgs * a.HR; i += 256) s_vec[i] = s_pool[i] * inv;
    } else {
      for (int i = tid; i < a.imgs * a.HR; i += 256) {
        const int im = i / a.HR, c = i % a.HR;
        a.pool[(size_t)(n0 + im) * a.hid + h0 + c] = s_pool[i] * inv;
      }
    }
  }

  // ---------------- squeeze-excite, once per image group (last CTA to arrive;
  // in fused mode the CTA owns the whole group and skips the global handshake)
  if (!FUSED) __threadfence();  // publish this CTA's pool slice before arriving
  tc_fence_before();
  __syncthreads();
  if (FUSED && a.bands > 1) {
    cluster_sync_all();  // both bands' partial pools delivered
    float* s_gt = reinterpret_cast<float*>(smem + a.s_gate);
    float* s_vec = s_gt + a.hid;
    const float inv = 1.f / (float)(a.Ho_img * a.Wo);
    for (int i = threadIdx.x; i < a.hid; i += blockDim.x) s_vec[i] = (s_pool[i] + s_gt[i]) * inv;
    __syncthreads();
  }
  const int a_tile = 128 * a.HCb * 2, a_stage = a.bulk ? a.a_stage_b : a.n_pt * a_tile;
  uint8_t* s_pa = smem + a.s_pa;
  uint8_t* s_pv = smem + a.s_pv;
  const uint8_t* vch = a.wback + align_up(a.K * 4, 128) + (FUSED ? (size_t)h0 * a.K * 2 : 0);  // this range's W_prj rows
  auto load_a = [&](int j) {  // h2 rows of chunk j (re-read from L2) -> A stage
    const int ab = j % a.sa;
    if (a.bulk) {  // planes [HCb/8][P_out][8], contiguous in global
      const uint32_t bytes = a.P_out * a.HCb * 2;
      mbar_arrive_expect_tx(&B.pa_full[ab], bytes);
      bulk_g2s(s_pa + ab * a_stage, a.h2 + ((size_t)group * a.hid + h0 + (size_t)j * a.HCb) * a.P_out, bytes,
               &B.pa_full[ab]);
      return;
    }
    mbar_arrive_expect_tx(&B.pa_full[ab], a_stage);
    for (int t = 0; t < a.n_pt; ++t)  // 2-D box (64 channels x 128 rows), 128-byte swizzle
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
          "%3}], [%4];" ::"r"(smem_u32(s_pa + ab * a_stage + t * a_tile)),
          "l"(&tmap_h2l), "r"(j * 64), "r"(group * a.P_out + t * 128), "r"(smem_u32(&B.pa_full[ab]))
          : "memory");
  };
  auto load_v = [&](int j) {
    const int vs = j % 3;
    mbar_arrive_expect_tx(&B.pv_full[vs], a.vchunk_bytes);
    bulk_g2s(s_pv + vs * a.vchunk_bytes, vch + (size_t)j * a.vchunk_bytes, a.vchunk_bytes, &B.pv_full[vs]);
  };
  if (threadIdx.x == 0) {
    if (FUSED) {
      B.last = 1;
    } else {
      __threadfence();
      const int old = atomicAdd(&a.counters[group], 1);
      B.last = (old == a.ranges - 1);
    }
    if (FUSED) {  // the projection's first operand loads overlap the squeeze-excite
      asm volatile("fence.proxy.async.global;" ::: "memory");  // h2 TMA stores -> TMA loads
      for (int j = 0; j < a.nchb && j < a.sa; ++j) load_a(j);
      for (int j = 0; j < a.nchb && j < 3; ++j) load_v(j);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) WL_TRACE(9);
  if (B.last) {
    if (!FUSED) __threadfence();
    // fp16 weights: w_sq [hid][SQP], w_ex^T [hid][SQP] (SQP = sq padded to a power of two >= 8)
    const uint8_t* seb = a.wpack;
    if (FUSED && a.se_pref) {  // prefetched into the weight ring
      mbar_wait(&B.se_full, 0);
      seb = smem + a.se_off;
    }
    const __half* wsq = reinterpret_cast<const __half*>(seb + a.o_wsq);
    const float* bsq = reinterpret_cast<const float*>(seb + a.o_bsq);
    const __half* wexT = reinterpret_cast<const __half*>(seb + a.o_wex);
    // w_ex^T rows hold their 16-byte blocks XOR-swizzled by (row >> 1): the
    // excite's row-per-thread loads then hit 8 distinct bank groups per 8 lanes
    auto wex_blk = [&](int h, int b8) -> uint4 {
      return *reinterpret_cast<const uint4*>(wexT + (size_t)h * a.SQP + (b8 ^ ((h >> 1) & (a.SQP / 8 - 1))) * 8);
    };
    const float* bex = reinterpret_cast<const float*>(seb + a.o_bex);
    float* s_vec = reinterpret_cast<float*>(smem + a.s_gate) + a.imgs * a.hid;  // [imgs][hid] pool
    float* s_red = s_vec + a.imgs * a.hid;                                       // [20 warps][imgs][SQP]
    float* s_sq = s_red + 20 * a.imgs * a.SQP;                                   // [imgs][SQP]
    float* s_sqx = s_sq + a.imgs * a.SQP;  // the pair peer's partial squeeze (cluster mode)
    float* s_gt = reinterpret_cast<float*>(smem + a.s_gate);
    const int tid = threadIdx.x, nt = blockDim.x, nw = nt / 32;
    // fused: this CTA's hidden range [h0, h0 + HR) (all of hid unless paired);
    // the split CTAs exchange partial squeezes through distributed shared memory
    const int SEH = FUSED ? a.HR : a.hid, seh0 = FUSED ? h0 : 0;
    const bool paired = FUSED && a.ranges == 2;
    // excite weights of this thread's hidden channel, fetched now so their
    // latency overlaps the squeeze (SQP <= 32: four 16-byte rows)
    const int JB = a.SQP / 8;
    uint4 wx[4];
    if (JB <= 4 && tid < SEH)
#pragma unroll
      for (int b8 = 0; b8 < 4; ++b8)
        if (b8 < JB) wx[b8] = wex_blk(seh0 + tid, b8);
    if (!FUSED) {
      for (int i = tid; i < a.imgs * a.hid; i += nt) {
        const int im = i / a.hid;
        s_vec[i] = __ldcg(a.pool + (size_t)(n0 + im) * a.hid + (i - im * a.hid));
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) WL_TRACE(124);
    // squeeze: lane = (row sub-index, 8-column block jb); each thread walks rows
    const int sub = 32 / JB;
    const int jb = lane % JB, isub = lane / JB;
    float acc[2][8];
#pragma unroll
    for (int im = 0; im < 2; ++im)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[im][k] = 0.f;
    for (int i0 = warp * sub + isub; i0 < SEH; i0 += 4 * nw * sub) {
      uint4 wq[4];  // four independent 16-byte loads in flight
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nw * sub;
        wq[u] = i < SEH ? *reinterpret_cast<const uint4*>(wsq + (size_t)(seh0 + i) * a.SQP + jb * 8)
                        : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nw * sub;
        if (i >= SEH) break;
        float wv[8];
        unpack8(wq[u], wv);
        const float p0 = s_vec[i], p1 = a.imgs > 1 ? s_vec[SEH + i] : 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          acc[0][k] += p0 * wv[k];
          acc[1][k] += p1 * wv[k];
        }
      }
    }
#pragma unroll
    for (int m = JB; m < 32; m <<= 1)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc[0][k] += __shfl_xor_sync(0xffffffffu, acc[0][k], m);
        acc[1][k] += __shfl_xor_sync(0xffffffffu, acc[1][k], m);
      }
    if (isub == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) s_red[(warp * a.imgs) * a.SQP + jb * 8 + k] = acc[0][k];
      if (a.imgs > 1)
#pragma unroll
        for (int k = 0; k < 8; ++k) s_red[(warp * a.imgs + 1) * a.SQP + jb * 8 + k] = acc[1][k];
    }
    __syncthreads();
    if (paired) {  // partial squeezes of the two hidden halves meet in both CTAs
      const uint32_t peer = blockIdx.x & 1 ? 0u : 1u;
      for (int i = tid; i < a.imgs * a.SQP; i += nt) {
        const int im = i / a.SQP, j = i - im * a.SQP;
        float v = 0.f;
        for (int w2 = 0; w2 < nw; ++w2) v += s_red[(w2 * a.imgs + im) * a.SQP + j];
        s_sq[i] = v;
        st_peer_f32(peer_smem(s_sqx + i, peer), v);
      }
      if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {  // per-CTA: partial squeeze ready
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        a.trace[2560 + 2 * blockIdx.x] = (long long)gt;
      }
      cluster_sync_all();
      if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {  // per-CTA: pair met
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        a.trace[2560 + 2 * blockIdx.x + 1] = (long long)gt;
      }
      for (int i = tid; i < a.imgs * a.SQP; i += nt) s_sq[i] = fmaxf(s_sq[i] + s_sqx[i] + bsq[i % a.SQP], 0.f);
    } else {
      for (int i = tid; i < a.imgs * a.SQP; i += nt) {
        const int im = i / a.SQP, j = i - im * a.SQP;
        float v = bsq[j];
        for (int w2 = 0; w2 < nw; ++w2) v += s_red[(w2 * a.imgs + im) * a.SQP + j];
        s_sq[i] = fmaxf(v, 0.f);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) WL_TRACE(125);
    // excite: one hidden channel per thread, its SQP weights as 16-byte vectors
    __half* s_gh = reinterpret_cast<__half*>(s_vec);  // [imgs][hid] half gates (pool is dead now)
    for (int i = tid; i < SEH; i += nt) {
      const int hch = seh0 + i;
      float e0 = bex[hch], e1 = bex[hch];
      uint4 wq[8];
      if (JB <= 4 && i == tid) {
#pragma unroll
        for (int b8 = 0; b8 < 4; ++b8) wq[b8] = wx[b8];
      } else {
#pragma unroll
        for (int b8 = 0; b8 < 8; ++b8)
          if (b8 < JB) wq[b8] = wex_blk(hch, b8);
      }
      for (int b8 = 0; b8 < JB; ++b8) {
        float wv[8];
        unpack8(b8 < 8 ? wq[b8] : wex_blk(hch, b8), wv);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          e0 += s_sq[b8 * 8 + k] * wv[k];
          if (a.imgs > 1) e1 += s_sq[a.SQP + b8 * 8 + k] * wv[k];
        }
      }
      for (int im = 0; im < a.imgs; ++im) {
        const float gv = __fdividef(1.f, 1.f + __expf(-(im ? e1 : e0)));
        if (!FUSED) a.gates[(size_t)(n0 + im) * a.hid + i] = gv;
        s_gt[im * SEH + i] = gv;
        s_gh[im * SEH + i] = __float2half_rn(gv);
      }
    }
    if (threadIdx.x == 0 && !FUSED) a.counters[group] = 0;  // self-cleaning for the next launch
  }
  if (threadIdx.x == 0) WL_TRACE(10);
  __syncthreads();
  if (FUSED) {
    // ---------------- projection: z = (h2 . gate) W_prj + b_prj (+ x). The
    // phase-1 buffers are dead: A (h2 rows, re-read by TMA from L2) and V
    // rings overlay them; Z accumulates in the expand/conv TMEM columns.
    const float* s_gate = reinterpret_cast<const float*>(smem + a.s_gate);
    const int pix_img = a.Ho * a.Wo;
    if (threadIdx.x == 0) WL_TRACE(11);
    if (warp == 0) {
      if (lane == 0) {
        if (a.zst && a.residual) {  // residual rows (the SE weights there are dead now)
          mbar_arrive_expect_tx(&B.res_full, (a.K / 64) * a.P_out * 128);
          for (int cb = 0; cb < a.K / 64; ++cb)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3}], [%4];" ::"r"(smem_u32(smem + a.se_off + cb * a.zst_rows * 128)),
                "l"(&tmap_h2l), "r"(cb * 64), "r"(group * a.P_out), "r"(smem_u32(&B.res_full))
                : "memory");
        }
        for (int j = 0; j < a.nchb; ++j) {
          const int jn = j + a.sa, jv = j + 3;  // refill the stage chunk j frees
          if (jn < a.nchb) {
            mbar_wait(&B.pa_empty[j % a.sa], (j / a.sa) & 1);
            load_a(jn);
          }
          if (jv < a.nchb) {
            mbar_wait(&B.pv_empty[j % 3], (j / 3) & 1);
            load_v(jv);
          }
        }
      }
    } else if (warp == 1) {
      if (lane == 0) {
        const uint32_t idesc = make_idesc_f16(128, a.K);
        for (int j = 0; j < a.nchb; ++j) {
          const int ab = j % a.sa, vs = j % 3;
          mbar_wait(&B.pa_ready[ab], (j / a.sa) & 1);
          if (j < 8) WL_TRACE(96 + j);
          mbar_wait(&B.pv_full[vs], (j / 3) & 1);
          if (j < 8) WL_TRACE(104 + j);
          tc_fence_after();
          const uint32_t vbase = smem_u32(s_pv + vs * a.vchunk_bytes);
          const int vsub = a.K * 64 * 2;  // one packed 64-row W_prj chunk
          for (int t = 0; t < a.n_pt; ++t) {
            if (a.bulk) {
              const uint64_t a_base = make_sdesc(smem_u32(s_pa + ab * a_stage) + t * 2048, a.P_out * 16, 128);
              for (int kk = 0; kk < a.HCb / 16; ++kk) {
                const uint64_t bd = make_sdesc(vbase + (kk / 4) * vsub + (kk % 4) * 2 * a.K * 16, a.K * 16, 128);
                mma_ss(tmem + a.t_z + t * a.K, a_base + (uint64_t)(kk * 2 * a.P_out), bd, idesc, (j > 0 || kk > 0));
              }
            } else {
              const uint64_t b_base = make_sdesc(vbase, a.K * 16, 128);
              const uint64_t a_base = make_sdesc_sw128(smem_u32(s_pa + ab * a_stage + t * a_tile));
              for (int kk = 0; kk < 4; ++kk)
                mma_ss(tmem + a.t_z + t * a.K, a_base + (uint64_t)(kk * 2), b_base + (uint64_t)(kk * 2 * a.K), idesc,
                       (j > 0 || kk > 0));
            }
          }
          mma_commit(&B.pa_empty[ab]);
          mma_commit(&B.pv_empty[vs]);
        }
        mma_commit(&B.z_full);
      }
    } else if (warp >= 4 && warp < 12) {
      // gate the staged h2 rows in place (packed half): each thread owns one
      // 16-byte column (8 channels) and walks rows, so a warp touches 4 whole
      // 128-byte swizzled rows per step (conflict-free) and the gates are one
      // broadcast 16-byte load
      const int tid = (warp - 4) * 32 + lane;
      const int c8 = tid & 7;
      const __half* s_gh = reinterpret_cast<const __half*>(s_gate + a.imgs * a.hid);  // half gates [imgs][HR] (SE scratch)
      for (int j = 0; j < a.nchb; ++j) {
        const int ab = j % a.sa;
        mbar_wait(&B.pa_full[ab], (j / a.sa) & 1);
        if (tid == 0 && j < 8) WL_TRACE(112 + j);
        if (a.bulk) {  // planes [HCb/8][P_out][8]: item = plane * P_out + pixel, 2 per step
          uint8_t* base = s_pa + ab * a_stage;
          const __half* gj = s_gh + j * a.HCb;  // [imgs][HR] gates of this hidden range
          const int nitems = (a.HCb / 8) * a.P_out;
          int c8p = tid / a.P_out, p = tid - c8p * a.P_out;  // walked incrementally
          const int dq = 256 / a.P_out, dr = 256 - dq * a.P_out;
          for (int idx = tid; idx < nitems; idx += 512) {
            int c8b = c8p + dq, pb = p + dr;
            if (pb >= a.P_out) {
              pb -= a.P_out;
              ++c8b;
            }
            const bool two = idx + 256 < nitems;
            const int ia = (a.imgs == 1 || p < pix_img) ? 0 : 1, ib = (a.imgs == 1 || pb < pix_img) ? 0 : 1;
            uint4* pa = reinterpret_cast<uint4*>(base + ((size_t)c8p * a.P_out + p) * 16);
            uint4* pb2 = reinterpret_cast<uint4*>(base + ((size_t)c8b * a.P_out + pb) * 16);
            uint4 va = *pa, vb = two ? *pb2 : va;
            const uint4 ga = *reinterpret_cast<const uint4*>(gj + ia * a.HR + c8p * 8);
            const uint4 gb = *reinterpret_cast<const uint4*>(gj + ib * a.HR + (two ? c8b : c8p) * 8);
            __half2* ha = reinterpret_cast<__half2*>(&va);
            __half2* hb = reinterpret_cast<__half2*>(&vb);
            const __half2* g1 = reinterpret_cast<const __half2*>(&ga);
            const __half2* g2 = reinterpret_cast<const __half2*>(&gb);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              ha[i] = __hmul2(ha[i], g1[i]);
              hb[i] = __hmul2(hb[i], g2[i]);
            }
            *pa = va;
            if (two) *pb2 = vb;
            c8p = c8b + dq;
            p = pb + dr;
            if (p >= a.P_out) {
              p -= a.P_out;
              ++c8p;
            }
          }
          fence_async_smem();
          mbar_arrive(&B.pa_ready[ab]);
          continue;
        }
        for (int r = tid >> 3; r < a.n_pt * 128; r += 32) {
          const int t = r >> 7, m = r & 127;
          const int p = min(t * 128 + m, a.P_out - 1);
          const uint4 gv = *reinterpret_cast<const uint4*>(s_gh + (p / pix_img) * a.HR + j * a.HCb + c8 * 8);
          uint4* ptr = reinterpret_cast<uint4*>(s_pa + ab * a_stage + t * a_tile + sw128_off(m, c8));
          uint4 v = *ptr;
          __half2* h = reinterpret_cast<__half2*>(&v);
          const __half2* g = reinterpret_cast<const __half2*>(&gv);
#pragma unroll
          for (int i = 0; i < 4; ++i) h[i] = __hmul2(h[i], g[i]);
          *ptr = v;
        }
        fence_async_smem();
        mbar_arrive(&B.pa_ready[ab]);
      }
    } else if (warp >= 12) {
      const int q = warp % 4, hh = (warp - 12) / 4;
      const float* bprj = reinterpret_cast<const float*>(a.wback);
      if (a.ranges == 2) {  // paired: the two partial Z meet after the projection (below)
        mbar_wait_sleep(&B.z_full, 0);
        tc_fence_after();
      } else if (a.zst) {
        // z = Z + b_prj (+ x) in shared memory: pixel p, 16-byte chunk c of the
        // 64-channel block cb at (p/8)*1024 + (p%8)*128 + (c ^ p%8)*16
        uint8_t* zs = smem + a.se_off;
        mbar_wait_sleep(&B.z_full, 0);
        if (a.residual) mbar_wait_sleep(&B.res_full, 0);
        tc_fence_after();
        if (warp == 12 && lane == 0) WL_TRACE(120);
        for (int t = 0; t < a.n_pt; ++t) {
          const int p = t * 128 + q * 32 + lane;
          const bool inside = p < a.P_out;
          uint8_t* rowb = zs + (p >> 3) * 1024 + (p & 7) * 128;
          for (int c0 = hh * 16; c0 < a.K; c0 += 32) {
            uint32_t v[16];
            WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_z + t * a.K + c0), v);
            tmem_ld_wait();
            if (!inside) continue;
            uint8_t* rb = rowb + (c0 / 64) * a.zst_rows * 128;
            const int ch = (c0 % 64) / 8;
            uint4* p0 = reinterpret_cast<uint4*>(rb + ((ch ^ (p & 7)) << 4));
            uint4* p1 = reinterpret_cast<uint4*>(rb + (((ch + 1) ^ (p & 7)) << 4));
            float f[16];
            float pb16[16];
            load16f(bprj + c0, pb16);
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) + pb16[i];
            if (a.residual) {
              float r[16];
              unpack8(lds128(p0), r);
              unpack8(lds128(p1), r + 8);
#pragma unroll
              for (int i = 0; i < 16; ++i) f[i] += r[i];
            }
            *p0 = pack8(f);
            *p1 = pack8(f + 8);
          }
        }
        fence_async_smem();
        named_bar(1, 256);
        if (warp == 12 && lane == 0) {
          for (int cb = 0; cb < a.K / 64; ++cb)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tmap_h2),
                         "r"(smem_u32(zs + cb * a.zst_rows * 128)), "r"(cb * 64), "r"(group * a.P_out)
                         : "memory");
          bulk_commit();
          bulk_wait0();
        }
        tc_fence_before();
      } else {
      // z = Z + b_prj (+ x). Each thread owns one pixel row and the 16-column
      // blocks hh, hh+2, ... (two per group); the residual rows of the next
      // group are loaded while this group is combined (the first group's are
      // issued before Z is even complete).
      const int nblk = (a.K - hh * 16 + 31) / 32;
      const int ngrp = (nblk + 1) / 2;
      uint4 res[4];
      auto fetch_res = [&](int t, int gi) {
        const int p = t * 128 + q * 32 + lane;
        if (!a.residual || p >= a.P_out) return;
        const uint4* xp = reinterpret_cast<const uint4*>(a.x + ((size_t)group * a.P_out + p) * a.K + hh * 16);
#pragma unroll
        for (int b = 0; b < 2; ++b)
          if (gi * 2 + b < nblk) {
            res[2 * b] = __ldg(xp + (gi * 2 + b) * 4);
            res[2 * b + 1] = __ldg(xp + (gi * 2 + b) * 4 + 1);
          }
      };
      fetch_res(0, 0);
      mbar_wait_sleep(&B.z_full, 0);
      tc_fence_after();
      if (warp == 12 && lane == 0) WL_TRACE(120);
      for (int t = 0; t < a.n_pt; ++t) {
        if (warp == 12 && lane == 0 && t < 3) WL_TRACE(121 + t);
        const int p = t * 128 + q * 32 + lane;
        const bool inside = p < a.P_out;
        const size_t gp = (size_t)group * a.P_out + (inside ? p : 0);  // dense (n, Ho*Wo) pixel
        for (int gi = 0; gi < ngrp; ++gi) {
          uint32_t v[2][16];
#pragma unroll
          for (int b = 0; b < 2; ++b)
            if (gi * 2 + b < nblk) WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_z + t * a.K + hh * 16 + (gi * 2 + b) * 32), v[b]);
          tmem_ld_wait();
          uint4 cur[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) cur[i] = res[i];
          if (gi + 1 < ngrp) fetch_res(t, gi + 1);  // next group's residual rows in flight
          else if (t + 1 < a.n_pt) fetch_res(t + 1, 0);
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            if (gi * 2 + b >= nblk || !inside) continue;
            const int c0 = hh * 16 + (gi * 2 + b) * 32;
            float f[16];
            float pb16[16];
            load16f(bprj + c0, pb16);
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[b][i]) + pb16[i];
            if (a.residual) {
              float r[16];
              unpack8(cur[2 * b], r);
              unpack8(cur[2 * b + 1], r + 8);
#pragma unroll
              for (int i = 0; i < 16; ++i) f[i] += r[i];
            }
            uint4* zp = reinterpret_cast<uint4*>(a.z + gp * a.K + c0);
            zp[0] = pack8(f);
            zp[1] = pack8(f + 8);
          }
        }
      }
      tc_fence_before();
      }
      if (warp == 12 && lane == 0) WL_TRACE(12);
    }
    __syncthreads();
    if (threadIdx.x == 0) WL_TRACE(13);
    if (a.ranges == 2) {
      // ---- paired CTAs: each holds Z over its hidden half. CTA r finishes the
      // output channels [r K/2, (r+1) K/2): it receives the peer's partial for
      // them (fp32, distributed shared memory, rows padded by 16 bytes) into
      // the dead projection-operand region, then adds its own, b_prj and x.
      const int rank = blockIdx.x & 1, KH = a.K / 2, RS = KH + 4;
      float* s_zr = reinterpret_cast<float*>(smem);  // [n_pt * 128][RS]
      cluster_sync_all();                            // both projections done: operand regions free
      if (warp >= 12) {
        const int q = warp % 4, hh = (warp - 12) / 4, m = q * 32 + lane;
        const int pc0 = (1 - rank) * KH;
        for (int t = 0; t < a.n_pt; ++t)
          for (int c0 = hh * 16; c0 < KH; c0 += 32) {
            uint32_t v[16];
            WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_z + t * a.K + pc0 + c0), v);
            tmem_ld_wait();
            const uint32_t dst = peer_smem(s_zr + (size_t)(t * 128 + m) * RS + c0, 1u - rank);
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) st_peer_v4(dst + 16 * k4, v + 4 * k4);
          }
      }
      cluster_sync_all();  // partials delivered
      if (warp >= 12) {
        const int q = warp % 4, hh = (warp - 12) / 4, m = q * 32 + lane;
        const int oc0 = rank * KH;
        const float* bprj = reinterpret_cast<const float*>(a.wback);
        for (int t = 0; t < a.n_pt; ++t) {
          const int p = t * 128 + m;
          const bool inside = p < a.P_out;
          const size_t gp = (size_t)group * a.P_out + (inside ? p : 0);
          for (int c0 = hh * 16; c0 < KH; c0 += 32) {
            uint32_t v[16];
            WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_z + t * a.K + oc0 + c0), v);
            tmem_ld_wait();
            if (!inside) continue;
            float f[16], r[16];
            const float* zr = s_zr + (size_t)(t * 128 + m) * RS + c0;
            float pb16[16], zr16[16];
            load16f(bprj + oc0 + c0, pb16);
            load16f(zr, zr16);  // the peer's partial (rows padded to 16-byte multiples)
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) + zr16[i] + pb16[i];
            if (a.residual) {
              const uint4* xp = reinterpret_cast<const uint4*>(a.x + gp * a.K + oc0 + c0);
              unpack8(__ldg(xp), r);
              unpack8(__ldg(xp + 1), r + 8);
#pragma unroll
              for (int i = 0; i < 16; ++i) f[i] += r[i];
            }
            uint4* zp = reinterpret_cast<uint4*>(a.z + gp * a.K + oc0 + c0);
            zp[0] = pack8(f);
            zp[1] = pack8(f + 8);
          }
        }
      }
      tc_fence_before();
      __syncthreads();
    }
  }
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {  // per-CTA span: end
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.trace[512 + 2 * blockIdx.x + 1] = (long long)gt;
  }
  if (warp == 2) tmem_dealloc_n(tmem, a.tmem_cols);
}

// ----------------------------------------------------------------- back
// CTA: 128 consecutive output pixels (any images) x output channels
// [k0, k0 + KR). Threads: w0 producer, w1 MMA, w2 alloc, w3 idle, w4-7
// gating + epilogue.
__global__ void __launch_bounds__(256, 1)
    mb_back_kernel(const __grid_constant__ CUtensorMap tmap_h2, const __grid_constant__ MbBackArgs a) {
  using namespace mbk;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_a = smem + a.s_a;                                // 2 x [HCb/8][128][8] fp16
  float* s_gate = reinterpret_cast<float*>(smem + a.s_gate);  // [4 imgs][hid]
  uint8_t* s_ring = smem + a.s_ring;
  BackBars& B = *reinterpret_cast<BackBars*>(smem + a.s_bar);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x / a.kranges, kr = blockIdx.x % a.kranges;
  const int p0 = tile * 128;
  const int k0 = kr * a.KR;
  const int S = a.ring_stages, nch = a.nchb, HCb = a.HCb;
  const int img_first = p0 / a.pix_per_img;
  const int img_last = min(a.P - 1, p0 + 127) / a.pix_per_img;
  const int nimg = img_last - img_first + 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.a_full[i], 1);
      mbar_init(&B.a_empty[i], 1);
      mbar_init(&B.a_ready[i], 128);
    }
    for (int i = 0; i < S; ++i) {
      mbar_init(&B.v_full[i], 1);
      mbar_init(&B.v_empty[i], 1);
    }
    mbar_init(&B.z_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_n(&B.tmem_base, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // (multi-wave grid: dependents launch as CTAs retire)
  pdl_wait();
  const uint32_t tmem = B.tmem_base;
  const int a_stage_bytes = 128 * HCb * 2;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmap_h2);
      const uint8_t* vchunks = a.wpack + a.o_bprj + align_up(a.K * 4, 128);
      for (int j = 0; j < nch; ++j) {
        const int ab = j & 1;
        mbar_wait(&B.a_empty[ab], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&B.a_full[ab], a_stage_bytes);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];" ::"r"(smem_u32(s_a + ab * a_stage_bytes)),
            "l"(&tmap_h2), "r"(0), "r"(p0), "r"(j * HCb / 8), "r"(smem_u32(&B.a_full[ab]))
            : "memory");
        const int slot = j % S;
        mbar_wait(&B.v_empty[slot], ((j / S) & 1) ^ 1);
        mbar_arrive_expect_tx(&B.v_full[slot], a.vchunk_bytes);
        bulk_g2s(s_ring + slot * a.vchunk_bytes, vchunks + (size_t)(kr * nch + j) * a.vchunk_bytes, a.vchunk_bytes,
                 &B.v_full[slot]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_f16(128, a.KR);
      const uint32_t a0 = smem_u32(s_a), ring0 = smem_u32(s_ring);
      for (int j = 0; j < nch; ++j) {
        const int ab = j & 1, slot = j % S;
        mbar_wait(&B.a_ready[ab], (j >> 1) & 1);
        mbar_wait(&B.v_full[slot], (j / S) & 1);
        tc_fence_after();
        for (int kk = 0; kk < HCb / 16; ++kk) {
          const uint64_t ad = make_sdesc(a0 + ab * a_stage_bytes + kk * 2 * 2048, 2048, 128);
          const uint64_t bd = make_sdesc(ring0 + slot * a.vchunk_bytes + kk * 2 * (a.KR * 16), a.KR * 16, 128);
          mma_ss(tmem + a.t_z, ad, bd, idesc, (j > 0 || kk > 0));
        }
        mma_commit(&B.a_empty[ab]);
        mma_commit(&B.v_empty[slot]);
      }
      mma_commit(&B.z_full);
    }
  } else if (warp >= 4) {
    const int q = warp - 4, tid = q * 32 + lane;
    for (int i = tid; i < nimg * a.hid; i += 128) s_gate[i] = a.gates[(size_t)img_first * a.hid + i];
    named_bar(1, 128);
    const int p = p0 + tid;
    const int im = min(p, a.P - 1) / a.pix_per_img - img_first;
    for (int j = 0; j < nch; ++j) {
      const int ab = j & 1;
      mbar_wait(&B.a_full[ab], (j >> 1) & 1);
      uint8_t* base = s_a + ab * a_stage_bytes;
      const float* g = s_gate + im * a.hid + j * HCb;
#pragma unroll 2
      for (int c8 = 0; c8 < HCb / 8; ++c8) {
        uint4* ptr = reinterpret_cast<uint4*>(base + (c8 * 128 + tid) * 16);
        uint4 v = *ptr;
        __half2* h = reinterpret_cast<__half2*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __hmul2(h[i], __floats2half2_rn(g[c8 * 8 + 2 * i], g[c8 * 8 + 2 * i + 1]));
        *ptr = v;
      }
      fence_async_smem();
      mbar_arrive(&B.a_ready[ab]);
    }
    // ---- epilogue: z = Z + b_prj (+ x)
    mbar_wait(&B.z_full, 0);
    tc_fence_after();
    const float* bprj = reinterpret_cast<const float*>(a.wpack + a.o_bprj);
    const bool inside = p < a.P;
    for (int c0 = 0; c0 < a.KR; c0 += 16) {
      uint32_t v[16];
      WL_TMEM_LD16(tmem_lane_addr(tmem, q, a.t_z + c0), v);
      tmem_ld_wait();
      if (!inside) continue;
      float f[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) + bprj[k0 + c0 + i];
      if (a.residual) {
        float r[16];
        const uint4* xp = reinterpret_cast<const uint4*>(a.x + (size_t)p * a.K + k0 + c0);
        unpack8(xp[0], r);
        unpack8(xp[1], r + 8);
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] += r[i];
      }
      uint4* zp = reinterpret_cast<uint4*>(a.z + (size_t)p * a.K + k0 + c0);
      zp[0] = pack8(f);
      zp[1] = pack8(f + 8);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc_n(tmem, a.tmem_cols);
}

}  // namespace wl

// =================================================================== host
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include "launch.h"

namespace wl {
// stride-1 T=8 MBConv with the grouped conv on mma.sync (mb_s1.cu)
bool mb1_eligible(const wl_block_desc& d);
int64_t mb1_packed_bytes(const wl_block_desc& d);
int64_t mb1_workspace(const wl_block_desc& d);
int mb1_pack(const wl_block_desc& d, const float* const* w, uint8_t* out);
int mb1_forward(const wl_block_desc& d, const void* x, const void* packed, void* z, void* ws, cudaStream_t st);
int mb1_init();
void mb1_set_trace(void* p);

namespace {

constexpr int kSmemMaxMb = 232448;
long long* g_mb_trace = nullptr;
constexpr int64_t kCounterBytes = 4096;  // workspace header: per-group arrival counters

struct MbPlanH {
  MbFrontArgs f;
  MbBackArgs b;
  int64_t front_bytes, back_bytes;
  int64_t h2_bytes, pool_bytes, gate_bytes;
};

// planner debug knobs, read ONCE per process: the plan is recomputed by
// validate / pack / workspace / forward and must not change between them
static bool env_dw_cuda() {
  static const bool v = getenv("WL_MB_DW_CUDA") != nullptr;
  return v;
}
static const int* env_force() {  // WL_MB_FORCE="xt,eb,cb,hc" pins the TMEM / chunk choice
  static int f[4] = {-1, -1, -1, -1};
  static const bool once = [] {
    if (const char* e = getenv("WL_MB_FORCE")) sscanf(e, "%d,%d,%d,%d", &f[0], &f[1], &f[2], &f[3]);
    return true;
  }();
  (void)once;
  return f;
}
// WL_MB_DEBUG=1 names the planner check that rejected a configuration
static bool mb_plan_fail(int id, int line) {
  if (getenv("WL_MB_DEBUG")) fprintf(stderr, "mb plan: rejected at check %d (mbconv.cu:%d)\n", id, line);
  return false;
}
bool mb_plan_try(const wl_block_desc& d, MbPlanH& P, bool want_fused, int bands = 1, int max_imgs = 2,
                 bool pair = true, int hc_cap = 128) {
  memset(&P, 0, sizeof(P));
  MbFrontArgs& f = P.f;
  MbBackArgs& b = P.b;
  const int C = d.c, hid = d.expansion * d.c, K = d.k;
  if (C % 16 || hid % 16 || K % 16) return mb_plan_fail(1, __LINE__);
  f.C = C;
  f.hid = hid;
  f.sq = d.se_sq;
  // depthwise (T=1) convs run on the same tensor-core path as T=8: each 8x8
  // block of the block-diagonal B is itself diagonal (exact, zeros elsewhere)
  f.T8 = d.group_width == 8 || (d.group_width == 1 && !env_dw_cuda());
  f.stride = d.stride;
  f.H = d.h;
  f.W = d.w;
  f.bands = bands;
  f.H_img = d.h;
  f.Ho_img = d.h / d.stride;
  if (bands > 1) {  // two row bands of Ob output rows: stride 1 convs Ob rows, stride 2 2*Ob+1 (blur halo)
    if (bands != 2 || !want_fused || f.Ho_img % 2) return mb_plan_fail(14, __LINE__);
    const int Ob = f.Ho_img / 2;
    f.H = d.stride == 1 ? Ob : 2 * Ob + 1;
  }
  f.imgs = (bands == 1 && max_imgs > 1 && d.h * d.w <= 64 && d.n % 2 == 0) ? 2 : 1;
  f.Wp = d.w + 1;  // stacked images must start 128-byte aligned (TMA)
  while (f.imgs > 1 && ((d.h + 1) * f.Wp) % 8) ++f.Wp;
  f.Ho = bands > 1 ? f.Ho_img / 2 : d.h / d.stride;
  f.Wo = d.w / d.stride;
  // whole images: [top halo + H rows] per image, one zero row below the stack;
  // bands: the band's H rows between two loaded halo rows (real image rows or
  // TMA zero fill at the image border)
  f.total_rows = bands > 1 ? f.H + 2 : f.imgs * (f.H + 1) + 1;
  const int x_valid = bands > 1 ? (f.H + 2) * f.Wp : f.imgs * (f.H + 1) * f.Wp;
  f.n_et = (x_valid + 127) / 128;
  f.x_alloc = x_valid;  // plane stride = the loaded rows (one TMA box); tile overrun reads are masked
  f.conv_base = f.Wp + 1;
  const int conv_end = (f.total_rows - 1) * f.Wp;
  f.n_ct = (conv_end - f.conv_base + 127) / 128;
  f.flat_h1 = align_up(f.conv_base + f.n_ct * 128 + f.Wp + 2, 8);
  f.groups = d.n / f.imgs * bands;  // CTAs per range
  f.P_out = f.imgs * f.Ho * f.Wo;
  f.P_full = f.imgs * f.H * f.W;
  f.st_stores = (f.P_out + 255) / 256;
  while (f.P_out % f.st_stores) ++f.st_stores;
  f.st_rows = f.P_out / f.st_stores;
  // arrival counters exist only in the two-launch (unfused) form
  if (!want_fused && f.groups > (int)(kCounterBytes / 4)) return mb_plan_fail(2, __LINE__);
  if (f.sq < 1 || f.sq > 128) return mb_plan_fail(3, __LINE__);
  // fused mode: the CTA owns every hidden channel of its images, or - when the
  // image groups would leave over half the SMs idle - a cluster pair splits them
  f.ranges = (want_fused && pair && bands == 1 && 2 * f.groups <= kNumSMs && hid % 128 == 0 && K % 64 == 0 && K <= 256) ? 2 : 1;
  while (!want_fused && f.groups * f.ranges < kNumSMs && hid % (f.ranges * 2 * 16) == 0) f.ranges *= 2;
  f.HR = hid / f.ranges;
  f.HC = 0;
  // room for either staging: [C/8 planes][x_valid rows] (+ tile overrun) or
  // [C/64 blocks][n_et * 128 rows][128 B] (swizzled pixel rows)
  const int x_bytes = std::max(align_up((C / 8) * f.x_alloc * 16 + (f.n_et * 128 - x_valid) * 16, 128),
                               (C % 64 == 0) ? C * 2 * f.n_et * 128 : 0);
  const int se_scratch = align_up((hid + 640 + f.sq) * 4, 16);
  // planner experiments: WL_MB_FORCE="xt,eb,cb,hc" pins the TMEM / chunk choice
  const int* force = env_force();
  for (int hc = hc_cap; hc >= 16; hc -= 16) {
    if (f.HR % hc || (force[3] > 0 && hc != force[3])) continue;
    const int tiles1 = f.T8 ? f.n_et + f.n_ct : f.n_et;
    if (tiles1 * hc > 512) continue;
    const int h1_bytes = std::max((hc / 8) * f.flat_h1 * 16, se_scratch);
    const int st = f.P_out * hc * 2;
    const int full = f.stride == 2 ? f.P_full * hc * 2 : 0;
    const int hdr = align_up(f.HR * 4, 16) * 2 + (f.T8 ? 0 : align_up(9 * f.HR * 4, 16));
    const int chunk = hc * C * 2 + (f.T8 ? (2 * (hc / 16) * 9 + 1) * 128 : 0);
    const int total = x_bytes + h1_bytes + st + full + hdr + 2 * chunk + f.imgs * f.HR * 4 + 2048 +
                      f.n_ct * 128 * 4 + f.n_et * 128;
    if (total <= kSmemMaxMb) {
      f.HC = hc;
      break;
    }
  }
  if (!f.HC) return mb_plan_fail(4, __LINE__);
  f.nch = f.HR / f.HC;
  // double-buffer the expand / conv accumulators when TMEM allows
  // TMEM: x tile (A of a TS-mode expansion, T=8 only) + expand / conv
  // accumulators, double-buffered when the 512 columns allow
  const int x_cols = f.n_et * (C / 2);
  auto cols = [&]() {
    return (f.x_tmem ? x_cols : 0) + (f.e_bufs * f.n_et + (f.T8 ? f.c_bufs * f.n_ct : 0)) * f.HC;
  };
  bool placed = false;
  for (int xt = f.T8 ? 1 : 0; xt >= 0 && !placed; --xt) {
    const int combos[4][2] = {{2, 2}, {1, 2}, {2, 1}, {1, 1}};
    for (auto& cb : combos) {
      if (force[0] >= 0 && (xt != force[0] || cb[0] != force[1] || cb[1] != force[2])) continue;
      f.x_tmem = xt;
      f.e_bufs = (f.T8 && f.nch > 1) ? cb[0] : 1;  // T=1: the MMA warp cannot observe E consumption early
      f.c_bufs = (f.T8 && f.nch > 1) ? cb[1] : 1;
      if (cols() <= 512) {
        placed = true;
        break;
      }
    }
  }
  if (!placed) return mb_plan_fail(5, __LINE__);
  f.xsw = f.x_tmem && C % 64 == 0;
  f.t_x = 0;
  f.t_e = f.x_tmem ? x_cols : 0;
  f.t_c = f.t_e + f.e_bufs * f.n_et * f.HC;
  f.tmem_cols = 32;
  while (f.tmem_cols < cols()) f.tmem_cols *= 2;
  f.h1_bytes = std::max((f.HC / 8) * f.flat_h1 * 16, se_scratch);
  f.st_bytes = f.P_out * f.HC * 2;
  f.full_bytes = f.stride == 2 ? f.P_full * f.HC * 2 : 0;
  f.o_bconv = align_up(f.HR * 4, 16);
  f.o_convw = f.o_bconv + align_up(f.HR * 4, 16);
  f.hdr_bytes = f.o_convw + (f.T8 ? 0 : align_up(9 * f.HR * 4, 16));
  f.u_bytes = f.HC * C * 2;
  f.chunk_bytes = f.u_bytes + (f.T8 ? (2 * (f.HC / 16) * 9 + 1) * 128 : 0);
  f.ring_stages = 2;  // raised to 3 below when shared memory allows
  // SE section at the start of the front blob: fp16 w_sq [hid][SQP] and
  // w_ex^T [hid][SQP] (SQP = squeeze width padded to a power of two >= 8,
  // zero-filled), fp32 biases
  f.SQP = 8;
  while (f.SQP < f.sq) f.SQP *= 2;
  if (f.SQP > 256) return mb_plan_fail(6, __LINE__);
  int so = 0;
  f.o_wsq = so;
  so = align_up(so + hid * f.SQP * 2, 16);
  f.o_bsq = so;
  so = align_up(so + f.SQP * 4, 16);
  f.o_wex = so;
  so = align_up(so + hid * f.SQP * 2, 16);
  f.o_bex = so;
  so = align_up(so + hid * 4, 16);
  f.se_bytes = align_up(so, 128);
  int o = 0;
  f.s_x = o;
  o = align_up(o + x_bytes, 128);
  f.s_h1 = o;
  o = align_up(o + f.h1_bytes, 128);
  f.s_st = o;
  o = align_up(o + f.st_bytes, 128);
  f.s_full = o;
  o = align_up(o + f.full_bytes, 128);
  f.s_hdr = o;
  o = align_up(o + f.hdr_bytes, 128);
  f.s_ring = o;
  o = align_up(o + f.ring_stages * f.chunk_bytes, 128);
  f.s_pool = o;
  o = align_up(o + f.imgs * f.HR * 4, 128);
  f.s_map = o;
  o = align_up(o + f.n_ct * 128 * 4 + f.n_et * 128, 128);
  if (o + f.chunk_bytes + 512 <= kSmemMaxMb && f.nch > 2) {  // third weight stage
    // shift everything after the ring by one chunk
    f.ring_stages = 3;
    f.s_pool += f.chunk_bytes;
    f.s_map += f.chunk_bytes;
    o += f.chunk_bytes;
  }
  // second h1 buffer: the x region once x lives in TMEM, else a new region if it fits
  const int h1_one = (f.HC / 8) * f.flat_h1 * 16;
  f.h1_bufs = 1;
  f.s_h1b = f.s_h1;
  if (f.nch > 1 && f.x_tmem && x_bytes >= h1_one) {
    f.h1_bufs = 2;
    f.s_h1b = f.s_x;
  } else if (f.nch > 1 && o + align_up(h1_one, 128) + 512 <= kSmemMaxMb) {
    f.h1_bufs = 2;
    f.s_h1b = o;
    o = align_up(o + h1_one, 128);
  }
  f.s_gate = o;  // SE gates (read by the fused projection) + squeeze-excite scratch
  o = align_up(o + (2 * f.imgs * hid + 22 * f.imgs * f.SQP) * 4, 128);
  f.s_bar = o;
  o += 512;
  f.smem = o;
  if (o > kSmemMaxMb) {  // the chunk-width estimate above was optimistic: next narrower chunk
    if (f.HC > 16) return mb_plan_try(d, P, want_fused, bands, max_imgs, pair, f.HC - 16);
    return mb_plan_fail(7, __LINE__);
  }
  P.front_bytes = f.se_bytes + (int64_t)f.ranges * f.hdr_bytes + (int64_t)f.ranges * f.nch * f.chunk_bytes;
  f.fused = 0;
  if (want_fused) {
    // projection overlays the dead phase-1 buffers: A ring (2 stages of the
    // CTA's h2 rows), V ring (3 stages); Z in the expand/conv TMEM columns
    f.K = K;
    if (hid % 64) return mb_plan_fail(8, __LINE__);  // W_prj packed in 64-row chunks
    f.bulk = f.st_stores == 1;
    if (f.ranges > 1 && !f.bulk) return mb_plan_fail(9, __LINE__);
    f.n_pt = (f.P_out + 127) / 128;
    f.residual = d.stride == 1;
    f.t_z = 0;  // x tile, expand and conv accumulators are all dead by the projection
    f.s_pa = 0;
    if (K > 256 || f.n_pt * K > 512) return mb_plan_fail(10, __LINE__);
    while (f.tmem_cols < f.n_pt * K) f.tmem_cols *= 2;
    // projection chunk width: whole conv chunks (lcm(HC, 64)) when its A / V
    // rings fit, else 64 channels (bulk h2 is plane-contiguous, [hidden/8][P_out][8],
    // so any 64-channel range is one copy whatever the conv chunk width)
    int pc = 64;
    if (f.bulk)
      while (pc % f.HC) pc += 64;
    f.sa = 0;
    for (int hcb : {pc, 64}) {
      if (f.sa || f.HR % hcb || (hcb != 64 && !f.bulk)) continue;
      f.HCb = hcb;
      f.nchb = f.HR / f.HCb;
      f.vchunk_bytes = K * f.HCb * 2;
      // bulk stages hold [HCb/8][P_out][8] plus the slack the last plane's
      // 128-row tiles read past P_out
      f.a_stage_b = align_up((f.HCb / 8) * f.P_out * 16 + (f.n_pt * 128 - f.P_out) * 16, 128);
      const int a_stage = f.bulk ? f.a_stage_b : f.n_pt * 128 * f.HCb * 2;
      for (int sa = std::min(4, std::max(2, f.nchb)); sa >= 2 && !f.sa; --sa) {
        f.s_pv = align_up(sa * a_stage, 128);
        if (f.s_pv + 3 * f.vchunk_bytes <= f.s_gate) f.sa = sa;
      }
    }
    if (!f.sa) return mb_plan_fail(11, __LINE__);
    const int a_stage = f.bulk ? f.a_stage_b : f.n_pt * 128 * f.HCb * 2;
    f.fused = 1;
    // SE weights at the tail of the weight ring, clear of the projection's A / V
    // rings (give up A stages for it, down to two)
    f.se_off = (f.s_ring + f.ring_stages * f.chunk_bytes - f.se_bytes) / 1024 * 1024;
    f.se_pref = 0;
    if (f.se_off >= f.s_ring)
      for (int sa = f.sa; sa >= 2 && !f.se_pref; --sa) {
        const int spv = align_up(sa * a_stage, 128);
        if (f.se_off >= spv + 3 * f.vchunk_bytes) {
          f.sa = sa;
          f.s_pv = spv;
          f.se_pref = 1;
        }
      }
    f.zst_rows = align_up(f.P_out, 8);
    f.zst = f.se_pref && f.bulk && f.ranges == 1 && f.imgs == 1 && K % 64 == 0 && f.P_out <= 256 &&
            f.se_off + (K / 64) * f.zst_rows * 128 <= f.s_ring + f.ring_stages * f.chunk_bytes;
  }

  // ---- back
  b.hid = hid;
  b.K = K;
  b.stride = d.stride;
  b.P = d.n * f.Ho_img * f.Wo;
  b.pix_per_img = f.Ho * f.Wo;
  b.residual = d.stride == 1;
  const int ntiles = (b.P + 127) / 128;
  b.KR = K;
  while (!f.fused && (b.KR > 256 || (ntiles * (K / b.KR) < kNumSMs && b.KR % 32 == 0 && b.KR >= 64))) b.KR /= 2;
  if (K % b.KR || b.KR % 16) return mb_plan_fail(12, __LINE__);
  b.kranges = K / b.KR;
  b.HCb = hid % 64 == 0 ? 64 : (hid % 32 == 0 ? 32 : 16);
  b.nchb = hid / b.HCb;
  b.o_bprj = 0;
  b.vchunk_bytes = b.KR * b.HCb * 2;
  b.ring_stages = 3;
  o = 0;
  b.s_a = o;
  o += 2 * 128 * b.HCb * 2;
  b.s_gate = o;
  o = align_up(o + 4 * hid * 4, 128);
  b.s_ring = o;
  o = align_up(o + b.ring_stages * b.vchunk_bytes, 128);
  b.s_bar = o;
  o += 512;
  b.smem = o;
  if (o > kSmemMaxMb) return mb_plan_fail(13, __LINE__);
  b.t_z = 0;
  b.tmem_cols = 32;
  while (b.tmem_cols < b.KR) b.tmem_cols *= 2;
  P.back_bytes = align_up(K * 4, 128) + (int64_t)b.kranges * b.nchb * b.vchunk_bytes;
  P.h2_bytes = (int64_t)d.n * f.Ho_img * f.Wo * hid * 2;
  P.pool_bytes = (int64_t)d.n * hid * 4;
  P.gate_bytes = (int64_t)d.n * hid * 4;
  return true;
}

// one launch per block when the projection fits (fused); else front + back
bool mb_plan(const wl_block_desc& d, MbPlanH& P) {
  return mb_plan_try(d, P, true) || mb_plan_try(d, P, false) || mb_plan_try(d, P, true, 1, 1) ||
         mb_plan_try(d, P, true, 1, 1, false) || mb_plan_try(d, P, true, 2);
}

using FrontK = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const MbFrontArgs);

template <int ACT>
FrontK front_kernel_act(bool t8, bool s2, bool fused) {
  const int k = (t8 ? 4 : 0) + (s2 ? 2 : 0) + (fused ? 1 : 0);
  static const FrontK tab[8] = {
      mb_front_kernel<ACT, false, false, false>, mb_front_kernel<ACT, false, false, true>,
      mb_front_kernel<ACT, false, true, false>,  mb_front_kernel<ACT, false, true, true>,
      mb_front_kernel<ACT, true, false, false>,  mb_front_kernel<ACT, true, false, true>,
      mb_front_kernel<ACT, true, true, false>,   mb_front_kernel<ACT, true, true, true>};
  return tab[k];
}
FrontK front_kernel(int act, bool t8 = true, bool s2 = false, bool fused = true) {
  switch (act) {
    case kRelu: return front_kernel_act<kRelu>(t8, s2, fused);
    case kSilu: return front_kernel_act<kSilu>(t8, s2, fused);
    case kGelu: return front_kernel_act<kGelu>(t8, s2, fused);
  }
  return nullptr;
}

int mb_validate(const wl_block_desc& d) {
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c < 1 || d.k < 1) return set_error(WL_EINVAL, "dims must be positive");
  if (d.expansion < 1) return set_error(WL_EINVAL, "expansion must be at least 1");
  const int hid = d.expansion * d.c;
  if (d.group_width < 1 || hid % d.group_width)
    return set_error(WL_EINVAL, "group width %d does not divide %d hidden channels", d.group_width, hid);
  if (d.stride != 1 && d.stride != 2) return set_error(WL_EINVAL, "stride must be 1 or 2");
  if (d.stride == 1 && d.k != d.c) return set_error(WL_EINVAL, "stride-1 blocks keep their channel count");
  if (d.stride == 2 && (d.h % 2 || d.w % 2)) return set_error(WL_EINVAL, "stride 2 needs an even resolution");
  if (d.se_sq < 1) return set_error(WL_EINVAL, "se_ratio must give at least one squeeze channel");
  if (d.ksize != 3) return set_error(WL_EUNSUPPORTED, "MBConv conv is 3x3 (complexity.py:38)");
  if (d.group_width != 8 && d.group_width != 1)
    return set_error(WL_EUNSUPPORTED, "MBConv kernel supports group width 8 or 1, got %d", d.group_width);
  if (!front_kernel(d.act)) return set_error(WL_EUNSUPPORTED, "MBConv supports relu/silu/gelu");
  if (mb1_eligible(d)) return WL_OK;
  MbPlanH P;
  if (!mb_plan(d, P)) return set_error(WL_EUNSUPPORTED, "no MBConv launch plan for C=%d hid=%d %dx%d", d.c, hid, d.h, d.w);
  return WL_OK;
}

int mb_weight_count(const wl_block_desc&) { return 10; }

int64_t mb_weight_numel(const wl_block_desc& d, int i) {
  const int64_t c = d.c, hid = (int64_t)d.expansion * d.c, sq = d.se_sq, k = d.k;
  switch (i) {
    case 0: return c * hid;                  // w_exp (C, hid)
    case 1: return hid;                      // b_exp
    case 2: return hid * 9 * d.group_width;  // w_conv (hid, 3, 3, T)
    case 3: return hid;                      // b_conv
    case 4: return hid * sq;                 // w_sq (hid, sq)
    case 5: return sq;                       // b_sq
    case 6: return sq * hid;                 // w_ex (sq, hid)
    case 7: return hid;                      // b_ex
    case 8: return hid * k;                  // w_prj (hid, K)
    case 9: return k;                        // b_prj
  }
  return set_error(WL_EINVAL, "weight index %d out of range", i);
}

int64_t mb_packed_bytes(const wl_block_desc& d) {
  if (mb1_eligible(d)) return mb1_packed_bytes(d);
  MbPlanH P;
  mb_plan(d, P);
  return P.front_bytes + P.back_bytes;
}

// workspace: [counters 4 KiB][h2][pool][gates]; zero it once before first use
int64_t mb_workspace(const wl_block_desc& d) {
  if (mb1_eligible(d)) return mb1_workspace(d);
  MbPlanH P;
  mb_plan(d, P);
  return kCounterBytes + ((P.h2_bytes + 255) / 256) * 256 + P.pool_bytes + P.gate_bytes;
}

int mb_pack(const wl_block_desc& d, const float* const* w, uint8_t* out) {
  if (mb1_eligible(d)) return mb1_pack(d, w, out);
  MbPlanH P;
  mb_plan(d, P);
  const MbFrontArgs& f = P.f;
  const MbBackArgs& b = P.b;
  memset(out, 0, (size_t)(P.front_bytes + P.back_bytes));
  const int C = d.c, hid = f.hid, T = d.group_width, K = d.k, sq = d.se_sq;
  const float *wexp = w[0], *bexp = w[1], *wconv = w[2], *bconv = w[3];
  for (int i = 0; i < hid; ++i)
    for (int j = 0; j < sq; ++j) {
      put_h(out + f.o_wsq, ((size_t)i * f.SQP + j) * 2, w[4][(size_t)i * sq + j]);   // w_sq (hid, sq)
      // w_ex (sq, hid)^T, 16-byte blocks of row i XOR-swizzled by (i >> 1) (see the excite)
      const int jp = ((j / 8) ^ ((i >> 1) & (f.SQP / 8 - 1))) * 8 + j % 8;
      put_h(out + f.o_wex, ((size_t)i * f.SQP + jp) * 2, w[6][(size_t)j * hid + i]);
    }
  memcpy(out + f.o_bsq, w[5], sizeof(float) * sq);
  memcpy(out + f.o_bex, w[7], sizeof(float) * hid);
  for (int r = 0; r < f.ranges; ++r) {
    uint8_t* hdr = out + f.se_bytes + (size_t)r * f.hdr_bytes;
    float* fb = reinterpret_cast<float*>(hdr);
    float* fc = reinterpret_cast<float*>(hdr + f.o_bconv);
    float* fw = reinterpret_cast<float*>(hdr + f.o_convw);
    for (int i = 0; i < f.HR; ++i) {
      const int h = r * f.HR + i;
      fb[i] = bexp[h];
      fc[i] = bconv[h];
      if (!f.T8)
        for (int t = 0; t < 9; ++t) fw[t * f.HR + i] = wconv[(size_t)h * 9 + t];
    }
    for (int j = 0; j < f.nch; ++j) {
      uint8_t* ch = out + f.se_bytes + (size_t)f.ranges * f.hdr_bytes + (size_t)(r * f.nch + j) * f.chunk_bytes;
      const int hb = r * f.HR + j * f.HC;
      for (int n = 0; n < f.HC; ++n)
        for (int k = 0; k < C; ++k) put_h(ch, core_off_h(n, k, f.HC * 16), wexp[(size_t)k * hid + hb + n]);
      if (f.T8) {
        uint8_t* cw = ch + f.u_bytes;
        const int E = (f.HC / 16) * 9;
        uint8_t* z = cw + E * 128;  // shared zero block
        for (int pr = 0; pr < f.HC / 16; ++pr)
          for (int t = 0; t < 9; ++t) {
            const int e = pr * 9 + t;
            for (int half = 0; half < 2; ++half) {
              uint8_t* blk = half ? z + (e + 1) * 128 : z - (e + 1) * 128;
              for (int nn = 0; nn < 8; ++nn)
                for (int kk = 0; kk < 8; ++kk) {
                  const int oc = hb + 16 * pr + 8 * half + nn;
                  const float wv = T == 8 ? wconv[((size_t)oc * 9 + t) * T + kk] : (kk == nn ? wconv[(size_t)oc * 9 + t] : 0.f);
                  put_h(blk, nn * 16 + kk * 2, wv);
                }
            }
          }
      }
    }
  }
  uint8_t* bk = out + P.front_bytes;
  memcpy(bk + b.o_bprj, w[9], sizeof(float) * K);
  const float* wprj = w[8];
  uint8_t* vbase = bk + align_up(K * 4, 128);
  for (int kr = 0; kr < b.kranges; ++kr)
    for (int j = 0; j < b.nchb; ++j) {
      uint8_t* vc = vbase + (size_t)(kr * b.nchb + j) * b.vchunk_bytes;
      for (int n = 0; n < b.KR; ++n)
        for (int k = 0; k < b.HCb; ++k)
          put_h(vc, core_off_h(n, k, b.KR * 16), wprj[(size_t)(j * b.HCb + k) * K + kr * b.KR + n]);
    }
  return WL_OK;
}

int mb_forward(const wl_block_desc& d, const void* x, const void* packed, void* z, void* ws, cudaStream_t st) {
  if (mb1_eligible(d)) return mb1_forward(d, x, packed, z, ws, st);
  MbPlanH P;
  mb_plan(d, P);
  MbFrontArgs f = P.f;
  MbBackArgs b = P.b;
  uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
  __half* h2 = reinterpret_cast<__half*>(wsb + kCounterBytes);
  float* pool = reinterpret_cast<float*>(wsb + kCounterBytes + ((P.h2_bytes + 255) / 256) * 256);
  f.wpack = reinterpret_cast<const uint8_t*>(packed);
  f.pool = pool;
  f.gates = pool + (size_t)d.n * f.hid;
  f.counters = reinterpret_cast<int*>(wsb);
  f.trace = g_mb_trace;
  CUtensorMap tx, th_store, th_load;
  {
    // dims (8 ch, W, H, image, channel group): one box = every plane of the CTA's images
    if (f.xsw) {
      const uint64_t dims[4] = {(uint64_t)d.c, (uint64_t)d.w, (uint64_t)d.h, (uint64_t)d.n};
      const uint64_t strides[3] = {(uint64_t)d.c * 2, (uint64_t)d.w * d.c * 2, (uint64_t)d.h * d.w * d.c * 2};
      const uint32_t box[4] = {64, (uint32_t)f.Wp, (uint32_t)(f.bands > 1 ? f.H + 2 : f.H + 1), (uint32_t)f.imgs};
      if (int e = encode_tmap(&tx, x, 4, dims, strides, box, true)) return e;
    } else {
      const uint64_t dims[5] = {8, (uint64_t)d.w, (uint64_t)d.h, (uint64_t)d.n, (uint64_t)(d.c / 8)};
      const uint64_t strides[4] = {(uint64_t)d.c * 2, (uint64_t)d.w * d.c * 2, (uint64_t)d.h * d.w * d.c * 2, 16};
      const uint32_t box[5] = {8, (uint32_t)f.Wp, (uint32_t)(f.bands > 1 ? f.H + 2 : f.H + 1), (uint32_t)f.imgs,
                               (uint32_t)(d.c / 8)};
      if (int e = encode_tmap(&tx, x, 5, dims, strides, box)) return e;
    }
  }
  {
    const uint64_t dims[3] = {8, (uint64_t)b.P, (uint64_t)(f.hid / 8)};
    const uint64_t strides[2] = {(uint64_t)f.hid * 2, 16};
    const uint32_t box_s[3] = {8, (uint32_t)f.st_rows, (uint32_t)(f.HC / 8)};
    if (int e = encode_tmap(&th_store, h2, 3, dims, strides, box_s)) return e;
    const uint32_t box_l[3] = {8, 128, (uint32_t)(b.HCb / 8)};
    if (int e = encode_tmap(&th_load, h2, 3, dims, strides, box_l)) return e;
  }
  f.wback = reinterpret_cast<const uint8_t*>(packed) + P.front_bytes;
  f.h2 = h2;
  f.x = reinterpret_cast<const __half*>(x);
  f.z = reinterpret_cast<__half*>(z);
  CUtensorMap th_fused = th_load;
  if (f.fused) {
    const uint64_t dims[2] = {(uint64_t)f.hid, (uint64_t)b.P};
    const uint64_t strides[1] = {(uint64_t)f.hid * 2};
    const uint32_t box[2] = {64, 128};
    if (int e = encode_tmap(&th_fused, h2, 2, dims, strides, box, true)) return e;
  }
  if (f.zst) {  // [pixels][K] rows of z and of the residual x, 64-channel 128B-swizzled boxes
    const uint64_t dims[2] = {(uint64_t)d.k, (uint64_t)d.n * f.Ho_img * f.Wo};
    const uint64_t strides[1] = {(uint64_t)d.k * 2};
    const uint32_t box[2] = {64, (uint32_t)f.P_out};
    if (int e = encode_tmap(&th_store, z, 2, dims, strides, box, true)) return e;
    if (f.residual)
      if (int e = encode_tmap(&th_fused, x, 2, dims, strides, box, true)) return e;
  }
  if (int e = launch_pdl_cluster(front_kernel(d.act, f.T8 != 0, f.stride == 2, f.fused != 0), f.groups * f.ranges,
                                 mbk::kThreads, f.smem, st, "mb_front launch",
                                 (f.fused && (f.ranges == 2 || f.bands == 2)) ? 2 : 1, tx,
                                 th_store, th_fused, f))
    return e;
  if (f.fused) return WL_OK;
  b.wpack = reinterpret_cast<const uint8_t*>(packed) + P.front_bytes;
  b.gates = f.gates;
  b.x = reinterpret_cast<const __half*>(x);
  b.z = reinterpret_cast<__half*>(z);
  const int ntiles = (b.P + 127) / 128;
  return launch_pdl(mb_back_kernel, ntiles * b.kranges, 256, b.smem, st, "mb_back launch", th_load, b);
}

int mb_init() {
  if (int e = mb1_init()) return e;
  for (int a : {kRelu, kSilu, kGelu})
    for (int k = 0; k < 8; ++k)
      if (int e = check_cuda(cudaFuncSetAttribute(front_kernel(a, k & 4, k & 2, k & 1),
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxMb),
                             "cudaFuncSetAttribute(mb_front)"))
        return e;
  return check_cuda(cudaFuncSetAttribute(mb_back_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMaxMb),
                    "cudaFuncSetAttribute(mb_back)");
}

}  // namespace

int mb_kernel_launches(const wl_block_desc& d) {
  if (mb1_eligible(d)) return 1;
  MbPlanH P;
  if (!mb_plan(d, P)) return set_error(WL_EUNSUPPORTED, "no MBConv launch plan");
  return P.f.fused ? 1 : 2;
}

void mb_set_trace(void* p) {
  g_mb_trace = reinterpret_cast<long long*>(p);
  mb1_set_trace(p);
}

const Family kMbFamily = {mb_validate, mb_weight_count, mb_weight_numel, mb_packed_bytes,
                          mb_pack,     mb_workspace,    mb_forward,      mb_init};

}  // namespace wl
