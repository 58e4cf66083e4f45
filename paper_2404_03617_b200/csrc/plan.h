// plan.h — launch plans shared by the host launcher (abi.cu) and the kernels.
// A plan fixes tile shapes, hidden-chunk widths, the packed-weight layout and
// the shared-memory / TMEM carve-up for one block descriptor.
#pragma once
#include <cstdint>

namespace wl {

constexpr int kTileM = 128;      // pixels per tile = one tcgen05 M=128 accumulator
constexpr int kCoreBytes = 128;  // 8 rows x 16 B core matrix
constexpr int kNumSMs = 148;

__host__ __device__ constexpr int align_up(int v, int a) { return (v + a - 1) / a * a; }

// Conv-first fused block (ConvFirst / ConvNeXt-style), stride 1.
//   tile: 16 output rows x 8 output columns (M-block i = output row i)
//   packed blob: [hdr][chunk 0][chunk 1]... ; chunk j = [U_j][V_j]
struct CfPlan {
  int C, KS, T8, hid, r, nchunks;
  int TH, TW, HH, HW, G;
  int halo_bytes, xc_bytes;
  int hdr_bytes, chunk_bytes, u_bytes;
  int o_convw, o_bconv, o_lng, o_lnb, o_a, o_b;  // byte offsets in hdr
  int ring_stages, resident;
  int s_halo, s_xc, s_hdr, s_ring, s_bar, smem_bytes;
  int t_z, t_cacc, t_e, t_h, h_stride, tmem_cols;
  int ctas_per_sm;
  int halo_bufs;  // TMA halo ring depth (2..8)
};

// Stride-2 ConvFirst fused block (BlurPool along H then W).
struct Cf2Plan {
  int C, K, hid, r, nchunks;
  int W, Wq, rows_out;  // input width, output width, output rows per CTA
  int HW;               // padded halo row width (W + 2)
  int conv_rows;        // full-res conv rows per CTA = 2*rows_out + 1
  int G;
  int halo_bytes, xc_bytes, hq_bytes, hstage_bytes;
  int hdr_bytes, chunk_bytes, u_bytes;
  int o_convw, o_bconv, o_a, o_b;
  int s_halo, s_xc, s_hstage, s_hq, s_hdr, s_ring, s_bar, smem_bytes;
  int ring_stages;
  int t_z, t_cacc, t_e, tmem_cols;
};

// MBConv front (expand -> conv -> act [-> blur]) and back (SE -> gated project).
struct MbPlan {
  int C, K, hid, sq, T8, stride;
  int H, W, Ho, Wo;
  int hc, nchunks;  // hidden channels per chunk
  // front tile: output rows [y0, y0+rows) of one image in flat padded layout
  int rows, Wp, flat_out, x_rows, flat_x;
  int hdr_bytes, chunk_bytes, u_bytes, cw_bytes;
  int o_bexp, o_bconv, o_convw1;  // hdr offsets
  int s_x, s_h1, s_hdr, s_ring, s_bar, smem_bytes;
  int h1_plane_bytes, h1_bytes;
  int ring_stages;
  int t_e, t_c, tmem_cols;
  // back
  int vb_hdr_bytes, vchunk_bytes, vchunks, vr;
};

}  // namespace wl
