"""CPU parity oracle for the block-fusion hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the numeric semantics the reference
``waterline`` package defines for fused blocks (``machine.py``), and extends
them with the pieces the reference cannot execute (LayerNorm, GELU, k x k
depthwise blocks, stride-2 BlurPool blocks, stem, head, whole networks).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import it, and only as the *checker* or the timed CPU reference. The
product path (``paper_2404_03617_b200``) never imports it and has no CPU
fallback.

Parity status
-------------
* pinned: ConvFirst / MBConv / FFN stride-1 blocks — checked bit-for-bit
  (to fp32 rounding) against golden vectors produced by the reference's own
  ``execute_numeric`` (``tests/golden/make_golden.py``).
* unpinned (restatement only, the reference has no executable form):
  LayerNorm + GELU ConvNeXt-style blocks, stride-2 BlurPool blocks, stem,
  head. Their restatements reuse the pinned primitives, and the tests check
  the shared special cases (e.g. LN off + ReLU + 3x3 == reference ConvFirst).
"""

from .blocks import (  # noqa: F401
    blurpool_h,
    blurpool_w,
    blurpool_2d,
    convfirst_block,
    convfirst_s2_block,
    convnext_block,
    downsample_block,
    ln_head_block,
    patch_stem_block,
    ffn_block,
    grouped_conv2d,
    head_block,
    layer_norm,
    mbconv_block,
    phi,
    stem_block,
)
