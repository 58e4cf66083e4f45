"""ConvNeXt-T end to end (BASELINE config 4: "ConvNeXt-T 224x224 batch 128 fp16
inference (paper baseline architecture) with fused blocks").

The reference has no ConvNeXt constructor: ConvNeXt enters it
only as a measured row of the efficiency-gap table (PAPER.md:1696,
``data/model_speed_accuracy.csv:10``) and, through PAPER.md:919-921, as "the
same block with different normalization, group-width, and kernel-size" as
ConvFirst. This module builds the published architecture (Liu et al. 2022,
ConvNeXt-T: depths 3/3/9/3, widths 96/192/384/768) from this package's units:

* ``PatchifyStem(96)``: 4x4 stride-4 conv + LayerNorm;
* ``ConvNeXtBlock``: dw7x7 + LayerNorm + 1x1 4x + GELU + 1x1 + residual — the
  fused conv-first kernel at C = 96, the wide path (dwln + L2-resident hidden,
  ``csrc/cnx.cu``) at C = 192 / 384 / 768;
* ``Downsample``: LayerNorm + 2x2 stride-2 conv between stages;
* ``LNHead``: global average pool + LayerNorm + linear classifier.

Layer scale (gamma, init 1e-6 in the original) multiplies the projection
output channel-wise; it is folded into the projection weights and bias at
weight-load time (like BatchNorm folding for ConvFirst),
so the unit ABI has no separate tensor for it. Drop path is identity at
inference.

MACs per image (the efficiency numerator) count the convolutions and linear
layers (4.456 GMAC at 224, the figure SURVEY.md 8(d) quotes); LayerNorm,
GELU, bias and residual adds are not counted, as in the paper's MAC column.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import BlockInstance, ConvNeXtBlock, Downsample, LNHead, PatchifyStem


@dataclass(frozen=True)
class ConvNeXtSpec:
    name: str
    input_resolution: tuple[int, int]
    depths: tuple[int, ...] = (3, 3, 9, 3)
    dims: tuple[int, ...] = (96, 192, 384, 768)
    num_classes: int = 1000
    kernel_size: int = 7
    expansion: int = 4
    patch: int = 4
    layer_norm_eps: float = 1e-6

    def __post_init__(self):
        object.__setattr__(self, "input_resolution", tuple(self.input_resolution))
        object.__setattr__(self, "depths", tuple(self.depths))
        object.__setattr__(self, "dims", tuple(self.dims))
        if len(self.depths) != len(self.dims) or not self.depths:
            raise ValueError("depths and dims must be non-empty and of equal length")
        h, w = self.input_resolution
        total = self.patch * 2 ** (len(self.dims) - 1)
        if h % total or w % total:
            raise ValueError(f"input {h}x{w} must be divisible by {total} (patch x downsamples)")

    def plan(self) -> list[BlockInstance]:
        """Ordered units, the same BlockInstance records ``core.plan_blocks``
        returns for ConvFirstNet (labels stem, s{i}b{j}, ds{i}, head)."""
        eps = self.layer_norm_eps
        h, w = self.input_resolution
        units = [BlockInstance("stem", PatchifyStem(self.dims[0], self.patch, eps), 3, self.dims[0], h, w,
                               self.patch)]
        h, w = h // self.patch, w // self.patch
        block = ConvNeXtBlock(self.kernel_size, self.expansion, "gelu", eps)
        for si, (depth, c) in enumerate(zip(self.depths, self.dims), start=1):
            if si > 1:
                prev = self.dims[si - 2]
                units.append(BlockInstance(f"ds{si - 1}", Downsample(c, eps), prev, c, h, w, 2))
                h, w = h // 2, w // 2
            for bi in range(depth):
                units.append(BlockInstance(f"s{si}b{bi}", block, c, c, h, w, 1))
        units.append(BlockInstance("head", LNHead(self.num_classes, eps), self.dims[-1], self.num_classes, h, w, 1))
        return units


def convnext_tiny(resolution: int = 224) -> ConvNeXtSpec:
    return ConvNeXtSpec(f"convnext-tiny@{resolution}", (resolution, resolution))


def unit_macs(inst: BlockInstance) -> int:
    """Multiply-accumulates of one unit for ONE image."""
    b = inst.block
    hw = inst.in_h * inst.in_w
    c = inst.in_channels
    if isinstance(b, PatchifyStem):
        return (hw // (b.patch * b.patch)) * inst.out_channels * b.patch * b.patch * c
    if isinstance(b, ConvNeXtBlock):
        return hw * c * b.kernel_size ** 2 + 2 * hw * c * b.expansion * c
    if isinstance(b, Downsample):
        return (hw // 4) * inst.out_channels * 4 * c
    if isinstance(b, LNHead):
        return c * b.num_classes
    raise ValueError(f"unknown ConvNeXt unit {type(b).__name__}")


def network_macs(spec: ConvNeXtSpec) -> int:
    return sum(unit_macs(u) for u in spec.plan())


def fold_layer_scale(weights: dict, gamma) -> dict:
    """Fold ConvNeXt's layer scale into a block's projection: gamma * (h V + b)
    = h (V diag(gamma)) + gamma * b."""
    import numpy as np

    g = np.asarray(gamma, dtype=np.float32)
    out = dict(weights)
    out["v"] = (np.asarray(weights["v"], dtype=np.float32) * g[None, :]).astype(np.float32)
    out["b"] = (np.asarray(weights["b"], dtype=np.float32) * g).astype(np.float32)
    return out


__all__ = ["ConvNeXtSpec", "convnext_tiny", "network_macs", "unit_macs", "fold_layer_scale"]
