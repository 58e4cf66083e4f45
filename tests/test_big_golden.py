"""BASELINE.json configs at full size against outputs of the UNMODIFIED
reference (tests/golden/make_golden.py -> tests/golden/big/): 56x56x96 b8
ConvFirst (config 1's reference form), MBConv(1,4,.25) 28x28x80 b128
(config 2) and the Pico 14x14x128 MBConv at b128. The whole batch is
regenerated from the seed through machine.random_inputs (the reference's
stream); the reference was evaluated on the picked images only."""

import numpy as np
import pytest

import oracle
from oracle.fixtures import big_golden_names, load_big_golden
from paper_2404_03617_b200.core import ConvFirst, ExecutionScheme, MBConv, TensorDims
from paper_2404_03617_b200.machine import build_schedule, random_inputs

KINDS = {"ConvFirst": ConvFirst, "MBConv": MBConv}
CF_ORDER = ["x", "w_conv", "b_conv", "u", "a", "v", "b"]
MB_ORDER = ["x", "w_exp", "b_exp", "w_conv", "b_conv", "w_sq", "b_sq", "w_ex", "b_ex", "w_prj", "b_prj"]


def regenerate(meta):
    block = KINDS[meta["block"]](**meta["params"])
    s = build_schedule(block, TensorDims(*meta["dims"]), ExecutionScheme.LAYER_WISE)
    ins = random_inputs(s, np.random.default_rng(meta["seed"]))
    ins = {k: v.astype(np.float16).astype(np.float32) for k, v in ins.items()}
    assert float(ins["x"].astype(np.float64).sum()) == meta["x_checksum"]
    assert float(sum(v.astype(np.float64).sum() for k, v in ins.items() if k != "x")) == meta["w_checksum"]
    return block, ins


@pytest.mark.parametrize("name", big_golden_names())
def test_oracle_matches_reference_at_config_size(name):
    meta, ref = load_big_golden(name)
    block, ins = regenerate(meta)
    sub = dict(ins, x=ins["x"][meta["picks"]])
    if meta["block"] == "ConvFirst":
        got = oracle.convfirst_block(*[sub[k] for k in CF_ORDER], activation=block.activation)
    else:
        got = oracle.mbconv_block(*[sub[k] for k in MB_ORDER], activation=block.activation)
    assert np.abs(got - ref).max() <= 2e-6 * np.abs(ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", [ExecutionScheme.BLOCK_FUSION, ExecutionScheme.LAYER_WISE], ids=["fused", "lw"])
@pytest.mark.parametrize("name", big_golden_names())
def test_gpu_full_batch_matches_reference(name, scheme):
    """The fused kernel runs the WHOLE batch (its full-size launch plan);
    so does the device layer-wise schedule (layerwise.cu); the picked
    images must match the reference within the fp16 budget
    (max-rel 1e-2, L2-rel 2e-3)."""
    from paper_2404_03617_b200.machine import execute_numeric

    meta, ref = load_big_golden(name)
    block, ins = regenerate(meta)
    s = build_schedule(block, TensorDims(*meta["dims"]), scheme)
    got = execute_numeric(s, ins)[meta["picks"]].astype(np.float64)
    m = np.abs(got - ref).max() / np.abs(ref).max()
    l2 = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert np.isfinite(got).all()
    assert m <= 1e-2 and l2 <= 2e-3, (m, l2)
