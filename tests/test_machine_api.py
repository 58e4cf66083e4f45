"""The execute_numeric drop-in's host logic (no GPU): schedules, tensor
tables and seeded inputs match the reference's."""

import numpy as np
import pytest

from oracle.fixtures import golden_names, load_golden
from paper_2404_03617_b200.core import ConvFirst, FFN, MBConv, PlainConv, ConvSpec, TensorDims
from paper_2404_03617_b200.machine import (
    ScheduleError, build_schedule, execute_numeric, fused_dram_bytes, microbatch_plan, random_inputs,
)
from paper_2404_03617_b200.core import DeviceSpec, StageSpec


@pytest.mark.parametrize("name", golden_names())
def test_random_inputs_reproduce_the_reference_stream(name):
    meta, ins, _, _ = load_golden(name)
    p = meta["params"]
    kinds = {"ConvFirst": ConvFirst, "MBConv": MBConv, "FFN": FFN}
    block = kinds[meta["block"]](**p)
    s = build_schedule(block, TensorDims(*meta["dims"]))
    ours = random_inputs(s, np.random.default_rng(meta["seed"]))
    assert list(ours) == [k for k in ins]
    for k, v in ours.items():
        assert np.array_equal(v.astype(np.float16).astype(np.float32), ins[k]), k
    assert fused_dram_bytes(s) == meta["fused_dram_bytes"]


def test_build_schedule_errors_match_reference():
    with pytest.raises(ValueError):
        build_schedule(PlainConv(ConvSpec(8, 8)), TensorDims(1, 4, 4, 8))
    with pytest.raises(ValueError):
        build_schedule(ConvFirst(8, 6), TensorDims(1, 4, 4, 16), out_channels=32)
    with pytest.raises(ValueError):
        build_schedule(ConvFirst(8, 6), TensorDims(1, 4, 4, 16), chunk=7)
    # partitioned schedules follow the reference's rules (machine.py:469-474, 655-657)
    assert build_schedule(ConvFirst(8, 6), TensorDims(1, 4, 4, 32), processors=4).processors == 4
    with pytest.raises(ValueError):
        build_schedule(ConvFirst(8, 6), TensorDims(1, 4, 4, 32), processors=3)
    with pytest.raises(ValueError):
        build_schedule(ConvFirst(8, 6), TensorDims(1, 4, 4, 32), processors=8)  # 4 channels per part < T
    with pytest.raises(ValueError):
        build_schedule(ConvFirst(8, 6, 2), TensorDims(1, 4, 4, 32), out_channels=48, processors=2)
    with pytest.raises(ValueError):
        build_schedule(MBConv(8, 4, 0.25), TensorDims(1, 4, 4, 32), processors=5)


def test_execute_numeric_input_checks():
    s = build_schedule(ConvFirst(8, 6), TensorDims(1, 8, 8, 16))
    ins = random_inputs(s, np.random.default_rng(0))
    bad = dict(ins)
    del bad["u"]
    with pytest.raises(ScheduleError, match="missing input tensor 'u'"):
        execute_numeric(s, bad)
    bad = dict(ins, a=np.zeros(3, np.float32))
    with pytest.raises(ScheduleError, match="has shape"):
        execute_numeric(s, bad)


def test_microbatch_plan_reference_example():
    # SPEC.md:420 worked example: C=128, 16x16, alpha 4, d=10, 6 MiB -> n_mb 22, weights 3,358,720 B
    dev = DeviceSpec("a5000", 76.7e12, 479.375e9, l2_bytes=6 * 2**20)
    plan = microbatch_plan(StageSpec(MBConv(8, 4, 0.25), 10, 128), TensorDims(128, 16, 16, 128), dev)
    assert plan.feasible and plan.micro_batch == 22 and plan.weights_bytes == 3_358_720


def test_simulate_without_gpu_is_a_usage_error(capsys):
    """The B200 simulate leg (reference cli.py:283-325) has no CPU path."""
    import torch

    from paper_2404_03617_b200 import simulate

    if torch.cuda.is_available():
        pytest.skip("CPU-only behaviour")
    assert simulate.main(["--block", "convfirst", "--channels", "16"]) == simulate.EXIT_USAGE
    assert "no CPU path" in capsys.readouterr().err
