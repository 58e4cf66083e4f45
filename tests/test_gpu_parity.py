"""Parity of the sm_100a kernels (through the C ABI) with the reference's
golden vectors and the CPU oracle. Tolerance (fp16 storage, fp32
accumulation): max|gpu - ref| / max|ref| <= 1e-2 and ||gpu - ref||_2 /
||ref||_2 <= 2e-3."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import model as om  # noqa: E402
from oracle.fixtures import golden_names, load_golden  # noqa: E402
from paper_2404_03617_b200 import zoo  # noqa: E402
from paper_2404_03617_b200.blocks import FusedBlock, init_weights  # noqa: E402
from paper_2404_03617_b200.core import FFN, ConvFirst, ConvNeXtBlock, Head, MBConv, Stem, TensorDims  # noqa: E402
from paper_2404_03617_b200.machine import ScheduleError, build_schedule, execute_numeric, random_inputs  # noqa: E402
from paper_2404_03617_b200.scheduler import FusedNetwork  # noqa: E402

MAX_REL, L2_REL = 1e-2, 2e-3


def close(got, ref, max_rel=MAX_REL, l2_rel=L2_REL):
    got = np.asarray(got, np.float64).reshape(np.shape(ref))
    ref = np.asarray(ref, np.float64)
    m = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-12)
    l2 = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-12)
    assert np.isfinite(got).all()
    assert m <= max_rel and l2 <= l2_rel, (m, l2)


def r16(rng, shape, scale=1.0):
    return (scale * rng.standard_normal(shape)).astype(np.float16).astype(np.float32)


def oracle_unit(block, w, x):
    return om.unit_forward(block, w, x)


@pytest.mark.parametrize("name", golden_names())
def test_golden_vectors(name):
    meta, ins, out_lw, _ = load_golden(name)
    kinds = {"ConvFirst": ConvFirst, "MBConv": MBConv, "FFN": FFN}
    s = build_schedule(kinds[meta["block"]](**meta["params"]), TensorDims(*meta["dims"]),
                       processors=meta.get("processors"))
    close(execute_numeric(s, ins), out_lw)


def _block_case(block, dims, k=None, seed=0):
    rng = np.random.default_rng(seed)
    s = build_schedule(block, dims, out_channels=k)
    w = init_weights(s, rng)
    w = {n: v.astype(np.float16).astype(np.float32) for n, v in w.items()}
    x = r16(rng, (dims.n, dims.h, dims.w, dims.c))
    return s, w, x


CASES = [
    ("convfirst_pico_s1", ConvFirst(8, 3), TensorDims(2, 112, 112, 16), None),
    ("convfirst_partial_tiles", ConvFirst(8, 6), TensorDims(3, 20, 12, 32), None),
    ("convfirst_c96_ring", ConvFirst(8, 6), TensorDims(1, 28, 28, 96), None),
    ("convfirst_dw3x3", ConvFirst(1, 4), TensorDims(2, 15, 9, 64), None),
    ("convnext_c1_config", ConvNeXtBlock(7, 4, "gelu"), TensorDims(8, 56, 56, 96), None),
    ("convfirst_s2_112", ConvFirst(8, 6, 2), TensorDims(2, 112, 112, 16), 32),
    ("convfirst_s2_56", ConvFirst(8, 6, 2), TensorDims(2, 56, 56, 32), 48),
    ("mbconv_14", MBConv(8, 4, 0.25), TensorDims(2, 14, 14, 128), None),
    ("mbconv_7_odd_batch", MBConv(8, 4, 0.25), TensorDims(3, 7, 7, 128), None),
    # the pitch-8 7x7 path at other widths / activations, and a hidden width it
    # does not take (6 chunks: the block-diagonal kernel runs it)
    ("mbconv_7_c64", MBConv(8, 4, 0.25), TensorDims(3, 7, 7, 64), None),
    ("mbconv_7_c128_a2_relu", MBConv(8, 2, 0.25, 1, "relu"), TensorDims(2, 7, 7, 128), None),
    ("mbconv_7_hid384_fallback", MBConv(8, 3, 0.25), TensorDims(2, 7, 7, 128), None),
    ("mbconv_c2_config_shape", MBConv(1, 4, 0.25), TensorDims(4, 28, 28, 80), None),
    ("mbconv_small_c256", MBConv(8, 4, 0.25), TensorDims(2, 14, 14, 256), None),
    ("mbconv_s2_28", MBConv(8, 4, 0.25, 2), TensorDims(2, 28, 28, 48), 128),
    ("mbconv_s2_14", MBConv(8, 4, 0.25, 2), TensorDims(2, 14, 14, 128), 128),
    # the stride-2 14x14 -> 7x7 variant of the mma.sync kernel: other widths, ReLU, odd batch
    ("mbconv_s2_14_c64_k128_relu", MBConv(8, 4, 0.25, 2, "relu"), TensorDims(3, 14, 14, 64), 128),
    ("mbconv_s2_14_c128_k64", MBConv(8, 2, 0.25, 2), TensorDims(2, 14, 14, 128), 64),
    ("mbconv_s2_14_b129", MBConv(8, 4, 0.25, 2), TensorDims(129, 14, 14, 128), 128),
    ("stem_224", Stem(16), TensorDims(2, 224, 224, 3), None),
    ("stem_c32", Stem(32), TensorDims(1, 64, 48, 3), None),
    ("head_pico", Head(1280, 1000), TensorDims(5, 7, 7, 128), None),
    ("head_batch_over_128", Head(1280, 1000), TensorDims(130, 7, 7, 128), None),
    # ConvFirstNet-Nano/Tiny widths: C % 16 != 0 runs zero-padded to 16
    ("stem_c24_padded", Stem(24), TensorDims(2, 64, 64, 3), None),
    ("convfirst_c24_padded", ConvFirst(8, 3), TensorDims(2, 56, 56, 24), None),
    ("convfirst_s2_24_48_padded_in", ConvFirst(8, 6, 2), TensorDims(2, 56, 56, 24), 48),
    ("convfirst_s2_48_72_padded_out", ConvFirst(8, 6, 2), TensorDims(2, 56, 56, 48), 72),
    ("convfirst_c72_padded", ConvFirst(8, 6), TensorDims(2, 28, 28, 72), None),
    ("mbconv_s2_72_192_padded_in", MBConv(8, 4, 0.25, 2), TensorDims(2, 28, 28, 72), 192),
    ("mbconv_c192_hc48", MBConv(8, 4, 0.25), TensorDims(2, 14, 14, 192), None),
    ("mbconv_c160", MBConv(8, 4, 0.25), TensorDims(2, 14, 14, 160), None),
    # ConvFirstNet-Pico at the reference's native 256: 8x8 stage, two images per CTA pair
    ("mbconv_8x8_c128", MBConv(8, 4, 0.25), TensorDims(4, 8, 8, 128), None),
    # row bands: a cluster pair splits one image (whole tile exceeds shared memory)
    ("mbconv_s2_28_c96_bands", MBConv(8, 4, 0.25, 2), TensorDims(2, 28, 28, 96), 256),
    ("mbconv_s2_32_c64_bands", MBConv(8, 4, 0.25, 2), TensorDims(2, 32, 32, 64), 160),
    ("mbconv_16_c256_bands", MBConv(8, 4, 0.25), TensorDims(2, 16, 16, 256), None),
    ("mbconv_8x8_c256_one_image", MBConv(8, 4, 0.25), TensorDims(2, 8, 8, 256), None),
    # wide conv-first blocks (C > 128, no LayerNorm): grouped conv kernel + FFN rows
    ("convfirst_wide_c192", ConvFirst(8, 6), TensorDims(2, 28, 28, 192), None),
    ("convfirst_wide_c256_silu", ConvFirst(8, 4, 1, "silu"), TensorDims(3, 14, 14, 256), None),
    ("convfirst_wide_c384_dw", ConvFirst(1, 4), TensorDims(2, 14, 14, 384), None),
    # ConvFirstNet-Small s3b0: FFN weights streamed through a chunk ring
    ("convfirst_s2_64_96_streamed", ConvFirst(8, 6, 2), TensorDims(2, 56, 56, 64), 96),
]


@pytest.mark.parametrize("name,block,dims,k", CASES, ids=[c[0] for c in CASES])
def test_block_vs_oracle(name, block, dims, k):
    s, w, x = _block_case(block, dims, k)
    got = execute_numeric(s, dict(w, x=x))
    close(got, oracle_unit(block, w, x))


def test_device_module_matches_host_abi():
    s, w, x = _block_case(MBConv(8, 4, 0.25), TensorDims(2, 14, 14, 128))
    host = execute_numeric(s, dict(w, x=x))
    mod = FusedBlock(s.block, s.dims, weights=w)
    dev = mod(torch.from_numpy(x).half().cuda()).float().cpu().numpy()
    close(dev, host, max_rel=2e-3, l2_rel=5e-4)


def test_deterministic_and_graph_equals_eager():
    net = zoo.at_resolution(zoo.from_name("convfirstnet-pico"), 224)
    m = FusedNetwork(net, batch=4, seed=3)
    m.x.normal_()
    m.launch_all()
    eager = m.output.clone()
    m.capture()
    m.replay()
    a = m.output.clone()
    m.replay()
    torch.cuda.synchronize()
    assert torch.equal(eager, a) and torch.equal(a, m.output)


@pytest.mark.parametrize("model,res", [("convfirstnet-pico", 224), ("convfirstnet-nano", 224),
                                       ("convfirstnet-tiny", 224), ("convfirstnet-small", 224),
                                       ("convfirstnet-pico", 256), ("convfirstnet-nano", 256),
                                       ("convfirstnet-tiny", 256), ("convfirstnet-small", 256)])
def test_network_per_unit_and_logits(model, res):
    net = zoo.at_resolution(zoo.from_name(model), res)
    m = FusedNetwork(net, batch=2, seed=11, stages=False)  # every unit's output materialised
    rng = np.random.default_rng(1)
    x = r16(rng, (2, res, res, 3))
    out = m(torch.from_numpy(x).half().cuda())
    torch.cuda.synchronize()
    src = x
    for u, inst in zip(m.units, m.instances):
        dev = u.out.float().cpu().numpy()
        got = u.module.binding.real_output(dev)
        ref = oracle_unit(inst.block, u.module.weights, src)
        close(got, ref)
        if dev.ndim == 4 and dev.shape[3] > got.shape[3]:
            assert not dev[..., got.shape[3]:].any(), f"{u.label}: padded channels are not zero"
        src = np.ascontiguousarray(got).reshape(ref.shape)
    ref = om.network_forward(m.instances, m.weights(), x)
    close(out.float().cpu().numpy(), ref, max_rel=2e-2, l2_rel=1e-2)


@pytest.mark.parametrize("model,res", [("convfirstnet-pico", 224), ("convfirstnet-small", 224),
                                       ("convfirstnet-tiny", 256)])
def test_full_size_b128_sampled_images(model, res):
    """BASELINE config 3 at full size (and the padded / row-band plans at the
    same batch): images 0, 63 and 127 of the b128 forward match the oracle
    unit by unit (the oracle runs on the three images)."""
    net = zoo.at_resolution(zoo.from_name(model), res)
    m = FusedNetwork(net, batch=128, seed=5, stages=False)
    m.x.normal_()
    m.replay()
    torch.cuda.synchronize()
    pick = [0, 63, 127]
    src = m.x.float().cpu().numpy()[pick]
    for u, inst in zip(m.units, m.instances):
        got = u.module.binding.real_output(u.out.float().cpu().numpy()[pick])
        ref = oracle_unit(inst.block, u.module.weights, src)
        close(got, ref)
        src = np.ascontiguousarray(got).reshape(ref.shape)


def test_unsupported_configs_fail_loudly():
    # a 56x56x256 MBConv: even a row band's tile exceeds shared memory -> refused, never approximated
    with pytest.raises(ScheduleError):
        FusedBlock(MBConv(8, 4, 0.25), TensorDims(2, 56, 56, 256))
    with pytest.raises(ScheduleError):
        FusedBlock(ConvFirst(4, 6), TensorDims(1, 8, 8, 16))  # no T=4 kernel
    with pytest.raises(ScheduleError):  # LayerNorm statistics cannot absorb zero padding
        FusedBlock(ConvNeXtBlock(7, 4, "gelu"), TensorDims(1, 8, 8, 24))


def test_pipelined_host_batches_match_single_calls():
    """run_host_batches (double-buffered H2D / forward overlap, the e2e path of
    bench.py) returns exactly the logits of one-at-a-time calls."""
    net = zoo.at_resolution(zoo.from_name("convfirstnet-pico"), 224)
    m = FusedNetwork(net, batch=4, seed=9)
    rng = np.random.default_rng(4)
    hosts = [torch.from_numpy(r16(rng, (4, 224, 224, 3))).half().pin_memory() for _ in range(3)]
    ref = []
    for h in hosts:
        ref.append(m(h.cuda()).clone())
    outs = [torch.empty(m.output.shape, dtype=torch.float16).pin_memory() for _ in hosts]
    m.run_host_batches(hosts, outs)
    torch.cuda.synchronize()
    for r, o in zip(ref, outs):
        assert torch.equal(r.cpu(), o)


@pytest.mark.parametrize("batch", [4, 128])
def test_stage_launches_match_per_block_launches(batch):
    """Per-stage persistent launches (wl_stage_forward: consecutive stride-1
    MBConv blocks with the image kept in shared memory) give exactly the
    logits of one launch per block, with fewer launches."""
    net = zoo.at_resolution(zoo.from_name("convfirstnet-pico"), 224)
    staged = FusedNetwork(net, batch=batch, seed=17)
    single = FusedNetwork(net, batch=batch, seed=17, stages=False)
    assert any(k == "stage" for _, _, k in staged.steps) and any(k == "pair" for _, _, k in staged.steps)
    assert staged.launch_count() < single.launch_count()
    staged.x.normal_()
    single.x.copy_(staged.x)
    staged.replay()
    single.replay()
    torch.cuda.synchronize()
    # the stem + s1b0 pair kernel (mma.sync, fp32 accumulation in another
    # order) is not bitwise identical to the two tcgen05 launches
    close(staged.output.float().cpu().numpy(), single.output.float().cpu().numpy(), max_rel=2e-2, l2_rel=1e-2)


def test_stem_block_pair_vs_oracle():
    """The fused stem + first ConvFirst block (wl_pair_forward, stem_cf.cu)
    against the oracle's stem then block, at Pico's 224 input and at a ragged
    resolution (partial 8 x 16 tiles)."""
    import ctypes

    from paper_2404_03617_b200 import _lib

    for hw in ((224, 224), (40, 72)):
        net_in = TensorDims(2, hw[0], hw[1], 3)
        s0, w0, x = _block_case(Stem(16), net_in, seed=5)
        s1, w1, _ = _block_case(ConvFirst(8, 3), TensorDims(2, hw[0] // 2, hw[1] // 2, 16), seed=6)
        m0 = FusedBlock(s0.block, s0.dims, weights=w0)
        m1 = FusedBlock(s1.block, s1.dims, weights=w1)
        L = _lib.lib()
        assert L.wl_pair_supported(ctypes.byref(m0.desc), ctypes.byref(m1.desc)) == 1
        nb = L.wl_pair_packed_bytes(ctypes.byref(m0.desc), ctypes.byref(m1.desc))
        packed = np.zeros(nb, np.uint8)
        c0 = [np.ascontiguousarray(v, np.float32) for v in m0.binding.device_weights(w0)]
        c1 = [np.ascontiguousarray(v, np.float32) for v in m1.binding.device_weights(w1)]
        fp0, fp1 = _lib.float_ptr_array(c0), _lib.float_ptr_array(c1)
        _lib.check(L.wl_pair_pack(ctypes.byref(m0.desc), ctypes.byref(m1.desc), fp0[1], len(c0),
                                  fp1[1], len(c1), packed.ctypes.data_as(ctypes.c_void_p)))
        pd = torch.from_numpy(packed).cuda()
        xd = torch.from_numpy(x).half().cuda()
        out = torch.empty(m1.out_shape, dtype=torch.float16, device="cuda")
        _lib.check(L.wl_pair_forward(ctypes.byref(m0.desc), ctypes.byref(m1.desc), xd.data_ptr(), pd.data_ptr(),
                                     out.data_ptr(), torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        h = om.unit_forward(Stem(16), w0, x).astype(np.float16).astype(np.float32)
        ref = om.unit_forward(ConvFirst(8, 3), w1, h)
        close(out.float().cpu().numpy(), ref)


def test_stage_forward_abi_three_blocks():
    """wl_stage_forward over three different-weight 14x14 MBConv blocks equals
    the oracle applied block by block."""
    import ctypes

    from paper_2404_03617_b200 import _lib

    dims = TensorDims(3, 14, 14, 128)
    mods, ws = [], []
    rng = np.random.default_rng(8)
    for i in range(3):
        s, w, _ = _block_case(MBConv(8, 4, 0.25), dims, seed=30 + i)
        mods.append(FusedBlock(s.block, s.dims, weights=w))
        ws.append(w)
    x = r16(rng, (3, 14, 14, 128))
    xd = torch.from_numpy(x).half().cuda()
    out = torch.empty_like(xd)
    ptrs = (ctypes.c_void_p * 3)(*[m.packed.data_ptr() for m in mods])
    _lib.check(_lib.lib().wl_stage_forward(ctypes.byref(mods[0].desc), 3, xd.data_ptr(), ptrs, out.data_ptr(),
                                           mods[0].workspace.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ref = x
    for w in ws:
        ref = om.unit_forward(MBConv(8, 4, 0.25), w, ref).astype(np.float16).astype(np.float32)
    close(out.float().cpu().numpy(), ref)
