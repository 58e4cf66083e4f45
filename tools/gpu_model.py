import sys, os, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_03617_b200 import zoo, complexity
from paper_2404_03617_b200.scheduler import FusedNetwork
from oracle import model as om

for name in ["convfirstnet-pico", "convfirstnet-small"]:
    net = zoo.at_resolution(zoo.from_name(name), 224)
    fn = FusedNetwork(net, batch=2, seed=1)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 224, 224, 3)).astype(np.float16)
    fn.x.copy_(torch.from_numpy(x).cuda())
    fn.launch_all(); torch.cuda.synchronize()
    # per-unit parity: oracle fed with the GPU's own unit input
    src = x.astype(np.float32); worst = 0
    for u, inst in zip(fn.units, fn.instances):
        got = u.out.float().cpu().numpy()
        ref = om.unit_forward(inst.block, u.module.weights, src)
        got = got.reshape(ref.shape)
        err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-6)
        worst = max(worst, err)
        if err > 1e-2: print("  unit", u.label, "maxrel", err)
        src = got
    logits = fn.output.float().cpu().numpy().reshape(2, 1000)
    ref = om.network_forward(fn.instances, fn.weights(), x.astype(np.float32)).reshape(2, 1000)
    e2e = np.abs(logits - ref).max() / np.abs(ref).max()
    print(name, "units", len(fn.units), "worst unit maxrel %.3g" % worst, "end-to-end logits maxrel %.3g" % e2e, flush=True)
    del fn
    # timing at b128
    fn = FusedNetwork(net, batch=128, seed=1)
    fn.x.normal_()
    g = fn.capture()
    for _ in range(5): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): g.replay()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    macs = complexity.network_macs(net)
    eff = 2 * macs * 128 / (ms / 1e3) / 2.25e15
    print(f"{name} b128: {ms:.3f} ms/batch, {128/(ms/1e3):.0f} img/s, eff {eff*100:.1f}% of 2.25 PF", flush=True)
    ts = fn.time_units(10)
    tot = sum(ts)
    for u, inst, t in zip(fn.units, fn.instances, ts):
        ops = complexity.block_ops(inst.block, inst.dims(128), inst.out_channels)
        print(f"   {u.label:6s} {type(inst.block).__name__:10s} {inst.in_h:4d}x{inst.in_w:<4d} c{inst.in_channels:4d}->{inst.out_channels:4d}  {t*1e6:8.1f} us  {ops/t/1e12:7.1f} TF/s  {100*t/tot:5.1f}%")
    del fn
