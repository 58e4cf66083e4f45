"""Model-level kernel scheduler: replaces the reference's per-layer path
(``expand_network(..., LAYER_WISE)``, core.py:401-429) with one fused launch
per ``plan_blocks`` unit (core.py:362-398), all stream-ordered on one CUDA
stream and captured into a single CUDA graph.

Memory plan (HBM): one fp16 NHWC activation buffer per unit boundary
(the unit's output), one shared workspace sized to the largest unit
(MBConv's L2-resident hidden + SE pool, the head's pooled embedding), packed
weights per unit. Batch sharding across GPUs is by independent image shards
(no collective on the path; see bench.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .blocks import FusedBlock, init_weights
from .core import DeviceSpec, ExecutionScheme, NetworkSpec, TensorDims, expand_network, plan_blocks
from .machine import build_schedule


@dataclass
class Unit:
    label: str
    block: object
    module: FusedBlock
    out: torch.Tensor


class FusedNetwork:
    """A NetworkSpec bound to a per-GPU batch, ready to launch.

    ``weights`` (optional) maps unit labels (``stem``, ``s1b0`` ...,
    ``head``) to reference-named float32 tensors; otherwise fan-in-scaled
    synthetic weights are drawn with seed ``seed + unit index``.
    """

    def __init__(self, net: NetworkSpec, batch: int, device: str | torch.device = "cuda", seed: int = 0,
                 weights: dict | None = None, stages: bool = True, dtype: torch.dtype = torch.float16):
        self.net = net
        self.batch = batch
        self.device = torch.device(device)
        # a ConvFirstNet NetworkSpec plans through core.plan_blocks; a
        # ConvNeXtSpec (convnext.py) carries its own unit plan
        self.instances = net.plan() if hasattr(net, "plan") else plan_blocks(net)
        self.units: list[Unit] = []
        ws_bytes = 256
        for i, inst in enumerate(self.instances):
            dims = inst.dims(batch)
            sched = build_schedule(inst.block, dims, out_channels=inst.out_channels)
            wts = None
            if weights is not None:
                wts = weights[inst.label]
            else:
                wts = init_weights(sched, np.random.default_rng(seed + i))
            mod = FusedBlock(inst.block, dims, inst.out_channels, weights=wts, device=self.device, dtype=dtype)
            ws_bytes = max(ws_bytes, mod.workspace.numel())
            out = torch.empty(mod.out_shape, dtype=dtype, device=self.device)
            self.units.append(Unit(inst.label, inst.block, mod, out))
        # the static input carries the first unit's DEVICE width (a stem-less
        # stack at C % 16 != 0 runs zero-padded); __call__ pads into it
        self.dtype = dtype
        self.x = torch.zeros(self.units[0].module.in_shape, dtype=dtype, device=self.device)
        self.in_channels = self.instances[0].in_channels
        # one workspace shared by every unit (launches are stream-ordered)
        self.workspace = torch.zeros(ws_bytes, dtype=torch.uint8, device=self.device)
        for u in self.units:
            u.module.workspace = self.workspace
        self.graph: torch.cuda.CUDAGraph | None = None
        self.steps = self._plan_steps(stages)

    def _plan_steps(self, stages: bool) -> list[tuple[int, int, str]]:
        """Launch plan: [(first unit, unit count, kind)]. With ``stages``:
        * "pair": a unit pair with one fused kernel (``wl_pair_supported``:
          the stem + first ConvFirst block of ConvFirstNet-Pico), the stem
          output kept on chip;
        * "stage": a run of consecutive units sharing one descriptor with a
          stage kernel (``wl_stage_max_blocks``) — ONE launch, each block's
          output stays on chip as the next block's input (the per-stage
          persistent kernel, machine.py:1091-1120);
        * "unit": one launch per unit.
        Only a step's last output is written; the intermediate units' ``out``
        tensors are then not produced."""
        L = _lib.lib()
        steps, i = [], 0
        self._pair_packed = {}
        while i < len(self.units):
            d = self.units[i].module.desc
            if stages and i + 1 < len(self.units) and \
                    L.wl_pair_supported(ctypes.byref(d), ctypes.byref(self.units[i + 1].module.desc)):
                self._pair_packed[i] = self._pack_pair(i)
                steps.append((i, 2, "pair"))
                i += 2
                continue
            cap = L.wl_stage_max_blocks(ctypes.byref(d)) if stages else 0
            j = i + 1
            while cap and j < len(self.units) and j - i < cap and \
                    self.units[j].module.desc.as_tuple() == d.as_tuple():
                j += 1
            steps.append((i, j - i, "stage" if j - i > 1 else "unit"))
            i = j
        return steps

    def _pack_pair(self, i: int) -> torch.Tensor:
        m0, m1 = self.units[i].module, self.units[i + 1].module
        w0 = m0.binding.device_weights(m0.weights)
        w1 = m1.binding.device_weights(m1.weights)
        L = _lib.lib()
        nb = _lib.check(L.wl_pair_packed_bytes(ctypes.byref(m0.desc), ctypes.byref(m1.desc)), "wl_pair_packed_bytes")
        out = np.zeros(nb, dtype=np.uint8)
        c0 = [np.ascontiguousarray(w, dtype=np.float32) for w in w0]
        c1 = [np.ascontiguousarray(w, dtype=np.float32) for w in w1]
        fp0, fp1 = _lib.float_ptr_array(c0), _lib.float_ptr_array(c1)
        _lib.check(L.wl_pair_pack(ctypes.byref(m0.desc), ctypes.byref(m1.desc), fp0[1], len(c0),
                                  fp1[1], len(c1), out.ctypes.data_as(ctypes.c_void_p)),
                   "wl_pair_pack")
        return torch.from_numpy(out).to(self.device)

    def _launch_step(self, first: int, count: int, kind: str, x: torch.Tensor, stream=None) -> torch.Tensor:
        u = self.units[first + count - 1]
        if kind == "unit":
            u.module.launch(x, u.out, self.workspace, stream)
        elif kind == "stage":
            self._launch_stage(first, count, x, u.out, stream)
        else:
            st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
            m0, m1 = self.units[first].module, self.units[first + 1].module
            _lib.check(_lib.lib().wl_pair_forward(ctypes.byref(m0.desc), ctypes.byref(m1.desc), x.data_ptr(),
                                                  self._pair_packed[first].data_ptr(), u.out.data_ptr(), st),
                       "wl_pair_forward")
        return u.out

    # ----------------------------------------------------------- execution
    @property
    def output(self) -> torch.Tensor:
        """The last unit's output at the reference channel count (a view)."""
        return self.units[-1].module.binding.real_output(self.units[-1].out)

    def _load_input(self, dst: torch.Tensor, src: torch.Tensor, non_blocking=True) -> None:
        if src.shape[-1] == dst.shape[-1]:
            dst.copy_(src, non_blocking=non_blocking)
        else:  # reference width -> zero-padded device width (pad channels stay zero)
            dst[..., : src.shape[-1]].copy_(src, non_blocking=non_blocking)

    def launch_all(self, stream=None, x: torch.Tensor | None = None) -> None:
        src = self.x if x is None else x
        for first, count, kind in self.steps:
            src = self._launch_step(first, count, kind, src, stream)

    def _launch_stage(self, first: int, count: int, x: torch.Tensor, out: torch.Tensor, stream=None) -> None:
        mods = [self.units[k].module for k in range(first, first + count)]
        ptrs = (ctypes.c_void_p * count)(*[m.packed.data_ptr() for m in mods])
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        _lib.check(_lib.lib().wl_stage_forward(ctypes.byref(mods[0].desc), count, x.data_ptr(), ptrs, out.data_ptr(),
                                               self.workspace.data_ptr(), st), "wl_stage_forward")

    def _capture_on(self, x: torch.Tensor) -> torch.cuda.CUDAGraph:
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.launch_all(s, x)
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch_all(x=x)
        return g

    def capture(self) -> torch.cuda.CUDAGraph:
        """Capture the whole forward into one CUDA graph (warm-up first)."""
        self.graph = self._capture_on(self.x)
        return self.graph

    def run_host_batches(self, batches, outs) -> None:
        """Serve a sequence of host batches (pinned NHWC fp16) into host logit
        buffers (pinned). Two input slots, each with its own captured graph:
        the host->device copy of batch i+1 runs on a copy stream while the
        forward of batch i runs, and each batch's logits are read back right
        behind its forward on the compute stream."""
        if not hasattr(self, "_slots"):
            self._slots = [self.x, torch.zeros_like(self.x)]
            self._graphs = [self.graph or self.capture(), self._capture_on(self._slots[1])]
            self._copy = torch.cuda.Stream(device=self.device)
            self._d2h = torch.cuda.Stream(device=self.device)
            self._h2d = [torch.cuda.Event(), torch.cuda.Event()]
            self._free = [torch.cuda.Event(), torch.cuda.Event()]
            self._done = [torch.cuda.Event(), torch.cuda.Event()]
            self._logits = [torch.empty(self.output.shape, dtype=self.output.dtype, device=self.device)
                            for _ in range(2)]
        comp = torch.cuda.current_stream(self.device)
        for b in range(2):
            self._free[b].record(comp)
            self._done[b].record(comp)
        for i, (hb, ho) in enumerate(zip(batches, outs)):
            b = i & 1
            with torch.cuda.stream(self._copy):
                self._copy.wait_event(self._free[b])  # slot's previous forward has read it
                self._load_input(self._slots[b], hb)
                self._h2d[b].record(self._copy)
            comp.wait_event(self._h2d[b])
            comp.wait_event(self._done[b])  # the slot's logits of batch i-2 have left the device
            self._graphs[b].replay()
            self._free[b].record(comp)
            # logits to a per-slot buffer (on device), read back on a third
            # stream so neither the next forward nor the next upload queues
            # behind the PCIe transfer
            self._logits[b].copy_(self.output, non_blocking=True)
            fwd = torch.cuda.Event()
            fwd.record(comp)
            with torch.cuda.stream(self._d2h):
                self._d2h.wait_event(fwd)
                ho.copy_(self._logits[b], non_blocking=True)
                self._done[b].record(self._d2h)
        comp.wait_stream(self._d2h)  # every read-back complete before the caller syncs

    def replay(self) -> None:
        if self.graph is None:
            self.capture()
        self.graph.replay()

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        """Forward on an NHWC fp16 batch (copied into the static input)."""
        self._load_input(self.x, x)
        self.replay()
        return self.output

    # ------------------------------------------------------- accounting
    def workloads(self, device: DeviceSpec, scheme=ExecutionScheme.BLOCK_FUSION):
        return expand_network(self.net, self.batch, scheme, device)

    def launch_count(self) -> int:
        """Kernels this forward launches, as the library plans them
        (``wl_kernel_launches``: 1 per fused block, 2 for the head; one per
        stage launch)."""
        n = 0
        for first, count, kind in self.steps:
            if kind != "unit":
                n += 1
                continue
            k = _lib.lib().wl_kernel_launches(ctypes.byref(self.units[first].module.desc))
            _lib.check(k if k < 0 else 0, "wl_kernel_launches")
            n += k
        return n

    def weights(self) -> dict:
        return {u.label: u.module.weights for u in self.units}

    def time_units(self, iters: int = 20) -> list[float]:
        """Per-unit device time (seconds, mean over ``iters``) with CUDA
        events on the launching stream — the measured column beside the
        waterline's attainable latency."""
        torch.cuda.synchronize(self.device)
        times = []
        src = self.x
        for first, count, kind in self.steps:
            u = self.units[first + count - 1]
            go = lambda s=src, f=first, c=count, k=kind: self._launch_step(f, c, k, s)  # noqa: E731
            for _ in range(3):
                go()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
            for _ in range(iters):
                go()
            ev1.record()
            ev1.synchronize()
            # a stage / pair launch's time is shared equally by its units
            times += [ev0.elapsed_time(ev1) / iters / 1e3 / count] * count
            src = u.out
        return times


def ctypes_ref(x):
    return ctypes.byref(x)


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous image shard of ``rank`` (near-equal split; images never
    interact, so no collective is needed on the data path)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)
