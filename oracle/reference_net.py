"""CPU reference forward of a whole network — BASELINE INFRASTRUCTURE (the
``--impl reference`` arm and the ``cpu_baseline`` leg of bench.py only).

Every stride-1 ConvFirst / MBConv unit runs through the UNMODIFIED
reference: ``waterline.machine.execute_numeric`` on the LAYER_WISE schedule
(machine.py:1053, the reference's fastest executable form of the block),
installed offline under ``baseline/_ref``. The units the reference cannot
execute (stem, stride-2 blocks, head: machine.py:423-425, 753-754,
1055-1059) run through the oracle port (oracle/blocks.py). Images are
independent, so throughput uses every host core: one worker process per
core, one image per worker, single-threaded BLAS each.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The installed reference package, or None when it is absent."""
    if os.path.isdir(os.path.join(REF_DIR, "waterline")) and REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import waterline.core as wcore  # noqa: F401
        import waterline.machine as wmach  # noqa: F401
    except Exception:
        return None
    return wcore, wmach


def _ref_block(wcore, block):
    if block.kind == "convfirst" and block.stride == 1:
        return wcore.ConvFirst(block.group_width, block.expansion, 1, block.activation)
    if block.kind == "mbconv" and block.stride == 1:
        return wcore.MBConv(block.group_width, block.expansion, block.se_ratio, 1, block.activation)
    return None


def unit_forward(inst, weights, x, ref):
    """One plan_blocks unit: the reference where it can execute, else the port."""
    from . import model as om

    if ref is not None:
        wcore, wmach = ref
        rb = _ref_block(wcore, inst.block)
        if rb is not None:
            n, h, w, c = x.shape
            s = wmach.build_schedule(rb, wcore.TensorDims(n, h, w, c), wcore.ExecutionScheme.LAYER_WISE)
            return wmach.execute_numeric(s, dict(weights, x=x))
    return om.unit_forward(inst.block, weights, x)


def network_forward(units, weights, x, ref):
    h = np.asarray(x, dtype=np.float32)
    for u in units:
        h = unit_forward(u, weights[u.label], h, ref).astype(np.float16).astype(np.float32)
    return h


# ------------------------------------------------------------ worker pool

_W = {}


def _init_worker(model: str, seed: int):
    sys.path.insert(0, ROOT)
    from paper_2404_03617_b200 import zoo
    from paper_2404_03617_b200.blocks import init_weights
    from paper_2404_03617_b200.core import plan_blocks
    from paper_2404_03617_b200.machine import build_schedule

    net = zoo.at_resolution(zoo.from_name(model), 224)
    units = plan_blocks(net)
    weights = {}
    for i, u in enumerate(units):
        s = build_schedule(u.block, u.dims(1), out_channels=u.out_channels)
        weights[u.label] = init_weights(s, np.random.default_rng(seed + i))
    _W.update(units=units, weights=weights, ref=load_reference(),
              x=np.random.default_rng(seed).standard_normal((1, 224, 224, 3)).astype(np.float16).astype(np.float32))


def _one_image(_):
    t0 = time.perf_counter()
    network_forward(_W["units"], _W["weights"], _W["x"], _W["ref"])
    return time.perf_counter() - t0


class ReferencePool:
    """``workers`` single-threaded processes, each holding the network."""

    def __init__(self, model: str, workers: int | None = None, seed: int = 0):
        import concurrent.futures as cf
        import multiprocessing as mp

        self.workers = workers or int(os.environ.get("WL_REF_WORKERS", "0")) or max(1, min(os.cpu_count() or 1, 64))
        env_keys = ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")
        saved = {k: os.environ.get(k) for k in env_keys}
        for k in env_keys:  # inherited by the spawned workers: one BLAS thread each
            os.environ[k] = "1"
        try:
            self.pool = cf.ProcessPoolExecutor(self.workers, mp_context=mp.get_context("spawn"),
                                               initializer=_init_worker, initargs=(model, seed))
            list(self.pool.map(_one_image, range(self.workers)))  # warm every worker
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        self.kind = "reference" if load_reference() is not None else "port"

    def step(self) -> float:
        """Wall seconds for one image on every worker (``workers`` images)."""
        t0 = time.perf_counter()
        list(self.pool.map(_one_image, range(self.workers)))
        return time.perf_counter() - t0

    def close(self):
        self.pool.shutdown()
