"""Golden-fixture loading (TEST INFRASTRUCTURE)."""

import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    inputs = {k[3:]: z[k].astype(np.float32) for k in z.files if k.startswith("in_")}
    return meta, inputs, z["out_layerwise"], z["out_fused"]


def golden_names(prefix=""):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def load_costs():
    with open(os.path.join(GOLDEN, "costs.json")) as fh:
        return json.load(fh)


def big_golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "big", "*.npz")))


def load_big_golden(name):
    """A full-size BASELINE-config case: (meta, reference outputs of the picked
    images). The inputs are regenerated from meta['seed'] with
    machine.random_inputs (the reference's stream) and fp16-rounded."""
    z = np.load(os.path.join(GOLDEN, "big", name + ".npz"))
    return json.loads(str(z["meta"])), z["out_picked"]
